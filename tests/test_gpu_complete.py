"""GPU parity for the completion path (chm_monitor_complete)
against the reference's golden vectors: batch 1, record_completion of a
shuffled subset of the live requests (batch rows and pre-seeded entries),
batch 2 -- in-flight sums bit-exact after the removals, decisions bit-exact
after them."""

import numpy as np
import pytest
import torch

from paper_2603_22206_b200 import _lib, errors as E
from paper_2603_22206_b200.scheduler import RowBatch
from paper_2603_22206_b200.state import request_key
from tests import harness as H
from tests.test_gpu_schedule import make_scheduler

pytestmark = pytest.mark.gpu


def _batch(gs, rt, pr, sc):
    dev = gs.device
    rt.set(torch.as_tensor(sc["q"], device=dev))
    pr.set(torch.as_tensor(sc["yhat"], device=dev))
    n = len(sc["prog"])
    b = RowBatch.from_numpy(dev, program=sc["prog"], stage=sc["stage"], arrival=sc["arrival"],
                            out_tokens=sc["out_tok"], handle=np.arange(n))
    gs.run_rows(b, n_iterations=0)
    gs.check_errors()
    buf = gs.buf
    return dict(model=buf.model[:n].cpu().numpy(), priority=buf.priority[:n].cpu().numpy(),
                cached=(buf.dflags[:n].cpu().numpy() & 1).astype(np.int8),
                loads=buf.loads[:n * sc["k"]].view(n, sc["k"]).cpu().numpy())


def _complete(gs, models, keys):
    st, buf = gs.state, gs.buf
    dev = gs.device
    cm = torch.as_tensor(np.asarray(models, np.int32), device=dev)
    ck = torch.as_tensor(np.asarray(keys, np.int64), device=dev)
    buf.error.copy_(buf.error_init)
    _lib.check(gs.lib.chm_monitor_complete(st.pool_c, st.monitor_c, cm.data_ptr(), ck.data_ptr(),
                                           int(cm.numel()), buf.n_complete.data_ptr(),
                                           buf.error.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream),
               "chm_monitor_complete")
    torch.cuda.synchronize()


@pytest.mark.parametrize("name", H.complete_names())
def test_completion_matches_reference(name):
    d, b1, b2 = H.load_complete(name)
    decay = bool(int(d["decay"]))
    gs, rt, pr = make_scheduler(b1, max_rows=max(len(b1["prog"]), len(b2["prog"])),
                                decay_in_flight=decay)
    r1 = _batch(gs, rt, pr, b1)
    for key in ("model", "priority", "cached"):
        np.testing.assert_array_equal(r1[key], d[f"out1_{key}"], err_msg=key)
    if decay:  # note_progress (monitor.py:108-111), then the decayed sums (122-129)
        gs.note_progress(d["p_model"], d["p_key"], d["p_emitted"])
        torch.cuda.synchronize()
        gs.check_errors("progress")
        assert np.array(gs.state.in_flight_sums()).tobytes() == d["prog_p"].tobytes()
    _complete(gs, d["c_model"], d["c_key"])
    gs.check_errors("completions")
    st = gs.state
    assert np.array(st.in_flight_sums()).tobytes() == d["mid_p"].tobytes()
    np.testing.assert_array_equal(st.inflight_count.cpu().numpy(), d["mid_cnt"])
    np.testing.assert_array_equal(gs.buf.n_complete.cpu().numpy(),
                                  np.bincount(d["c_model"], minlength=b1["k"]))
    r2 = _batch(gs, rt, pr, b2)
    for key in ("model", "priority", "cached"):
        np.testing.assert_array_equal(r2[key], d[f"out2_{key}"], err_msg=key)
    routed = d["out2_cached"] == 0  # loads are estimated on the routing branch only
    assert r2["loads"][routed].tobytes() == d["out2_loads"][routed].tobytes()
    assert np.array(st.in_flight_sums()).tobytes() == d["final_p"].tobytes()


def test_completion_unknown_request():
    """errors.UnknownRequest (monitor.py:104-105): not in flight on that model."""
    d, b1, _ = H.load_complete("c3_nondyadic")
    gs, rt, pr = make_scheduler(b1)
    r1 = _batch(gs, rt, pr, b1)
    m0 = int(r1["model"][0])
    key0 = request_key(b1["prog"][0], b1["stage"][0])
    wrong = (m0 + 1) % b1["k"]
    _complete(gs, [wrong], [key0])
    with pytest.raises(E.UnknownRequest):
        gs.check_errors()
    # completing it on its own model works, twice does not
    _complete(gs, [m0], [key0])
    gs.check_errors()
    _complete(gs, [m0], [key0])
    with pytest.raises(E.UnknownRequest):
        gs.check_errors()


def test_redispatch_after_completion():
    """A completed (program, stage) may be dispatched again (its in-flight bit
    is cleared); without the completion it is a DuplicateRequest."""
    d, b1, _ = H.load_complete("c4_all")
    gs, rt, pr = make_scheduler(b1)
    _batch(gs, rt, pr, b1)
    one = {k: (v[:1] if isinstance(v, np.ndarray) and v.ndim and len(v) == len(b1["prog"])
               else v) for k, v in b1.items()}
    one["arrival"] = np.array([100.0])
    dev = gs.device
    rt.set(torch.as_tensor(one["q"], device=dev))
    pr.set(torch.as_tensor(one["yhat"], device=dev))
    b = RowBatch.from_numpy(dev, program=one["prog"], stage=one["stage"],
                            arrival=one["arrival"], out_tokens=one["out_tok"], handle=np.zeros(1))
    gs.run_rows(b, n_iterations=0)
    with pytest.raises(E.DuplicateRequest):
        gs.check_errors()
    gs2, rt2, pr2 = make_scheduler(b1)
    r = _batch(gs2, rt2, pr2, b1)
    _complete(gs2, [int(r["model"][0])], [request_key(one["prog"][0], one["stage"][0])])
    gs2.check_errors()
    rt2.set(torch.as_tensor(one["q"], device=dev))
    pr2.set(torch.as_tensor(one["yhat"], device=dev))
    gs2.run_rows(b, n_iterations=0)
    gs2.check_errors()
