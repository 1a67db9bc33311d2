"""GPU parity: K5/K6/K7 through the C-ABI against the reference's golden vectors
and the oracle port (bit-exact decisions, loads, in-flight sums, queue state)."""

import math

import numpy as np
import pytest
import torch

from paper_2603_22206_b200 import errors as E
from paper_2603_22206_b200.config import AgingConfig, BalancerConfig
from paper_2603_22206_b200.predictor import PrecomputedPredictor
from paper_2603_22206_b200.router import ScoreTableRouter
from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch
from tests import harness as H

pytestmark = pytest.mark.gpu

ERR_CLASS = {"ValidationError": E.ValidationError, "ValueError": ValueError,
             "DuplicateRequest": E.DuplicateRequest}


def make_scheduler(sc, max_rows=None, aging=AgingConfig(), decay_in_flight=False):
    pool = H.pool_of(sc)
    rt, pr = ScoreTableRouter(), PrecomputedPredictor()
    n = len(sc["prog"])
    gs = GpuScheduler(pool, BalancerConfig(sc["tau"], sc["margin"]), aging, router=rt,
                      predictor=pr, n_programs=sc["n_prog"], max_rows=max_rows or max(n, 1),
                      queue_capacity=10240, decay_in_flight=decay_in_flight)
    st = gs.state
    per_model = {m: [] for m in sc["ids"]}
    for m, v in sc["p0"]:
        per_model[sc["ids"][int(m)]].append(float(v))
    st.seed_inflight(per_model)
    if len(sc["pre"]):
        st.preassign(sc["pre"][:, 0], sc["pre"][:, 1])
    pr_run = sc["pre_running"].astype(np.int32)
    st.set_engine_counters(running=pr_run, seq=pr_run.astype(np.int64))
    return gs, rt, pr


def run_gpu(sc):
    gs, rt, pr = make_scheduler(sc)
    dev = gs.device
    rt.set(torch.as_tensor(sc["q"], device=dev))
    pr.set(torch.as_tensor(sc["yhat"], device=dev))
    n = len(sc["prog"])
    batch = RowBatch.from_numpy(dev, program=sc["prog"], stage=sc["stage"],
                                arrival=sc["arrival"], out_tokens=sc["out_tok"],
                                handle=np.arange(n))
    gs.run_rows(batch, n_iterations=0)
    torch.cuda.synchronize()
    buf = gs.buf
    res = dict(
        model=buf.model[:n].cpu().numpy(), priority=buf.priority[:n].cpu().numpy(),
        flags=buf.dflags[:n].cpu().numpy(), seq=buf.seq[:n].cpu().numpy(),
        loads=buf.loads[:n * sc["k"]].view(n, sc["k"]).cpu().numpy(),
        n_committed=int(buf.n_committed.item()), error=buf.error.cpu().tolist(),
        final_p=np.array(gs.state.in_flight_sums()),
        final_cnt=gs.state.inflight_count.cpu().numpy(),
        running=gs.state.engine_running.cpu().numpy(),
        queued=gs.state.engine_queued.cpu().numpy(),
        assign=gs.state.assignment.cpu().numpy(),
    )
    return gs, res


@pytest.mark.parametrize("name", H.schedule_names())
def test_schedule_matches_reference(name):
    sc = H.load_schedule(name)
    gs, res = run_gpu(sc)
    n = sc["err_row"] if sc["err_kind"] else len(sc["prog"])
    assert res["n_committed"] == n
    np.testing.assert_array_equal(res["model"][:n], sc["out_model"][:n])
    np.testing.assert_array_equal(res["priority"][:n], sc["out_priority"][:n])
    np.testing.assert_array_equal(res["flags"][:n] & 1, sc["out_cached"][:n])
    np.testing.assert_array_equal((res["flags"][:n] >> 1) & 1, sc["out_admitted"][:n])
    np.testing.assert_array_equal(res["seq"][:n], sc["out_seq"][:n])
    routed = sc["out_cached"][:n] == 0
    assert res["loads"][:n][routed].tobytes() == sc["out_loads"][:n][routed].tobytes()
    # bit-exact Neumaier in-flight sums, counts, engine counters, assignments
    assert res["final_p"].tobytes() == sc["out_final_p"].tobytes()
    np.testing.assert_array_equal(res["final_cnt"], sc["out_final_cnt"])
    np.testing.assert_array_equal(res["running"], sc["out_running"])
    np.testing.assert_array_equal(res["queued"], sc["out_queued"])
    np.testing.assert_array_equal(res["assign"], sc["out_assign"])
    if sc["err_kind"]:
        with pytest.raises(ERR_CLASS[sc["err_kind"]]):
            gs.check_errors()
        assert res["error"][1] == sc["err_row"]
    else:
        assert res["error"][0] == 0


def test_schedule_batch_object_api():
    """schedule_batch(reqs, recs) -> Decision list equal to the oracle port's."""
    sc = H.load_schedule("k5_nondyadic_p0")
    gs, rt, pr = make_scheduler(sc)
    reqs, recs = H.requests_of(sc)
    rt.set(torch.as_tensor(sc["q"], device=gs.device))
    pr.set(torch.as_tensor(sc["yhat"], device=gs.device))
    for p in range(sc["n_prog"]):  # dense program index = numeric suffix
        gs.program_index(f"p{p:06d}")
    decs = gs.schedule_batch(reqs, recs)
    port, err = H.run_port_schedule(sc)
    assert err is None
    for i, d in enumerate(decs):
        assert d.model == sc["ids"][port["model"][i]]
        assert d.priority == port["priority"][i]
        assert d.used_cached_assignment == bool(port["cached"][i])
        if not d.used_cached_assignment:
            assert [d.estimated_loads[m] for m in sc["ids"]] == port["loads"][i].tolist()
            assert d.scores == {m: float(np.float32(sc["q"][i, k]))
                                for k, m in enumerate(sc["ids"])}


def test_nan_prediction_rejected():
    sc = H.load_schedule("k3_basic")
    sc["yhat"] = sc["yhat"].copy()
    sc["yhat"][17, :] = math.nan
    gs, res = run_gpu(sc)
    assert res["n_committed"] == 17
    with pytest.raises(ValueError):
        gs.check_errors()


def test_two_batches_continue_state():
    """Splitting a batch in two gives the same decisions (state carries over)."""
    sc = H.load_schedule("k8_mixed")
    gs, rt, pr = make_scheduler(sc)
    dev = gs.device
    n = len(sc["prog"])
    cut = n // 3
    outs = []
    for lo, hi in ((0, cut), (cut, n)):
        rt.set(torch.as_tensor(sc["q"][lo:hi], device=dev))
        pr.set(torch.as_tensor(sc["yhat"][lo:hi], device=dev))
        b = RowBatch.from_numpy(dev, program=sc["prog"][lo:hi], stage=sc["stage"][lo:hi],
                                arrival=sc["arrival"][lo:hi], out_tokens=sc["out_tok"][lo:hi],
                                handle=np.arange(lo, hi))
        gs.run_rows(b, n_iterations=0)
        outs.append(gs.buf.model[:hi - lo].cpu().numpy().copy())
    np.testing.assert_array_equal(np.concatenate(outs), sc["out_model"])
    assert np.array(gs.state.in_flight_sums()).tobytes() == sc["out_final_p"].tobytes()
