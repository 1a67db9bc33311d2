"""GPU parity for the engine execution clock: golden
EngineSim scripts (enqueue with input / output tokens, scheduling
iterations, advance_to), written by the unmodified reference with prefill and
decode times, replayed through GpuScheduler(engine_clock=True). Completions
and their finish times, the admission order, the running set's stint ends,
the final queue and the engine counters must be bit-exact."""

import math

import numpy as np
import pytest
import torch

from paper_2603_22206_b200.config import AgingConfig, BalancerConfig, ModelProfile, Pool
from paper_2603_22206_b200.predictor import PrecomputedPredictor
from paper_2603_22206_b200.router import ScoreTableRouter
from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch
from tests import harness as H

pytestmark = pytest.mark.gpu


def replay_engine(ed, capacity=10240):
    S = ed["S"] if ed["S"] else math.inf
    pool = Pool((ModelProfile("m0", ed["d"], ed["b"], prefill_ms_per_token=ed["p"]),))
    rt, pr = ScoreTableRouter(), PrecomputedPredictor()
    enq = ed["enq"]
    gs = GpuScheduler(pool, BalancerConfig(), AgingConfig(starvation_threshold=S), router=rt,
                      predictor=pr, n_programs=len(enq) + 1, max_rows=max(len(enq), 1),
                      queue_capacity=capacity, engine_clock=True)
    dev = gs.device
    admitted, done = [], []
    pos = 0

    def rows(n):
        nonlocal pos
        o = enq[pos:pos + n]
        pos += n
        rt.set(torch.full((n, 1), 0.5, dtype=torch.float32, device=dev))
        pr.set(torch.as_tensor(o[:, 1] if n else np.zeros(0), device=dev).reshape(-1, 1))
        return o, RowBatch.from_numpy(dev, program=o[:, 0].astype(np.int32), stage=np.ones(n),
                                      arrival=o[:, 2], out_tokens=o[:, 4:5].astype(np.int32),
                                      handle=o[:, 0].astype(np.int64),
                                      input_tokens=o[:, 3].astype(np.int32))

    def tick(n_rows=0, n_iter=0):
        o, b = rows(n_rows)
        gs.run_rows(b, n_iterations=n_iter)
        gs.check_errors()
        fl = gs.buf.dflags[:n_rows].cpu().numpy()
        admitted.extend(int(x) for x in o[(fl & 2) != 0, 0])
        admitted.extend(int(x) for x in gs.state.admitted(0))

    t = 0.0
    tick(n_rows=ed["n_pre"])
    for step in ed["script"]:
        if step[0] == "enq":
            t += step[2]
            tick(n_rows=step[1])
        elif step[0] == "iter":
            tick(n_iter=step[1])
        else:
            t += step[1]
            gs.advance_to(t)
            gs.check_errors()
            h, tm = gs.state.completions(0)
            done.extend(zip(h.tolist(), tm.tolist()))
            admitted.extend(int(x) for x in gs.state.admitted(0))
    st = gs.state
    nq = int(st.engine_queued[0])
    order_idx = st.q_order[:nq].long()
    return dict(
        admitted=np.array(admitted),
        done=np.array(done, dtype=np.float64).reshape(-1, 2),
        order=st.q_handle[:nq][order_idx].cpu().numpy(),
        level=st.q_level[:nq][order_idx].cpu().numpy(),
        count=st.q_count[:nq][order_idx].cpu().numpy(),
        running=np.array(st.running_set(0), dtype=np.float64).reshape(-1, 3),
        now=float(st.engine_clock[0]),
        tokens=int(st.tokens_emitted[0]),
        served=int(st.served[0]),
        iterations=int(st.engine_iterations[0]),
        n_running=int(st.engine_running[0]),
    )


@pytest.mark.parametrize("capacity", [10240, 20480])  # smem / global-memory keys
@pytest.mark.parametrize("name", H.engine_names())
def test_engine_clock_matches_reference(name, capacity):
    ed = H.load_engine(name)
    res = replay_engine(ed, capacity)
    np.testing.assert_array_equal(res["admitted"], ed["admitted"])
    # completions: same requests, same finish times (float64 bit patterns)
    assert res["done"].shape == ed["done"].shape
    assert res["done"].tobytes() == ed["done"].tobytes()
    np.testing.assert_array_equal(res["order"], ed["order"])
    np.testing.assert_array_equal(res["level"], ed["level"])
    np.testing.assert_array_equal(res["count"], ed["count"])
    assert res["running"].tobytes() == ed["running"].tobytes()
    assert res["n_running"] == len(ed["running"])
    assert res["now"] == ed["now"]
    assert res["tokens"] == ed["tokens"]
    assert res["served"] == ed["served"]
    assert res["iterations"] == ed["iterations"]


def test_advance_backwards_raises():
    """advance_to a target before the clock: ValueError (engine.py:140-143)."""
    ed = H.load_engine("e_basic")
    pool = Pool((ModelProfile("m0", ed["d"], ed["b"], prefill_ms_per_token=ed["p"]),))
    gs = GpuScheduler(pool, router=ScoreTableRouter(), predictor=PrecomputedPredictor(),
                      n_programs=8, max_rows=4, engine_clock=True)
    gs.advance_to(10.0)
    gs.check_errors()
    gs.advance_to(5.0)
    with pytest.raises(ValueError):
        gs.check_errors()
