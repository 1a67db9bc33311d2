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
from oracle import hetsched_port as hp
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
    # tie band (flag bits 3 / 4) against the oracle's definition on the same keys
    ids = sc["ids"]
    want_rank = np.zeros(n, np.uint8)
    want_gate = np.zeros(n, np.uint8)
    for i in np.nonzero(routed)[0]:
        q = {m: float(sc["q"][i, k]) for k, m in enumerate(ids)}
        loads = {m: float(sc["out_loads"][i, k]) for k, m in enumerate(ids)}
        rk, gt = hp.port_tie_band(q, loads, ids[sc["out_model"][i]], sc["tau"], sc["margin"],
                                  gs.tie_tolerance)
        want_rank[i], want_gate[i] = rk, gt
    np.testing.assert_array_equal((res["flags"][:n] >> 3) & 1, want_rank)
    np.testing.assert_array_equal((res["flags"][:n] >> 4) & 1, want_gate)
    tb = gs.tie_band()
    assert (tb["rank"], tb["gate"], tb["any"]) == (
        int(want_rank.sum()), int(want_gate.sum()), int((want_rank | want_gate).sum()))


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
            assert d.scores == {m: float(sc["q"][i, k]) for k, m in enumerate(sc["ids"])}


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


@pytest.mark.parametrize("exact_chain", [False, True])
def test_select_kat_through_k6(exact_chain):
    """Every select_model case of tests/golden/select_kat.npz (5,006: SPEC
    examples, AC2 random instances with ties, tau in {0, 1e6}, margin in
    {0, 1}, decimal table scores) as a one-row batch through K6: loads are
    installed as in-flight sums with d = b = 1 (L = P exactly). exact_chain
    adds a repeat row so the batch takes K6's exact (erroring) chain instead
    of the fast one. balancer.py:63-77."""
    import os
    z = np.load(os.path.join(H.GOLDEN, "select_kat.npz"))
    from paper_2603_22206_b200.config import ModelProfile, Pool
    n_cases = len(z["k"])
    by_k = {}
    for k in range(1, 9):
        pool = Pool(tuple(ModelProfile(f"m{i}", 1.0, 1) for i in range(k)))
        rt, pr = ScoreTableRouter(), PrecomputedPredictor()
        gs = GpuScheduler(pool, BalancerConfig(0.5, 0.1), AgingConfig(), router=rt, predictor=pr,
                          n_programs=2 * n_cases + 2, max_rows=2, queue_capacity=16)
        by_k[k] = (gs, rt, pr)
    dev = torch.device("cuda")
    got = np.full(n_cases, -1, np.int32)
    for i in range(n_cases):
        k = int(z["k"][i])
        gs, rt, pr = by_k[k]
        st = gs.state
        tau, dm = (float(x) for x in z["cfg"][i])
        gs.bal_c.latency_slack, gs.bal_c.confidence_margin = tau, dm
        st.inflight_sum.copy_(torch.as_tensor(z["loads"][i, :k]))
        st.inflight_comp.zero_()
        st.engine_running.zero_()
        st.engine_queued.zero_()
        rows = 2 if exact_chain else 1
        rt.set(torch.as_tensor(np.repeat(z["q"][i:i + 1, :k], rows, 0), device=dev))
        pr.set(torch.zeros((rows, k), dtype=torch.float64, device=dev))
        batch = RowBatch.from_numpy(dev, program=[2 * i] * rows, stage=list(range(1, rows + 1)),
                                    arrival=[0.0] * rows, out_tokens=np.zeros((rows, k)),
                                    handle=np.arange(rows))
        gs.run_rows(batch, n_iterations=0)
        got[i] = int(gs.buf.model[0].item())
        assert int(gs.buf.n_committed.item()) == rows
    np.testing.assert_array_equal(got, z["chosen"])


def test_schedule_batch_with_encoder_router():
    """The drop-in as INTEGRATION.md binds it: reference-style Request /
    TraceRecord objects, the sm_100a encoder as the Router (token ids from a
    caller-supplied source, ragged lengths packed to S), the Predictor
    shim -> schedule_batch -> Decisions equal to the oracle port's serial
    schedule_request loop fed the same router scores (balancer.py:89-129,
    router.py:34-45). Router.score(req, rec, pool) on one request returns
    the same ConfidenceVector as the batched forward."""
    from oracle import hetsched_port as hp
    from paper_2603_22206_b200.encoder import SMALL, GpuEncoderRouter
    from paper_2603_22206_b200.router import ConfidenceVector

    sc = H.load_schedule("k5_nondyadic_p0")
    n = len(sc["prog"])
    rng = np.random.default_rng(11)
    toks = {}
    for p in set(int(x) for x in sc["prog"]):
        ln = int(rng.integers(16, 129))
        toks[f"p{p:06d}"] = [101] + rng.integers(1000, 30522, ln - 1).tolist()
    router = GpuEncoderRouter(SMALL, sc["k"], max_rows=n, seed=3, head_std=0.2,
                              tokens=lambda req, rec: toks[req.program_id])
    gs, rt, pr = make_scheduler(sc)
    gs.router = router
    pr.set(torch.as_tensor(sc["yhat"], device=gs.device))
    for p in range(sc["n_prog"]):
        gs.program_index(f"p{p:06d}")
    reqs, recs = H.requests_of(sc)
    decs = gs.schedule_batch(reqs, recs)
    assert len(decs) == n
    pool = H.pool_of(sc)
    ids = sc["ids"]
    q_batch = gs.buf.scores[:n * sc["k"]].view(n, sc["k"]).cpu().numpy()
    # the port replays the serial loop with the scores the device computed
    mon = hp.PortMonitor(ids)
    for j, (m, v) in enumerate(sc["p0"]):
        mon.record_dispatch(ids[int(m)], f"seed:{j}", float(v))
    for p, m in sc["pre"]:
        mon.assign(f"p{int(p):06d}", ids[int(m)])
    engines = {mid: hp.PortEngine(pool[mid].max_batch_size) for mid in ids}
    for i, (r, rec) in enumerate(zip(reqs, recs)):
        d = hp.port_schedule_request(r, rec, pool, mon, engines,
                                     lambda rq, rc, i=i: {m: float(q_batch[i, k])
                                                          for k, m in enumerate(ids)},
                                     lambda rq, rc, m, i=i: float(sc["yhat"][i, ids.index(m)]),
                                     sc["tau"], sc["margin"])
        assert decs[i].model == d.model, i
        assert decs[i].priority == d.priority
        assert decs[i].used_cached_assignment == d.used_cached_assignment
        if not d.used_cached_assignment:
            assert decs[i].estimated_loads == d.estimated_loads
            assert decs[i].scores == d.scores
    # Router.score on single requests: same encoder, same scores
    routed = [i for i, d in enumerate(decs) if not d.used_cached_assignment][:8]
    for i in routed:
        cv = router.score(reqs[i], recs[i], pool)
        assert isinstance(cv, ConfidenceVector)
        got = np.array([cv[m] for m in ids])
        assert np.abs(got - q_batch[i]).max() <= 1e-6, (i, got, q_batch[i])
