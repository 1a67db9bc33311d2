"""Full-size tick parity on BASELINE.json's configurations: one scheduling
tick of the synthetic workload through the GPU path (router on device, K5,
K6, K7) against the oracle port fed the GPU's own router output -- every
decision, priority, in-flight sum, engine counter, final STJF queue order,
level and count bit-exact -- plus the router against the fp32 restatement
(every row at S = 128, 512 rows at S = 512) with the achieved max |dq|
recorded, and the tie-band report checked against a replay of the selection
with the fp32 restatement's scores.

CHM_PARITY_LOG=<path> appends one JSON line per config (max |dq|, tie band,
flips) -- profiles/r2_parity.jsonl holds the GPU box's."""

import json
import os

import numpy as np
import pytest
import torch

from oracle import hetsched_port as hp
from oracle.replay import port_state as _port_state
from oracle.replay import replay_batch as _replay
from oracle.replay import router_fp32
from workloads import synth
from paper_2603_22206_b200.scheduler import GpuScheduler

pytestmark = pytest.mark.gpu


def _record(entry):
    path = os.environ.get("CHM_PARITY_LOG")
    print(json.dumps(entry))
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(entry) + "\n")


# (config, router rows compared with the fp32 restatement, chunk)
CASES = [("cfg1", None, 1000), ("cfg2", None, 512), ("cfg3", None, 512), ("cfg4", None, 1024),
         ("cfg5", 512, 32)]


@pytest.mark.parametrize("name,n_ref,chunk", CASES, ids=[c[0] for c in CASES])
def test_full_tick_matches_oracle(name, n_ref, chunk):
    wl = synth.make_workload(name)
    gs = GpuScheduler(wl.pool, wl.balancer, wl.aging, router=wl.router, predictor=wl.predictor,
                      n_programs=wl.n_programs, max_rows=wl.batch_size,
                      queue_capacity=wl.queue_capacity)
    wl.seed_state(gs.state)
    batch = wl.batch(0)
    gs.run_rows(batch, n_iterations=1, completions=wl.completions())
    torch.cuda.synchronize()
    gs.check_errors(name)
    B, K = batch.n_rows, gs.K
    ids = wl.pool.model_ids
    q = gs.buf.scores[:B * K].view(B, K).cpu().numpy()
    # router vs the fp32 restatement (north star: <= 1e-2 absolute)
    n_ref = B if n_ref is None else n_ref
    q_ref = router_fp32(wl, batch.token_ids, n_ref, chunk)
    dq = np.abs(q[:n_ref] - q_ref)
    assert dq.max() <= 1e-2, dq.max()
    # everything downstream of the router: bit-exact against the port
    mon, engines = _port_state(wl)
    want_m, want_p, want_l = _replay(wl, batch, q, mon, engines)
    got_m = gs.buf.model[:B].cpu().numpy()
    np.testing.assert_array_equal(got_m, want_m)
    assert gs.buf.priority[:B].cpu().numpy().tobytes() == want_p.tobytes()
    assert gs.buf.loads[:B * K].view(B, K).cpu().numpy().tobytes() == want_l.tobytes()
    want_p = np.array([mon.in_flight_sum(m) for m in ids])
    assert np.array(gs.state.in_flight_sums()).tobytes() == want_p.tobytes()
    np.testing.assert_array_equal(gs.state.inflight_count.cpu().numpy(),
                                  [len(mon.live[m]) for m in ids])
    t_end = float(batch.arrival.max().item())
    for m in ids:  # the tick's explicit scheduling iteration
        engines[m].scheduling_iteration(max(t_end, engines[m].now))
    st = gs.state
    for k, m in enumerate(ids):
        e = engines[m]
        assert int(st.engine_running[k]) == e.running_count
        assert int(st.engine_queued[k]) == e.waiting_count
        assert int(st.engine_seq[k]) == e.next_seq
        assert int(st.engine_iterations[k]) == e.iterations
        port_q = e.queue_order()
        np.testing.assert_array_equal(st.queue_order(k), [x.rid for x in port_q])
        n, b = int(st.engine_queued[k]), k * st.capacity
        order = st.q_order[b:b + n].long()
        np.testing.assert_array_equal(st.q_level[b:b + n][order].cpu().numpy(),
                                      [x.level for x in port_q])
        np.testing.assert_array_equal(st.q_count[b:b + n][order].cpu().numpy(),
                                      [x.count for x in port_q])
    # tie band: device flags == the definition on the same keys; and replaying
    # the selection with the fp32 restatement's scores, the first decision
    # that differs must be one the band flagged (|dq| <= 1e-2 on each score)
    fl = gs.buf.dflags[:B].cpu().numpy()
    routed = (fl & 1) == 0
    want_tb = np.zeros(B, np.uint8)
    for i in np.nonzero(routed)[0]:
        rk, gt = hp.port_tie_band({m: float(q[i, k]) for k, m in enumerate(ids)},
                                  {m: float(want_l[i, k]) for k, m in enumerate(ids)},
                                  ids[want_m[i]], wl.balancer.latency_slack,
                                  wl.balancer.confidence_margin, gs.tie_tolerance)
        want_tb[i] = (8 if rk else 0) | (16 if gt else 0)
    np.testing.assert_array_equal(fl & 24, want_tb)
    tb = gs.tie_band()
    entry = {"config": name, "rows": B, "router_rows_compared": n_ref,
             "router_max_abs_dq": float(dq.max()), "router_mean_abs_dq": float(dq.mean()),
             "tie_band": tb}
    # local flips: each routed row re-decided with the fp32 scores but the
    # loads the device saw (no cascade through the in-flight state); every one
    # must lie in the band
    local = 0
    for i in np.nonzero(routed[:n_ref])[0]:
        sq = {m: float(q_ref[i, k]) for k, m in enumerate(ids)}
        sl = {m: float(want_l[i, k]) for k, m in enumerate(ids)}
        if ids.index(hp.port_select_model(sq, sl, wl.balancer.latency_slack,
                                          wl.balancer.confidence_margin)) != got_m[i]:
            local += 1
            assert fl[i] & 24, f"row {i} flips with the fp32 scores outside the tie band"
    entry["fp32_local_flips"] = local
    if n_ref == B:
        mon2, eng2 = _port_state(wl)
        ref_m, _, _ = _replay(wl, batch, q_ref, mon2, eng2)
        diff = np.nonzero(ref_m != got_m)[0]
        entry["fp32_replay_flips"] = int(len(diff))
        entry["first_flip_row"] = int(diff[0]) if len(diff) else None
        if len(diff):
            assert fl[diff[0]] & 24, f"first flip at row {diff[0]} outside the tie band"
    _record(entry)
