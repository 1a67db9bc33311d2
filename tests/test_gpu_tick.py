"""Full-size tick parity on BASELINE.json's configurations: one scheduling
tick of the synthetic workload through the GPU path (router on device, K5,
K6, K7) against the oracle port fed the GPU's own router output -- every
decision, priority, in-flight sum, engine counter and final STJF queue order
bit-exact -- plus the router against the fp32 restatement on a row sample."""

import numpy as np
import pytest
import torch

from oracle import hetsched_port as hp
from oracle.encoder_ref import encoder_forward_fp32
from paper_2603_22206_b200 import synth
from paper_2603_22206_b200.scheduler import GpuScheduler

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3"])
def test_full_tick_matches_oracle(name):
    wl = synth.make_workload(name)
    gs = GpuScheduler(wl.pool, wl.balancer, wl.aging, router=wl.router, predictor=wl.predictor,
                      n_programs=wl.n_programs, max_rows=wl.batch_size,
                      queue_capacity=wl.queue_capacity)
    batch = wl.batch(0)
    gs.run_rows(batch, n_iterations=1)
    torch.cuda.synchronize()
    gs.check_errors(name)
    B, K = batch.n_rows, gs.K
    q = gs.buf.scores[:B * K].view(B, K).cpu().numpy()
    # router vs the fp32 restatement on a sample of rows (north-star 1e-2)
    r = wl.router
    n_s = 64
    want_q = encoder_forward_fp32(r.weights, batch.token_ids[:n_s], r.cfg.n_layers,
                                  r.cfg.n_heads, r.cfg.ln_eps).cpu().numpy()
    assert np.abs(q[:n_s] - want_q).max() <= 1e-2
    # everything downstream of the router: bit-exact against the port
    want = synth.oracle_tick(wl, batch, q, hp)
    np.testing.assert_array_equal(gs.buf.model[:B].cpu().numpy(), want["model"])
    assert gs.buf.priority[:B].cpu().numpy().tobytes() == want["priority"].tobytes()
    ids = wl.pool.model_ids
    mon, engines = want["monitor"], want["engines"]
    want_p = np.array([mon.in_flight_sum(m) for m in ids])
    assert np.array(gs.state.in_flight_sums()).tobytes() == want_p.tobytes()
    t_end = float(batch.arrival.max().item())
    for m in ids:  # the tick's explicit scheduling iteration
        engines[m].scheduling_iteration(max(t_end, engines[m].now))
    st = gs.state
    prog = batch.program.cpu().numpy()
    row_of = {f"p{int(p)}:1": i for i, p in enumerate(prog)}
    for k, m in enumerate(ids):
        e = engines[m]
        assert int(st.engine_running[k]) == e.running_count
        assert int(st.engine_queued[k]) == e.waiting_count
        port_order = [row_of[x.rid] for x in sorted(e.queued.values(), key=lambda x: x.key())]
        np.testing.assert_array_equal(st.queue_order(k), np.array(port_order, dtype=np.int64))
