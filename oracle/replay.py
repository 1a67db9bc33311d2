"""Replay a synthetic workload's tick on the oracle port -- TEST INFRASTRUCTURE.

Used by tests/test_gpu_tick.py (full-tick parity) and by bench.py's
cpu_baseline leg (tie-band replay). Duck-typed on the workload object
(`pool`, `seed_state(state)`, `completions()`, `training`, `balancer`,
`predictor.workflow_index`) and on the batch (torch or numpy columns); it
imports nothing from the product package.

  port_state(wl)                  PortMonitor + PortEngines holding the
                                  workload's pre-tick state (cfg4: 64k in
                                  flight, 64k queued, engines full) with the
                                  tick's completions applied
  replay_batch(wl, batch, q, ...) schedule_request (balancer.py:89-129) over
                                  the batch rows with router scores q
  router_fp32(wl, token_ids, n)   the fp32 encoder restatement's scores
"""

from __future__ import annotations

import heapq

import numpy as np

from . import hetsched_port as hp


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


class _Recorder:
    """Captures Workload.seed_state's calls so the port sees the same state."""

    def __init__(self):
        self.inflight, self.queues, self.counters = None, {}, None

    def seed_inflight(self, per_model):
        self.inflight = per_model

    def load_queue(self, m, prio, arr, seq, handle, out_tokens=None, count=None):
        self.queues[m] = (prio, arr, seq, handle, out_tokens, count)

    def set_engine_counters(self, **kw):
        self.counters = kw


def port_state(wl):
    ids = wl.pool.model_ids
    mon = hp.PortMonitor(ids)
    engines = {m: hp.PortEngine(wl.pool[m].max_batch_size,
                                starvation_threshold=wl.aging.starvation_threshold,
                                running_quantum=wl.aging.running_quantum) for m in ids}
    rec = _Recorder()
    wl.seed_state(rec)
    if rec.inflight is None:
        return mon, engines
    for m, vals in rec.inflight.items():
        for j, v in enumerate(vals):  # seeded entry j+1 has log key -(j+1)
            mon.record_dispatch(m, f"seed:{m}:{j + 1}", float(v))
    for k, m in enumerate(ids):
        prio, arr, seq, handle, out_tok, count = rec.queues[k]
        e = engines[m]
        for j in range(len(prio)):
            ent = hp.PortEntry(int(handle[j]), float(prio[j]), float(arr[j]), int(seq[j]),
                               int(out_tok[j]), count=int(count[j]))
            e.queued[ent.seq] = ent
            e.heap.append((ent.key(), ent.seq))
        heapq.heapify(e.heap)
        e.next_seq = int(rec.counters["seq"][k])
        e.now = float(rec.counters["clock"][k])
        for j in range(int(rec.counters["running"][k])):
            e.running[-1 - j] = hp.PortEntry(("run", j), 0.0, 0.0, -1 - j, 0)
    comp = wl.completions()
    if comp is not None:
        c_model, c_key = (_np(t) for t in comp)
        n_done = {m: 0 for m in ids}
        for k, key in zip(c_model.tolist(), c_key.tolist()):
            m = ids[k]
            mon.record_completion(m, f"seed:{m}:{-key}")
            n_done[m] += 1
        for m in ids:  # each completion frees a slot and runs one iteration
            engines[m].complete(n_done[m], engines[m].now)
    return mon, engines


def replay_batch(wl, batch, q, mon, engines):
    """Returns (model index, priority, estimated loads [B, K]) per row."""
    ids = wl.pool.model_ids
    port_pred = hp.PortQuantilePredictor(wl.training, 0.5)
    prog = _np(batch.program)
    stage = _np(batch.stage)
    arr = _np(batch.arrival)
    wf_idx = _np(batch.workflow)
    handle = _np(batch.handle)
    inv_wf = {v: k for k, v in wl.predictor.workflow_index.items()}
    out_tok = _np(batch.out_tokens)

    class _Req:
        __slots__ = ("program_id", "stage_index", "arrival_time", "workflow_id", "request_id")

    class _Rec:
        def __init__(self, row):
            self.row = row

        def out_tokens(self, stage, m):
            return int(out_tok[self.row, ids.index(m)])

    n = len(prog)
    models = np.empty(n, np.int32)
    prios = np.empty(n)
    loads = np.zeros((n, len(ids)))
    for i in range(n):
        r = _Req()
        r.program_id = f"p{int(prog[i])}"
        r.stage_index = int(stage[i])
        r.arrival_time = float(arr[i])
        r.workflow_id = inv_wf.get(int(wf_idx[i]), "?")
        r.request_id = int(handle[i])
        d = hp.port_schedule_request(
            r, _Rec(i), wl.pool, mon, engines,
            lambda rq, rc, i=i: {m: float(q[i, k]) for k, m in enumerate(ids)},
            port_pred, wl.balancer.latency_slack, wl.balancer.confidence_margin)
        models[i] = ids.index(d.model)
        prios[i] = d.priority
        if d.estimated_loads:
            loads[i] = [d.estimated_loads[m] for m in ids]
    return models, prios, loads


def router_fp32(wl, token_ids, n_rows=None, chunk=256):
    """Scores of the fp32 encoder restatement for the first n_rows sequences
    (same weights as the device router), fp64 numpy [n, K]."""
    from .encoder_ref import encoder_forward_fp32
    r = wl.router
    n_rows = token_ids.shape[0] if n_rows is None else n_rows
    out = []
    for a in range(0, n_rows, chunk):
        out.append(encoder_forward_fp32(r.weights, token_ids[a:min(n_rows, a + chunk)],
                                        r.cfg.n_layers, r.cfg.n_heads, r.cfg.ln_eps)
                   .cpu().numpy())
    return np.concatenate(out).astype(np.float64)
