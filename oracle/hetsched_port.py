"""Pure-Python restatement of the reference scheduling path -- TEST INFRASTRUCTURE.

This is the oracle the GPU path is checked against and the CPU arm bench.py
times. It restates, with the same algorithm and the same cost structure, the
reference functions under /root/reference/pkg/src/hetsched:

  PortMonitor            monitor.py:40-140  (assignment map, in-flight map,
                                             P_m = sum(values) re-summed on
                                             every read, monitor.py:122-129)
  port_estimate_load     balancer.py:49-60
  port_select_model      balancer.py:63-77
  port_schedule_request  balancer.py:89-129 (Algorithm 1)
  PortEngine             engine.py:55-69, 108-143, 265-394 (EngineSim queue:
                                             lazy-deletion heap keyed by
                                             (level, priority, arrival, seq),
                                             _iterate, _age_queued,
                                             _tick_running_quantum)
  PortQuantilePredictor  predictor.py:65-108 (np.quantile 'linear' tables with
                                             the (wf,stage,m)->(stage,m)->(m)
                                             ->global fallback chain)
  port_oracle_predict    predictor.py:30-36
  port_input_length      predictor.py:39-45

Inputs are duck-typed: any objects with the reference's attribute names
(Request.program_id/stage_index/input_tokens/arrival_time/workflow_id,
TraceRecord.stages/remaining_tokens/out_tokens, Pool.model_ids/__getitem__).
Nothing here imports the product package.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field

import numpy as np


class PortError(Exception):
    """Raised with `.kind` naming the hetsched exception the reference raises."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# activity monitor (monitor.py:40-140)
# --------------------------------------------------------------------------
class PortMonitor:
    def __init__(self, model_ids, decay_in_flight: bool = False):  # monitor.py:40-48
        self.live: dict[str, dict[str, float]] = {m: {} for m in sorted(model_ids)}
        self.progress: dict[str, dict[str, float]] = {m: {} for m in self.live}
        self.owner: dict[str, str] = {}
        self.assignments: dict[str, str] = {}
        self.decay_in_flight = decay_in_flight

    def assignment(self, program_id):
        return self.assignments.get(program_id)

    def assign(self, program_id, model_id):  # monitor.py:55-63
        prev = self.assignments.get(program_id)
        if prev is not None and prev != model_id:
            raise PortError("AssignmentConflict", f"{program_id}: {prev} -> {model_id}")
        self.assignments[program_id] = model_id

    def record_dispatch(self, model_id, request_id, predicted):  # monitor.py:86-96
        if model_id not in self.live:
            raise PortError("UnknownModel", model_id)
        if predicted < 0:
            raise PortError("ValueError", f"predicted_tokens must be >= 0, got {predicted}")
        if request_id in self.owner:
            raise PortError("DuplicateRequest", request_id)
        self.live[model_id][request_id] = predicted
        self.owner[request_id] = model_id

    def record_completion(self, model_id, request_id):  # monitor.py:98-106
        if model_id not in self.live:
            raise PortError("UnknownModel", model_id)
        if self.live[model_id].pop(request_id, None) is None:
            raise PortError("UnknownRequest", request_id)
        del self.owner[request_id]
        self.progress[model_id].pop(request_id, None)

    def note_progress(self, model_id, request_id, emitted):  # monitor.py:108-111
        if request_id in self.live.get(model_id, {}):
            self.progress[model_id][request_id] = emitted

    def in_flight_sum(self, model_id):  # monitor.py:122-129
        # builtin sum(): Neumaier-compensated on CPython >= 3.12, re-evaluated
        # over every live entry on every call -- the reference's cost.
        if not self.decay_in_flight:
            return sum(self.live[model_id].values())
        prog = self.progress[model_id]
        return sum(max(y - prog.get(rid, 0.0), 0.0) for rid, y in self.live[model_id].items())


# --------------------------------------------------------------------------
# load estimate + selection + Algorithm 1 (balancer.py:49-129)
# --------------------------------------------------------------------------
def port_estimate_load(pool, monitor) -> dict:
    out = {}
    for mid in pool.model_ids:
        prof = pool[mid]
        out[mid] = monitor.in_flight_sum(mid) * prof.decode_ms_per_token / prof.max_batch_size
    return out


def port_select_model(scores: dict, loads: dict, latency_slack: float,
                      confidence_margin: float) -> str:
    if set(scores) != set(loads):
        raise PortError("ValidationError", "scores and loads must cover the same model set")
    fastest = min(loads, key=lambda mid: (loads[mid], mid))
    ceiling = (1.0 + latency_slack) * loads[fastest]
    need = scores[fastest]
    for mid in sorted(loads, key=lambda x: (-scores[x], x)):
        if loads[mid] <= ceiling and scores[mid] >= need + confidence_margin:
            return mid
    return fastest


def port_tie_band(scores: dict, loads: dict, chosen: str, latency_slack: float,
                  confidence_margin: float, tol: float = 2e-2) -> tuple[bool, bool]:
    """Tie band of one routed decision (north star: "ties inside the tolerance
    band are reported"; the reference has no such report, this is the
    definition the device flags are checked against). Inside the latency
    slack of m_fast (balancer.py:71-72):
      gate  some model m != m_fast has |q_m - (q_fast + margin)| <= tol, so a
            router error of tol could flip its confidence gate (balancer.py:75)
      rank  the chosen candidate and another candidate have q within tol, so
            the descending-q order (balancer.py:73) could flip between them
    Returns (rank, gate)."""
    fastest = min(loads, key=lambda mid: (loads[mid], mid))
    ceiling = (1.0 + latency_slack) * loads[fastest]
    need = scores[fastest] + confidence_margin
    ok = [m for m in loads if loads[m] <= ceiling]
    gate = any(m != fastest and abs(scores[m] - need) <= tol for m in ok)
    cand = [m for m in ok if scores[m] >= need]
    rank = bool(cand) and any(m != chosen and scores[chosen] - scores[m] <= tol for m in cand)
    return rank, gate


@dataclass
class PortDecision:
    model: str
    priority: float
    estimated_loads: dict
    used_cached_assignment: bool
    scores: dict | None


def port_schedule_request(req, rec, pool, monitor, engines, score_fn, predict_fn,
                          latency_slack: float, confidence_margin: float) -> PortDecision:
    """One call of schedule_request. score_fn(req, rec) -> {model: q};
    predict_fn(req, rec, model) -> float; engines[model].enqueue(...)."""
    prior = monitor.assignment(req.program_id)
    if prior is None:
        loads = port_estimate_load(pool, monitor)
        q = score_fn(req, rec)
        for mid, v in q.items():  # ConfidenceVector.__post_init__ (router.py:24-28)
            if not 0.0 <= v <= 1.0:
                raise PortError("ValidationError", f"score for {mid!r} outside [0,1]: {v}")
        model = port_select_model(q, loads, latency_slack, confidence_margin)
        monitor.assign(req.program_id, model)
    else:
        model, loads, q = prior, {}, None
    yhat = predict_fn(req, rec, model)
    monitor.record_dispatch(model, req.request_id, yhat)
    engines[model].enqueue(req.request_id, yhat, rec.out_tokens(req.stage_index, model),
                           req.arrival_time)
    return PortDecision(model, yhat, loads, prior is not None, q)


# --------------------------------------------------------------------------
# STJF + aging engine queue (engine.py:36-69, 108-158, 265-394)
# --------------------------------------------------------------------------
@dataclass
class PortEntry:
    rid: object
    priority: float
    arrival: float
    seq: int
    out_tokens: int
    count: int = 0
    level: int = 0
    quantum: int = 0

    def key(self):
        return (self.level, self.priority, self.arrival, self.seq)


class PortEngine:
    def __init__(self, max_batch_size: int, starvation_threshold=8, running_quantum=4,
                 demote_while_queued=False):
        self.b = max_batch_size
        self.S = starvation_threshold
        self.Q = running_quantum
        self.demote_while_queued = demote_while_queued
        self.now = 0.0
        self.next_seq = 0
        self.heap: list = []
        self.queued: dict[int, PortEntry] = {}
        self.running: dict[int, PortEntry] = {}
        self.iterations = 0
        self.admitted_log: list = []
        self.promotions = 0

    @property
    def waiting_count(self):
        return len(self.queued)

    @property
    def running_count(self):
        return len(self.running)

    def _clock(self, now):  # engine.py:140-143
        if now < self.now - 1e-9:
            raise PortError("ValueError", f"time going backwards ({now} < {self.now})")
        self.now = max(self.now, now)

    def enqueue(self, rid, priority, out_tokens, now):  # engine.py:145-158
        self._clock(now)
        if out_tokens < 0:
            raise PortError("ValidationError", f"out_tokens must be >= 0, got {out_tokens}")
        e = PortEntry(rid, priority, now, self.next_seq, out_tokens)
        self.next_seq += 1
        self.queued[e.seq] = e
        heapq.heappush(self.heap, (e.key(), e.seq))
        if len(self.running) < self.b:
            self._iterate(now)

    def scheduling_iteration(self, now):  # engine.py:160-163
        self._clock(now)
        return self._iterate(now)

    def complete(self, n: int, now: float):
        """n running requests finish at `now`; each completion runs one
        iteration (engine.py:232-241). The earliest-admitted ones finish."""
        self._clock(now)
        out = []
        for _ in range(n):
            if not self.running:
                break
            del self.running[min(self.running)]
            out += self._iterate(now)
        return out

    def _pop(self):  # engine.py:314-326
        while self.heap:
            key, seq = self.heap[0]
            e = self.queued.get(seq)
            heapq.heappop(self.heap)
            if e is None or e.key() != key:
                continue
            del self.queued[seq]
            return e
        return None

    def _iterate(self, now):  # engine.py:328-338
        self.iterations += 1
        got = []
        while len(self.running) < self.b:
            e = self._pop()
            if e is None:
                break
            self.running[e.seq] = e
            got.append(e.rid)
        self.admitted_log += got
        self._age()
        self._tick_running()
        return got

    def _age(self):  # engine.py:340-374
        if self.S == math.inf or not self.queued:
            return
        for seq in sorted(self.queued):
            e = self.queued[seq]
            e.count += 1
            if e.count >= self.S:
                e.count = 0
                e.level -= 1
                e.quantum = 0
                self.promotions += 1
                heapq.heappush(self.heap, (e.key(), e.seq))
            elif self.demote_while_queued and e.level < 0:
                e.quantum += 1
                if e.quantum >= self.Q:
                    e.quantum = 0
                    e.level += 1
                    heapq.heappush(self.heap, (e.key(), e.seq))

    def _tick_running(self):  # engine.py:376-394
        if self.S == math.inf:
            return
        for seq in sorted(self.running):
            e = self.running[seq]
            if e.level < 0:
                e.quantum += 1
                if e.quantum >= self.Q:
                    e.quantum = 0
                    e.level += 1

    def queue_order(self):
        """Queued entries in pop order (ascending sort_key)."""
        return sorted(self.queued.values(), key=PortEntry.key)


# --------------------------------------------------------------------------
# predictors (predictor.py:30-108)
# --------------------------------------------------------------------------
def port_oracle_predict(req, rec, model_id) -> float:
    return float(rec.remaining_tokens(req.stage_index, model_id))


def port_input_length(req, rec, model_id) -> float:
    return float(req.input_tokens)


class PortQuantilePredictor:
    def __init__(self, training, quantile: float = 0.5):
        if not 0.0 < quantile < 1.0:
            raise PortError("ValidationError", f"quantile must be in (0,1), got {quantile}")
        buckets: dict = {"k": {}, "sm": {}, "m": {}, "all": []}
        for rec in training:
            for st in rec.stages:
                for mid in sorted(st.models):
                    y = float(rec.remaining_tokens(st.stage_index, mid))
                    buckets["k"].setdefault((rec.workflow_id, st.stage_index, mid), []).append(y)
                    buckets["sm"].setdefault((st.stage_index, mid), []).append(y)
                    buckets["m"].setdefault(mid, []).append(y)
                    buckets["all"].append(y)
        if not buckets["all"]:
            raise PortError("EmptyTrainingSet", "no training values")
        qf = lambda v: float(np.quantile(v, quantile))  # noqa: E731
        self.by_key = {k: qf(v) for k, v in buckets["k"].items()}
        self.by_stage_model = {k: qf(v) for k, v in buckets["sm"].items()}
        self.by_model = {k: qf(v) for k, v in buckets["m"].items()}
        self.global_q = qf(buckets["all"])

    def lookup(self, workflow_id, stage_index, model_id) -> float:
        v = self.by_key.get((workflow_id, stage_index, model_id))
        if v is not None:
            return v
        v = self.by_stage_model.get((stage_index, model_id))
        if v is not None:
            return v
        v = self.by_model.get(model_id)
        return self.global_q if v is None else v

    def __call__(self, req, rec, model_id) -> float:
        return self.lookup(req.workflow_id, req.stage_index, model_id)


# --------------------------------------------------------------------------
# one scheduling tick (B decisions in arrival order + one iteration per engine)
# --------------------------------------------------------------------------
def port_tick(reqs, recs, pool, monitor, engines, score_fn, predict_fn, latency_slack,
              confidence_margin, n_iterations: int = 1, now: float | None = None):
    decisions = [
        port_schedule_request(r, rec, pool, monitor, engines, score_fn, predict_fn,
                              latency_slack, confidence_margin)
        for r, rec in zip(reqs, recs)
    ]
    t = now if now is not None else (reqs[-1].arrival_time if reqs else 0.0)
    for _ in range(n_iterations):
        for mid in pool.model_ids:
            engines[mid].scheduling_iteration(max(t, engines[mid].now))
    return decisions
