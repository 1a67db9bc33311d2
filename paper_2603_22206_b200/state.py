"""Device-resident scheduler state: activity monitor, engine counters, queues.

Everything is a torch tensor on one CUDA device (PyTorch owns memory; the
kernels only see raw pointers). Layout in HBM:

  monitor   inflight_sum/comp f64[K]   Neumaier (s, c) of live predictions
            inflight_count    i64[K]
            assignment        i8[NP]   model index per program, -1 = none
            stage_bits        i32[NP]  bit (stage-1) while (program, stage) in flight
            batch_stamp       i64[NP]  per-batch repeat detection scratch
  engines   clock f64[K], seq i64[K], running i32[K], queued i32[K], iterations i64[K]
  queues    SoA segments of `capacity` entries per engine, kept in seq order:
            priority f64, arrival f64, seq i64, handle i64, out_tokens i32,
            level i32, count i32, quantum i32; order i32 (STJF order output)

NP (number of programs) bounds the dense program index space; at 1 byte of
assignment + 4 of stage bits + 8 of stamp per program, 10^8 programs take
1.3 GB of the 180 GB HBM.
"""

from __future__ import annotations

import ctypes

import math

import numpy as np
import torch

from . import _lib
from .config import AgingConfig, BalancerConfig, Pool


def neumaier_state(values) -> tuple[float, float]:
    """(s, c) after summing `values` in order the way CPython 3.12 sum() does."""
    s = 0.0
    c = 0.0
    for x in values:
        x = float(x)
        t = s + x
        if abs(s) >= abs(x):
            c += (s - t) + x
        else:
            c += (x - t) + s
        s = t
    return s, c


def neumaier_value(s: float, c: float) -> float:
    return s + c if (c and math.isfinite(c)) else s


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class DeviceState:
    """Monitor + engine + queue state for one pool on one device."""

    def __init__(self, pool: Pool, n_programs: int, queue_capacity: int = 10240,
                 device: str | torch.device = "cuda", inflight_capacity: int | None = None,
                 decay_in_flight: bool = False):
        self.pool = pool
        self.ids = pool.model_ids
        self.K = len(self.ids)
        if not 1 <= self.K <= _lib.MAX_MODELS:
            raise ValueError(f"pool size {self.K} outside 1..{_lib.MAX_MODELS}")
        self.n_programs = int(n_programs)
        self.capacity = int(queue_capacity)
        self.device = torch.device(device)
        d, K, NP, C = self.device, self.K, self.n_programs, self.capacity
        f64, i64, i32 = torch.float64, torch.int64, torch.int32
        # (s, c) of every engine in one buffer: the Mode B relay moves it as is
        self.inflight_sc = torch.zeros(2 * K, dtype=f64, device=d)
        self.inflight_sum = self.inflight_sc[:K]
        self.inflight_comp = self.inflight_sc[K:]
        self.inflight_count = torch.zeros(K, dtype=i64, device=d)
        self.assignment = torch.full((NP,), -1, dtype=torch.int8, device=d)
        self.stage_bits = torch.zeros(NP, dtype=i32, device=d)
        self.batch_stamp = torch.full((NP,), -1, dtype=i64, device=d)
        self.epoch = torch.zeros(1, dtype=i32, device=d)
        self.engine_clock = torch.zeros(K, dtype=f64, device=d)
        self.engine_seq = torch.zeros(K, dtype=i64, device=d)
        self.engine_running = torch.zeros(K, dtype=i32, device=d)
        self.engine_queued = torch.zeros(K, dtype=i32, device=d)
        self.engine_iterations = torch.zeros(K, dtype=i64, device=d)
        # live in-flight log (insertion order) for the completion path
        self.inflight_capacity = int(inflight_capacity if inflight_capacity is not None
                                     else min(max(NP, 65536), 1 << 22))
        self.inflight_key = torch.zeros(K * self.inflight_capacity, dtype=i64, device=d)
        self.inflight_yhat = torch.zeros(K * self.inflight_capacity, dtype=f64, device=d)
        # ActivityMonitor(decay_in_flight=True): emitted tokens per live entry
        self.decay_in_flight = bool(decay_in_flight)
        self.inflight_progress = (torch.zeros(K * self.inflight_capacity, dtype=f64, device=d)
                                  if self.decay_in_flight else None)
        # request-sharded runs: global insertion stamps of the live log
        # (enable_stamps(); dist.ShardedScheduler sets stamp_base every tick)
        self.inflight_stamp = None
        self.stamp_base = torch.zeros(1, dtype=i64, device=d)
        n = K * C
        self.q_priority = torch.zeros(n, dtype=f64, device=d)
        self.q_arrival = torch.zeros(n, dtype=f64, device=d)
        self.q_seq = torch.zeros(n, dtype=i64, device=d)
        self.q_handle = torch.zeros(n, dtype=i64, device=d)
        self.q_out_tokens = torch.zeros(n, dtype=i32, device=d)
        self.q_level = torch.zeros(n, dtype=i32, device=d)
        self.q_count = torch.zeros(n, dtype=i32, device=d)
        self.q_quantum = torch.zeros(n, dtype=i32, device=d)
        self.q_order = torch.zeros(n, dtype=i32, device=d)
        self.q_admitted = torch.zeros(n, dtype=i64, device=d)
        self.q_n_admitted = torch.zeros(K, dtype=i32, device=d)
        self.q_n_promoted = torch.zeros(K, dtype=i32, device=d)
        self.q_arrival_unsorted = torch.zeros(K, dtype=torch.uint8, device=d)
        self.q_scratch = None
        per_engine = int(_lib.load().chm_queue_scratch_bytes(C))
        if per_engine:
            self.q_scratch = torch.empty(K * per_engine, dtype=torch.uint8, device=d)
        self.pool_c = _lib.Pool()
        self.pool_c.n_models = K
        for i, mid in enumerate(self.ids):
            self.pool_c.max_batch_size[i] = pool[mid].max_batch_size
            self.pool_c.decode_ms_per_token[i] = pool[mid].decode_ms_per_token
        self.monitor_c = _lib.MonitorState(
            NP, _ptr(self.inflight_sum), _ptr(self.inflight_comp), _ptr(self.inflight_count),
            _ptr(self.assignment), _ptr(self.stage_bits), _ptr(self.batch_stamp),
            _ptr(self.engine_clock), _ptr(self.engine_seq), _ptr(self.engine_running),
            _ptr(self.engine_queued), _ptr(self.engine_iterations), self.inflight_capacity,
            _ptr(self.inflight_key), _ptr(self.inflight_yhat), _ptr(self.inflight_progress),
            None, _ptr(self.stamp_base))
        self.queue_c = _lib.QueueState(
            C, _ptr(self.q_priority), _ptr(self.q_arrival), _ptr(self.q_seq),
            _ptr(self.q_handle), _ptr(self.q_out_tokens), _ptr(self.q_level),
            _ptr(self.q_count), _ptr(self.q_quantum), _ptr(self.q_order),
            _ptr(self.q_admitted), _ptr(self.q_n_admitted), _ptr(self.q_n_promoted),
            _ptr(self.q_arrival_unsorted), _ptr(self.q_scratch))

    def enable_stamps(self) -> None:
        """Keep a global insertion stamp per live entry (request-sharded
        runs: the ranks' logs merge into one insertion order). Entries
        already in the log (seeded) get stamps before every tick's."""
        if self.inflight_stamp is not None:
            return
        K, cap = self.K, self.inflight_capacity
        self.inflight_stamp = torch.full((K * cap,), -(1 << 62), dtype=torch.int64,
                                         device=self.device)
        n = self.inflight_count.cpu().tolist()
        for k in range(K):
            self.inflight_stamp[k * cap:k * cap + n[k]] = torch.arange(
                n[k], dtype=torch.int64) - (1 << 62)
        self.monitor_c.inflight_stamp = _ptr(self.inflight_stamp)

    # -- engine execution clock ----------------------------
    run_c = None

    def enable_engine_run(self, done_capacity: int) -> None:
        """Allocate the per-engine running sets (EngineSim.running) and the
        completion lists, and attach them to the queue state: from now on
        every admission starts a stint and chm_engine_advance finishes them."""
        d, K = self.device, self.K
        cap = max(self.pool[mid].max_batch_size for mid in self.ids)
        f64, i64, i32 = torch.float64, torch.int64, torch.int32
        self.q_input_tokens = torch.ones(K * self.capacity, dtype=i32, device=d)
        self.run_handle = torch.zeros(K * cap, dtype=i64, device=d)
        self.run_seq = torch.zeros(K * cap, dtype=i64, device=d)
        self.run_stint_end = torch.zeros(K * cap, dtype=f64, device=d)
        self.run_decode_start = torch.zeros(K * cap, dtype=f64, device=d)
        self.run_stint_tokens = torch.zeros(K * cap, dtype=i32, device=d)
        self.run_n = torch.zeros(K, dtype=i32, device=d)
        self.tokens_emitted = torch.zeros(K, dtype=i64, device=d)
        self.served = torch.zeros(K, dtype=i64, device=d)
        self.done_capacity = int(done_capacity)
        self.done_handle = torch.zeros(K * self.done_capacity, dtype=i64, device=d)
        self.done_time = torch.zeros(K * self.done_capacity, dtype=f64, device=d)
        self.run_n_done = torch.zeros(K, dtype=i32, device=d)
        self.run_capacity = cap
        er = _lib.EngineRun()
        er.capacity = cap
        er.done_capacity = self.done_capacity
        for i, mid in enumerate(self.ids):
            er.prefill_ms_per_token[i] = self.pool[mid].prefill_ms_per_token
        for name, t in (("queue_input_tokens", self.q_input_tokens),
                        ("handle", self.run_handle), ("seq", self.run_seq),
                        ("stint_end", self.run_stint_end),
                        ("decode_start", self.run_decode_start),
                        ("stint_tokens", self.run_stint_tokens), ("n", self.run_n),
                        ("tokens_emitted", self.tokens_emitted), ("served", self.served),
                        ("done_handle", self.done_handle), ("done_time", self.done_time),
                        ("n_done", self.run_n_done)):
            setattr(er, name, _ptr(t))
        self.run_c = er
        self.queue_c.run = ctypes.addressof(er)

    def completions(self, model: int) -> tuple[np.ndarray, np.ndarray]:
        """(handles, finish times) of engine `model`'s completions, in order."""
        n = int(self.run_n_done[model])
        b = model * self.done_capacity
        return (self.done_handle[b:b + n].cpu().numpy(), self.done_time[b:b + n].cpu().numpy())

    def running_set(self, model: int) -> list[tuple[int, int, float]]:
        """(seq, handle, stint_end) of engine `model`'s running requests by seq."""
        n = int(self.run_n[model])
        b = model * self.run_capacity
        rows = zip(self.run_seq[b:b + n].tolist(), self.run_handle[b:b + n].tolist(),
                   self.run_stint_end[b:b + n].tolist())
        return sorted(rows)

    # -- host-side setup (not on the tick path) ------------------------------
    def seed_inflight(self, per_model_values: dict[str, list[float]]) -> None:
        """Install pre-existing in-flight predictions (insertion order kept)."""
        s = self.inflight_sum.cpu().numpy()
        c = self.inflight_comp.cpu().numpy()
        n = self.inflight_count.cpu().numpy()
        cap = self.inflight_capacity
        for mid, vals in per_model_values.items():
            k = self.ids.index(mid)
            ss, cc = float(s[k]), float(c[k])
            for x in vals:
                x = float(x)
                t = ss + x
                cc += ((ss - t) + x) if abs(ss) >= abs(x) else ((x - t) + ss)
                ss = t
            n0 = int(n[k])
            if n0 + len(vals) > cap:
                raise ValueError(f"in-flight log of {mid} exceeds capacity {cap}")
            # log entries keyed -(n0 + j + 1): seeded requests (see seed_key)
            b = k * cap + n0
            self.inflight_key[b:b + len(vals)] = torch.arange(
                -(n0 + 1), -(n0 + len(vals) + 1), -1, dtype=torch.int64)
            self.inflight_yhat[b:b + len(vals)] = torch.as_tensor(
                np.asarray(vals, dtype=np.float64))
            if self.inflight_stamp is not None:  # seeded entries precede every tick's
                self.inflight_stamp[b:b + len(vals)] = torch.arange(
                    n0, n0 + len(vals), dtype=torch.int64) - (1 << 62)
            s[k], c[k], n[k] = ss, cc, n0 + len(vals)
        self.inflight_sum.copy_(torch.from_numpy(s))
        self.inflight_comp.copy_(torch.from_numpy(c))
        self.inflight_count.copy_(torch.from_numpy(n))

    def preassign(self, programs, models) -> None:
        idx = torch.as_tensor(np.asarray(programs, dtype=np.int64), device=self.device)
        val = torch.as_tensor(np.asarray(models, dtype=np.int8), device=self.device)
        self.assignment[idx] = val

    def set_engine_counters(self, running=None, queued=None, seq=None, clock=None) -> None:
        for src, dst in ((running, self.engine_running), (queued, self.engine_queued),
                         (seq, self.engine_seq), (clock, self.engine_clock)):
            if src is not None:
                dst.copy_(torch.as_tensor(np.asarray(src), dtype=dst.dtype))

    def load_queue(self, model: int, priority, arrival, seq, handle, out_tokens=None,
                   level=None, count=None) -> None:
        """Install a queue segment (entries must be in seq order)."""
        n = len(priority)
        if n > self.capacity:
            raise ValueError("queue segment exceeds capacity")
        b = model * self.capacity
        put = lambda dst, v, dt: dst[b:b + n].copy_(torch.as_tensor(np.asarray(v), dtype=dt))  # noqa: E731
        put(self.q_priority, priority, torch.float64)
        put(self.q_arrival, arrival, torch.float64)
        put(self.q_seq, seq, torch.int64)
        put(self.q_handle, handle, torch.int64)
        put(self.q_out_tokens, out_tokens if out_tokens is not None else np.zeros(n), torch.int32)
        put(self.q_level, level if level is not None else np.zeros(n), torch.int32)
        put(self.q_count, count if count is not None else np.zeros(n), torch.int32)
        self.q_quantum[b:b + n].zero_()
        self.engine_queued[model] = n

    # -- snapshot / restore (device-to-device copies, graph-capturable) ------
    _MUTABLE = ("inflight_sc", "inflight_count", "inflight_key",
                "inflight_yhat", "assignment", "stage_bits",
                "engine_clock", "engine_seq", "engine_running", "engine_queued",
                "engine_iterations", "q_priority", "q_arrival", "q_seq", "q_handle",
                "q_out_tokens", "q_level", "q_count", "q_quantum")

    def _mutable(self):
        return (self._MUTABLE + (("inflight_progress",) if self.decay_in_flight else ())
                + (("inflight_stamp",) if self.inflight_stamp is not None else ()))

    def snapshot(self) -> dict:
        return {k: getattr(self, k).clone() for k in self._mutable()}

    def restore(self, snap: dict) -> None:
        missing = [k for k in self._mutable() if k not in snap]
        if missing:
            raise KeyError(f"snapshot taken before {missing} existed (e.g. before "
                           "ShardedScheduler enabled the in-flight stamps); take it again")
        for k in self._mutable():
            getattr(self, k).copy_(snap[k], non_blocking=True)

    # -- views ---------------------------------------------------------------
    def in_flight_sums(self) -> list[float]:
        s = self.inflight_sum.cpu().tolist()
        c = self.inflight_comp.cpu().tolist()
        return [neumaier_value(a, b) for a, b in zip(s, c)]

    def queue_order(self, model: int) -> np.ndarray:
        """Handles of engine `model`'s queue in STJF order (after the last tick)."""
        n = int(self.engine_queued[model])
        b = model * self.capacity
        order = self.q_order[b:b + n].long()
        return self.q_handle[b:b + n][order].cpu().numpy()

    def admitted(self, model: int) -> np.ndarray:
        n = int(self.q_n_admitted[model])
        b = model * self.capacity
        return self.q_admitted[b:b + n].cpu().numpy()


def request_key(program: int, stage: int) -> int:
    """In-flight log key of request (program, stage) (request_id "p:stage")."""
    return int(program) * 32 + (int(stage) - 1)


def balancer_struct(cfg: BalancerConfig, tie_tolerance: float = 2e-2) -> _lib.BalancerCfg:
    return _lib.BalancerCfg(float(cfg.latency_slack), float(cfg.confidence_margin),
                            float(tie_tolerance))


def aging_struct(aging: AgingConfig) -> _lib.AgingCfg:
    """EngineSim compares integer counters with the thresholds (`count >= S`,
    `quantum >= Q`, engine.py:346-374), so fractional thresholds act as their
    ceilings. A NaN threshold never promotes, like S = inf."""
    S = float(aging.starvation_threshold)
    Q = math.ceil(float(aging.running_quantum))
    if aging.enabled and not math.isnan(S):
        return _lib.AgingCfg(1, int(math.ceil(S)), int(Q), int(aging.demote_while_queued))
    return _lib.AgingCfg(0, 0, int(Q), 0)
