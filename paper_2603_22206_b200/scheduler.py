"""Batched drop-in for hetsched's scheduling hot path.

`GpuScheduler.schedule_batch(reqs, recs)` returns exactly the list of
`Decision`s that B serial calls of `hetsched.balancer.schedule_request`
(balancer.py:89-129) would return, and leaves the activity monitor and the
engine queues in the same state. Per batch it enqueues on one CUDA stream:

  chm_queue_complete   (optional) engine completions freeing slots (K7 phase A)
  chm_prepare_rows     assignment lookup, in-batch repeats, router row list
  router.score_rows    K1-K4 encoder (or a lookup router) on the routed rows
  predictor.predict_rows   K5
  chm_schedule_rows    K6 serial-exact monitor + load + selection + dispatch
  chm_queue_tick       K7 append + aging iterations + STJF order

The columnar entry point `run_rows(RowBatch)` is the hot path (no per-request
Python objects); `schedule_batch` converts reference-style Request/TraceRecord
objects to columns first. Everything is asynchronous until results are read;
the whole sequence is CUDA-graph capturable for a fixed batch shape
(see tick.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import AgingConfig, BalancerConfig, Decision, Pool
from .state import DeviceState, aging_struct, balancer_struct

INT32_MAX = 2**31 - 1


def _p(t):
    return None if t is None else t.data_ptr()


@dataclass
class RowBatch:
    """Columnar batch of requests in arrival order (device tensors)."""

    program: torch.Tensor        # i32[B] dense program index
    stage: torch.Tensor          # i32[B] 1-based stage index
    arrival: torch.Tensor        # f64[B]
    out_tokens: torch.Tensor     # i32[B, K] rec.out_tokens(stage, m)
    handle: torch.Tensor         # i64[B]
    workflow: torch.Tensor | None = None      # i32[B] predictor workflow index
    input_tokens: torch.Tensor | None = None  # i32[B]
    token_ids: torch.Tensor | None = None     # i32[B, S] router input
    n_stages: torch.Tensor | None = None      # i32[B] (oracle predictor)
    stage_out: torch.Tensor | None = None     # i32[B, MAXST, K] (oracle predictor)

    @property
    def n_rows(self) -> int:
        return int(self.program.shape[0])

    def rows_struct(self) -> _lib.Rows:
        return _lib.Rows(self.n_rows, _p(self.program), _p(self.stage), _p(self.arrival),
                         _p(self.out_tokens), _p(self.handle), _p(self.input_tokens))

    @staticmethod
    def from_numpy(device, **cols) -> "RowBatch":
        conv = {}
        dtypes = dict(program=np.int32, stage=np.int32, arrival=np.float64,
                      out_tokens=np.int32, handle=np.int64, workflow=np.int32,
                      input_tokens=np.int32, token_ids=np.int32, n_stages=np.int32,
                      stage_out=np.int32)
        for k, v in cols.items():
            if v is None:
                conv[k] = None
                continue
            conv[k] = torch.as_tensor(np.ascontiguousarray(np.asarray(v, dtype=dtypes[k])),
                                      device=device)
        return RowBatch(**conv)


class HostStaging:
    """Pinned host columns of one batch + pinned decision outputs.

    `upload()` enqueues the host->device copies of the batch, `download()` the
    device->host copies of the decisions (model, priority, flags), both
    asynchronous on the current stream: what an end-to-end caller pays per tick.
    """

    _DT = dict(program=np.int32, stage=np.int32, arrival=np.float64, out_tokens=np.int32,
               handle=np.int64, workflow=np.int32, input_tokens=np.int32, token_ids=np.int32,
               n_stages=np.int32, stage_out=np.int32)

    def __init__(self, cols: dict, device):
        self.host = {k: torch.from_numpy(np.ascontiguousarray(np.asarray(v, dtype=self._DT[k])))
                     .pin_memory() for k, v in cols.items() if v is not None}
        self.batch = RowBatch(**{k: torch.empty(v.shape, dtype=v.dtype, device=device)
                                 for k, v in self.host.items()})
        B = self.batch.n_rows
        self.model = torch.empty(B, dtype=torch.int32).pin_memory()
        self.priority = torch.empty(B, dtype=torch.float64).pin_memory()
        self.flags = torch.empty(B, dtype=torch.uint8).pin_memory()

    @property
    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.host.values())

    @property
    def d2h_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.model, self.priority, self.flags))

    def upload(self) -> RowBatch:
        for k, h in self.host.items():
            getattr(self.batch, k).copy_(h, non_blocking=True)
        return self.batch

    def download(self, buf: "BatchBuffers") -> None:
        B = self.batch.n_rows
        self.model.copy_(buf.model[:B], non_blocking=True)
        self.priority.copy_(buf.priority[:B], non_blocking=True)
        self.flags.copy_(buf.dflags[:B], non_blocking=True)


class BatchBuffers:
    """Per-batch scratch and outputs for up to `max_rows` rows."""

    def __init__(self, K: int, max_rows: int, device):
        d, B = device, int(max_rows)
        self.K, self.max_rows = K, B
        self.first_row = torch.empty(B, dtype=torch.int32, device=d)
        self.pre_model = torch.empty(B, dtype=torch.int8, device=d)
        self.route_rows = torch.empty(B, dtype=torch.int32, device=d)
        self.n_route = torch.zeros(1, dtype=torch.int32, device=d)
        self.qual = torch.empty(B, dtype=torch.int64, device=d)
        self.rank = torch.empty(B, dtype=torch.int32, device=d)
        self.flags = torch.empty(B, dtype=torch.int32, device=d)
        self.scores = torch.zeros(B * K, dtype=torch.float64, device=d)  # fp64 like ConfidenceVector
        self.yhat = torch.zeros(B * K, dtype=torch.float64, device=d)
        self.model = torch.full((B,), -1, dtype=torch.int32, device=d)
        self.priority = torch.zeros(B, dtype=torch.float64, device=d)
        self.dflags = torch.zeros(B, dtype=torch.uint8, device=d)
        self.seq = torch.zeros(B, dtype=torch.int64, device=d)
        self.loads = torch.zeros(B * K, dtype=torch.float64, device=d)
        self.n_committed = torch.zeros(1, dtype=torch.int32, device=d)
        self.n_complete = torch.zeros(K, dtype=torch.int32, device=d)
        self.lnew = torch.zeros(B, dtype=torch.float64, device=d)
        self.tie_counts = torch.zeros(3, dtype=torch.int32, device=d)
        # error words: the batch's (predictor / K6 / K7, lowest row wins) and
        # the completions' (record_completion runs before the batch)
        self.error = torch.zeros(4, dtype=torch.int32, device=d)
        self.error_complete = torch.zeros(4, dtype=torch.int32, device=d)
        self.error_init = torch.tensor([0, INT32_MAX, -1, 0], dtype=torch.int32, device=d)
        self.error_complete.copy_(self.error_init)
        self.scratch_c = _lib.RowScratch(
            _p(self.first_row), _p(self.pre_model), _p(self.route_rows), _p(self.n_route),
            _p(self.qual), _p(self.rank), _p(self.flags), _p(self.lnew))

    def decisions_struct(self, with_loads: bool = True) -> _lib.Decisions:
        return _lib.Decisions(_p(self.model), _p(self.priority), _p(self.dflags), _p(self.seq),
                              _p(self.loads) if with_loads else None, _p(self.n_committed),
                              _p(self.error), _p(self.tie_counts))


class GpuScheduler:
    """Serial-exact batched Algorithm 1 on one B200."""

    def __init__(self, pool: Pool, balancer: BalancerConfig = BalancerConfig(),
                 aging: AgingConfig = AgingConfig(), *, router=None, predictor=None,
                 n_programs: int = 1 << 20, max_rows: int = 16384,
                 queue_capacity: int = 10240, device="cuda", inflight_capacity=None,
                 decay_in_flight: bool = False, engine_clock: bool = False,
                 completion_capacity: int | None = None, tie_tolerance: float = 2e-2):
        self.lib = _lib.load()
        self.pool = pool
        self.ids = pool.model_ids
        self.K = len(self.ids)
        self.cfg = balancer
        self.aging = aging
        self.router = router
        self.predictor = predictor
        self.device = torch.device(device)
        self.state = DeviceState(pool, n_programs, queue_capacity, self.device,
                                 inflight_capacity=inflight_capacity,
                                 decay_in_flight=decay_in_flight)
        if engine_clock:
            # running sets + stint clock on the device
            self.state.enable_engine_run(
                completion_capacity if completion_capacity is not None
                else queue_capacity + max(p.max_batch_size for p in pool.profiles))
        self.buf = BatchBuffers(self.K, max_rows, self.device)
        self.tie_tolerance = float(tie_tolerance)
        self.bal_c = balancer_struct(balancer, self.tie_tolerance)
        self.aging_c = aging_struct(aging)
        self._program_index: dict[str, int] = {}
        self._handles: list = []

    # ------------------------------------------------------------------ core
    def run_rows(self, batch: RowBatch, n_iterations: int = 1, n_complete=None,
                 with_loads: bool = True, stream=None, completions=None,
                 keep_admitted: bool = False) -> None:
        """Enqueue one tick for `batch` on `stream` (default: current stream).

        completions: optional (model int32[n], key int64[n]) device tensors of
        requests that finished since the last tick (key = request_key(program,
        stage)): removed from the in-flight log (record_completion) and their
        engines' slots freed, before the batch is scheduled. n_complete: the
        engine side only (int32[K] finished-per-engine counts).
        keep_admitted: append to the admission lists instead of resetting
        them (the sharded protocol runs merged iterations before the batch).

        The tick is three phases, also callable one by one (dist.py runs the
        P-independent ones on every GPU before the serial chain's exchange):
        begin_tick (error words, completions), route_predict (prepare, router,
        predictor) and select_enqueue (K6 chain + K7 queues)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.begin_tick(completions=completions, n_complete=n_complete,
                        keep_admitted=keep_admitted, stream=s)
        self.route_predict(batch, stream=s)
        self.select_enqueue(batch, n_iterations=n_iterations, with_loads=with_loads, stream=s)

    def begin_tick(self, completions=None, n_complete=None, keep_admitted: bool = False,
                   stream=None) -> None:
        """Reset the tick's error words and admission lists; apply completions
        (record_completion -> in-flight log + sums, then the engines' freed
        slots). On a request shard the recomputed sums cover only the local
        log; dist.ShardedScheduler replaces them with the global exact sum."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        sh = s.cuda_stream
        st, buf, lib = self.state, self.buf, self.lib
        with torch.cuda.stream(s):
            buf.error.copy_(buf.error_init)
            buf.error_complete.copy_(buf.error_init)
            if not keep_admitted:
                st.q_n_admitted.zero_()
                st.q_n_promoted.zero_()
            if completions is not None:
                # monitor side (record_completion) -> per-engine counts -> engines
                if n_complete is not None:
                    raise ValueError("give either completions or n_complete")
                c_model, c_key = completions
                _lib.check(lib.chm_monitor_complete(st.pool_c, st.monitor_c, _p(c_model),
                                                    _p(c_key), int(c_model.numel()),
                                                    _p(buf.n_complete), _p(buf.error_complete),
                                                    sh),
                           "chm_monitor_complete")
                n_complete = buf.n_complete
            if n_complete is not None:
                _lib.check(lib.chm_queue_complete(st.pool_c, self.aging_c, st.monitor_c,
                                                  st.queue_c, _p(n_complete),
                                                  _p(buf.error_complete), sh),
                           "chm_queue_complete")

    def route_predict(self, batch: RowBatch, stream=None) -> None:
        """The in-flight-independent half of the tick: assignment lookup and
        router row list (chm_prepare_rows), router (K1-K4), predictor (K5)."""
        B = batch.n_rows
        if B > self.buf.max_rows:
            raise ValueError(f"batch of {B} rows exceeds max_rows={self.buf.max_rows}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        st, buf, lib = self.state, self.buf, self.lib
        rows_c = batch.rows_struct()
        with torch.cuda.stream(s):
            _lib.check(lib.chm_prepare_rows(st.monitor_c, rows_c, buf.scratch_c,
                                            _p(st.epoch), s.cuda_stream), "chm_prepare_rows")
            if self.router is None:
                raise RuntimeError("GpuScheduler needs a router")
            self.router.score_rows(batch, buf.route_rows, buf.n_route, buf.scores, s)
            if self.predictor is None:
                raise RuntimeError("GpuScheduler needs a predictor")
            self.predictor.predict_rows(batch, self.K, buf.yhat, buf.error, s)

    def select_enqueue(self, batch: RowBatch, n_iterations: int = 1, with_loads: bool = True,
                       stream=None) -> None:
        """The serial half: K6 (monitor + load + selection + dispatch, in row
        order from the current in-flight state) and K7 (append + aging
        iterations + STJF order)."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        sh = s.cuda_stream
        st, buf, lib = self.state, self.buf, self.lib
        rows_c = batch.rows_struct()
        dec_c = buf.decisions_struct(with_loads)
        self._dec_c = dec_c  # kept alive for callers that pack the decisions
        _lib.check(lib.chm_schedule_rows(st.pool_c, self.bal_c, st.monitor_c, rows_c,
                                         buf.scratch_c, _p(buf.scores), _p(buf.yhat),
                                         dec_c, sh), "chm_schedule_rows")
        _lib.check(lib.chm_queue_tick(st.pool_c, self.aging_c, st.monitor_c, st.queue_c,
                                      rows_c, dec_c, int(n_iterations), _p(buf.error), sh),
                   "chm_queue_tick")

    def note_progress(self, models, keys, emitted, stream=None) -> None:
        """ActivityMonitor.note_progress (monitor.py:108-111) for a batch of
        (model index, request key, emitted tokens) updates, then the decayed
        in-flight sums (decay_in_flight=True schedulers only). Keys are
        `state.request_key(program, stage)` (negative for seeded entries)."""
        if not self.state.decay_in_flight:
            raise ValueError("note_progress needs GpuScheduler(decay_in_flight=True)")
        d = self.device
        m = torch.as_tensor(np.asarray(models, np.int32), device=d)
        k = torch.as_tensor(np.asarray(keys, np.int64), device=d)
        e = torch.as_tensor(np.asarray(emitted, np.float64), device=d)
        s = stream if stream is not None else torch.cuda.current_stream(d)
        self.buf.error.copy_(self.buf.error_init)
        _lib.check(self.lib.chm_monitor_note_progress(
            self.state.pool_c, self.state.monitor_c, _p(m), _p(k), _p(e), int(m.numel()),
            _p(self.buf.error), s.cuda_stream), "chm_monitor_note_progress")
        self._keep = (m, k, e)  # alive until the stream has consumed them

    def scheduling_iteration(self, n_iterations: int = 1, stream=None) -> None:
        """EngineSim.scheduling_iteration on every engine, n times, with no new
        arrivals (engine.py:160-163): chm_queue_tick on an empty batch, at
        each engine's current clock. Admissions go to `state.admitted(m)`."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        st, buf = self.state, self.buf
        rows_c = _lib.Rows(0, None, None, None, None, None, None)
        with torch.cuda.stream(s):
            buf.error.copy_(buf.error_init)
            buf.n_committed.zero_()
            st.q_n_admitted.zero_()
            st.q_n_promoted.zero_()
            _lib.check(self.lib.chm_queue_tick(st.pool_c, self.aging_c, st.monitor_c,
                                               st.queue_c, rows_c,
                                               buf.decisions_struct(False), int(n_iterations),
                                               _p(buf.error), s.cuda_stream), "chm_queue_tick")

    # -- engine execution clock ----------------------------
    def advance_to(self, target, stream=None, keep_completions: bool = False):
        """EngineSim.advance_to(target) on every engine (engine.py:174-183):
        finish the stints ending by `target` (float, or float64[K] per engine),
        each running one scheduling iteration at its end. Returns nothing; the
        completions are in `state.completions(m)` (appended to the previous
        call's when keep_completions)."""
        st = self.state
        if st.run_c is None:
            raise RuntimeError("GpuScheduler(engine_clock=True) is required")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        if not torch.is_tensor(target):
            target = torch.full((self.K,), float(target), dtype=torch.float64,
                                device=self.device)
        with torch.cuda.stream(s):
            if not keep_completions:
                st.run_n_done.zero_()
            st.q_n_admitted.zero_()
            st.q_n_promoted.zero_()
            self.buf.error.copy_(self.buf.error_init)
            _lib.check(self.lib.chm_engine_advance(st.pool_c, self.aging_c, st.monitor_c,
                                                   st.queue_c, _p(target), _p(self.buf.error),
                                                   s.cuda_stream), "chm_engine_advance")

    # -- sharded engine queues: cross-GPU admission --------
    def candidate_width(self) -> int:
        """F of chm_queue_candidates: the largest max_batch_size in the pool."""
        return max(self.pool[mid].max_batch_size for mid in self.ids)

    def queue_candidates(self, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        """This rank's STJF head of every engine sub-queue, as chm_queue_key
        records in an int64 tensor [K, F, 5] (level, priority bits, arrival
        bits, seq, handle; level INT64_MAX = no candidate)."""
        F = self.candidate_width()
        if out is None:
            out = torch.empty((self.K, F, 5), dtype=torch.int64, device=self.device)
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        st = self.state
        _lib.check(self.lib.chm_queue_candidates(st.pool_c, st.monitor_c, st.queue_c, F,
                                                 _p(out), s.cuda_stream),
                   "chm_queue_candidates")
        return out

    def queue_admit_merged(self, gathered: torch.Tensor, rank: int, release=None,
                           stream=None) -> None:
        """One scheduling iteration of every engine against the gathered
        candidates of all G ranks ([G, K, F, 5], rank-major): admit this
        rank's share of the global top, count the global admissions as
        running, age the rest. release: optional int32[K] device tensor
        (1 = a running request finished first, -1 = engine idle this call)."""
        G, K, F = int(gathered.shape[0]), int(gathered.shape[1]), int(gathered.shape[2])
        if K != self.K or F != self.candidate_width() or gathered.dtype != torch.int64:
            raise ValueError("gathered candidates do not match this pool")
        gathered = gathered.contiguous()
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        st = self.state
        _lib.check(self.lib.chm_queue_admit_merged(st.pool_c, self.aging_c, st.monitor_c,
                                                   st.queue_c, _p(gathered), G, F, int(rank),
                                                   _p(release), _p(self.buf.error),
                                                   s.cuda_stream), "chm_queue_admit_merged")

    def check_errors(self, context: str = "") -> None:
        """Raise the reference exception for the last tick, if any: a
        completion error first (record_completion ran before the batch),
        then the batch's lowest-row error."""
        _lib.raise_device_error(self.buf.error_complete.cpu().tolist(),
                                (context + " completions").strip())
        _lib.raise_device_error(self.buf.error.cpu().tolist(), context)

    def tie_band(self) -> dict:
        """Tie-band report of the last batch (north star: "ties inside the
        tolerance band are reported"): routed decisions whose descending-q
        choice (`rank`) or confidence gate q_m >= q_fast + margin (`gate`)
        compares two router outputs that are within `tie_tolerance`, and
        either (`any`). The default 2e-2 is twice the router's 1e-2 tolerance
        (both sides of each comparison carry router error), so every decision
        a router error <= 1e-2 could flip is counted. Per-row bits: Decision
        flags 8 / 16 (`buf.dflags`)."""
        r, g, a = (int(x) for x in self.buf.tie_counts.cpu().tolist())
        return {"tolerance": self.tie_tolerance, "rank": r, "gate": g, "any": a,
                "routed": int(self.buf.n_route.item())}

    # ------------------------------------------------------ reference-style API
    def program_index(self, program_id: str) -> int:
        idx = self._program_index.get(program_id)
        if idx is None:
            idx = len(self._program_index)
            if idx >= self.state.n_programs:
                raise ValueError("program index space exhausted (raise n_programs)")
            self._program_index[program_id] = idx
        return idx

    def rows_from_requests(self, reqs, recs) -> RowBatch:
        K = self.K
        B = len(reqs)
        prog = np.empty(B, np.int32)
        stage = np.empty(B, np.int32)
        arr = np.empty(B, np.float64)
        out = np.empty((B, K), np.int32)
        handle = np.empty(B, np.int64)
        inp = np.empty(B, np.int32)
        for i, (r, rec) in enumerate(zip(reqs, recs)):
            prog[i] = self.program_index(r.program_id)
            stage[i] = r.stage_index
            arr[i] = r.arrival_time
            out[i] = [rec.out_tokens(r.stage_index, mid) for mid in self.ids]
            handle[i] = len(self._handles)
            self._handles.append(r.request_id)
            inp[i] = r.input_tokens
        extra = {}
        if hasattr(self.predictor, "columns_for"):
            extra = self.predictor.columns_for(reqs, recs, self.ids)
        if hasattr(self.router, "columns_for"):
            extra.update(self.router.columns_for(reqs, recs))
        return RowBatch.from_numpy(self.device, program=prog, stage=stage, arrival=arr,
                                   out_tokens=out, handle=handle, input_tokens=inp, **extra)

    def schedule_batch(self, reqs, recs, n_iterations: int = 0) -> list[Decision]:
        """B serial schedule_request calls (balancer.py:89-129), batched.

        n_iterations explicit EngineSim.scheduling_iteration calls per engine
        follow the batch (0 = just the enqueues, like the reference loop)."""
        batch = self.rows_from_requests(reqs, recs)
        self.run_rows(batch, n_iterations=n_iterations)
        return self.collect(batch)

    def collect(self, batch: RowBatch) -> list[Decision]:
        """Read back decisions (syncs) and raise the reference's exception, if any."""
        buf, K = self.buf, self.K
        B = batch.n_rows
        n_ok = int(buf.n_committed.item())
        err_code, err_row = (int(x) for x in buf.error[:2].cpu().tolist())
        if err_code:
            # the reference raised at err_row: no decisions for it or later rows
            n_ok = min(n_ok, err_row)
        model = buf.model[:n_ok].cpu().numpy()
        prio = buf.priority[:n_ok].cpu().numpy()
        fl = buf.dflags[:n_ok].cpu().numpy()
        loads = buf.loads[:n_ok * K].view(-1, K).cpu().numpy() if n_ok else np.zeros((0, K))
        scores = buf.scores[:n_ok * K].view(-1, K).cpu().numpy() if n_ok else np.zeros((0, K))
        out = []
        for i in range(n_ok):
            cached = bool(fl[i] & 1)
            out.append(Decision(
                model=self.ids[int(model[i])],
                priority=float(prio[i]),
                estimated_loads={} if cached else {m: float(loads[i, k]) for k, m in enumerate(self.ids)},
                used_cached_assignment=cached,
                scores=None if cached else {m: float(scores[i, k]) for k, m in enumerate(self.ids)},
            ))
        try:
            self.check_errors("schedule_batch")
        except Exception as exc:  # the reference raised after applying rows < n_ok
            exc.decisions = out
            raise
        if n_ok != B:
            raise RuntimeError(f"batch stopped at row {n_ok} without an error code")
        return out
