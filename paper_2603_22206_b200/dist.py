"""Request-sharded multi-GPU scheduling: one process per GPU.

Requests shard by program (`shard_of`), so every stage of a program lands on
the same GPU and the assignment map stays local. Router, predictor, the
per-row precompute, the in-flight logs and the engine sub-queues are
shard-local; the only cross-GPU state is the per-engine in-flight
predicted-token vector P (K doubles, the Neumaier (s, c) of
ActivityMonitor.in_flight_sum, monitor.py:122-129).

Every tick runs the P-independent half (prepare, router, predictor:
`GpuScheduler.route_predict`) on all GPUs at once; only the serial selection
chain (`select_enqueue`, record_dispatch inside every schedule_request,
balancer.py:116) depends on P. Two decision semantics:

  Mode A (north-star literal): every GPU runs its chain from the tick-start
      global P; afterwards the ranks' committed (model, yhat) rows are
      all-gathered and folded on the device in rank order
      (chm_allreduce_inflight). Decisions equal G independent serial replays
      that all start from P_prev; the tick-end P is exactly the state of one
      serial replay of the concatenated batch (rank 0's rows, then rank 1's..).
  Mode B (serial-exact relay): rank g receives (s, c) from rank g-1 right
      before its selection kernel and forwards it after; the last rank
      broadcasts the tick-end state (chm_inflight_relay_recv / _send). The
      routers and predictors are already enqueued, so they overlap the
      predecessors' chains. Decisions equal ONE serial replay of the
      concatenated batch, bit for bit.

Both modes end every tick in the same state, so they can be mixed tick by
tick and `divergence` counts how many decisions Mode A changes.

Completions are sharded too: each rank removes its own finished requests from
its own log, reduces the survivors exactly (int64 units of 2^-8) and the K
sums are all-reduced (chm_inflight_local_sum / chm_comm_allreduce_i64 /
chm_inflight_set_sum); when a survivor is not dyadic, the ranks' survivor
lists (with global insertion stamps) are all-gathered and merged, and the
Neumaier recurrence replays them in the reference's insertion order
(chm_inflight_pack_live / chm_inflight_merge_sum).

Transport: `NcclComm` drives the C-ABI's NCCL entry points (the product path,
NCCL over NVLink); `TorchComm` runs the same packing / folding kernels over a
torch.distributed group (gloo in the tests: two ranks can share one GPU, NCCL
refuses that).
"""

from __future__ import annotations

import ctypes
import hashlib

import torch
import torch.distributed as dist

from . import _lib


def shard_of(program_id: str, world: int) -> int:
    """Stable program -> rank map (all stages of a program on one GPU)."""
    h = hashlib.blake2b(program_id.encode("utf-8"), digest_size=8).digest()
    return int.from_bytes(h, "big") % world


def _p(t):
    return None if t is None else t.data_ptr()


def _global(rank: int, group) -> int:
    return rank if group is None else dist.get_global_rank(group, rank)


class TorchComm:
    """Exchange over a torch.distributed group (gloo: host staging copies)."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.host = dist.get_backend(group) == "gloo"

    def _buf(self, t):
        return t.cpu() if (t.is_cuda and self.host) else t

    def allgather(self, send: torch.Tensor, recv: torch.Tensor, stream) -> None:
        """recv [world, *send.shape] <- every rank's send."""
        b = self._buf(send)
        parts = [torch.empty_like(b) for _ in range(self.world)]
        dist.all_gather(parts, b, group=self.group)
        recv.copy_(torch.stack(parts).view_as(recv))

    def allreduce_i64(self, buf: torch.Tensor, stream) -> None:
        b = self._buf(buf)
        dist.all_reduce(b, group=self.group)
        if b is not buf:
            buf.copy_(b)

    def relay_recv(self, state: torch.Tensor, stream) -> None:
        if self.rank > 0:
            b = self._buf(state)
            dist.recv(b, src=_global(self.rank - 1, self.group), group=self.group)
            if b is not state:
                state.copy_(b)

    def relay_send(self, state: torch.Tensor, stream) -> None:
        b = self._buf(state)
        if self.rank + 1 < self.world:
            dist.send(b, dst=_global(self.rank + 1, self.group), group=self.group)
        dist.broadcast(b, src=_global(self.world - 1, self.group), group=self.group)
        if b is not state:
            state.copy_(b)


class NcclComm:
    """NCCL communicator owned by libchimera_sm100a.so (chm_comm_*). The unique
    id travels over an existing torch.distributed group once, at setup."""

    def __init__(self, device, group=None):
        self.lib = _lib.load()
        _lib.check(self.lib.chm_comm_available(), "chm_comm_available")
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        uid = (ctypes.c_uint8 * _lib.COMM_ID_BYTES)()
        if self.rank == 0:
            _lib.check(self.lib.chm_comm_unique_id(ctypes.addressof(uid)), "chm_comm_unique_id")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=_global(0, group), group=group)
        uid = (ctypes.c_uint8 * _lib.COMM_ID_BYTES).from_buffer_copy(obj[0])
        self.handle = ctypes.c_void_p()
        dev = torch.device(device)
        _lib.check(self.lib.chm_comm_init(ctypes.addressof(uid), self.rank, self.world,
                                          dev.index if dev.index is not None else -1,
                                          ctypes.byref(self.handle)), "chm_comm_init")

    def close(self) -> None:
        if self.handle:
            self.lib.chm_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def allgather(self, send, recv, stream) -> None:
        _lib.check(self.lib.chm_comm_allgather(self.handle, _p(send), _p(recv),
                                               send.numel() * send.element_size(),
                                               stream.cuda_stream), "chm_comm_allgather")

    def allreduce_i64(self, buf, stream) -> None:
        _lib.check(self.lib.chm_comm_allreduce_i64(self.handle, _p(buf), buf.numel(),
                                                   stream.cuda_stream), "chm_comm_allreduce_i64")

    def relay_recv(self, state, stream) -> None:
        _lib.check(self.lib.chm_inflight_relay_recv(self.handle, _p(state), state.numel(),
                                                    stream.cuda_stream), "chm_inflight_relay_recv")

    def relay_send(self, state, stream) -> None:
        _lib.check(self.lib.chm_inflight_relay_send(self.handle, _p(state), state.numel(),
                                                    stream.cuda_stream), "chm_inflight_relay_send")


def make_comm(device, group=None):
    """NCCL (C-ABI) when the group's backend is NCCL, else the torch group."""
    if dist.get_backend(group) == "nccl":
        return NcclComm(device, group)
    return TorchComm(group)


def sharded_iteration(gs, comm, stream, release=None) -> None:
    """One scheduling iteration of every engine over the G sub-queues
    (global admission): each rank's STJF head candidates
    are all-gathered, then every rank admits its share of the global top and
    ages its sub-queue (chm_queue_admit_merged). Equal to one
    EngineSim._iterate on the union queue (engine.py:328-338)."""
    cand = gs.queue_candidates(stream=stream)
    gathered = torch.empty((comm.world,) + tuple(cand.shape), dtype=cand.dtype,
                           device=cand.device)
    comm.allgather(cand, gathered, stream)
    gs.queue_admit_merged(gathered, comm.rank, release, stream=stream)


# Engine counters relayed with (s, c) under global admission: they make the
# enqueue-time admission (running < max_batch_size), the seq tie-break and the
# clock check (engine.py:140-158) see the one reference engine.
_RELAYED = ("engine_running", "engine_seq", "engine_clock", "engine_iterations")


class ShardedScheduler:
    """A per-rank GpuScheduler with the Mode A / Mode B exchange.

    global_admission (Mode B only): each engine's queue is the union of the
    ranks' sub-queues, served in the reference's global STJF order. The relay
    also carries the engine counters, and every scheduling iteration, whether
    an explicit one or one per completion, is a `sharded_iteration`. Then the
    decisions, admissions and queue orders equal one serial replay of the
    concatenated batch through one EngineSim per model."""

    def __init__(self, scheduler, mode: str = "B", group=None, global_admission: bool = False,
                 comm=None, completion_sums: str = "auto"):
        if mode not in ("A", "B"):
            raise ValueError("mode must be 'A' or 'B'")
        if global_admission and mode != "B":
            raise ValueError("global admission needs the Mode B relay")
        self.gs = scheduler
        self.mode = mode
        self.group = group
        self.global_admission = global_admission
        self.comm = comm if comm is not None else make_comm(scheduler.device, group)
        st = scheduler.state
        K = st.K
        dev = st.device
        self.lib = _lib.load()
        if global_admission:
            self.packed = torch.empty((2 + len(_RELAYED)) * K, dtype=torch.float64, device=dev)
        self.s0 = torch.empty(2 * K, dtype=torch.float64, device=dev)
        # the Mode A records are all-gathered: every rank needs the same size
        mr = torch.tensor([scheduler.buf.max_rows], dtype=torch.int64, device=dev)
        all_mr = torch.empty((self.comm.world, 1), dtype=torch.int64, device=dev)
        self.comm.allgather(mr, all_mr, torch.cuda.current_stream(dev))
        if int(all_mr.min()) != int(all_mr.max()):
            raise ValueError(f"ranks use different max_rows {all_mr.view(-1).tolist()}: the "
                             "sharded exchange needs one batch capacity on every rank")
        rb = int(self.lib.chm_inflight_record_bytes(K, scheduler.buf.max_rows))
        self.rec_bytes = rb
        self.record = torch.empty(rb, dtype=torch.uint8, device=dev)
        self.gathered = torch.empty((self.comm.world, rb), dtype=torch.uint8, device=dev)
        self.sums = torch.zeros(K + 1, dtype=torch.int64, device=dev)
        # completion sums: "auto" = the exact dyadic all-reduce when every
        # survivor is dyadic (checked on the host after it), else the
        # stamp-ordered merge; "dyadic" = the all-reduce only (non-dyadic
        # survivors raise); "merge" = always the merge
        if completion_sums not in ("auto", "dyadic", "merge"):
            raise ValueError("completion_sums must be auto, dyadic or merge")
        self.completion_sums = completion_sums
        st.enable_stamps()
        self.tick = 0

    # -- exchange pieces ------------------------------------------------------
    def _pack(self) -> None:
        st, K = self.gs.state, self.gs.state.K
        self.packed[:2 * K].copy_(st.inflight_sc)
        for i, name in enumerate(_RELAYED):
            self.packed[(2 + i) * K:(3 + i) * K].copy_(getattr(st, name))

    def _unpack(self) -> None:
        st, K = self.gs.state, self.gs.state.K
        st.inflight_sc.copy_(self.packed[:2 * K])
        for i, name in enumerate(_RELAYED):
            getattr(st, name).copy_(self.packed[(2 + i) * K:(3 + i) * K])

    def _relay_state(self):
        return self.packed if self.global_admission else self.gs.state.inflight_sc

    def _allreduce_inflight(self, stream) -> None:
        """Mode A tick end: pack -> all-gather -> fold (chm_allreduce_inflight)."""
        gs, st = self.gs, self.gs.state
        K = st.K
        dec_c = gs.buf.decisions_struct(False)
        if isinstance(self.comm, NcclComm):
            ws = self._ws if hasattr(self, "_ws") else torch.empty(
                (self.comm.world + 1) * self.rec_bytes, dtype=torch.uint8, device=st.device)
            self._ws = ws
            _lib.check(self.lib.chm_allreduce_inflight(
                self.comm.handle, st.pool_c, st.monitor_c, _p(self.s0), _p(self.s0[K:]), dec_c,
                gs.buf.max_rows, _p(ws), _p(gs.buf.error), stream.cuda_stream),
                "chm_allreduce_inflight")
            return
        _lib.check(self.lib.chm_inflight_pack(st.pool_c, dec_c, gs.buf.max_rows,
                                              _p(self.record), stream.cuda_stream),
                   "chm_inflight_pack")
        self.comm.allgather(self.record, self.gathered, stream)
        _lib.check(self.lib.chm_inflight_fold(st.pool_c, st.monitor_c, _p(self.s0),
                                              _p(self.s0[K:]), _p(self.gathered),
                                              self.comm.world, gs.buf.max_rows,
                                              _p(gs.buf.error), stream.cuda_stream),
                   "chm_inflight_fold")

    def _sum_completions(self, stream) -> None:
        """Global exact in-flight sums after sharded record_completion
        (monitor.py:98-129): the dyadic all-reduce, or the merge of every
        rank's survivors in the global insertion order."""
        st = self.gs.state
        K = st.K
        if self.completion_sums != "merge":
            _lib.check(self.lib.chm_inflight_local_sum(st.pool_c, st.monitor_c, _p(self.sums),
                                                       stream.cuda_stream),
                       "chm_inflight_local_sum")
            self.comm.allreduce_i64(self.sums, stream)
            err = _p(self.gs.buf.error_complete) if self.completion_sums == "dyadic" else None
            _lib.check(self.lib.chm_inflight_set_sum(st.pool_c, st.monitor_c, _p(self.sums),
                                                     err, stream.cuda_stream),
                       "chm_inflight_set_sum")
            if self.completion_sums == "dyadic":
                return
            s = self.sums.cpu()  # host check (syncs the stream)
            if int(s[K]) == 0 and int(s[:K].max()) < (1 << 53):
                return
        # merge path: every rank's (stamp, term) lists, all-gathered
        counts = torch.empty((self.comm.world, K), dtype=torch.int64, device=st.device)
        self.comm.allgather(st.inflight_count.contiguous(), counts, stream)
        cap = int(counts.max().item())
        rec = torch.empty(K * max(cap, 1) * 2, dtype=torch.int64, device=st.device)
        _lib.check(self.lib.chm_inflight_pack_live(st.pool_c, st.monitor_c, cap, _p(rec),
                                                   stream.cuda_stream), "chm_inflight_pack_live")
        gathered = torch.empty((self.comm.world, rec.numel()), dtype=torch.int64,
                               device=st.device)
        self.comm.allgather(rec, gathered, stream)
        _lib.check(self.lib.chm_inflight_merge_sum(st.pool_c, st.monitor_c, _p(gathered),
                                                   _p(counts), self.comm.world, cap,
                                                   stream.cuda_stream), "chm_inflight_merge_sum")
        self._keep = (counts, rec, gathered)

    # -- the tick ---------------------------------------------------------------
    def run_rows(self, batch, n_iterations: int = 1, completions=None, n_complete=None,
                 stream=None, with_loads: bool = True) -> None:
        """One sharded tick. completions: this rank's finished requests (model,
        key) -- the ones it dispatched; with them every rank must pass a
        (possibly empty) tensor pair, since the sums are all-reduced.
        n_complete: engine slots freed without monitor records (int32[K]);
        under global admission it is the global per-engine count and
        completions only update the monitor."""
        gs = self.gs
        s = stream if stream is not None else torch.cuda.current_stream(gs.device)
        st = gs.state
        # global insertion stamps of this tick's dispatches: (tick, rank, row)
        st.stamp_base.fill_((self.tick << 40) | (self.comm.rank << 32))
        self.tick += 1
        if self.global_admission:
            gs.begin_tick(completions=None, keep_admitted=False, stream=s)
            if completions is not None:
                self._monitor_complete(completions, s)
            if n_complete is not None:
                # each completion frees a slot and runs one iteration of its engine
                # (engine.py:232-241); n_complete is global, equal on all ranks
                for r in range(int(n_complete.max().item()) if n_complete.numel() else 0):
                    release = torch.where(n_complete > r, 1, -1).to(torch.int32)
                    sharded_iteration(gs, self.comm, s, release)
            gs.route_predict(batch, stream=s)
            self._pack()
            self.comm.relay_recv(self.packed, s)
            self._unpack()
            gs.select_enqueue(batch, n_iterations=0, with_loads=with_loads, stream=s)
            self._pack()
            self.comm.relay_send(self.packed, s)
            self._unpack()
            for _ in range(n_iterations):
                sharded_iteration(gs, self.comm, s)
            return
        gs.begin_tick(completions=completions, n_complete=n_complete, stream=s)
        if completions is not None:
            self._sum_completions(s)
        gs.route_predict(batch, stream=s)
        if self.mode == "A":
            self.s0.copy_(st.inflight_sc)
            gs.select_enqueue(batch, n_iterations=n_iterations, with_loads=with_loads, stream=s)
            self._allreduce_inflight(s)
            return
        self.comm.relay_recv(st.inflight_sc, s)
        gs.select_enqueue(batch, n_iterations=n_iterations, with_loads=with_loads, stream=s)
        self.comm.relay_send(st.inflight_sc, s)

    def _monitor_complete(self, completions, stream) -> None:
        gs, st = self.gs, self.gs.state
        c_model, c_key = completions
        _lib.check(self.lib.chm_monitor_complete(
            st.pool_c, st.monitor_c, _p(c_model), _p(c_key), int(c_model.numel()),
            _p(gs.buf.n_complete), _p(gs.buf.error_complete), stream.cuda_stream),
            "chm_monitor_complete")
        self._sum_completions(stream)


def divergence(models_a: torch.Tensor, models_b: torch.Tensor, comm, stream) -> int:
    """Decisions that differ between a Mode A and a Mode B run of the same
    sharded tick, summed over the ranks."""
    d = torch.tensor([int((models_a != models_b).sum().item())], dtype=torch.int64,
                     device=models_a.device)
    comm.allreduce_i64(d, stream)
    return int(d.item())
