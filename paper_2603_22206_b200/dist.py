"""Request-sharded multi-GPU scheduling: one process per GPU.

Requests shard by program (`shard_of`), so every stage of a program lands on
the same GPU and the assignment map stays local. Router, predictor and the
per-row precompute are shard-local; the only cross-GPU state is the
per-engine in-flight predicted-token vector P (K doubles, Neumaier (s, c)).

Two decision semantics (the caller picks one):

  Mode A (north-star literal): every GPU runs its shard's serial chain from
      the tick-start global P; afterwards the per-engine deltas are summed
      with one all-reduce (NCCL over NVLink, 64 B for K = 8). Decisions equal
      G independent serial replays that all start from P0.
  Mode B (serial-exact relay): the chains run in rank order; rank g receives
      (s, c) from rank g-1 before its selection kernel, sends its final
      (s, c) to rank g+1, and the last rank broadcasts the tick-end state.
      Decisions equal ONE serial replay of the concatenated batch (rank 0's
      rows, then rank 1's, ...) -- bit for bit, because (s, c) is exactly
      the reference's Neumaier state. Routers and predictors still run in
      parallel; only the short serial chains are ordered.

The functions below operate on torch tensors on any device, so the same
protocol code runs over NCCL on GPUs and over gloo on CPUs (tests).
"""

from __future__ import annotations

import hashlib

import torch
import torch.distributed as dist


def shard_of(program_id: str, world: int) -> int:
    """Stable program -> rank map (all stages of a program on one GPU)."""
    h = hashlib.blake2b(program_id.encode("utf-8"), digest_size=8).digest()
    return int.from_bytes(h, "big") % world


def neumaier_value_t(s: torch.Tensor, c: torch.Tensor) -> torch.Tensor:
    """Elementwise CPython-sum value of (s, c): s + c when c is finite and != 0."""
    use = torch.isfinite(c) & (c != 0)
    return torch.where(use, s + c, s)


def mode_a_allreduce(s: torch.Tensor, c: torch.Tensor, s0: torch.Tensor,
                     c0: torch.Tensor, group=None) -> None:
    """Mode A tick end: P = P0 + sum_g (P_g - P0); (s, c) <- (P, 0) in place."""
    p0 = neumaier_value_t(s0, c0)
    delta = neumaier_value_t(s, c) - p0
    dist.all_reduce(delta, group=group)
    s.copy_(p0 + delta)
    c.zero_()


def _p2p_buffer(state: torch.Tensor, group) -> torch.Tensor:
    # gloo point-to-point needs host tensors (NCCL takes the device tensor)
    if state.is_cuda and dist.get_backend(group) == "gloo":
        return state.cpu()
    return state


def relay_receive(state: torch.Tensor, group=None) -> None:
    """Mode B: before the selection chain, rank g > 0 receives the packed
    monitor state [2K] = (s, c) from rank g-1 (in place)."""
    rank = dist.get_rank(group)
    if rank > 0:
        buf = _p2p_buffer(state, group)
        dist.recv(buf, src=_global(rank - 1, group), group=group)
        if buf is not state:
            state.copy_(buf)


def relay_forward(state: torch.Tensor, group=None) -> None:
    """Mode B: after the chain, pass (s, c) on; the last rank broadcasts the
    tick-end state so every rank starts the next tick from it."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    buf = _p2p_buffer(state, group)
    if rank + 1 < world:
        dist.send(buf, dst=_global(rank + 1, group), group=group)
    dist.broadcast(buf, src=_global(world - 1, group), group=group)
    if buf is not state:
        state.copy_(buf)


def sharded_iteration(gs, group=None, release=None) -> None:
    """One scheduling iteration of every engine over the G sub-queues
    (global admission): each rank's STJF head candidates
    are all-gathered (NCCL; gloo over host copies), then every rank admits its
    share of the global top and ages its sub-queue (chm_queue_admit_merged).
    Equal to one EngineSim._iterate on the union queue (engine.py:328-338)."""
    cand = gs.queue_candidates()
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    send = _p2p_buffer(cand, group)
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    gathered = torch.stack(parts).to(cand.device)
    gs.queue_admit_merged(gathered, rank, release)


def _global(rank: int, group) -> int:
    return rank if group is None else dist.get_global_rank(group, rank)


# Engine counters relayed with (s, c) under global admission: they make the
# enqueue-time admission (running < max_batch_size), the seq tie-break and the
# clock check (engine.py:140-158) see the one reference engine.
_RELAYED = ("engine_running", "engine_seq", "engine_clock", "engine_iterations")


class ShardedScheduler:
    """Wraps a per-rank GpuScheduler with the Mode A / Mode B exchange.

    global_admission (Mode B only): each engine's queue is the union of the
    ranks' sub-queues, served in the reference's global STJF order. The relay
    also carries the engine counters, and every scheduling iteration, whether
    an explicit one or one per completion, is a `sharded_iteration`. Then the
    decisions, admissions and queue orders equal one serial replay of the
    concatenated batch through one EngineSim per model."""

    def __init__(self, scheduler, mode: str = "B", group=None, global_admission: bool = False):
        if mode not in ("A", "B"):
            raise ValueError("mode must be 'A' or 'B'")
        if global_admission and mode != "B":
            raise ValueError("global admission needs the Mode B relay")
        self.gs = scheduler
        self.mode = mode
        self.group = group
        self.global_admission = global_admission
        st = scheduler.state
        n = (2 + len(_RELAYED)) * st.K if global_admission else 2 * st.K
        self.packed = torch.empty(n, dtype=torch.float64, device=st.device)

    def _pack(self) -> None:
        st, K = self.gs.state, self.gs.state.K
        self.packed[:K].copy_(st.inflight_sum)
        self.packed[K:2 * K].copy_(st.inflight_comp)
        if self.global_admission:
            for i, name in enumerate(_RELAYED):
                self.packed[(2 + i) * K:(3 + i) * K].copy_(getattr(st, name))

    def _unpack(self) -> None:
        st, K = self.gs.state, self.gs.state.K
        st.inflight_sum.copy_(self.packed[:K])
        st.inflight_comp.copy_(self.packed[K:2 * K])
        if self.global_admission:
            for i, name in enumerate(_RELAYED):
                getattr(st, name).copy_(self.packed[(2 + i) * K:(3 + i) * K])

    def _run_global(self, batch, n_iterations: int, n_complete, kw) -> None:
        st = self.gs.state
        st.q_n_admitted.zero_()
        st.q_n_promoted.zero_()
        if n_complete is not None:
            # each completion frees a slot and runs one iteration of its engine
            # (engine.py:232-241); n_complete is the global count, equal on all ranks
            for r in range(int(n_complete.max().item()) if n_complete.numel() else 0):
                release = torch.where(n_complete > r, 1, -1).to(torch.int32)
                sharded_iteration(self.gs, self.group, release)
        self._pack()
        relay_receive(self.packed, self.group)
        self._unpack()
        self.gs.run_rows(batch, n_iterations=0, keep_admitted=True, **kw)
        self._pack()
        relay_forward(self.packed, self.group)
        self._unpack()
        for _ in range(n_iterations):
            sharded_iteration(self.gs, self.group)

    def run_rows(self, batch, n_iterations: int = 1, **kw) -> None:
        st = self.gs.state
        K = st.K
        if self.global_admission:
            if kw.get("completions") is not None:
                raise NotImplementedError("monitor completions are single-GPU; pass n_complete")
            self._run_global(batch, n_iterations, kw.pop("n_complete", None), kw)
            return
        if kw.get("completions") is not None:
            # each GPU's log holds only its own dispatches while (s, c) carries
            # the global volume: recomputing from the local log would drop the
            # other shards' contributions
            raise NotImplementedError("monitor completions are single-GPU; pass n_complete")
        if self.mode == "A":
            s0 = st.inflight_sum.clone()
            c0 = st.inflight_comp.clone()
            self.gs.run_rows(batch, n_iterations=n_iterations, **kw)
            mode_a_allreduce(st.inflight_sum, st.inflight_comp, s0, c0, self.group)
            return
        # Mode B: receive the predecessor's (s, c), run, forward.
        self.packed[:K].copy_(st.inflight_sum)
        self.packed[K:].copy_(st.inflight_comp)
        relay_receive(self.packed, self.group)
        st.inflight_sum.copy_(self.packed[:K])
        st.inflight_comp.copy_(self.packed[K:])
        self.gs.run_rows(batch, n_iterations=n_iterations, **kw)
        self.packed[:K].copy_(st.inflight_sum)
        self.packed[K:].copy_(st.inflight_comp)
        relay_forward(self.packed, self.group)
        st.inflight_sum.copy_(self.packed[:K])
        st.inflight_comp.copy_(self.packed[K:])
