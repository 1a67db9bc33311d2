"""One scheduling tick captured as a CUDA graph.

`TickGraph` captures (state restore) -> chm_prepare_rows -> router ->
predictor -> chm_schedule_rows -> chm_queue_tick for a fixed batch shape on
one stream and replays it; per tick the caller only refreshes the captured
input tensors (device-to-device or host-to-device copies) before `replay()`.
Every pointer and size the kernels see is baked into the graph (the library
allocates nothing and its epoch counter lives in device memory), so replays
are exactly the eager sequence without the ~100-300 host launches.
"""

from __future__ import annotations

import torch

from . import _lib
from .scheduler import RowBatch


class TickGraph:
    def __init__(self, scheduler, batch: RowBatch, n_iterations: int = 1,
                 restore_snapshot: dict | None = None, warmup: int = 1, n_complete=None,
                 completions=None):
        self.gs = scheduler
        self.batch = batch
        self.snapshot = restore_snapshot
        self.n_iterations = n_iterations
        self.n_complete = n_complete
        self.completions = completions
        dev = scheduler.device
        self.stream = torch.cuda.Stream(dev)
        _lib.profile_enable(False)
        # warm up on the capture stream (allocator, attributes, tensor maps)
        self.stream.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(self.stream):
            for _ in range(warmup):
                self._body()
        torch.cuda.current_stream(dev).wait_stream(self.stream)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=self.stream):
            self._body()
        torch.cuda.synchronize(dev)

    def _body(self):
        if self.snapshot is not None:
            self.gs.state.restore(self.snapshot)
        self.gs.run_rows(self.batch, n_iterations=self.n_iterations, n_complete=self.n_complete,
                         stream=torch.cuda.current_stream(), completions=self.completions)

    def replay(self) -> None:
        self.graph.replay()
