"""Routers: per-model confidence q[m] in [0, 1] for the rows that need routing.

Protocol (device side): `score_rows(batch, route_rows, n_route, scores, stream)`
writes the fp64 scores[row * K + m] for every row listed in
route_rows[:n_route] (chm_prepare_rows compacts the rows with no assignment;
the reference calls the router only on that branch, balancer.py:104-114).
Each router also keeps the reference's `score(req, rec, pool) ->
ConfidenceVector` (router.py:34-45), and routers whose inputs come from the
request objects provide `columns_for(reqs, recs)` so
`GpuScheduler.schedule_batch(reqs, recs)` can build the device batch.

  GpuEncoderRouter   the semantic router: BERT-style encoder + CLS sigmoid
                     head on hand-written sm_100a kernels (encoder.py)
  ConstantRouter     router.py:57-68, filled on device
  ScoreTableRouter   scores supplied per batch as a [B, K] tensor (the parity
                     harness's stand-in for the reference Router shims)
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .errors import ValidationError

try:  # the reference's own class when hetsched is importable
    from hetsched.router import ConfidenceVector  # pragma: no cover
except ImportError:
    @dataclass(frozen=True)
    class ConfidenceVector:
        """hetsched.router.ConfidenceVector (router.py:21-31)."""

        scores: dict[str, float]

        def __post_init__(self):
            for mid, q in self.scores.items():
                if not 0.0 <= q <= 1.0:
                    raise ValidationError(f"score for {mid!r} outside [0,1]: {q}")

        def __getitem__(self, model_id: str) -> float:
            return self.scores[model_id]


class ConstantRouter:
    name = "constant"

    def __init__(self, value: float):
        if not 0.0 <= value <= 1.0:
            raise ValidationError(f"constant score must be in [0,1], got {value}")
        self.value = float(value)

    def score(self, req, rec, pool) -> ConfidenceVector:
        return ConfidenceVector({mid: self.value for mid in pool.model_ids})

    def score_rows(self, batch, route_rows, n_route, scores, stream) -> None:
        scores.fill_(self.value)


class ScoreTableRouter:
    name = "score-table"

    def __init__(self):
        self.values: torch.Tensor | None = None

    def set(self, values: torch.Tensor) -> None:
        self.values = values

    def score_rows(self, batch, route_rows, n_route, scores, stream) -> None:
        n = self.values.numel()
        scores[:n].copy_(self.values.reshape(-1), non_blocking=True)
