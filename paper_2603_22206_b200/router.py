"""Routers: per-model confidence q[m] in [0, 1] for the rows that need routing.

Protocol (device side): `score_rows(batch, route_rows, n_route, scores, stream)`
writes scores[row * K + m] for every row listed in route_rows[:n_route]
(chm_prepare_rows compacts the rows with no assignment; the reference calls
the router only on that branch, balancer.py:104-114). Each router also keeps
the reference's `score(req, rec, pool)` (router.py:39-42).

  GpuEncoderRouter   the semantic router: BERT-style encoder + CLS sigmoid
                     head on hand-written sm_100a kernels (encoder.py)
  ConstantRouter     router.py:57-68, filled on device
  ScoreTableRouter   scores supplied per batch as a [B, K] tensor (the parity
                     harness's stand-in for the reference Router shims)
"""

from __future__ import annotations

import torch

from .errors import ValidationError


class ConstantRouter:
    name = "constant"

    def __init__(self, value: float):
        if not 0.0 <= value <= 1.0:
            raise ValidationError(f"constant score must be in [0,1], got {value}")
        self.value = float(value)

    def score(self, req, rec, pool) -> dict:
        return {mid: self.value for mid in pool.model_ids}

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
