"""Pool, balancer and aging configuration plus the Decision record.

Mirrors hetsched.profiles.ModelProfile/Pool (profiles.py:17-71),
hetsched.balancer.BalancerConfig/Decision (balancer.py:26-46) and
hetsched.engine.AgingConfig (engine.py:36-52): same fields, same validation.
Model index order on the device is `Pool.model_ids` = sorted(model_id), the
reference's tie-break order (profiles.py:56-59).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

from .errors import ValidationError


@dataclass(frozen=True)
class ModelProfile:
    model_id: str
    decode_ms_per_token: float
    max_batch_size: int
    prefill_ms_per_token: float = 0.0

    def __post_init__(self):
        if self.decode_ms_per_token <= 0:
            raise ValidationError(f"{self.model_id}: decode_ms_per_token must be > 0")
        if self.max_batch_size < 1:
            raise ValidationError(f"{self.model_id}: max_batch_size must be >= 1")
        if self.prefill_ms_per_token < 0:
            raise ValidationError(f"{self.model_id}: prefill_ms_per_token must be >= 0")


@dataclass(frozen=True)
class Pool:
    profiles: tuple[ModelProfile, ...]
    quality_order: tuple[str, ...] | None = None

    def __post_init__(self):
        if not self.profiles:
            raise ValidationError("pool must contain at least one model")
        ids = [p.model_id for p in self.profiles]
        if len(set(ids)) != len(ids):
            raise ValidationError(f"duplicate model ids in pool: {ids}")

    @property
    def model_ids(self) -> list[str]:
        return sorted(p.model_id for p in self.profiles)

    def __getitem__(self, model_id: str) -> ModelProfile:
        for p in self.profiles:
            if p.model_id == model_id:
                return p
        raise KeyError(model_id)

    def __contains__(self, model_id: str) -> bool:
        return any(p.model_id == model_id for p in self.profiles)

    def __len__(self) -> int:
        return len(self.profiles)


@dataclass(frozen=True)
class BalancerConfig:
    latency_slack: float = 0.5
    confidence_margin: float = 0.1

    def __post_init__(self):
        if self.latency_slack < 0:
            raise ValidationError(f"latency_slack must be >= 0, got {self.latency_slack}")
        if not 0.0 <= self.confidence_margin <= 1.0:
            raise ValidationError(
                f"confidence_margin must be in [0,1], got {self.confidence_margin}"
            )


@dataclass(frozen=True)
class AgingConfig:
    starvation_threshold: float = 8
    running_quantum: int = 4
    demote_while_queued: bool = False

    def __post_init__(self):
        if self.starvation_threshold < 1:
            raise ValidationError("starvation_threshold must be >= 1 (or inf)")
        if self.running_quantum < 1:
            raise ValidationError("running_quantum must be >= 1")

    @property
    def enabled(self) -> bool:
        return not math.isinf(self.starvation_threshold)


AGING_DISABLED = AgingConfig(starvation_threshold=math.inf)


try:  # the reference's own record when hetsched is importable (balancer.py:40-46)
    from hetsched.balancer import Decision  # pragma: no cover
except ImportError:
    @dataclass(frozen=True)
    class Decision:
        model: str
        priority: float
        estimated_loads: dict[str, float]
        used_cached_assignment: bool
        scores: dict[str, float] | None = None
