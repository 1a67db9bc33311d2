"""Request / trace data model and the seeded synthetic trace generator.

Field names and semantics follow hetsched.workload
(/root/reference/pkg/src/hetsched/workload.py) so that objects built here can
be handed to the reference functions (and vice versa) in parity tests:
  Request            workload.py:87-108   (request_id = "pid:stage")
  TraceRecord        workload.py:125-165  (remaining_tokens = suffix sum)
  WorkflowSpec       workload.py:42-58, templates 67-77
  synthesize_trace   workload.py:314-416  (same RNG call order => same trace)
  first/next_stage_request  workload.py:454-495

Only the accessors the scheduling path reads are kept; trace file I/O and
arrival processes are harness concerns outside the hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2603_22206_b200.errors import InvalidStats, UnknownStage, ValidationError


@dataclass(frozen=True)
class StageSpec:
    role: str
    index: int


@dataclass(frozen=True)
class WorkflowSpec:
    workflow_id: str
    stages: tuple[StageSpec, ...]

    def __post_init__(self):
        if not self.stages:
            raise ValidationError(f"workflow {self.workflow_id!r} has no stages")
        if [s.index for s in self.stages] != list(range(1, len(self.stages) + 1)):
            raise ValidationError(
                f"workflow {self.workflow_id!r}: stage indices must be contiguous from 1"
            )

    @property
    def n_stages(self) -> int:
        return len(self.stages)


def workflow(workflow_id: str, *roles: str) -> WorkflowSpec:
    return WorkflowSpec(workflow_id, tuple(StageSpec(r, k) for k, r in enumerate(roles, 1)))


CODE_WORKFLOWS = (
    workflow("code-4stage", "planner", "coder", "qa_agent", "coder"),
    workflow("code-2stage", "planner", "coder"),
    workflow("code-1stage", "coder"),
)
MATH_WORKFLOWS = (
    workflow("math-4stage", "planner", "solver", "verifier", "solver"),
    workflow("math-2stage", "planner", "solver"),
    workflow("math-1stage", "solver"),
)


@dataclass(frozen=True)
class Request:
    program_id: str
    stage_index: int
    input_tokens: int
    arrival_time: float
    workflow_id: str
    role: str

    def __post_init__(self):
        if self.stage_index < 1:
            raise ValidationError(f"stage_index must be >= 1, got {self.stage_index}")
        if self.input_tokens <= 0:
            raise ValidationError(f"input_tokens must be > 0, got {self.input_tokens}")
        if self.arrival_time < 0:
            raise ValidationError(f"arrival_time must be >= 0, got {self.arrival_time}")

    @property
    def request_id(self) -> str:
        return f"{self.program_id}:{self.stage_index}"


@dataclass(frozen=True)
class ModelStageOutput:
    out_tokens: int
    carried_context_tokens: int


@dataclass
class StageTrace:
    stage_index: int
    role: str
    base_input_tokens: int
    models: dict[str, ModelStageOutput]


@dataclass
class TraceRecord:
    program_id: str
    workflow_id: str
    user_arrival_time_ms: float
    stages: list[StageTrace]
    success: dict[str, int]
    difficulty: str

    @property
    def n_stages(self) -> int:
        return len(self.stages)

    def _stage(self, stage_index: int) -> StageTrace:
        if not 1 <= stage_index <= len(self.stages):
            raise UnknownStage(
                f"{self.program_id}: stage {stage_index} outside 1..{len(self.stages)}"
            )
        return self.stages[stage_index - 1]

    def base_input(self, stage_index: int) -> int:
        return self._stage(stage_index).base_input_tokens

    def out_tokens(self, stage_index: int, model_id: str) -> int:
        return self._stage(stage_index).models[model_id].out_tokens

    def carried_context(self, stage_index: int, model_id: str) -> int:
        return self._stage(stage_index).models[model_id].carried_context_tokens

    def remaining_tokens(self, from_stage: int, model_id: str) -> int:
        self._stage(from_stage)
        total = 0
        for st in self.stages[from_stage - 1:]:
            total += st.models[model_id].out_tokens
        return total


@dataclass(frozen=True)
class LengthStats:
    mean: float
    std: float

    def __post_init__(self):
        if self.mean <= 0:
            raise InvalidStats(f"mean must be > 0, got {self.mean}")
        if self.std < 0:
            raise InvalidStats(f"std must be >= 0, got {self.std}")


def _moment_matched_lognormal(mean: float, std: float) -> tuple[float, float]:
    var_log = math.log(1.0 + (std / mean) ** 2)
    return math.log(mean) - var_log / 2.0, math.sqrt(var_log)


def _largest_remainder(total: int, weights: list[float]) -> list[int]:
    wsum = sum(weights)
    shares = [total * w / wsum for w in weights]
    parts = [int(math.floor(x)) for x in shares]
    leftover = total - sum(parts)
    by_fraction = sorted(range(len(shares)), key=lambda k: (-(shares[k] - parts[k]), k))
    for k in by_fraction[:leftover]:
        parts[k] += 1
    return parts


def synthesize_trace(templates, stats, success_rates, n, seed, *, difficulty_mix=None,
                     template_mix=None, role_weights=None,
                     input_stats=LengthStats(256.0, 128.0)) -> list[TraceRecord]:
    """Seeded lognormal trace, draw-for-draw identical to workload.py:334-416."""
    if n <= 0:
        raise ValidationError(f"n must be > 0, got {n}")
    if not templates or not stats:
        raise ValidationError("templates and stats must be non-empty")
    models = sorted(stats)
    mix = difficulty_mix or {"easy": 0.5, "hard": 0.5}
    diffs = sorted(mix)
    p_diff = np.array([mix[d] for d in diffs], dtype=float)
    p_diff = p_diff / p_diff.sum()
    p_tmpl = np.array(template_mix or [1.0] * len(templates), dtype=float)
    p_tmpl = p_tmpl / p_tmpl.sum()
    for mid in models:
        if mid not in success_rates or any(d not in success_rates[mid] for d in diffs):
            raise ValidationError(f"missing success rates for model {mid!r}")
    rng = np.random.default_rng(seed)
    ln_params = {mid: _moment_matched_lognormal(stats[mid].mean, stats[mid].std) for mid in models}
    in_mu, in_sigma = _moment_matched_lognormal(
        input_stats.mean, max(input_stats.std, 0.0) or 1e-12
    )
    out: list[TraceRecord] = []
    for k in range(n):
        wf = templates[int(rng.choice(len(templates), p=p_tmpl))]
        diff = diffs[int(rng.choice(len(diffs), p=p_diff))]
        weights = [(role_weights or {}).get(s.role, 1.0) for s in wf.stages]
        base = [max(1, int(round(rng.lognormal(in_mu, in_sigma)))) for _ in wf.stages]
        per_stage: list[dict[str, ModelStageOutput]] = [{} for _ in wf.stages]
        success: dict[str, int] = {}
        for mid in models:
            if stats[mid].std == 0:
                total = max(1, int(round(stats[mid].mean)))
            else:
                total = max(1, int(round(rng.lognormal(*ln_params[mid]))))
            for j, tok in enumerate(_largest_remainder(total, weights)):
                per_stage[j][mid] = ModelStageOutput(tok, tok)
            success[mid] = int(rng.random() < success_rates[mid][diff])
        stages = [StageTrace(s.index, s.role, base[s.index - 1], per_stage[s.index - 1])
                  for s in wf.stages]
        out.append(TraceRecord(f"p{k:06d}", wf.workflow_id, 0.0, stages, success, diff))
    return out


def first_stage_request(rec: TraceRecord, arrival_time: float | None = None) -> Request:
    st = rec.stages[0]
    t = rec.user_arrival_time_ms if arrival_time is None else arrival_time
    return Request(rec.program_id, 1, st.base_input_tokens, t, rec.workflow_id, st.role)


def next_stage_request(rec: TraceRecord, completed_stage: int, completion_time: float,
                       assigned_model: str) -> Request | None:
    if not 1 <= completed_stage <= rec.n_stages:
        raise UnknownStage(
            f"{rec.program_id}: completed stage {completed_stage} outside 1..{rec.n_stages}"
        )
    if completed_stage == rec.n_stages:
        return None
    nxt = completed_stage + 1
    carried = sum(rec.carried_context(j, assigned_model) for j in range(1, nxt))
    st = rec.stages[nxt - 1]
    return Request(rec.program_id, nxt, st.base_input_tokens + carried, completion_time,
                   rec.workflow_id, st.role)
