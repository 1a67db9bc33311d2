"""Columnar trace store on the device.

hetsched keeps a trace as a list of TraceRecord objects
(/root/reference/pkg/src/hetsched/workload.py:111-253) and answers
`remaining_tokens`, `out_tokens`, `first_stage_request` and
`next_stage_request` (workload.py:160-165, 154-155, 454-495) by walking those
objects per call. Here the same fields are dense SoA columns in HBM, indexed
by a dense program number, and the derived columns (output-token suffix sums,
carried-context prefix sums) are computed once by chm_trace_derive. Per tick
the scheduling path then gathers what it needs by (program, stage) on the
device: `out_tokens` for EngineSim.enqueue, the OraclePredictor prediction,
the next stage's request for every completion.

`load_ndjson` reads the reference's trace file format (workload.py:9-20,
load_trace 256-291) with the same validation and error types; records built
in memory (workload.TraceRecord or the reference's own) go through
`TraceStore.from_records`.
"""

from __future__ import annotations

import json

import numpy as np
import torch

from . import _lib
from .errors import ParseError, ValidationError


def _p(t):
    return None if t is None else t.data_ptr()


class TraceColumns:
    """Host (numpy) columns of a trace, program-major, stages padded to S."""

    def __init__(self, n_programs: int, max_stages: int, model_ids):
        self.model_ids = list(model_ids)
        NP, S, K = n_programs, max_stages, len(self.model_ids)
        self.program_ids: list[str] = [""] * NP
        self.workflow_ids: list[str] = [""] * NP
        self.n_stages = np.zeros(NP, np.int32)
        self.user_arrival = np.zeros(NP, np.float64)
        self.base_input = np.zeros((NP, S), np.int32)
        self.out_tokens = np.zeros((NP, S, K), np.int32)
        self.carried = np.zeros((NP, S, K), np.int32)

    @property
    def max_stages(self) -> int:
        return self.base_input.shape[1]


def _i32(v, what: str) -> int:
    v = int(v)
    if not -(2**31) <= v < 2**31:
        raise ValidationError(f"{what} {v} does not fit the int32 trace columns")
    return v


def columns_from_records(records, model_ids=None, max_stages: int | None = None) -> TraceColumns:
    """TraceRecord objects (this package's or hetsched's) -> columns. The
    pool order is sorted(model_id) (profiles.py:48-52); every record must carry
    every pool model (TraceRecord.validate, workload.py:180-183)."""
    if model_ids is None:
        model_ids = sorted(records[0].success) if records else []
    S = max_stages or max((len(r.stages) for r in records), default=1)
    cols = TraceColumns(len(records), S, model_ids)
    for p, rec in enumerate(records):
        _fill(cols, p, rec.program_id, rec.workflow_id, rec.user_arrival_time_ms,
              [(st.stage_index, st.base_input_tokens,
                {m: (o.out_tokens, o.carried_context_tokens) for m, o in st.models.items()})
               for st in rec.stages], set(rec.success), f"{rec.program_id}")
    return cols


def _fill(cols: TraceColumns, p: int, pid, wid, arrival, stages, models: set, where: str):
    S = cols.max_stages
    if len(stages) > S:
        raise ValidationError(f"{where}: {len(stages)} stages exceed max_stages={S}")
    missing = set(cols.model_ids) - models
    if missing:
        raise ValidationError(f"{where}: missing model entries {sorted(missing)}")
    cols.program_ids[p] = pid
    cols.workflow_ids[p] = wid
    cols.n_stages[p] = len(stages)
    cols.user_arrival[p] = float(arrival)
    for j, (idx, base, outs) in enumerate(stages):
        if idx != j + 1:
            raise ValidationError(f"{where}: stage indices must be contiguous from 1")
        cols.base_input[p, j] = _i32(base, "base_input_tokens")
        for k, m in enumerate(cols.model_ids):
            o, c = outs[m]
            cols.out_tokens[p, j, k] = _i32(o, "out_tokens")
            cols.carried[p, j, k] = _i32(c, "carried_context_tokens")


def load_ndjson(path: str, model_ids=None, max_stages: int | None = None,
                expected_models: set | None = None) -> TraceColumns:
    """Read a trace file into columns with load_trace's checks and errors
    (workload.py:256-291): ParseError(line) for bad JSON / non-objects /
    missing or ill-typed fields, ValidationError("line N: ...") for records
    that fail TraceRecord.validate (workload.py:170-200), and for a model set
    differing from earlier records."""
    parsed = []
    model_set = None
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                obj = json.loads(line)
            except json.JSONDecodeError as exc:
                raise ParseError(lineno, f"invalid JSON: {exc.msg}")
            if not isinstance(obj, dict):
                raise ParseError(lineno, "record is not a JSON object")
            try:  # TraceRecord.from_json_dict (workload.py:227-253)
                stages = [(int(s["stage_index"]), int(s["base_input_tokens"]),
                           {mid: (int(o["out_tokens"]), int(o["carried_context_tokens"]))
                            for mid, o in s["models"].items()})
                          for s in obj["stages"]]
                rec = (str(obj["program_id"]), str(obj["workflow_id"]),
                       float(obj["user_arrival_time_ms"]), stages,
                       {mid: int(v) for mid, v in obj["success"].items()})
                str(obj["difficulty"])
            except (KeyError, TypeError, ValueError) as exc:
                raise ParseError(lineno, f"bad trace record: {exc}")
            try:
                _validate(rec, expected_models)
            except ValidationError as exc:
                raise ValidationError(f"line {lineno}: {exc}")
            models = set(rec[4])
            if model_set is None:
                model_set = models
            elif models != model_set:
                raise ValidationError(
                    f"line {lineno}: model set {sorted(models)} differs from "
                    f"earlier records {sorted(model_set)}")
            parsed.append(rec)
    if model_ids is None:
        model_ids = sorted(model_set or [])
    S = max_stages or max((len(r[3]) for r in parsed), default=1)
    cols = TraceColumns(len(parsed), S, model_ids)
    for p, (pid, wid, arr, stages, success) in enumerate(parsed):
        _fill(cols, p, pid, wid, arr, stages, set(success), pid)
    return cols


def _validate(rec, expected_models):
    """TraceRecord.validate (workload.py:170-200) on a parsed tuple."""
    pid, _, arrival, stages, success = rec
    if not stages:
        raise ValidationError(f"{pid}: no stages")
    if arrival < 0:
        raise ValidationError(f"{pid}: negative user_arrival_time_ms")
    models = set(success)
    if not models:
        raise ValidationError(f"{pid}: empty success map")
    if expected_models is not None and not set(expected_models) <= models:
        missing = sorted(set(expected_models) - models)
        raise ValidationError(f"{pid}: missing model entries {missing}")
    for flag in success.values():
        if flag not in (0, 1):
            raise ValidationError(f"{pid}: success flags must be 0 or 1")
    for i, (idx, base, outs) in enumerate(stages, start=1):
        if idx != i:
            raise ValidationError(f"{pid}: stage indices must be contiguous from 1")
        if base < 1:
            raise ValidationError(f"{pid}: stage {i} base_input_tokens < 1")
        if set(outs) != models:
            raise ValidationError(
                f"{pid}: stage {i} model entries {sorted(outs)} do not match success map "
                f"{sorted(models)}")
        for mid, (o, c) in outs.items():
            if o < 0 or c < 0:
                raise ValidationError(f"{pid}: stage {i} model {mid}: negative token count")


class TraceStore:
    """Device-resident trace columns + derived columns for one pool."""

    def __init__(self, cols: TraceColumns, device="cuda", workflow_index: dict | None = None,
                 stream=None):
        self.cols = cols
        self.device = torch.device(device)
        self.model_ids = cols.model_ids
        self.K = len(self.model_ids)
        self.S = cols.max_stages
        self.n_programs = len(cols.program_ids)
        self.program_index = {pid: i for i, pid in enumerate(cols.program_ids)}
        wf = np.array([(workflow_index or {}).get(w, -1) for w in cols.workflow_ids], np.int32)
        d = self.device
        up = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=d)  # noqa: E731
        self.n_stages = up(cols.n_stages)
        self.workflow = up(wf)
        self.user_arrival = up(cols.user_arrival)
        self.base_input = up(cols.base_input)
        self.out_tokens = up(cols.out_tokens)
        self.carried = up(cols.carried)
        shape = (self.n_programs, self.S, self.K)
        self.remaining = torch.empty(shape, dtype=torch.int64, device=d)
        self.carried_prefix = torch.empty(shape, dtype=torch.int64, device=d)
        self.error = torch.zeros(4, dtype=torch.int32, device=d)
        self.t = _lib.Trace(self.n_programs, self.S, self.K, _p(self.n_stages), _p(self.workflow),
                            _p(self.user_arrival), _p(self.base_input), _p(self.out_tokens),
                            _p(self.carried), _p(self.remaining), _p(self.carried_prefix))
        self.lib = _lib.load()
        self.derive(stream)

    @classmethod
    def from_records(cls, records, model_ids=None, device="cuda", max_stages=None,
                     workflow_index=None):
        return cls(columns_from_records(records, model_ids, max_stages), device, workflow_index)

    @classmethod
    def from_ndjson(cls, path, model_ids=None, device="cuda", max_stages=None,
                    workflow_index=None, expected_models=None):
        return cls(load_ndjson(path, model_ids, max_stages, expected_models), device,
                   workflow_index)

    # ---- device entry points -------------------------------------------------
    def _stream(self, stream):
        return (stream if stream is not None else torch.cuda.current_stream(self.device)).cuda_stream

    def _reset_error(self):
        self.error.copy_(torch.tensor([0, 2**31 - 1, -1, 0], dtype=torch.int32))

    def check_errors(self, context: str) -> None:
        err = self.error.cpu().tolist()
        if err[0] != _lib.CHM_OK:
            _lib.raise_device_error(err, context)

    def derive(self, stream=None) -> None:
        self._reset_error()
        _lib.check(self.lib.chm_trace_derive(self.t, _p(self.error), self._stream(stream)),
                   "chm_trace_derive")
        self.check_errors("trace")

    def gather_rows(self, program: torch.Tensor, stage: torch.Tensor, out_tokens=None,
                    workflow=None, n_stages=None, oracle=None, stream=None,
                    check: bool = True) -> None:
        """Fill the given [B, K] / [B] outputs for rows (program, stage)."""
        if check:
            self._reset_error()
        _lib.check(self.lib.chm_trace_gather_rows(
            self.t, _p(program), _p(stage), int(program.shape[0]), _p(out_tokens), _p(workflow),
            _p(n_stages), _p(oracle), _p(self.error), self._stream(stream)),
            "chm_trace_gather_rows")
        if check:
            self.check_errors("gather_rows")

    def next_stage(self, program, completed_stage, completion_time, model, stream=None,
                   check: bool = True) -> dict:
        """next_stage_request for every completion; returns device columns of
        the next-stage requests (compacted, completion order) and their count."""
        n = int(program.shape[0])
        d = self.device
        out = {
            "program": torch.empty(n, dtype=torch.int32, device=d),
            "stage": torch.empty(n, dtype=torch.int32, device=d),
            "arrival": torch.empty(n, dtype=torch.float64, device=d),
            "input_tokens": torch.empty(n, dtype=torch.int32, device=d),
            "workflow": torch.empty(n, dtype=torch.int32, device=d),
            "source_row": torch.empty(n, dtype=torch.int32, device=d),
            "n": torch.zeros(1, dtype=torch.int32, device=d),
        }
        if check:
            self._reset_error()
        _lib.check(self.lib.chm_trace_next_stage(
            self.t, _p(program), _p(completed_stage), _p(completion_time), _p(model), n,
            _p(out["program"]), _p(out["stage"]), _p(out["arrival"]), _p(out["input_tokens"]),
            _p(out["workflow"]), _p(out["source_row"]), _p(out["n"]), _p(self.error),
            self._stream(stream)), "chm_trace_next_stage")
        if check:
            self.check_errors("next_stage")
        return out

    def first_stage(self, program: torch.Tensor, arrival: torch.Tensor | None = None,
                    stream=None) -> dict:
        n = int(program.shape[0])
        d = self.device
        out = {"input_tokens": torch.empty(n, dtype=torch.int32, device=d),
               "arrival": torch.empty(n, dtype=torch.float64, device=d),
               "workflow": torch.empty(n, dtype=torch.int32, device=d)}
        self._reset_error()
        _lib.check(self.lib.chm_trace_first_stage(
            self.t, _p(program), _p(arrival), n, _p(out["input_tokens"]), _p(out["arrival"]),
            _p(out["workflow"]), _p(self.error), self._stream(stream)), "chm_trace_first_stage")
        self.check_errors("first_stage")
        return out

    def make_batch(self, program: torch.Tensor, stage: torch.Tensor, arrival: torch.Tensor,
                   handle: torch.Tensor | None = None, token_ids: torch.Tensor | None = None,
                   stream=None):
        """A scheduler RowBatch for rows (program, stage) whose per-model
        out_tokens (the EngineSim.enqueue argument, balancer.py:117-122) and
        workflow index are gathered from the store on the device."""
        from .scheduler import RowBatch
        B, d = int(program.shape[0]), self.device
        out_tokens = torch.empty(B, self.K, dtype=torch.int32, device=d)
        workflow = torch.empty(B, dtype=torch.int32, device=d)
        self.gather_rows(program, stage, out_tokens=out_tokens, workflow=workflow, stream=stream)
        if handle is None:
            handle = torch.arange(B, dtype=torch.int64, device=d)
        return RowBatch(program=program, stage=stage, arrival=arrival, out_tokens=out_tokens,
                        handle=handle, workflow=workflow, token_ids=token_ids)

    @property
    def bytes_derive(self) -> int:
        """Algorithmic HBM bytes of chm_trace_derive: out_tokens + carried
        read (4 + 4), remaining + carried_prefix written (8 + 8) per entry,
        base_input (4 per program-stage) and n_stages (4 per program) read for
        the validation."""
        return self.n_programs * (self.S * (self.K * 24 + 4) + 4)


def model_index(model_ids, model_id: str) -> int:
    try:
        return list(model_ids).index(model_id)
    except ValueError:
        raise ValidationError(f"unknown model {model_id!r}") from None


__all__ = ["TraceColumns", "TraceStore", "columns_from_records", "load_ndjson", "model_index"]
