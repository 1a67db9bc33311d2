"""CPU restatement of the reference's trace accessors -- TEST INFRASTRUCTURE.

Checker for the device trace store (paper_2603_22206_b200/trace.py,
csrc/trace.cu). Restates, on dense numpy columns (program p, 0-based stage s
padded to S, model k in pool order), the per-record functions of
/root/reference/pkg/src/hetsched/workload.py:

  ref_remaining     TraceRecord.remaining_tokens   workload.py:160-165
                    (sum of out_tokens of stages from_stage..N)
  ref_next_stage    next_stage_request             workload.py:467-495
                    (None after the final stage; input = base of the next
                    stage + carried context of stages 1..completed under the
                    assigned model; arrival = completion time)
  ref_first_stage   first_stage_request            workload.py:454-464

Pinned against tests/golden/trace_small.* (written by the unmodified
reference, tests/golden/make_golden.py::make_trace) in tests/test_trace.py.
"""

from __future__ import annotations

import numpy as np


def ref_remaining(n_stages, out_tokens):
    """[NP, S, K] int64: remaining[p, s, k] for s < n_stages[p], else 0."""
    NP, S, K = out_tokens.shape
    live = np.arange(S)[None, :] < np.asarray(n_stages)[:, None]            # [NP, S]
    o = np.where(live[..., None], out_tokens.astype(np.int64), 0)
    rem = np.flip(np.cumsum(np.flip(o, axis=1), axis=1), axis=1)
    return np.where(live[..., None], rem, 0)


def ref_carried_prefix(n_stages, carried):
    """[NP, S, K] int64: sum_{j < s} carried[p, j, k] for s < n_stages[p], else 0."""
    NP, S, K = carried.shape
    live = np.arange(S)[None, :] < np.asarray(n_stages)[:, None]
    c = np.where(live[..., None], carried.astype(np.int64), 0)
    pre = np.cumsum(c, axis=1) - c
    return np.where(live[..., None], pre, 0)


def ref_next_stage(n_stages, base_input, carried, program, completed, time, model):
    """Completions -> list of (source_row, program, stage, arrival, input) in
    completion order; raises ValueError('UnknownStage', row) like the
    reference's UnknownStage for a completed stage outside 1..N."""
    out = []
    for i, (p, s, t, m) in enumerate(zip(program, completed, time, model)):
        n = int(n_stages[p])
        if not 1 <= s <= n:
            raise ValueError("UnknownStage", i)
        if s == n:
            continue
        carried_sum = int(np.asarray(carried[p, :s, m], np.int64).sum())
        out.append((i, int(p), int(s) + 1, float(t), int(base_input[p, s]) + carried_sum))
    return out


def ref_first_stage(base_input, user_arrival, program, arrival=None):
    inp = np.asarray(base_input)[np.asarray(program), 0].astype(np.int64)
    arr = np.asarray(user_arrival)[np.asarray(program)] if arrival is None else np.asarray(arrival)
    return inp, arr
