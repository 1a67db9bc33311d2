"""Trace store host side, CPU only: the ndjson reader
against load_trace's golden behaviour, and the oracle restatement
(oracle/trace_ref.py) against the reference's answers for every
(program, stage, model) of tests/golden/trace_small.*."""

import json
import os

import numpy as np
import pytest

from oracle import trace_ref
from paper_2603_22206_b200 import errors
from paper_2603_22206_b200.trace import load_ndjson

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "trace_small.npz"))


@pytest.fixture(scope="module")
def cols():
    return load_ndjson(os.path.join(GOLD, "trace_small.ndjson"))


def test_columns_match_reference_reader(cols, gold):
    assert cols.model_ids == list(gold["model_ids"])
    assert cols.program_ids == list(gold["program_ids"])
    assert np.array_equal(cols.n_stages, gold["n_stages"])
    assert cols.max_stages == gold["remaining"].shape[1]


def test_oracle_remaining_and_first_stage(cols, gold):
    rem = trace_ref.ref_remaining(cols.n_stages, cols.out_tokens)
    want = gold["remaining"]
    live = want >= 0
    assert np.array_equal(rem[live], want[live])
    assert np.all(rem[~live] == 0)
    inp, arr = trace_ref.ref_first_stage(cols.base_input, cols.user_arrival,
                                         np.arange(len(cols.program_ids)))
    assert np.array_equal(inp, gold["first_input"])
    assert np.array_equal(arr, gold["first_arrival"])


def test_oracle_next_stage(cols, gold):
    NP, S, K = gold["remaining"].shape
    prog, comp, time, model = [], [], [], []
    for p in range(NP):
        for s in range(1, int(cols.n_stages[p]) + 1):
            for k in range(K):
                prog.append(p), comp.append(s), time.append(1000.0 + p + 0.25 * s)
                model.append(k)
    got = trace_ref.ref_next_stage(cols.n_stages, cols.base_input, cols.carried, prog, comp,
                                   time, model)
    emitted = {src for src, *_ in got}
    for src, p, st, t, inp in got:
        assert st == comp[src] + 1
        assert inp == gold["next_input"][p, comp[src] - 1, model[src]]
        assert t == gold["next_arrival"][p, comp[src] - 1, model[src]]
    for i in range(len(prog)):
        final = gold["next_input"][prog[i], comp[i] - 1, model[i]] < 0
        assert (i not in emitted) == final
    for s, name in gold["unknown"]:
        with pytest.raises(ValueError):
            trace_ref.ref_next_stage(cols.n_stages, cols.base_input, cols.carried, [0],
                                     [int(s)], [0.0], [0])
        assert name == "UnknownStage"


def test_carried_prefix_identity(cols):
    pre = trace_ref.ref_carried_prefix(cols.n_stages, cols.carried)
    for p in range(len(cols.program_ids)):
        for s in range(int(cols.n_stages[p])):
            assert np.array_equal(pre[p, s], cols.carried[p, :s].astype(np.int64).sum(0))


@pytest.mark.parametrize("case", sorted(json.load(open(os.path.join(GOLD,
                                                                    "trace_errors.json")))))
def test_reader_errors_match_reference(case, tmp_path):
    spec = json.load(open(os.path.join(GOLD, "trace_errors.json")))[case]
    path = tmp_path / "t.ndjson"
    path.write_text(spec["text"])
    if spec["error"] is None:
        assert len(load_ndjson(str(path)).program_ids) == spec["n"]
        return
    cls = getattr(errors, spec["error"])
    with pytest.raises(cls) as ei:
        load_ndjson(str(path))
    assert str(ei.value) == spec["message"]
    if spec["line"] is not None:
        assert ei.value.line == spec["line"]
