"""Device predictor evaluation (csrc/evaluate.cu) against the reference's
values (tests/golden/kendall.npz), bit-exact fp64, and against the oracle
restatement's integer counts."""

import os

import numpy as np
import pytest
import torch

from oracle import eval_ref
from paper_2603_22206_b200.evaluate import (LengthMismatch, arrival_order_distance,
                                            evaluate_predictor, kendall_tau_distance)

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "kendall.npz"))


def test_kendall_cases(gold):
    for name in gold["cases"]:
        p, t = gold[f"{name}_p"], gold[f"{name}_t"]
        d, counts = kendall_tau_distance(p, t, return_counts=True)
        assert d == float(gold[f"{name}_d"]), name
        if len(p) <= 1000:
            want, _ = eval_ref.ref_kendall_counts(p.tolist(), t.tolist())
            assert counts == want, name


def test_kendall_errors():
    with pytest.raises(LengthMismatch):
        kendall_tau_distance([1.0, 2.0], [1.0])
    with pytest.raises(LengthMismatch):
        kendall_tau_distance([1.0], [1.0])


def test_kendall_large_identities():
    """n = 2^21 + 3: identical rankings 0, reversed 1, symmetry in its
    arguments; integer-valued (heavily tied) data against pair counts."""
    n = (1 << 21) + 3
    g = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    assert kendall_tau_distance(x, x) == 0.0
    assert kendall_tau_distance(x, -x) == 1.0
    a = torch.randint(0, 1000, (n,), device="cuda", generator=g).double()
    b = torch.randint(0, 1000, (n,), device="cuda", generator=g).double()
    assert kendall_tau_distance(a, b) == kendall_tau_distance(b, a)
    _, c = kendall_tau_distance(a, a, return_counts=True)
    counts = torch.bincount(a.long()).double()
    assert c[1] == c[2] == c[3] == int((counts * (counts - 1) / 2).sum().item())
    assert c[0] == 0


def test_evaluate_predictor_on_trace(gold):
    from paper_2603_22206_b200.predictor import (GpuInputLengthPredictor, GpuOraclePredictor,
                                                 GpuQuantilePredictor)
    from paper_2603_22206_b200.trace import TraceStore, columns_from_records, load_ndjson
    from workloads.tracegen import ModelStageOutput, StageTrace, TraceRecord

    cols = load_ndjson(os.path.join(GOLD, "trace_small.ndjson"))
    ids = cols.model_ids
    tcols = load_ndjson(os.path.join(GOLD, "kendall_training.ndjson"))
    training = []  # TraceRecord objects for the quantile training (host, once)
    for p in range(len(tcols.program_ids)):
        st = [StageTrace(j + 1, "r", int(tcols.base_input[p, j]),
                         {m: ModelStageOutput(int(tcols.out_tokens[p, j, k]),
                                              int(tcols.carried[p, j, k]))
                          for k, m in enumerate(ids)})
              for j in range(int(tcols.n_stages[p]))]
        training.append(TraceRecord(tcols.program_ids[p], tcols.workflow_ids[p], 0.0, st,
                                    {m: 0 for m in ids}, "easy"))
    q50 = GpuQuantilePredictor(training, ids, 0.5)
    q90 = GpuQuantilePredictor(training, ids, 0.9)
    store = TraceStore(cols, "cuda", workflow_index=q50.workflow_index)
    preds = {"oracle": GpuOraclePredictor(trace=store), "input-length": GpuInputLengthPredictor(),
             "quantile": q50, "quantile90": q90}
    for name, pr in preds.items():
        got = [evaluate_predictor(pr, store, m) for m in ids]
        np.testing.assert_array_equal(got, gold[f"eval_{name}"], err_msg=name)
    got = [arrival_order_distance(store, m) for m in ids]
    np.testing.assert_array_equal(got, gold["eval_arrival"])
    _ = columns_from_records  # (records path covered in test_gpu_trace)


@pytest.mark.parametrize("q", [0.5, 0.9, 0.37])
def test_quantile_training_on_device(q):
    """chm_quantile_train from a trace store == the host np.quantile build and
    the reference's EmpiricalQuantilePredictor (tests/golden/quantile.npz grid)."""
    from paper_2603_22206_b200.predictor import GpuQuantilePredictor
    from paper_2603_22206_b200.trace import TraceStore
    from workloads.tracegen import MATH_WORKFLOWS, LengthStats, synthesize_trace
    from tests.test_oracle import MATH_STATS, MATH_SUCCESS  # the golden generator's inputs

    stats = {m: LengthStats(*v) for m, v in MATH_STATS.items()}
    tr = synthesize_trace(MATH_WORKFLOWS, stats, MATH_SUCCESS, 2000, 1)
    ids = ["m0", "m1", "m2"]
    host = GpuQuantilePredictor(tr, ids, q)
    dev = GpuQuantilePredictor.from_trace(TraceStore.from_records(tr, ids, "cuda"), q)
    assert dev.workflow_index == host.workflow_index and dev.s_cap == host.s_cap
    assert dev.table_host.tobytes() == host.table_host.tobytes()
    z = np.load(os.path.join(GOLD, "quantile.npz"))
    grid = z[f"q{q}"]
    for a, wf in enumerate(z["wfs"]):
        for st in range(1, 8):
            for m in range(3):
                assert dev.lookup(str(wf), st, f"m{m}") == grid[a, st - 1, m]
