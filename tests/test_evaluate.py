"""Predictor evaluation, CPU: the oracle restatement of
kendall_tau_distance (oracle/eval_ref.py) against the reference's values
(tests/golden/kendall.npz)."""

import os

import numpy as np
import pytest

from oracle import eval_ref

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "kendall.npz"))


def test_oracle_kendall_matches_reference(gold):
    for name in gold["cases"]:
        if name.endswith("20000"):
            continue  # the pure-Python restatement is slow; the GPU test covers it
        p, t = gold[f"{name}_p"].tolist(), gold[f"{name}_t"].tolist()
        _, d = eval_ref.ref_kendall_counts(p, t)
        assert d == float(gold[f"{name}_d"]), name
