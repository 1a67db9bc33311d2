"""Differential tests: the CPU oracle (oracle/hetsched_port.py) against the
UNMODIFIED reference itself on randomized inputs it has never seen (the
golden fixtures pin fixed scenarios; this draws new ones every seed). Runs
only where /root/reference exists (the build container); the GPU box has no
reference and skips it. CPU only, imports the reference read-only.

Covers select_model (balancer.py:63-77) on random K / q / loads / slack /
margin with ties, and whole schedule_request sequences (balancer.py:89-129
with the monitor and EngineSim side effects) through the golden generator's
scenario builder and reference driver (tests/golden/make_golden.py)."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "hetsched")),
                                reason="reference checkout not present")

sys.dont_write_bytecode = True


@pytest.fixture(scope="module")
def golden():
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    import make_golden  # imports hetsched from /root/reference read-only

    return make_golden


def test_select_model_random(golden):
    from oracle import hetsched_port as hp

    balancer, router = golden.balancer, golden.router
    rng = np.random.default_rng(20261017)
    for _ in range(3000):
        k = int(rng.integers(1, 9))
        ids = golden.model_ids(k)
        if rng.random() < 0.4:  # decimal table scores with exact ties
            q = rng.integers(0, 11, size=k) / 10.0
        else:
            q = rng.random(k)
        loads = (rng.integers(0, 5, size=k) * 250.0 if rng.random() < 0.5
                 else rng.lognormal(6, 1, size=k))
        tau = float(rng.choice([0.0, 0.1, 0.5, 2.0, 1e6]))
        dm = float(rng.choice([0.0, 0.05, 0.1, 0.25, 1.0]))
        want = balancer.select_model(router.ConfidenceVector(dict(zip(ids, q.tolist()))),
                                     dict(zip(ids, loads.tolist())),
                                     balancer.BalancerConfig(tau, dm))
        got = hp.port_select_model(dict(zip(ids, q.tolist())), dict(zip(ids, loads.tolist())),
                                   tau, dm)
        assert got == want, (k, q, loads, tau, dm)


@pytest.mark.parametrize("seed", [101, 102, 103, 104, 105, 106])
def test_schedule_sequences_random(golden, seed):
    from tests import harness as H

    rng = np.random.default_rng(seed)
    k = int(rng.integers(1, 9))
    spec = dict(dyadic=bool(rng.random() < 0.5), p0_entries=int(rng.integers(0, 400)),
                pre_assigned=float(rng.choice([0.0, 0.1, 0.3])),
                repeats=float(rng.choice([0.0, 0.1, 0.2])),
                tau=float(rng.choice([0.0, 0.5, 2.0])), margin=float(rng.choice([0.0, 0.1])),
                tied_q=bool(rng.random() < 0.3), table_q=bool(rng.random() < 0.3),
                pre_running=[int(x) for x in rng.integers(0, 4, size=k)])
    sc = golden.build_scenario(seed, k, int(rng.integers(50, 400)), **spec)
    want, err_ref = golden.run_reference(sc)
    # the harness's (fixture) layout: pre as sorted (program, model) pairs
    sc2 = dict(sc)
    sc2["pre"] = sorted(sc["pre"].items())
    sc2["p0"] = np.array(sc["p0"], dtype=np.float64).reshape(-1, 2)
    got, err_port = H.run_port_schedule(sc2)
    assert (err_ref is None) == (err_port is None)
    if err_ref is not None:
        assert err_ref["row"] == err_port["row"]
    n = len(sc["prog"]) if err_ref is None else err_ref["row"]
    for key in ("model", "priority", "cached", "seq", "admitted"):
        np.testing.assert_array_equal(got[key][:n], want[key][:n], err_msg=key)
    np.testing.assert_array_equal(got["loads"][:n], want["loads"][:n])
    assert got["final_p"].tobytes() == want["final_p"].tobytes()  # Neumaier order, bit-exact
    for key in ("final_cnt", "running", "queued", "assign"):
        np.testing.assert_array_equal(got[key], want[key], err_msg=key)
