"""Pin the CPU oracle (oracle/hetsched_port.py) against golden vectors produced
by the unmodified reference (tests/golden/make_golden.py). CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import hetsched_port as hp
from tests import harness as H


def test_select_model_kat():
    z = np.load(os.path.join(H.GOLDEN, "select_kat.npz"))
    n_bad = 0
    for i in range(len(z["k"])):
        k = int(z["k"][i])
        ids = [f"m{j}" for j in range(k)]
        q = dict(zip(ids, z["q"][i, :k].tolist()))
        loads = dict(zip(ids, z["loads"][i, :k].tolist()))
        tau, dm = z["cfg"][i]
        got = hp.port_select_model(q, loads, float(tau), float(dm))
        n_bad += ids.index(got) != int(z["chosen"][i])
    assert n_bad == 0


def test_spec_examples():
    # SPEC.md:319-321 and estimate_load SPEC.md:310
    assert hp.port_select_model({"A": 0.4, "B": 0.9}, {"A": 100.0, "B": 140.0}, 0.5, 0.1) == "B"
    assert hp.port_select_model({"A": 0.4, "B": 0.9}, {"A": 100.0, "B": 300.0}, 0.5, 0.1) == "A"
    assert hp.port_select_model({"A": 0.3, "B": 0.7, "C": 0.5},
                                {"A": 10.0, "B": 10.0, "C": 10.0}, 0.5, 0.0) == "B"
    assert 1000.0 * 20.0 / 8 == 2500.0


def test_tie_band_definition():
    """port_tie_band (the definition the device tie flags are checked against):
    a decision is flagged when a router error of tol could flip it."""
    # gate: B at 0.9 vs A's 0.4 + 0.1 = 0.5 -> clear by 0.4; no tie
    assert hp.port_tie_band({"A": 0.4, "B": 0.9}, {"A": 100.0, "B": 140.0}, "B", 0.5, 0.1) == \
        (False, False)
    # gate: B at 0.505 sits within 1e-2 of 0.5
    assert hp.port_tie_band({"A": 0.4, "B": 0.505}, {"A": 100.0, "B": 140.0}, "B", 0.5, 0.1) == \
        (False, True)
    # B outside the slack: its gate comparison cannot matter
    assert hp.port_tie_band({"A": 0.4, "B": 0.505}, {"A": 100.0, "B": 300.0}, "A", 0.5, 0.1) == \
        (False, False)
    # rank: B and C both qualify and differ by 0.005
    assert hp.port_tie_band({"A": 0.3, "B": 0.7, "C": 0.695}, {"A": 10.0, "B": 10.0, "C": 10.0},
                            "B", 0.5, 0.0) == (True, False)
    # exact q tie between candidates (broken by id) is a rank tie
    assert hp.port_tie_band({"A": 0.3, "B": 0.7, "C": 0.7}, {"A": 10.0, "B": 10.0, "C": 10.0},
                            "B", 0.5, 0.0)[0]
    # no candidate: m_fast chosen, no rank tie
    assert hp.port_tie_band({"A": 0.5, "B": 0.55}, {"A": 1.0, "B": 1.0}, "A", 0.0, 0.2) == \
        (False, False)


@pytest.mark.parametrize("name", H.schedule_names())
def test_schedule_port_matches_reference(name):
    sc = H.load_schedule(name)
    res, err = H.run_port_schedule(sc)
    n = len(sc["prog"]) if not sc["err_kind"] else sc["err_row"]
    if sc["err_kind"]:
        assert err is not None and err["kind"] == sc["err_kind"] and err["row"] == sc["err_row"]
    else:
        assert err is None
    for key in ("model", "priority", "cached", "seq", "admitted"):
        np.testing.assert_array_equal(res[key][:n], sc[f"out_{key}"][:n], err_msg=key)
    np.testing.assert_array_equal(res["loads"][:n], sc["out_loads"][:n])
    # bit-exact in-flight sums (Neumaier order) and engine/monitor state
    assert res["final_p"].tobytes() == sc["out_final_p"].tobytes()
    for key in ("final_cnt", "running", "queued", "assign"):
        np.testing.assert_array_equal(res[key], sc[f"out_{key}"], err_msg=key)


@pytest.mark.parametrize("name", H.complete_names())
def test_completion_port_matches_reference(name):
    """record_completion + the recomputed Neumaier sums + the next batch's
    decisions, against the real reference (tests/golden/complete_*.npz)."""
    d, r1, r2, mid_p, mid_cnt, final_p = H.run_port_complete(name)
    for key in ("model", "priority", "cached"):
        np.testing.assert_array_equal(r1[key], d[f"out1_{key}"], err_msg=key)
        np.testing.assert_array_equal(r2[key], d[f"out2_{key}"], err_msg=key)
    np.testing.assert_array_equal(r2["loads"], d["out2_loads"])
    assert mid_p.tobytes() == d["mid_p"].tobytes()
    np.testing.assert_array_equal(mid_cnt, d["mid_cnt"])
    assert final_p.tobytes() == d["final_p"].tobytes()


@pytest.mark.parametrize("name", H.queue_names())
def test_queue_port_matches_reference(name):
    qd = H.load_queue(name)
    res = H.run_port_queue(qd)
    np.testing.assert_array_equal(res["admitted"], qd["admitted"])
    np.testing.assert_array_equal(res["order"], qd["order"])
    np.testing.assert_array_equal(res["level"], qd["level"])
    np.testing.assert_array_equal(res["count"], qd["count"])
    assert res["running"] == qd["running"]
    assert res["iterations"] == qd["iterations"]


MATH_STATS = {"m0": (606.0, 2587.0), "m1": (657.5, 1651.0), "m2": (709.0, 715.0)}
MATH_SUCCESS = {"m0": {"easy": 0.55, "hard": 0.12}, "m1": {"easy": 0.72, "hard": 0.36},
                "m2": {"easy": 0.9, "hard": 0.6}}


def _math_trace():
    from workloads import tracegen as W
    stats = {m: W.LengthStats(*v) for m, v in MATH_STATS.items()}
    return W.synthesize_trace(W.MATH_WORKFLOWS, stats, MATH_SUCCESS, 2000, 1)


def _digest(tr):
    import hashlib
    h = hashlib.sha256()
    for rec in tr:
        d = {
            "program_id": rec.program_id, "workflow_id": rec.workflow_id,
            "user_arrival_time_ms": rec.user_arrival_time_ms,
            "stages": [{"stage_index": s.stage_index, "role": s.role,
                        "base_input_tokens": s.base_input_tokens,
                        "models": {m: {"out_tokens": o.out_tokens,
                                       "carried_context_tokens": o.carried_context_tokens}
                                   for m, o in sorted(s.models.items())}} for s in rec.stages],
            "success": {m: rec.success[m] for m in sorted(rec.success)},
            "difficulty": rec.difficulty,
        }
        h.update(json.dumps(d, sort_keys=True).encode())
    return h.hexdigest()


def test_synthesize_trace_matches_reference():
    from workloads import tracegen as W
    gold = json.load(open(os.path.join(H.GOLDEN, "synth.json")))
    assert _digest(_math_trace()) == gold["math_2000_1"]
    cs = {"fast": W.LengthStats(447, 1276), "strong": W.LengthStats(649, 534)}
    cr = {"fast": {"easy": 0.45, "hard": 0.08}, "strong": {"easy": 0.85, "hard": 0.55}}
    assert _digest(W.synthesize_trace(W.CODE_WORKFLOWS, cs, cr, 500, 3)) == gold["code_500_3"]
    assert _digest(W.synthesize_trace(W.CODE_WORKFLOWS, cs, cr, 300, 4,
                                      role_weights={"planner": 0.5, "coder": 2.0},
                                      template_mix=[1, 2, 3])) == gold["code_300_4_weights"]


@pytest.mark.parametrize("q", [0.5, 0.9, 0.37])
def test_quantile_tables(q):
    from paper_2603_22206_b200.predictor import GpuQuantilePredictor
    z = np.load(os.path.join(H.GOLDEN, "quantile.npz"))
    grid = z[f"q{q}"]
    wfs = [str(w) for w in z["wfs"]]
    tr = _math_trace()
    port = hp.PortQuantilePredictor(tr, q)
    for a, wf in enumerate(wfs):
        for st in range(1, 8):
            for m in range(3):
                assert port.lookup(wf, st, f"m{m}") == grid[a, st - 1, m]
    # the device table (built on the host) resolves the same fallback chain
    gp = GpuQuantilePredictor.__new__(GpuQuantilePredictor)
    GpuQuantilePredictor.__init__(gp, tr, ["m0", "m1", "m2"], q, device="cpu")
    tab = gp.table_host
    for a, wf in enumerate(wfs):
        wi = gp.workflow_index.get(wf, gp.n_wf)
        for st in range(1, 8):
            sti = st if st <= gp.s_cap else 0
            for m in range(3):
                assert tab[wi, sti, m] == grid[a, st - 1, m], (wf, st, m)
