"""Generate golden vectors by running the UNMODIFIED reference (hetsched).

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports /root/reference/pkg/src/hetsched read-only and writes small .npz /
.json fixtures next to this file. The GPU box has no /root/reference; the
tests there read only these committed fixtures.

Fixtures
  select_kat.npz      select_model on SPEC examples + random instances
                      (balancer.py:63-77, AC2 SPEC.md:533)
  schedule_*.npz      sequences of schedule_request calls (balancer.py:89-129)
                      fed precomputed scores/predictions through Router /
                      Predictor shims, with pre-seeded in-flight state,
                      pre-assigned programs, in-batch repeats and engines
                      with free / full slots
  errors.json         the exception class + row the reference raises
  queue_*.npz         EngineSim STJF + aging: enqueue / iterate / complete
                      scripts and the resulting admission and queue orders
                      (engine.py:265-394)
  e_*.npz             the engine execution clock: enqueue (with input / output
                      tokens) / iterate / advance_to scripts on one EngineSim
                      with prefill and decode times; completions with their
                      finish times, admissions, the running set's stint ends,
                      final queue, counters (engine.py:165-241)
  quantile.npz        EmpiricalQuantilePredictor on synthesize_trace(2000, 1)
                      (predictor.py:65-108) over a (wf, stage, model) grid
  synth.json          fingerprints of synthesize_trace outputs (workload.py:334-416)
  trace_small.ndjson  a mixed code/math trace written by save_trace (workload.py:294-297),
  trace_small.npz     carried context != out tokens for some stages, and the reference's
                      remaining_tokens / first_stage_request / next_stage_request answers
                      for every (program, stage, model) (workload.py:160-165, 454-495)
  trace_errors.json   malformed trace files and the error load_trace raises (256-291)
  kendall.npz         kendall_tau_distance cases + evaluate_predictor / arrival_order_distance
  kendall_training.ndjson  on trace_small per model and predictor (predictor.py:182-261)
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))
sys.dont_write_bytecode = True
sys.path.insert(0, REF)

from hetsched import balancer, engine, monitor, predictor, profiles, router, workload  # noqa: E402
from hetsched.errors import SimError  # noqa: E402


def model_ids(k):
    return [f"m{i}" for i in range(k)]


# ---------------------------------------------------------------- select KAT
def make_select_kat():
    rng = np.random.default_rng(7)
    cases = []
    # SPEC.md:319-321 examples (two models A<B as m0<m1)
    cases.append(([0.4, 0.9], [100.0, 140.0], 0.5, 0.1))
    cases.append(([0.4, 0.9], [100.0, 300.0], 0.5, 0.1))
    cases.append(([0.3, 0.7, 0.5], [10.0, 10.0, 10.0], 0.5, 0.0))
    for _ in range(4000):
        k = int(rng.integers(1, 9))
        q = rng.random(k).astype(np.float32).astype(np.float64)
        if rng.random() < 0.3:  # ties in q
            q[rng.integers(0, k, size=k)] = q[0]
        if rng.random() < 0.5:
            loads = rng.integers(0, 6, size=k).astype(np.float64) * 100.0  # ties in loads
        else:
            loads = rng.random(k) * 1000.0
        tau = float(rng.choice([0.0, 0.25, 0.5, 1.0, 3.0, 1e6]))
        dm = float(rng.choice([0.0, 0.05, 0.1, 0.3, 1.0]))
        cases.append((list(q), list(loads), tau, dm))
    # decimal table scores (TableRouter-style 0.1 steps, not fp32-representable):
    # with margin 0.1, (0.9 vs 0.8) and (0.4 vs 0.3) clear the margin in fp64
    # but (0.3 vs 0.2) does not -- fp32-rounded scores get each of them wrong
    cases.append(([0.8, 0.9], [100.0, 120.0], 0.5, 0.1))
    cases.append(([0.3, 0.4], [100.0, 120.0], 0.5, 0.1))
    cases.append(([0.2, 0.3], [100.0, 120.0], 0.5, 0.1))
    rng2 = np.random.default_rng(8)
    for _ in range(1000):
        k = int(rng2.integers(2, 9))
        q = rng2.integers(0, 11, size=k) / 10.0
        loads = rng2.integers(0, 6, size=k).astype(np.float64) * 100.0
        tau = float(rng2.choice([0.0, 0.5, 1.0, 1e6]))
        dm = float(rng2.choice([0.1, 0.2, 0.3]))
        cases.append((list(q), list(loads), tau, dm))
    K = 8
    Q = np.full((len(cases), K), np.nan)
    L = np.full((len(cases), K), np.nan)
    meta = np.zeros((len(cases), 2))
    kk = np.zeros(len(cases), dtype=np.int32)
    out = np.zeros(len(cases), dtype=np.int32)
    for i, (q, loads, tau, dm) in enumerate(cases):
        k = len(q)
        ids = model_ids(k)
        cv = router.ConfidenceVector(dict(zip(ids, q)))
        cfg = balancer.BalancerConfig(tau, dm)
        sel = balancer.select_model(cv, dict(zip(ids, loads)), cfg)
        Q[i, :k] = q
        L[i, :k] = loads
        meta[i] = (tau, dm)
        kk[i] = k
        out[i] = ids.index(sel)
    np.savez_compressed(os.path.join(OUT, "select_kat.npz"), q=Q, loads=L, cfg=meta, k=kk,
                        chosen=out)
    return len(cases)


# ----------------------------------------------------------- schedule shims
class ShimRouter(router.Router):
    name = "shim"

    def __init__(self, table):
        self.table = table  # request_id -> {model: q}

    def _score_one(self, req, rec, model_id):
        return self.table[req.request_id][model_id]


class ShimPredictor(predictor.Predictor):
    name = "shim"

    def __init__(self, table):
        self.table = table  # request_id -> {model: yhat}

    def predict(self, req, rec, model_id):
        return self.table[req.request_id][model_id]


def build_scenario(seed, k, n_rows, *, dyadic=True, p0_entries=0, pre_assigned=0.0,
                   repeats=0.0, batch=None, decode=None, pre_running=None, tau=0.5,
                   margin=0.1, spread=1.0, tied_q=False, table_q=False):
    rng = np.random.default_rng(seed)
    ids = model_ids(k)
    decode = decode or [5.0 * (i + 1) for i in range(k)]
    batch = batch or [max(1, 32 >> i) for i in range(k)]
    n_prog = n_rows + 8
    # programs for rows: mostly distinct, some repeats (later stage of an earlier row)
    prog = []
    stage = []
    used = {}
    for i in range(n_rows):
        if i > 0 and rng.random() < repeats:
            p = int(prog[int(rng.integers(0, i))])
            used[p] = used.get(p, 0) + 1
            prog.append(p)
            stage.append(used[p])
        else:
            p = i + 8
            used[p] = 1
            prog.append(p)
            stage.append(1)
    prog = np.array(prog, dtype=np.int32)
    stage = np.array(stage, dtype=np.int32)
    q = rng.random((n_rows, k))
    q = 0.5 + (q - 0.5) * spread
    if tied_q:
        q = np.round(q * 4) / 4
    q = np.clip(q, 0, 1).astype(np.float32)
    if table_q:  # TableRouter-style decimal scores, exact fp64 (router.py:71-88)
        q = rng.integers(0, 11, size=(n_rows, k)) / 10.0
    if dyadic:
        yhat = rng.integers(0, 4000, size=(n_rows, k)).astype(np.float64) / 2.0
    else:
        yhat = rng.lognormal(6.0, 1.0, size=(n_rows, k))
    out_tok = rng.integers(0, 2000, size=(n_rows, k)).astype(np.int32)
    arrival = np.sort(rng.random(n_rows) * 10.0) if rng.random() < 0.5 else np.full(n_rows, 3.0)
    # initial in-flight entries on each model (request ids "seed:j")
    p0 = []
    for j in range(p0_entries):
        m = int(rng.integers(0, k))
        v = float(rng.integers(1, 3000)) / (1.0 if dyadic else 7.0)
        p0.append((m, v))
    # pre-assigned programs (programs 0..7 and some row programs)
    pre = {}
    for p in range(8):
        pre[p] = int(rng.integers(0, k))
    for p in set(prog.tolist()):
        if rng.random() < pre_assigned:
            pre[p] = int(rng.integers(0, k))
    pre_running = pre_running if pre_running is not None else [0] * k
    return dict(seed=seed, k=k, ids=ids, decode=decode, batch=batch, n_prog=n_prog,
                prog=prog, stage=stage, q=q, yhat=yhat, out_tok=out_tok, arrival=arrival,
                p0=p0, pre=pre, pre_running=pre_running, tau=tau, margin=margin)


def run_reference(sc):
    ids = sc["ids"]
    k = sc["k"]
    pool = profiles.Pool(tuple(profiles.ModelProfile(ids[i], sc["decode"][i], sc["batch"][i])
                               for i in range(k)))
    mon = monitor.ActivityMonitor(ids)
    for j, (m, v) in enumerate(sc["p0"]):
        mon.record_dispatch(ids[m], f"seed:{j}", v)
    for p, m in sc["pre"].items():
        mon.assign(f"p{p:06d}", ids[m])
    aging = engine.AgingConfig()
    engines = {mid: engine.EngineSim(pool[mid], aging=aging) for mid in ids}
    for i, mid in enumerate(ids):
        for j in range(sc["pre_running"][i]):
            rq = workload.Request(f"r{i}x{j}", 1, 1, 0.0, "wf", "x")
            engines[mid].enqueue(rq, priority=1.0, out_tokens=10 ** 6, now=0.0)
    state = balancer.SchedulerState(pool=pool, monitor=mon, queues=engines)
    n = len(sc["prog"])
    qtab, ytab, recs, reqs = {}, {}, {}, []
    for i in range(n):
        pid = f"p{int(sc['prog'][i]):06d}"
        st = int(sc["stage"][i])
        req = workload.Request(pid, st, 10, float(sc["arrival"][i]), "wf", "r")
        qtab[req.request_id] = {ids[m]: float(sc["q"][i, m]) for m in range(k)}
        ytab[req.request_id] = {ids[m]: float(sc["yhat"][i, m]) for m in range(k)}
        rec = recs.get(pid)
        if rec is None or rec.n_stages < st:
            stages = [] if rec is None else rec.stages
            while len(stages) < st:
                stages.append(workload.StageTrace(len(stages) + 1, "r", 10, {
                    mid: workload.ModelStageOutput(0, 0) for mid in ids}))
            rec = workload.TraceRecord(pid, "wf", 0.0, stages, {mid: 0 for mid in ids}, "easy")
            recs[pid] = rec
        rec.stages[st - 1].models = {
            ids[m]: workload.ModelStageOutput(int(sc["out_tok"][i, m]), 0) for m in range(k)}
        reqs.append(req)
    rt, pr = ShimRouter(qtab), ShimPredictor(ytab)
    cfg = balancer.BalancerConfig(sc["tau"], sc["margin"])
    model = np.full(n, -1, dtype=np.int32)
    prio = np.zeros(n)
    cached = np.zeros(n, dtype=np.int8)
    loads = np.full((n, k), np.nan)
    seq = np.full(n, -1, dtype=np.int64)
    admitted = np.zeros(n, dtype=np.int8)
    err = None
    for i, req in enumerate(reqs):
        before = {mid: (engines[mid].running_count, engines[mid]._seq) for mid in ids}
        try:
            d = balancer.schedule_request(req, recs[req.program_id], state, rt, pr, cfg)
        except (SimError, ValueError) as exc:
            err = {"kind": type(exc).__name__, "row": i}
            break
        mi = ids.index(d.model)
        model[i] = mi
        prio[i] = d.priority
        cached[i] = int(d.used_cached_assignment)
        if d.estimated_loads:
            loads[i] = [d.estimated_loads[mid] for mid in ids]
        e = engines[d.model]
        for s, rr in e.running.items():
            if rr.entry.request.request_id == req.request_id:
                seq[i], admitted[i] = s, 1
        for s, qe in e._queued.items():
            if qe.request.request_id == req.request_id:
                seq[i] = s
    final_p = np.array([mon.in_flight_sum(mid) for mid in ids], dtype=np.float64)
    final_cnt = np.array([mon.in_flight_count(mid) for mid in ids], dtype=np.int64)
    running = np.array([engines[mid].running_count for mid in ids], dtype=np.int32)
    queued = np.array([engines[mid].waiting_count for mid in ids], dtype=np.int32)
    assign = np.full(sc["n_prog"], -1, dtype=np.int8)
    for p in range(sc["n_prog"]):
        a = mon.assignment(f"p{p:06d}")
        if a is not None:
            assign[p] = ids.index(a)
    return dict(model=model, priority=prio, cached=cached, loads=loads, seq=seq,
                admitted=admitted, final_p=final_p, final_cnt=final_cnt, running=running,
                queued=queued, assign=assign), err


def save_scenario(name, sc, res, err):
    p0 = np.array(sc["p0"], dtype=np.float64).reshape(-1, 2)
    pre = np.array(sorted(sc["pre"].items()), dtype=np.int64).reshape(-1, 2)
    np.savez_compressed(
        os.path.join(OUT, f"schedule_{name}.npz"),
        k=sc["k"], decode=np.array(sc["decode"]), batch=np.array(sc["batch"], dtype=np.int32),
        n_prog=sc["n_prog"], prog=sc["prog"], stage=sc["stage"], q=sc["q"], yhat=sc["yhat"],
        out_tok=sc["out_tok"], arrival=sc["arrival"], p0=p0, pre=pre,
        pre_running=np.array(sc["pre_running"], dtype=np.int32), tau=sc["tau"],
        margin=sc["margin"], err_kind=(err or {}).get("kind", ""),
        err_row=(err or {}).get("row", -1), **{f"out_{k}": v for k, v in res.items()})


def make_schedules():
    specs = {
        "k3_basic": dict(seed=1, k=3, n_rows=600),
        "k5_dyadic_p0": dict(seed=2, k=5, n_rows=2000, p0_entries=3000),
        "k5_nondyadic_p0": dict(seed=3, k=5, n_rows=2000, dyadic=False, p0_entries=500),
        "k8_mixed": dict(seed=4, k=8, n_rows=3000, pre_assigned=0.2, repeats=0.15,
                         dyadic=False, p0_entries=200),
        "k5_nonpow2": dict(seed=5, k=5, n_rows=1500, batch=[3, 7, 12, 5, 1],
                           decode=[4.7, 9.3, 13.1, 0.7, 21.0], dyadic=False, p0_entries=100),
        "k4_ties": dict(seed=6, k=4, n_rows=1200, tied_q=True, margin=0.0, tau=0.0),
        "k5_slack_big": dict(seed=7, k=5, n_rows=1000, tau=1e6, margin=0.0),
        "k2_spread": dict(seed=8, k=2, n_rows=800, spread=0.2, pre_running=[31, 0]),
        "k1_single": dict(seed=9, k=1, n_rows=300),
        "k3_table": dict(seed=11, k=3, n_rows=700, table_q=True, margin=0.1, tau=1.0),
        "k5_table": dict(seed=12, k=5, n_rows=900, table_q=True, margin=0.2, tau=0.5,
                         dyadic=False, p0_entries=40),
        "k6_running": dict(seed=10, k=6, n_rows=1000, pre_running=[5, 16, 8, 0, 2, 1],
                           repeats=0.1, pre_assigned=0.1),
    }
    out = {}
    for name, spec in specs.items():
        seed = spec.pop("seed")
        k = spec.pop("k")
        n = spec.pop("n_rows")
        sc = build_scenario(seed, k, n, **spec)
        res, err = run_reference(sc)
        save_scenario(name, sc, res, err)
        out[name] = err
    return out


def make_errors():
    """Scenarios where the reference raises mid-batch."""
    cases = {}
    # ValidationError: score outside [0,1] at row 5
    sc = build_scenario(21, 3, 20)
    sc["q"][5, 1] = 1.5
    res, err = run_reference(sc)
    save_scenario("err_score", sc, res, err)
    cases["err_score"] = err
    # ValueError: negative prediction for the chosen model at row 7 (all models negative)
    sc = build_scenario(22, 3, 20)
    sc["yhat"][7, :] = -1.0
    res, err = run_reference(sc)
    save_scenario("err_negative", sc, res, err)
    cases["err_negative"] = err
    # DuplicateRequest: same (program, stage) twice
    sc = build_scenario(23, 3, 20)
    sc["prog"][9] = sc["prog"][4]
    sc["stage"][9] = sc["stage"][4]
    # the shims key scores/predictions by request_id: keep both rows consistent
    sc["q"][9] = sc["q"][4]
    sc["yhat"][9] = sc["yhat"][4]
    res, err = run_reference(sc)
    save_scenario("err_duplicate", sc, res, err)
    cases["err_duplicate"] = err
    # ValueError: time going backwards (arrival decreases by > 1e-9)
    sc = build_scenario(24, 3, 20)
    sc["arrival"] = np.linspace(5, 10, 20)
    sc["arrival"][12] = 1.0
    sc["q"][:, :] = 0.5  # everything goes to the fastest model -> same engine
    sc["margin"] = 0.1
    res, err = run_reference(sc)
    save_scenario("err_backwards", sc, res, err)
    cases["err_backwards"] = err
    # ValidationError: negative out_tokens
    sc = build_scenario(25, 3, 20)
    sc["out_tok"][11, :] = -3
    res, err = run_reference(sc)
    save_scenario("err_outtok", sc, res, err)
    cases["err_outtok"] = err
    with open(os.path.join(OUT, "errors.json"), "w") as fh:
        json.dump(cases, fh, indent=1, sort_keys=True)
    return cases


# ------------------------------------------------------------------ queues
def run_queue_script(seed, b, S, n_pre, script, Q=4, demote=False):
    """Drive one EngineSim. `script` is a list of ("enq", n) / ("iter", n) /
    ("complete", n) steps. Returns admission order and final queue order as
    lists of request ordinals, plus the queued entries' (level, count)."""
    rng = np.random.default_rng(seed)
    prof = profiles.ModelProfile("m0", 1.0, b)
    aging = engine.AgingConfig(starvation_threshold=S if S else math.inf, running_quantum=Q,
                               demote_while_queued=demote)
    eng = engine.EngineSim(prof, aging=aging)
    t = 0.0
    ordinal = 0
    recs = []  # (ordinal, priority, out_tokens_completion_time)
    admitted = []
    prio_vals = rng.integers(1, 60, size=100000).astype(np.float64)
    if seed % 2:
        prio_vals = prio_vals / 3.0  # non-dyadic
    # the first b requests fill the batch; completion time controlled by out_tokens
    enq_log = []

    def enqueue(n):
        nonlocal ordinal
        for _ in range(n):
            p = float(prio_vals[ordinal])
            rq = workload.Request(f"q{ordinal}", 1, 1, t, "wf", "x")
            eng.enqueue(rq, priority=p, out_tokens=10 ** 9, now=t)
            enq_log.append((ordinal, p, t))
            ordinal += 1

    admit_events = []
    orig_admit = eng._admit

    def spy(entry, now):
        admit_events.append(int(entry.request.program_id[1:]))
        rr = orig_admit(entry, now)
        return rr
    eng._admit = spy
    enqueue(n_pre)
    for op, n in script:
        if op == "enq":
            t += 1.0
            enqueue(n)
        elif op == "iter":
            for _ in range(n):
                t += 1.0
                eng.scheduling_iteration(t)
        elif op == "complete":
            # complete the n earliest-admitted running requests at time t+1:
            # shorten their stint so they end exactly then
            t += 1.0
            victims = sorted(eng.running)[:n]
            for s in victims:
                eng.running[s].stint_end = t
            eng.advance_to(t)
    order = [int(e.request.program_id[1:]) for e in sorted(eng._queued.values(),
                                                             key=lambda e: e.sort_key())]
    lv = {int(e.request.program_id[1:]): (e.starvation_level, e.starvation_count)
          for e in eng._queued.values()}
    return dict(enq=np.array(enq_log, dtype=np.float64), admitted=np.array(admit_events),
                order=np.array(order), level=np.array([lv[o][0] for o in order]),
                count=np.array([lv[o][1] for o in order]), running=eng.running_count,
                iterations=eng.iterations)


def make_queues(only=None):
    scripts = {
        "q_basic": (1, 4, 8, 20, [("iter", 3), ("enq", 10), ("iter", 2)]),
        "q_promote": (2, 2, 3, 12, [("iter", 4), ("enq", 5), ("iter", 5)]),
        "q_complete": (3, 8, 4, 60, [("iter", 2), ("complete", 3), ("enq", 7),
                                      ("iter", 1), ("complete", 8), ("iter", 6)]),
        "q_noaging": (4, 3, 0, 40, [("iter", 20), ("complete", 3), ("enq", 4), ("iter", 2)]),
        "q_big": (5, 32, 8, 3000, [("iter", 7), ("complete", 32), ("enq", 500), ("iter", 3),
                                   ("complete", 16), ("iter", 9), ("complete", 32)]),
        "q_S1": (6, 2, 1, 30, [("iter", 3), ("complete", 2), ("iter", 2)]),
        # a fractional threshold: count >= 2.5 with integer counts
        "q_frac_s": (9, 3, 2.5, 25, [("iter", 4), ("enq", 6), ("complete", 2), ("iter", 3)]),
    }
    for name, (seed, b, S, n_pre, script) in scripts.items():
        if only is not None and name not in only:
            continue
        res = run_queue_script(seed, b, S, n_pre, script)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), seed=seed, b=b, S=S, n_pre=n_pre,
                            script=json.dumps(script), **res)
    # AgingConfig.demote_while_queued (engine.py:360-374): promoted entries that
    # stay queued lose a level every Q further iterations
    demote = {
        "q_demote": (7, 3, 2, 2, 30, [("iter", 6), ("complete", 2), ("enq", 6), ("iter", 5)]),
        "q_demote_big": (8, 16, 3, 3, 1500, [("iter", 9), ("complete", 16), ("enq", 100),
                                              ("iter", 7), ("complete", 5), ("iter", 4)]),
        "q_demote_frac": (10, 3, 1.5, 2.5, 30, [("iter", 6), ("complete", 2), ("enq", 6),
                                                 ("iter", 5)]),
    }
    for name, (seed, b, S, Q, n_pre, script) in demote.items():
        if only is not None and name not in only:
            continue
        res = run_queue_script(seed, b, S, n_pre, script, Q=Q, demote=True)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), seed=seed, b=b, S=S, n_pre=n_pre,
                            Q=Q, demote=1, script=json.dumps(script), **res)


# ---------------------------------------------------------------- quantile
MATH_STATS = {"m0": (606.0, 2587.0), "m1": (657.5, 1651.0), "m2": (709.0, 715.0)}
MATH_SUCCESS = {"m0": {"easy": 0.55, "hard": 0.12}, "m1": {"easy": 0.72, "hard": 0.36},
                "m2": {"easy": 0.9, "hard": 0.6}}


def make_quantile():
    stats = {m: workload.LengthStats(*v) for m, v in MATH_STATS.items()}
    tr = workload.synthesize_trace(workload.MATH_WORKFLOWS, stats, MATH_SUCCESS, 2000, 1)
    wfs = ["math-4stage", "math-2stage", "math-1stage", "unknown-wf"]
    out = {}
    for q in (0.5, 0.9, 0.37):
        pr = predictor.EmpiricalQuantilePredictor(tr, q)
        grid = np.zeros((len(wfs), 7, 3))
        for a, wf in enumerate(wfs):
            for st in range(1, 8):
                for m in range(3):
                    req = workload.Request("x", st, 1, 0.0, wf, "r")
                    grid[a, st - 1, m] = pr.predict(req, None, f"m{m}")
        out[f"q{q}"] = grid
    np.savez_compressed(os.path.join(OUT, "quantile.npz"), wfs=np.array(wfs), **out)


def trace_digest(tr):
    h = hashlib.sha256()
    for rec in tr:
        h.update(json.dumps(rec.to_json_dict(), sort_keys=True).encode())
    return h.hexdigest()


def make_synth():
    out = {}
    stats = {m: workload.LengthStats(*v) for m, v in MATH_STATS.items()}
    out["math_2000_1"] = trace_digest(
        workload.synthesize_trace(workload.MATH_WORKFLOWS, stats, MATH_SUCCESS, 2000, 1))
    code_stats = {"fast": workload.LengthStats(447, 1276), "strong": workload.LengthStats(649, 534)}
    code_succ = {"fast": {"easy": 0.45, "hard": 0.08}, "strong": {"easy": 0.85, "hard": 0.55}}
    out["code_500_3"] = trace_digest(
        workload.synthesize_trace(workload.CODE_WORKFLOWS, code_stats, code_succ, 500, 3))
    out["code_300_4_weights"] = trace_digest(workload.synthesize_trace(
        workload.CODE_WORKFLOWS, code_stats, code_succ, 300, 4,
        role_weights={"planner": 0.5, "coder": 2.0}, template_mix=[1, 2, 3]))
    with open(os.path.join(OUT, "synth.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


def make_trace():
    """A small mixed trace through the reference's own writer and readers."""
    code_stats = {f"m{i}": workload.LengthStats(300 + 150 * i, 200 + 50 * i) for i in range(3)}
    succ = {f"m{i}": {"easy": 0.5 + 0.1 * i, "hard": 0.1 + 0.1 * i} for i in range(3)}
    recs = workload.synthesize_trace(workload.CODE_WORKFLOWS, code_stats, succ, 30, 11)
    recs += workload.synthesize_trace(workload.MATH_WORKFLOWS, code_stats, succ, 30, 12)
    rng = np.random.default_rng(13)
    edited = []
    for p, rec in enumerate(recs):
        d = rec.to_json_dict()
        d["program_id"] = f"t{p:04d}"
        d["user_arrival_time_ms"] = float(rng.integers(0, 10**6)) / 8.0
        for st in d["stages"]:
            for mid, o in st["models"].items():
                if rng.random() < 0.5:  # carried context differs from the output
                    o["carried_context_tokens"] = int(rng.integers(0, 3 * o["out_tokens"] + 2))
        edited.append(workload.TraceRecord.from_json_dict(d))
    path = os.path.join(OUT, "trace_small.ndjson")
    workload.save_trace(edited, path)
    recs = workload.load_trace(path)
    ids = sorted(recs[0].model_ids)
    NP, S, K = len(recs), max(r.n_stages for r in recs), len(ids)
    remaining = np.full((NP, S, K), -1, np.int64)
    nxt_input = np.full((NP, S, K), -1, np.int64)   # -1: no next stage (final stage)
    nxt_arrival = np.full((NP, S, K), -1.0)
    first_input = np.zeros(NP, np.int64)
    first_arrival = np.zeros(NP)
    for p, rec in enumerate(recs):
        req = workload.first_stage_request(rec)
        first_input[p], first_arrival[p] = req.input_tokens, req.arrival_time
        for s in range(1, rec.n_stages + 1):
            for k, m in enumerate(ids):
                remaining[p, s - 1, k] = rec.remaining_tokens(s, m)
                nx = workload.next_stage_request(rec, s, 1000.0 + p + 0.25 * s, m)
                if nx is not None:
                    assert nx.stage_index == s + 1
                    nxt_input[p, s - 1, k] = nx.input_tokens
                    nxt_arrival[p, s - 1, k] = nx.arrival_time
    unknown = []
    for s in (0, recs[0].n_stages + 1):
        try:
            workload.next_stage_request(recs[0], s, 0.0, ids[0])
        except SimError as exc:
            unknown.append([s, type(exc).__name__])
    np.savez_compressed(os.path.join(OUT, "trace_small.npz"), model_ids=np.array(ids),
                        program_ids=np.array([r.program_id for r in recs]),
                        n_stages=np.array([r.n_stages for r in recs], np.int32),
                        remaining=remaining, next_input=nxt_input, next_arrival=nxt_arrival,
                        first_input=first_input, first_arrival=first_arrival,
                        unknown=np.array(unknown, dtype=object).astype(str))
    # malformed files: (name, content) -> reference exception, line, message
    good = open(path).read().splitlines()
    bad_rec = json.loads(good[1])
    cases = {
        "bad_json": good[0] + "\n{not json\n",
        "not_object": good[0] + "\n[1, 2]\n",
        "missing_field": good[0] + "\n" + json.dumps({k: v for k, v in bad_rec.items()
                                                       if k != "stages"}) + "\n",
        "negative_tokens": good[0] + "\n" + json.dumps(_edit(bad_rec, "neg")) + "\n",
        "bad_stage_index": "\n" + json.dumps(_edit(bad_rec, "idx")) + "\n",
        "model_mismatch": good[0] + "\n" + json.dumps(_edit(bad_rec, "models")) + "\n",
        "base_zero": json.dumps(_edit(bad_rec, "base")) + "\n",
        "blank_lines_ok": "\n" + good[0] + "\n\n" + good[1] + "\n",
    }
    out = {}
    tmp = os.path.join(OUT, "_tmp_trace.ndjson")
    for name, text in cases.items():
        with open(tmp, "w") as fh:
            fh.write(text)
        try:
            n = len(workload.load_trace(tmp))
            out[name] = {"text": text, "error": None, "n": n}
        except SimError as exc:
            out[name] = {"text": text, "error": type(exc).__name__,
                         "line": getattr(exc, "line", None), "message": str(exc)}
    os.remove(tmp)
    with open(os.path.join(OUT, "trace_errors.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    return NP


def make_kendall():
    """kendall_tau_distance on hand-made and random sequences (ties in one,
    the other and both; -0.0; identical and reversed), and evaluate_predictor /
    arrival_order_distance on trace_small with every predictor kind
    (predictor.py:182-261)."""
    rng = np.random.default_rng(31)
    cases = {
        "identical": ([1.0, 2.0, 3.0, 4.0], [1.0, 2.0, 3.0, 4.0]),
        "reversed": ([1.0, 2.0, 3.0, 4.0], [4.0, 3.0, 2.0, 1.0]),
        "pair": ([0.0, 1.0], [1.0, 0.0]),
        "ties_pred": ([1.0, 1.0, 2.0, 2.0, 3.0], [5.0, 3.0, 2.0, 9.0, 1.0]),
        "ties_both": ([1.0, 1.0, 1.0, 2.0, 2.0], [3.0, 3.0, 1.0, 0.5, 0.5]),
        "neg_zero": ([-0.0, 0.0, 1.0, -1.0], [0.0, -0.0, 2.0, 2.0]),
        "constant": ([7.0] * 6, [1.0, 2.0, 3.0, 4.0, 5.0, 6.0]),
    }
    for n in (17, 1000, 20000):
        cases[f"rand_{n}"] = (rng.normal(size=n).tolist(), rng.normal(size=n).tolist())
        cases[f"tied_{n}"] = (rng.integers(0, 20, n).astype(float).tolist(),
                              rng.integers(0, 50, n).astype(float).tolist())
    out = {}
    for name, (p, t) in cases.items():
        out[f"{name}_p"] = np.array(p)
        out[f"{name}_t"] = np.array(t)
        out[f"{name}_d"] = np.array(predictor.kendall_tau_distance(p, t))
    for bad, (p, t) in {"len": ([1.0, 2.0], [1.0]), "short": ([1.0], [1.0])}.items():
        try:
            predictor.kendall_tau_distance(p, t)
        except SimError as exc:
            out[f"err_{bad}"] = np.array(type(exc).__name__)
    recs = workload.load_trace(os.path.join(OUT, "trace_small.ndjson"))
    ids = sorted(recs[0].model_ids)
    stats = {m: workload.LengthStats(300 + 150 * i, 200 + 50 * i) for i, m in enumerate(ids)}
    succ = {m: {"easy": 0.6, "hard": 0.2} for m in ids}
    training = workload.synthesize_trace(workload.CODE_WORKFLOWS, stats, succ, 400, 41)
    training += workload.synthesize_trace(workload.MATH_WORKFLOWS, stats, succ, 400, 42)
    preds = {"oracle": predictor.OraclePredictor(), "input-length": predictor.InputLengthPredictor(),
             "quantile": predictor.EmpiricalQuantilePredictor(training, 0.5),
             "quantile90": predictor.EmpiricalQuantilePredictor(training, 0.9)}
    for pname, pr in preds.items():
        out[f"eval_{pname}"] = np.array([predictor.evaluate_predictor(pr, recs, m) for m in ids])
    out["eval_arrival"] = np.array([predictor.arrival_order_distance(recs, m) for m in ids])
    np.savez_compressed(os.path.join(OUT, "kendall.npz"), cases=np.array(sorted(cases)), **out)
    workload.save_trace(training, os.path.join(OUT, "kendall_training.ndjson"))
    return len(cases)


def _edit(rec, how):
    import copy
    d = copy.deepcopy(rec)
    if how == "neg":
        first = sorted(d["stages"][0]["models"])[0]
        d["stages"][0]["models"][first]["out_tokens"] = -3
    elif how == "idx":
        d["stages"][0]["stage_index"] = 2
    elif how == "models":
        first = sorted(d["success"])[0]
        del d["success"][first]
        for st in d["stages"]:
            del st["models"][first]
    elif how == "base":
        d["stages"][-1]["base_input_tokens"] = 0
    return d


def _reference_rows(sc, ids, state, engines, recs, rt_tab, pr_tab):
    """schedule_request over sc's rows against a live SchedulerState."""
    k = len(ids)
    n = len(sc["prog"])
    reqs = []
    for i in range(n):
        pid = f"p{int(sc['prog'][i]):06d}"
        st = int(sc["stage"][i])
        req = workload.Request(pid, st, 10, float(sc["arrival"][i]), "wf", "r")
        rt_tab[req.request_id] = {ids[m]: float(sc["q"][i, m]) for m in range(k)}
        pr_tab[req.request_id] = {ids[m]: float(sc["yhat"][i, m]) for m in range(k)}
        rec = recs.get(pid)
        if rec is None:
            rec = workload.TraceRecord(pid, "wf", 0.0, [], {mid: 0 for mid in ids}, "easy")
            recs[pid] = rec
        while rec.n_stages < st:
            rec.stages.append(workload.StageTrace(rec.n_stages + 1, "r", 10, {
                mid: workload.ModelStageOutput(0, 0) for mid in ids}))
        rec.stages[st - 1].models = {
            ids[m]: workload.ModelStageOutput(int(sc["out_tok"][i, m]), 0) for m in range(k)}
        reqs.append(req)
    rt, pr = ShimRouter(rt_tab), ShimPredictor(pr_tab)
    cfg = balancer.BalancerConfig(sc["tau"], sc["margin"])
    model = np.full(n, -1, dtype=np.int32)
    prio = np.zeros(n)
    cached = np.zeros(n, dtype=np.int8)
    loads = np.full((n, k), np.nan)
    err = None
    for i, req in enumerate(reqs):
        try:
            d = balancer.schedule_request(req, recs[req.program_id], state, rt, pr, cfg)
        except (SimError, ValueError) as exc:
            err = {"kind": type(exc).__name__, "row": i}
            break
        model[i] = ids.index(d.model)
        prio[i] = d.priority
        cached[i] = int(d.used_cached_assignment)
        if d.estimated_loads:
            loads[i] = [d.estimated_loads[mid] for mid in ids]
    return dict(model=model, priority=prio, cached=cached, loads=loads), err


COMPLETION_SPECS = {
    "c5_dyadic": dict(seed=21, k=5, n1=1500, n2=1500, p0=800, dyadic=True, frac=0.4),
    "c3_nondyadic": dict(seed=22, k=3, n1=1000, n2=800, p0=200, dyadic=False, frac=0.5),
    "c8_mixed": dict(seed=23, k=8, n1=2000, n2=1500, p0=300, dyadic=False, frac=0.3),
    "c4_all": dict(seed=24, k=4, n1=600, n2=600, p0=100, dyadic=True, frac=1.0),
    # ActivityMonitor(decay_in_flight=True) + note_progress before the completions
    "c5_decay": dict(seed=25, k=5, n1=1200, n2=1000, p0=300, dyadic=True, frac=0.3, decay=True),
    "c3_decay_nondyadic": dict(seed=26, k=3, n1=800, n2=700, p0=150, dyadic=False, frac=0.4,
                               decay=True),
}


def make_completions(only=None):
    """Completion path (monitor.py:98-129): batch 1 through schedule_request,
    then (decay specs) note_progress for a random subset of live requests plus
    unknown ids and repeats, then record_completion for a random subset of the
    live requests (batch-1 rows and pre-seeded entries, shuffled), then batch 2
    -- fresh programs and later stages of batch-1 programs -- against the
    reduced (decayed) in-flight sums."""
    out = {}
    for name, sp in COMPLETION_SPECS.items():
        if only is not None and name not in only:
            continue
        rng = np.random.default_rng(sp["seed"] + 1000)
        k, n1, n2 = sp["k"], sp["n1"], sp["n2"]
        sc1 = build_scenario(sp["seed"], k, n1, dyadic=sp["dyadic"], p0_entries=sp["p0"],
                             pre_assigned=0.1)
        sc2 = build_scenario(sp["seed"] + 100, k, n2, dyadic=sp["dyadic"])
        # batch 2 programs: half fresh, half the next stage of a batch-1 program
        last_stage = {}
        for p, s in zip(sc1["prog"].tolist(), sc1["stage"].tolist()):
            last_stage[p] = max(last_stage.get(p, 0), s)
        b1_progs = sorted(last_stage)
        prog2, stage2 = [], []
        for i in range(n2):
            if rng.random() < 0.5:
                p = int(b1_progs[int(rng.integers(0, len(b1_progs)))])
                last_stage[p] += 1
                prog2.append(p)
                stage2.append(last_stage[p])
            else:
                p = n1 + 16 + i
                last_stage[p] = 1
                prog2.append(p)
                stage2.append(1)
        sc2["prog"] = np.array(prog2, dtype=np.int32)
        sc2["stage"] = np.array(stage2, dtype=np.int32)
        sc2["arrival"] = np.sort(rng.random(n2) * 10.0) + 20.0
        n_prog = n1 + n2 + 32
        ids = sc1["ids"]
        pool = profiles.Pool(tuple(profiles.ModelProfile(ids[i], sc1["decode"][i],
                                                         sc1["batch"][i]) for i in range(k)))
        decay = bool(sp.get("decay", False))
        mon = monitor.ActivityMonitor(ids, decay_in_flight=decay)
        seed_pos = {m: 0 for m in range(k)}
        seed_keys = []
        for j, (m, v) in enumerate(sc1["p0"]):
            mon.record_dispatch(ids[m], f"seed:{j}", v)
            seed_pos[m] += 1
            seed_keys.append((m, -seed_pos[m], f"seed:{j}"))
        for p, m in sc1["pre"].items():
            mon.assign(f"p{p:06d}", ids[m])
        engines = {mid: engine.EngineSim(pool[mid], aging=engine.AgingConfig()) for mid in ids}
        state = balancer.SchedulerState(pool=pool, monitor=mon, queues=engines)
        recs, rt_tab, pr_tab = {}, {}, {}
        res1, err1 = _reference_rows(sc1, ids, state, engines, recs, rt_tab, pr_tab)
        assert err1 is None, err1
        live = [(int(res1["model"][i]), int(sc1["prog"][i]) * 32 + int(sc1["stage"][i]) - 1,
                 f"p{int(sc1['prog'][i]):06d}:{int(sc1['stage'][i])}") for i in range(n1)]
        live += seed_keys
        prog_upd = []  # (model, key, emitted) in call order
        if decay:
            for m, kk, rid in live:
                if rng.random() < 0.5:
                    y = mon._in_flight[ids[m]][rid]
                    e = float(rng.integers(0, int(2 * y) + 2)) / (2 if sp["dyadic"] else 3)
                    mon.note_progress(ids[m], rid, e)
                    prog_upd.append((m, kk, e))
            rows = [c for c in live if c[1] >= 0]  # program keys are unique across models
            for _ in range(20):  # not in flight on that model: ignored
                m, kk, rid = rows[int(rng.integers(0, len(rows)))]
                mon.note_progress(ids[(m + 1) % k], rid, 5.0)
                prog_upd.append(((m + 1) % k, kk, 5.0))
            for _ in range(30):  # repeats: the last call wins
                m, kk, rid = live[int(rng.integers(0, len(live)))]
                e = float(rng.integers(0, 50))
                mon.note_progress(ids[m], rid, e)
                prog_upd.append((m, kk, e))
        prog_p = np.array([mon.in_flight_sum(mid) for mid in ids], dtype=np.float64)
        pick = [c for c in live if rng.random() < sp["frac"]]
        rng.shuffle(pick)
        for m, _, rid in pick:
            mon.record_completion(ids[m], rid, 0, 0.0)
        mid_p = np.array([mon.in_flight_sum(mid) for mid in ids], dtype=np.float64)
        mid_cnt = np.array([mon.in_flight_count(mid) for mid in ids], dtype=np.int64)
        res2, err2 = _reference_rows(sc2, ids, state, engines, recs, rt_tab, pr_tab)
        final_p = np.array([mon.in_flight_sum(mid) for mid in ids], dtype=np.float64)
        final_cnt = np.array([mon.in_flight_count(mid) for mid in ids], dtype=np.int64)
        p0 = np.array(sc1["p0"], dtype=np.float64).reshape(-1, 2)
        pre = np.array(sorted(sc1["pre"].items()), dtype=np.int64).reshape(-1, 2)
        np.savez_compressed(
            os.path.join(OUT, f"complete_{name}.npz"),
            k=k, decode=np.array(sc1["decode"]), batch=np.array(sc1["batch"], dtype=np.int32),
            n_prog=n_prog, tau=sc1["tau"], margin=sc1["margin"], p0=p0, pre=pre,
            prog1=sc1["prog"], stage1=sc1["stage"], q1=sc1["q"], yhat1=sc1["yhat"],
            out_tok1=sc1["out_tok"], arrival1=sc1["arrival"],
            prog2=sc2["prog"], stage2=sc2["stage"], q2=sc2["q"], yhat2=sc2["yhat"],
            out_tok2=sc2["out_tok"], arrival2=sc2["arrival"],
            decay=int(decay), prog_p=prog_p,
            p_model=np.array([u[0] for u in prog_upd], dtype=np.int32),
            p_key=np.array([u[1] for u in prog_upd], dtype=np.int64),
            p_emitted=np.array([u[2] for u in prog_upd], dtype=np.float64),
            c_model=np.array([c[0] for c in pick], dtype=np.int32),
            c_key=np.array([c[1] for c in pick], dtype=np.int64),
            mid_p=mid_p, mid_cnt=mid_cnt, final_p=final_p, final_cnt=final_cnt,
            err2_kind=(err2 or {}).get("kind", ""), err2_row=(err2 or {}).get("row", -1),
            **{f"out1_{kk}": v for kk, v in res1.items()},
            **{f"out2_{kk}": v for kk, v in res2.items()})
        out[name] = (len(pick), err2)
    return out


# ------------------------------------------------------------- engine clock
def run_engine_script(seed, b, S, d, p, n_pre, script):
    """One EngineSim with decode d / prefill p ms per token. Steps: ("enq", n, dt)
    enqueue n requests at t += dt; ("iter", n) n scheduling iterations at the
    current clock; ("adv", dt) advance_to(t += dt)."""
    rng = np.random.default_rng(seed)
    prof = profiles.ModelProfile("m0", d, b, prefill_ms_per_token=p)
    aging = engine.AgingConfig(starvation_threshold=S if S else math.inf)
    eng = engine.EngineSim(prof, aging=aging)
    t = 0.0
    ordinal = 0
    enq_log, admitted, done = [], [], []
    orig_admit = eng._admit

    def spy(entry, now):
        admitted.append(int(entry.request.program_id[1:]))
        return orig_admit(entry, now)
    eng._admit = spy

    def enqueue(n):
        nonlocal ordinal
        for _ in range(n):
            prio = float(rng.integers(1, 400))
            if seed % 2:
                prio /= 3.0
            inp = int(rng.integers(1, 3000))
            out = int(rng.integers(1, 400))
            rq = workload.Request(f"e{ordinal}", 1, inp, t, "wf", "x")
            eng.enqueue(rq, priority=prio, out_tokens=out, now=t)
            enq_log.append((ordinal, prio, t, inp, out))
            ordinal += 1

    enqueue(n_pre)
    for step in script:
        if step[0] == "enq":
            t += step[2]
            enqueue(step[1])
        elif step[0] == "iter":
            for _ in range(step[1]):
                eng.scheduling_iteration(eng.now)
        else:
            t += step[1]
            for c in eng.advance_to(t):
                done.append((int(c.request.program_id[1:]), c.time))
    order = [int(e.request.program_id[1:]) for e in sorted(eng._queued.values(),
                                                             key=lambda e: e.sort_key())]
    lv = {int(e.request.program_id[1:]): (e.starvation_level, e.starvation_count)
          for e in eng._queued.values()}
    running = [(s, int(rr.entry.request.program_id[1:]), rr.stint_end)
               for s, rr in sorted(eng.running.items())]
    return dict(enq=np.array(enq_log, dtype=np.float64), admitted=np.array(admitted),
                done=np.array(done, dtype=np.float64).reshape(-1, 2),
                order=np.array(order), level=np.array([lv[o][0] for o in order]),
                count=np.array([lv[o][1] for o in order]),
                running=np.array(running, dtype=np.float64).reshape(-1, 3),
                now=eng.now, tokens=eng.tokens_emitted_total, served=eng.requests_served,
                iterations=eng.iterations)


def make_engines():
    scripts = {
        "e_basic": (11, 4, 8, 0.75, 0.02, 20,
                    [("adv", 50.0), ("iter", 2), ("enq", 10, 1.0), ("adv", 200.0),
                     ("adv", 150.0)]),
        "e_nondyadic": (12, 3, 3, 1.0 / 3.0, 0.013, 40,
                        [("adv", 30.0), ("enq", 7, 0.5), ("adv", 95.25), ("iter", 3),
                         ("adv", 400.0), ("enq", 12, 0.0), ("adv", 2500.0)]),
        "e_noaging": (13, 2, 0, 1.5, 0.0, 15,
                      [("adv", 100.0), ("enq", 5, 2.0), ("adv", 700.0), ("adv", 5000.0)]),
        "e_big": (15, 32, 8, 0.05, 0.001, 600,
                  [("adv", 5.0), ("adv", 20.0), ("enq", 200, 0.0), ("iter", 4), ("adv", 60.0),
                   ("adv", 150.0), ("enq", 50, 0.0), ("adv", 40.0)]),
        "e_S1": (17, 2, 1, 2.0, 0.5, 25, [("adv", 800.0), ("iter", 3), ("adv", 3000.0)]),
    }
    out = {}
    for name, (seed, b, S, d, p, n_pre, script) in scripts.items():
        res = run_engine_script(seed, b, S, d, p, n_pre, script)
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), seed=seed, b=b, S=S, d=d, p=p,
                            n_pre=n_pre, script=json.dumps(script), **res)
        out[name] = (len(res["done"]), len(res["order"]), len(res["running"]))
    return out


if __name__ == "__main__":
    if sys.argv[1:2] == ["queues"]:
        make_queues(sys.argv[2:] or None)
        sys.exit(0)
    if sys.argv[1:] == ["engines"]:
        print("engines:", make_engines())
        sys.exit(0)
    if sys.argv[1:] == ["select"]:
        print("select cases:", make_select_kat())
        print("schedule:", make_schedules())
        sys.exit(0)
    if sys.argv[1:] == ["completions"]:
        print("completions:", make_completions())
        sys.exit(0)
    print("completions:", make_completions())
    print("select cases:", make_select_kat())
    print("schedule:", make_schedules())
    print("errors:", make_errors())
    make_queues()
    print("engines:", make_engines())
    make_quantile()
    make_synth()
    print("trace programs:", make_trace())
    print("kendall cases:", make_kendall())
    print("done")
