"""Shared drivers for the parity tests: golden fixtures -> oracle port / GPU."""

from __future__ import annotations

import glob
import json
import os

import numpy as np

from oracle import hetsched_port as hp
from paper_2603_22206_b200.config import ModelProfile, Pool
from workloads.tracegen import ModelStageOutput, Request, StageTrace, TraceRecord

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def schedule_names(prefix="schedule_"):
    return sorted(os.path.basename(p)[len(prefix):-4]
                  for p in glob.glob(os.path.join(GOLDEN, f"{prefix}*.npz")))


def load_schedule(name):
    z = np.load(os.path.join(GOLDEN, f"schedule_{name}.npz"), allow_pickle=False)
    sc = {k: z[k] for k in z.files}
    sc["k"] = int(sc["k"])
    sc["n_prog"] = int(sc["n_prog"])
    sc["tau"] = float(sc["tau"])
    sc["margin"] = float(sc["margin"])
    sc["err_kind"] = str(sc["err_kind"])
    sc["err_row"] = int(sc["err_row"])
    sc["ids"] = [f"m{i}" for i in range(sc["k"])]
    return sc


def pool_of(sc):
    ids = sc["ids"]
    return Pool(tuple(ModelProfile(ids[i], float(sc["decode"][i]), int(sc["batch"][i]))
                      for i in range(sc["k"])))


def requests_of(sc):
    """Request / TraceRecord objects equivalent to the golden generator's."""
    ids, k = sc["ids"], sc["k"]
    recs, reqs = {}, []
    for i in range(len(sc["prog"])):
        pid = f"p{int(sc['prog'][i]):06d}"
        st = int(sc["stage"][i])
        reqs.append(Request(pid, st, 10, float(sc["arrival"][i]), "wf", "r"))
        rec = recs.get(pid)
        if rec is None:
            rec = TraceRecord(pid, "wf", 0.0, [], {m: 0 for m in ids}, "easy")
            recs[pid] = rec
        while rec.n_stages < st:
            rec.stages.append(StageTrace(rec.n_stages + 1, "r", 10,
                                         {m: ModelStageOutput(0, 0) for m in ids}))
        rec.stages[st - 1].models = {ids[m]: ModelStageOutput(int(sc["out_tok"][i, m]), 0)
                                     for m in range(k)}
    return reqs, [recs[r.program_id] for r in reqs]


def run_port_schedule(sc):
    ids, k = sc["ids"], sc["k"]
    pool = pool_of(sc)
    mon = hp.PortMonitor(ids)
    for j, (m, v) in enumerate(sc["p0"]):
        mon.record_dispatch(ids[int(m)], f"seed:{j}", float(v))
    for p, m in sc["pre"]:
        mon.assign(f"p{int(p):06d}", ids[int(m)])
    engines = {mid: hp.PortEngine(pool[mid].max_batch_size) for mid in ids}
    for i, mid in enumerate(ids):
        for j in range(int(sc["pre_running"][i])):
            engines[mid].enqueue(f"r{i}x{j}", 1.0, 10 ** 6, 0.0)
    reqs, recs = requests_of(sc)
    qtab = {r.request_id: {ids[m]: float(sc["q"][i, m]) for m in range(k)}
            for i, r in enumerate(reqs)}
    ytab = {r.request_id: {ids[m]: float(sc["yhat"][i, m]) for m in range(k)}
            for i, r in enumerate(reqs)}
    n = len(reqs)
    res = dict(model=np.full(n, -1, np.int32), priority=np.zeros(n), cached=np.zeros(n, np.int8),
               loads=np.full((n, k), np.nan), seq=np.full(n, -1, np.int64),
               admitted=np.zeros(n, np.int8))
    err = None
    for i, (r, rec) in enumerate(zip(reqs, recs)):
        try:
            d = hp.port_schedule_request(r, rec, pool, mon, engines,
                                         lambda rq, rc: qtab[rq.request_id],
                                         lambda rq, rc, m: ytab[rq.request_id][m],
                                         sc["tau"], sc["margin"])
        except hp.PortError as exc:
            err = {"kind": exc.kind, "row": i}
            break
        mi = ids.index(d.model)
        res["model"][i] = mi
        res["priority"][i] = d.priority
        res["cached"][i] = int(d.used_cached_assignment)
        if d.estimated_loads:
            res["loads"][i] = [d.estimated_loads[m] for m in ids]
        e = engines[d.model]
        for s, ent in e.running.items():
            if ent.rid == r.request_id:
                res["seq"][i], res["admitted"][i] = s, 1
        for s, ent in e.queued.items():
            if ent.rid == r.request_id:
                res["seq"][i] = s
    res["final_p"] = np.array([mon.in_flight_sum(m) for m in ids], dtype=np.float64)
    res["final_cnt"] = np.array([len(mon.live[m]) for m in ids], dtype=np.int64)
    res["running"] = np.array([engines[m].running_count for m in ids], np.int32)
    res["queued"] = np.array([engines[m].waiting_count for m in ids], np.int32)
    assign = np.full(sc["n_prog"], -1, np.int8)
    for p in range(sc["n_prog"]):
        a = mon.assignment(f"p{p:06d}")
        if a is not None:
            assign[p] = ids.index(a)
    res["assign"] = assign
    return res, err


# ----------------------------------------------------------------- completions
def complete_names():
    return schedule_names(prefix="complete_")


def load_complete(name):
    """A completion golden as two schedule-like batches sharing one state."""
    z = np.load(os.path.join(GOLDEN, f"complete_{name}.npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    k = int(d["k"])
    common = dict(k=k, decode=d["decode"], batch=d["batch"], n_prog=int(d["n_prog"]),
                  tau=float(d["tau"]), margin=float(d["margin"]), p0=d["p0"], pre=d["pre"],
                  pre_running=np.zeros(k, np.int32), ids=[f"m{i}" for i in range(k)])
    b1 = dict(common, prog=d["prog1"], stage=d["stage1"], q=d["q1"], yhat=d["yhat1"],
              out_tok=d["out_tok1"], arrival=d["arrival1"])
    b2 = dict(common, prog=d["prog2"], stage=d["stage2"], q=d["q2"], yhat=d["yhat2"],
              out_tok=d["out_tok2"], arrival=d["arrival2"], p0=np.zeros((0, 2)),
              pre=np.zeros((0, 2), np.int64))
    d.setdefault("decay", np.array(0))
    for key, dt in (("p_model", np.int32), ("p_key", np.int64), ("p_emitted", np.float64)):
        d.setdefault(key, np.zeros(0, dt))
    return d, b1, b2


def seed_request_ids(p0, k):
    """(model, log key) -> request id "seed:j" of the pre-seeded entries."""
    pos = {m: 0 for m in range(k)}
    out = {}
    for j, (m, _) in enumerate(p0):
        m = int(m)
        pos[m] += 1
        out[(m, -pos[m])] = f"seed:{j}"
    return out


def run_port_complete(name):
    """Replay a completion golden on the oracle port: batch 1, the
    record_completion list, batch 2 (one monitor / engine set throughout)."""
    d, b1, b2 = load_complete(name)
    ids, k = b1["ids"], b1["k"]
    pool = pool_of(b1)
    mon = hp.PortMonitor(ids, decay_in_flight=bool(int(d["decay"])))
    for j, (m, v) in enumerate(b1["p0"]):
        mon.record_dispatch(ids[int(m)], f"seed:{j}", float(v))
    for p, m in b1["pre"]:
        mon.assign(f"p{int(p):06d}", ids[int(m)])
    engines = {mid: hp.PortEngine(pool[mid].max_batch_size) for mid in ids}
    seeds = seed_request_ids(b1["p0"], k)

    def rid_of(m, key):
        return seeds[(m, key)] if key < 0 else f"p{key // 32:06d}:{key % 32 + 1}"

    def run(sc):
        reqs, recs = requests_of(sc)
        qtab = {r.request_id: {ids[m]: float(sc["q"][i, m]) for m in range(k)}
                for i, r in enumerate(reqs)}
        ytab = {r.request_id: {ids[m]: float(sc["yhat"][i, m]) for m in range(k)}
                for i, r in enumerate(reqs)}
        n = len(reqs)
        res = dict(model=np.full(n, -1, np.int32), priority=np.zeros(n),
                   cached=np.zeros(n, np.int8), loads=np.full((n, k), np.nan))
        for i, (r, rec) in enumerate(zip(reqs, recs)):
            dd = hp.port_schedule_request(r, rec, pool, mon, engines,
                                          lambda rq, rc: qtab[rq.request_id],
                                          lambda rq, rc, m: ytab[rq.request_id][m],
                                          sc["tau"], sc["margin"])
            res["model"][i] = ids.index(dd.model)
            res["priority"][i] = dd.priority
            res["cached"][i] = int(dd.used_cached_assignment)
            if dd.estimated_loads:
                res["loads"][i] = [dd.estimated_loads[m] for m in ids]
        return res

    r1 = run(b1)
    for m, key, e in zip(d["p_model"].tolist(), d["p_key"].tolist(), d["p_emitted"].tolist()):
        # (updates naming another model use program keys, unique across models)
        mon.note_progress(ids[m], rid_of(m, key) if key >= 0 else seeds[(m, key)], e)
    if len(d["p_model"]):
        assert np.array([mon.in_flight_sum(m) for m in ids]).tobytes() == d["prog_p"].tobytes()
    for m, key in zip(d["c_model"].tolist(), d["c_key"].tolist()):
        mon.record_completion(ids[m], rid_of(m, key))
    mid_p = np.array([mon.in_flight_sum(m) for m in ids], dtype=np.float64)
    mid_cnt = np.array([len(mon.live[m]) for m in ids], dtype=np.int64)
    r2 = run(b2)
    final_p = np.array([mon.in_flight_sum(m) for m in ids], dtype=np.float64)
    return d, r1, r2, mid_p, mid_cnt, final_p


# ----------------------------------------------------------------- queues
def queue_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "q_*.npz")))


def load_queue(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["script"] = json.loads(str(d["script"]))
    for k in ("seed", "b", "n_pre", "running", "iterations"):
        d[k] = int(d[k])
    d["S"] = float(d["S"])  # fractional thresholds compare count >= S (engine.py:348)
    d["Q"] = float(d["Q"]) if "Q" in d else 4
    d["demote"] = bool(int(d["demote"])) if "demote" in d else False
    return d


def run_port_queue(qd):
    """Replay a golden queue script on the oracle port engine."""
    import math
    S = qd["S"] if qd["S"] else math.inf
    eng = hp.PortEngine(qd["b"], starvation_threshold=S, running_quantum=qd["Q"],
                        demote_while_queued=qd["demote"])
    enq = qd["enq"]
    pos = 0
    t = 0.0

    def enqueue(n):
        nonlocal pos
        for _ in range(n):
            o, p, tt = enq[pos]
            eng.enqueue(int(o), float(p), 10 ** 9, float(tt))
            pos += 1

    enqueue(qd["n_pre"])
    for op, n in qd["script"]:
        t += 1.0
        if op == "enq":
            enqueue(n)
        elif op == "iter":
            for j in range(n):
                eng.scheduling_iteration(t + j)
            t += n - 1
        else:
            eng.complete(n, t)
    order = [e.rid for e in eng.queue_order()]
    return dict(admitted=np.array(eng.admitted_log), order=np.array(order),
                level=np.array([e.level for e in eng.queue_order()]),
                count=np.array([e.count for e in eng.queue_order()]),
                running=eng.running_count, iterations=eng.iterations)


# ------------------------------------------------------------ engine clock
def engine_names():
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "e_*.npz")))


def load_engine(name):
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)
    d = {k: z[k] for k in z.files}
    d["script"] = json.loads(str(d["script"]))
    for k in ("seed", "b", "S", "n_pre", "tokens", "served", "iterations"):
        d[k] = int(d[k])
    for k in ("d", "p", "now"):
        d[k] = float(d[k])
    return d
