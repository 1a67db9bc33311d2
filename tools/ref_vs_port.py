"""The unmodified reference (hetsched, imported read-only -- build container
only) against its oracle port (oracle/hetsched_port.py, the bench's CPU arm)
on the same cfg3 tick: B = 4096 first-stage requests, K = 5, the same router
scores (a precomputed table) and the same quantile predictor. Both run
schedule_request per row plus one scheduling iteration per engine, 1 thread.
Shows how the port's per-tick time relates to the reference's own.

  PYTHONDONTWRITEBYTECODE=1 python tools/ref_vs_port.py [--config cfg3] [--ticks 3]
"""

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.dont_write_bytecode = True


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="cfg3")
    p.add_argument("--ticks", type=int, default=3)
    a = p.parse_args()
    import numpy as np
    sys.path.insert(0, "/root/reference/pkg/src")
    from hetsched import balancer, engine, monitor, predictor, profiles, router, workload

    from oracle import hetsched_port as hp
    from workloads import synth
    wl = synth.make_workload(a.config, device="cpu", with_router=False)
    B, K = wl.batch_size, len(wl.pool)
    ids = wl.pool.model_ids
    pool = profiles.Pool(tuple(profiles.ModelProfile(m, wl.pool[m].decode_ms_per_token,
                                                     wl.pool[m].max_batch_size) for m in ids))
    q = np.random.default_rng(0).random((B, K))
    ref_t, port_t = [], []
    for t in range(a.ticks):
        cols = wl.host_columns(t)
        recs = cols["records"]
        reqs = [workload.first_stage_request(rec, float(cols["arrival"][i]))
                for i, rec in enumerate(recs)]
        qtab = {r.request_id: {m: float(q[i, k]) for k, m in enumerate(ids)}
                for i, r in enumerate(reqs)}

        class Shim(router.Router):
            def _score_one(self, req, rec, model_id):
                return qtab[req.request_id][model_id]

        pred = predictor.EmpiricalQuantilePredictor(wl.training, 0.5)
        mon = monitor.ActivityMonitor(ids)
        engines = {m: engine.EngineSim(pool[m]) for m in ids}
        st = balancer.SchedulerState(pool=pool, monitor=mon, queues=engines)
        cfg = balancer.BalancerConfig(wl.balancer.latency_slack, wl.balancer.confidence_margin)
        rt = Shim()
        t0 = time.perf_counter()
        for r, rec in zip(reqs, recs):
            balancer.schedule_request(r, rec, st, rt, pred, cfg)
        for m in ids:
            engines[m].scheduling_iteration(max(float(cols["arrival"].max()), engines[m].now))
        ref_t.append(time.perf_counter() - t0)
        # the port, same inputs
        pmon = hp.PortMonitor(ids)
        peng = {m: hp.PortEngine(wl.pool[m].max_batch_size) for m in ids}
        ppred = hp.PortQuantilePredictor(wl.training, 0.5)
        t0 = time.perf_counter()
        hp.port_tick(reqs, recs, wl.pool, pmon, peng, lambda rq, rc: qtab[rq.request_id], ppred,
                     wl.balancer.latency_slack, wl.balancer.confidence_margin, 1)
        port_t.append(time.perf_counter() - t0)
    r, pt = statistics.median(ref_t), statistics.median(port_t)
    print(json.dumps({"config": a.config, "rows": B, "reference_ms_per_tick": r * 1e3,
                      "port_ms_per_tick": pt * 1e3, "reference_over_port": r / pt,
                      "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0]
                      .strip(" :\t")}))


if __name__ == "__main__":
    main()
