# CPU side of tools/engine_bench.py: the unmodified reference EngineSim
# (hetsched, imported read-only from /root/reference -- build container only)
# on the same setup: K = 8 engines x 8192 queued, b = 32, 4 windows.
import math, sys, time
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import numpy as np
from hetsched import engine, profiles, workload
rng = np.random.default_rng(7)
K, Qn, b = 8, 8192, 32
d_ms = [0.5 + 0.5 * k for k in range(K)]
engs = []
for k in range(K):
    e = engine.EngineSim(profiles.ModelProfile(f"m{k}", d_ms[k], b, prefill_ms_per_token=0.02),
                         aging=engine.AgingConfig(starvation_threshold=8))
    engs.append(e)
pr = rng.integers(1, 4000, (K, Qn)); ot = rng.integers(16, 600, (K, Qn)); it = rng.integers(64, 2048, (K, Qn))
t0 = time.perf_counter()
for k, e in enumerate(engs):
    for i in range(Qn):
        e.enqueue(workload.Request(f"p{k}_{i}", 1, int(it[k, i]), 0.0, "wf", "x"),
                  priority=float(pr[k, i]), out_tokens=int(ot[k, i]), now=0.0)
t_enq = time.perf_counter() - t0
mean_stint = 0.02 * 1056 + np.mean(d_ms) * 308
dt = 256 * mean_stint / b
t = 0.0
n = 0
t0 = time.perf_counter()
for w in range(4):
    t += dt
    for e in engs:
        n += len(e.advance_to(t))
el = time.perf_counter() - t0
print(dict(completions=n, seconds=el, completions_per_s=n / el, enqueue_s=t_enq))
