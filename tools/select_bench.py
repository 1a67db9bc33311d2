"""K6 chain micro-benchmark: chm_schedule_rows alone on a cfg3-shaped batch
(B rows, K models, table scores, quantile-like dyadic or non-dyadic
predictions), timed with CUDA events; prints ns/decision per variant.

  python tools/select_bench.py [--rows 4096] [--k 5] [--reps 20]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--rows", type=int, default=4096)
    p.add_argument("--k", type=int, default=5)
    p.add_argument("--reps", type=int, default=20)
    a = p.parse_args()
    import numpy as np
    import torch

    from paper_2603_22206_b200 import _lib
    from paper_2603_22206_b200.config import BalancerConfig, ModelProfile, Pool
    from paper_2603_22206_b200.predictor import PrecomputedPredictor
    from paper_2603_22206_b200.router import ScoreTableRouter
    from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch

    B, K = a.rows, a.k
    rng = np.random.default_rng(0)
    out = {}
    for name, pow2, dyadic in (("dyadic_pow2", True, True), ("dyadic_pow2_clustered", True, True),
                               ("nondyadic_pow2", True, False), ("dyadic_nonpow2", False, True)):
        pool = Pool(tuple(ModelProfile(f"m{i}", 5.0 * (i + 1),
                                       max(1, 32 >> i) if pow2 else 3 + 2 * i)
                          for i in range(K)))
        rt, pr = ScoreTableRouter(), PrecomputedPredictor()
        gs = GpuScheduler(pool, BalancerConfig(0.5, 0.1), router=rt, predictor=pr,
                          n_programs=2 * B, max_rows=B)
        # clustered: router confidences near 0.5 (random-init router, cfg3): the
        # gate rarely passes and the chain is the argmin (m_fast) regime
        q = (np.clip(0.5 + 0.01 * rng.standard_normal((B, K)), 0, 1) if "clustered" in name
             else rng.random((B, K)))
        y = rng.integers(0, 4000, (B, K)) / 2.0 if dyadic else rng.lognormal(6, 1, (B, K))
        rt.set(torch.as_tensor(q, device="cuda"))
        pr.set(torch.as_tensor(y, device="cuda"))
        batch = RowBatch.from_numpy("cuda", program=np.arange(B), stage=np.ones(B),
                                    arrival=np.zeros(B), out_tokens=np.ones((B, K)),
                                    handle=np.arange(B))
        snap = gs.state.snapshot()
        ms = []
        for r in range(a.reps + 3):
            gs.state.restore(snap)
            _lib.profile_read()
            _lib.profile_enable(True)
            gs.run_rows(batch, n_iterations=0)
            torch.cuda.synchronize()
            prof = _lib.profile_read()
            _lib.profile_enable(False)
            if r >= 3:
                ms.append(prof["select"]["ms"])
        gs.check_errors()
        med = float(np.median(ms))
        out[name] = {"select_ms": med, "ns_per_decision": med * 1e6 / B}
    print(json.dumps({"rows": B, "K": K, **out}))


if __name__ == "__main__":
    main()
