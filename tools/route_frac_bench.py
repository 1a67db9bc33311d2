"""Router time vs routed fraction: the encoder runs only for the rows
chm_prepare_rows listed (the reference skips the router on the reuse branch,
balancer.py:104-114); n_route is read on the device, so the same launch
sequence (or CUDA graph) serves any cached fraction.

  python tools/route_frac_bench.py [--config cfg3] [--reps 5]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="cfg3")
    p.add_argument("--reps", type=int, default=5)
    a = p.parse_args()
    import torch

    from paper_2603_22206_b200.encoder import GpuEncoderRouter, synthetic_token_ids
    from workloads.synth import SPECS

    sp = SPECS[a.config]
    B, K, cfg = sp.batch, sp.n_models, sp.encoder
    r = GpuEncoderRouter(cfg, K, max_rows=B, seed=0)
    ids = torch.as_tensor(synthetic_token_ids(B, cfg.seq_len, 5), device="cuda")
    rows = torch.randperm(B, device="cuda").to(torch.int32)
    q = torch.zeros(B * K, dtype=torch.float64, device="cuda")
    n_dev = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = {"config": a.config, "batch": B}
    for frac in (1.0, 0.75, 0.5, 0.25, 0.0):
        n_dev.fill_(int(round(frac * B)))
        for _ in range(2):
            r.forward(ids, q, rows=rows, n_rows=n_dev, n_seq=B)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            r.forward(ids, q, rows=rows, n_rows=n_dev, n_seq=B)
        e1.record()
        torch.cuda.synchronize()
        out[f"routed_{frac:.2f}_ms"] = e0.elapsed_time(e1) / a.reps
    print(json.dumps(out))


if __name__ == "__main__":
    main()
