"""Run a few scheduling ticks of a config for ncu captures (no timing output).

  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python tools/profile_tick.py --ticks 2
  ncu --set full --clock-control none --import-source on -k regex:gemm_kernel \
      -s 48 -c 4 -o gpurun_out/gemm python tools/profile_tick.py --ticks 2
"""

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="cfg3")
    p.add_argument("--ticks", type=int, default=2)
    a = p.parse_args()
    import torch

    from workloads import synth
    from paper_2603_22206_b200.scheduler import GpuScheduler

    wl = synth.make_workload(a.config)
    gs = GpuScheduler(wl.pool, wl.balancer, wl.aging, router=wl.router, predictor=wl.predictor,
                      n_programs=wl.n_programs, max_rows=wl.batch_size,
                      queue_capacity=wl.queue_capacity)
    wl.seed_state(gs.state)  # cfg4: 64k in flight + 64k queued (as bench.py)
    snap = gs.state.snapshot()
    batches = [wl.batch(t) for t in range(2)]
    completions = wl.completions()  # cfg4: every engine's running batch turns over (as bench.py)
    kw = {"completions": completions} if completions is not None else {}
    for t in range(a.ticks):
        gs.state.restore(snap)
        gs.run_rows(batches[t % 2], n_iterations=1, **kw)
    torch.cuda.synchronize()
    gs.check_errors()
    print("ticks done")


if __name__ == "__main__":
    main()
