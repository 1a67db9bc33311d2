"""bench.py's N > 1 flow (request-sharded ticks, in-flight exchange, max over
ranks) end to end under torchrun with two ranks sharing the one GPU of the
test box (gloo; the measured path uses NCCL on one GPU per rank). Guards the
driver's scaling run: round 2 found the N > 1 path restoring a snapshot taken
before the sharded scheduler extended the state."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("mode", ["A", "B"])
def test_bench_two_ranks(mode):
    env = dict(os.environ, CHM_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29611 + (mode == "B")),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "cfg1", "--steps", "2",
           "--warmup", "3", "--mode", mode, "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["steps"] == 2
