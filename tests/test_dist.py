"""Multi-process (gloo, world_size 2, CPU) tests of the sharded-tick protocol
in paper_2603_22206_b200/dist.py: Mode B relay decisions equal one serial
replay of the reference path over the concatenated batch; Mode A equals
independent shard replays from P0 with the deltas all-reduced."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hetsched_port as hp
from tests import harness as H


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _chain(sc, rows, s, c):
    """Serial chain over `rows` from monitor state (s, c): the port's
    select_model plus the Neumaier state update (CPU stand-in for K6)."""
    from paper_2603_22206_b200.state import neumaier_value
    ids, k = sc["ids"], sc["k"]
    d = [float(x) for x in sc["decode"]]
    b = [int(x) for x in sc["batch"]]
    s, c = list(s), list(c)
    out = []
    for i in rows:
        loads = {ids[m]: neumaier_value(s[m], c[m]) * d[m] / b[m] for m in range(k)}
        q = {ids[m]: float(sc["q"][i, m]) for m in range(k)}
        mid = hp.port_select_model(q, loads, sc["tau"], sc["margin"])
        m = ids.index(mid)
        y = float(sc["yhat"][i, m])
        t = s[m] + y
        c[m] += ((s[m] - t) + y) if abs(s[m]) >= abs(y) else ((y - t) + s[m])
        s[m] = t
        out.append(m)
    return out, s, c


def _p0_state(sc):
    from paper_2603_22206_b200.state import neumaier_state
    k = sc["k"]
    s, c = [0.0] * k, [0.0] * k
    for m in range(k):
        vals = [float(v) for mm, v in sc["p0"] if int(mm) == m]
        s[m], c[m] = neumaier_state(vals)
    return s, c


def _worker(rank, world, port, mode, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_22206_b200 import dist as D
    sc = H.load_schedule(name)
    n = len(sc["prog"])
    bounds = np.linspace(0, n, world + 1).astype(int)
    rows = list(range(bounds[rank], bounds[rank + 1]))
    k = sc["k"]
    s0, c0 = _p0_state(sc)
    if mode == "B":
        packed = torch.tensor(s0 + c0, dtype=torch.float64)
        D.relay_receive(packed)
        models, s, c = _chain(sc, rows, packed[:k].tolist(), packed[k:].tolist())
        packed.copy_(torch.tensor(s + c, dtype=torch.float64))
        D.relay_forward(packed)
        final = packed.tolist()
    else:
        models, s, c = _chain(sc, rows, s0, c0)
        st = torch.tensor(s, dtype=torch.float64)
        ct = torch.tensor(c, dtype=torch.float64)
        D.mode_a_allreduce(st, ct, torch.tensor(s0, dtype=torch.float64),
                           torch.tensor(c0, dtype=torch.float64))
        final = st.tolist() + ct.tolist()
    gathered = [None] * world
    dist.all_gather_object(gathered, models)
    if rank == 0:
        q.put((gathered, final))
    dist.barrier()
    dist.destroy_process_group()


def _run(mode, name, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, name, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("name", ["k5_nondyadic_p0", "k3_basic"])
def test_mode_b_relay_equals_serial_replay(name):
    sc = H.load_schedule(name)
    gathered, final = _run("B", name)
    # the unmodified-reference-equivalent serial replay (golden fixture)
    from paper_2603_22206_b200.state import neumaier_value
    got = np.array(sum(gathered, []))
    np.testing.assert_array_equal(got, sc["out_model"])
    k = sc["k"]
    p = np.array([neumaier_value(a, b) for a, b in zip(final[:k], final[k:])])
    assert p.tobytes() == sc["out_final_p"].tobytes()


def test_mode_a_equals_shard_replays_from_p0():
    name = "k3_basic"
    sc = H.load_schedule(name)
    gathered, final = _run("A", name)
    n = len(sc["prog"])
    bounds = np.linspace(0, n, 3).astype(int)
    s0, c0 = _p0_state(sc)
    want, deltas = [], np.zeros(sc["k"])
    from paper_2603_22206_b200.state import neumaier_value
    for r in range(2):
        models, s, c = _chain(sc, range(bounds[r], bounds[r + 1]), s0, c0)
        want += models
        deltas += np.array([neumaier_value(a, b) for a, b in zip(s, c)]) - \
            np.array([neumaier_value(a, b) for a, b in zip(s0, c0)])
    assert sum(gathered, []) == want
    p0 = np.array([neumaier_value(a, b) for a, b in zip(s0, c0)])
    np.testing.assert_array_equal(np.array(final[:sc["k"]]), p0 + deltas)


def test_shard_of_is_stable_and_balanced():
    from paper_2603_22206_b200.dist import shard_of
    ranks = [shard_of(f"p{i:06d}", 8) for i in range(8000)]
    assert ranks == [shard_of(f"p{i:06d}", 8) for i in range(8000)]
    counts = np.bincount(ranks, minlength=8)
    assert counts.min() > 850 and counts.max() < 1150
