"""Multi-process (gloo, world_size 2, CPU) tests of the sharded-tick protocol
in paper_2603_22206_b200/dist.py over its TorchComm transport: Mode B relay
decisions equal one serial replay of the reference path over the
concatenated batch; Mode A equals independent shard replays from P0 with the
tick end folded in rank order (a restatement of chm_inflight_fold); the
global-admission queue protocol. The per-rank kernels are CPU stand-ins
here; tests/test_gpu_dist.py runs ShardedScheduler.run_rows with the real
kernels (two ranks sharing one GPU over gloo)."""

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


def _fold(s0, c0, records):
    """Restatement of chm_inflight_fold: the gathered (model, yhat) rows of
    every rank folded into (s, c) in rank order (Neumaier, monitor.py:127)."""
    s, c = list(s0), list(c0)
    for rows in records:
        for m, y in rows:
            t = s[m] + y
            c[m] += ((s[m] - t) + y) if abs(s[m]) >= abs(y) else ((y - t) + s[m])
            s[m] = t
    return s, c


def _worker(rank, world, port, mode, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_22206_b200 import dist as D
    comm = D.TorchComm()
    sc = H.load_schedule(name)
    n = len(sc["prog"])
    bounds = np.linspace(0, n, world + 1).astype(int)
    rows = list(range(bounds[rank], bounds[rank + 1]))
    k = sc["k"]
    s0, c0 = _p0_state(sc)
    if mode == "B":
        state = torch.tensor(s0 + c0, dtype=torch.float64)
        comm.relay_recv(state, None)
        models, s, c = _chain(sc, rows, state[:k].tolist(), state[k:].tolist())
        state.copy_(torch.tensor(s + c, dtype=torch.float64))
        comm.relay_send(state, None)
        final = state.tolist()
    else:
        models, s, c = _chain(sc, rows, s0, c0)
        # pack -> all-gather -> fold (the chm_allreduce_inflight protocol)
        rec = torch.tensor([[m, float(sc["yhat"][i, m])] for i, m in zip(rows, models)],
                           dtype=torch.float64)
        n_rec = torch.tensor([len(rows)], dtype=torch.int64)
        sizes = torch.zeros(world, dtype=torch.int64)
        comm.allgather(n_rec, sizes.view(world, 1), None)
        cap = int(sizes.max())
        pad = torch.zeros((cap, 2), dtype=torch.float64)
        pad[:len(rows)] = rec
        allrec = torch.zeros((world, cap, 2), dtype=torch.float64)
        comm.allgather(pad, allrec, None)
        recs = [[(int(m), float(y)) for m, y in allrec[g, :int(sizes[g])].tolist()]
                for g in range(world)]
        s, c = _fold(s0, c0, recs)
        final = s + c
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


@pytest.mark.parametrize("name", ["k3_basic", "k5_nondyadic_p0"])
def test_mode_a_shard_replays_and_canonical_state(name):
    """Mode A: each shard decides from P0; the tick end is the fold of every
    shard's dispatches in rank order -- the Neumaier state of the reference's
    monitor after the concatenated dispatches (same as Mode B's)."""
    sc = H.load_schedule(name)
    gathered, final = _run("A", name)
    n = len(sc["prog"])
    bounds = np.linspace(0, n, 3).astype(int)
    s0, c0 = _p0_state(sc)
    want = []
    mon = hp.PortMonitor(sc["ids"])
    for j, (m, v) in enumerate(sc["p0"]):
        mon.record_dispatch(sc["ids"][int(m)], f"seed:{j}", float(v))
    for r in range(2):
        models, _, _ = _chain(sc, range(bounds[r], bounds[r + 1]), s0, c0)
        want += models
        for i, m in zip(range(bounds[r], bounds[r + 1]), models):
            mon.record_dispatch(sc["ids"][m], f"r{i}", float(sc["yhat"][i, m]))
    assert sum(gathered, []) == want
    from paper_2603_22206_b200.state import neumaier_value
    k = sc["k"]
    p = np.array([neumaier_value(a, b) for a, b in zip(final[:k], final[k:])])
    assert p.tobytes() == np.array([mon.in_flight_sum(m) for m in sc["ids"]]).tobytes()


def test_shard_of_is_stable_and_balanced():
    from paper_2603_22206_b200.dist import shard_of
    ranks = [shard_of(f"p{i:06d}", 8) for i in range(8000)]
    assert ranks == [shard_of(f"p{i:06d}", 8) for i in range(8000)]
    counts = np.bincount(ranks, minlength=8)
    assert counts.min() > 850 and counts.max() < 1150


# ---------------------------------------------------------------------------
# Sharded engine queues with global admission (dist.sharded_iteration and the
# counter relay of ShardedScheduler(global_admission=True)) over gloo. The
# per-rank device kernels are replaced by a CPU sub-queue with the same
# contract (chm_queue_candidates / chm_queue_admit_merged, include/
# chimera_b200.h); the golden EngineSim scripts fix the expected result.

class _SubQueueShard:
    """CPU stand-in for one rank's GpuScheduler queue side (K = 1)."""

    def __init__(self, b, S):
        import types
        self.b, self.S = b, S
        self.entries = []  # dicts: level, prio, arr, seq, handle, count
        z = lambda dt: torch.zeros(1, dtype=dt)  # noqa: E731
        self.state = types.SimpleNamespace(
            K=1, device=torch.device("cpu"), inflight_sc=torch.zeros(2, dtype=torch.float64),
            engine_running=z(torch.int32),
            engine_seq=z(torch.int64), engine_clock=z(torch.float64),
            engine_iterations=z(torch.int64), q_n_admitted=z(torch.int32),
            q_n_promoted=z(torch.int32))
        self.admitted = []

    def _key(self, e):
        return (e["level"], e["prio"], e["arr"], e["seq"])

    def _age(self):
        for e in self.entries:
            e["count"] += 1
            if e["count"] >= self.S:
                e["level"] -= 1
                e["count"] = 0

    def run_rows(self, rows, n_iterations=0, keep_admitted=False):
        st = self.state
        for handle, prio, arr in rows:
            seq = int(st.engine_seq[0])
            st.engine_seq[0] += 1
            self.entries.append(dict(level=0, prio=prio, arr=arr, seq=seq, handle=handle, count=0))
            if int(st.engine_running[0]) < self.b:  # EngineSim.enqueue -> _iterate
                st.engine_iterations[0] += 1
                self.entries.sort(key=self._key)
                self.admitted.append(self.entries.pop(0)["handle"])
                st.engine_running[0] += 1
                self._age()

    def queue_candidates(self, stream=None):
        head = sorted(self.entries, key=self._key)[:self.b]
        out = torch.full((1, self.b, 5), 0, dtype=torch.int64)
        out[0, :, 0] = torch.iinfo(torch.int64).max
        for j, e in enumerate(head):
            out[0, j, 0] = e["level"]
            out[0, j, 1] = int(np.array([e["prio"]]).view(np.int64)[0])
            out[0, j, 2] = int(np.array([e["arr"]]).view(np.int64)[0])
            out[0, j, 3] = e["seq"]
            out[0, j, 4] = e["handle"]
        return out

    def queue_admit_merged(self, gathered, rank, release=None, stream=None):
        st = self.state
        rel = 0 if release is None else int(release[0])
        if rel < 0:
            return
        run = max(int(st.engine_running[0]) - rel, 0)
        cands = []
        for g in range(gathered.shape[0]):
            for c in gathered[g, 0].tolist():
                if c[0] == torch.iinfo(torch.int64).max:
                    continue
                pr = float(np.array([c[1]], dtype=np.int64).view(np.float64)[0])
                ar = float(np.array([c[2]], dtype=np.int64).view(np.float64)[0])
                cands.append(((c[0], pr, ar, c[3]), g, c[4]))
        cands.sort()
        take = cands[:max(0, min(self.b - run, len(cands)))]
        mine = {h for _, g, h in take if g == rank}
        self.entries.sort(key=self._key)
        for e in list(self.entries):
            if e["handle"] in mine:
                self.entries.remove(e)
        self.admitted.append([h for _, _, h in take])
        st.engine_running[0] = run + len(take)
        st.engine_iterations[0] += 1
        self._age()


def _queue_worker(rank, world, port, name, q):
    import math
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2603_22206_b200 import dist as D
    qd = H.load_queue(name)
    shard = _SubQueueShard(qd["b"], qd["S"] if qd["S"] else math.inf)
    comm = D.TorchComm()
    ss = D.ShardedScheduler.__new__(D.ShardedScheduler)
    ss.gs, ss.mode, ss.group, ss.global_admission, ss.comm = shard, "B", None, True, comm
    ss.packed = torch.empty((2 + len(D._RELAYED)) * 1, dtype=torch.float64)
    enq, pos = qd["enq"], 0
    log = []  # per step: handles admitted on enqueue (this rank) / per iteration (global)

    def enqueue(n):
        nonlocal pos
        o = enq[pos:pos + n]
        pos += n
        bounds = np.linspace(0, n, world + 1).astype(int)
        part = [(int(h), float(p), float(t)) for h, p, t in o[bounds[rank]:bounds[rank + 1]]]
        shard.admitted = []
        ss._pack()
        comm.relay_recv(ss.packed, None)
        ss._unpack()
        shard.run_rows(part)
        ss._pack()
        comm.relay_send(ss.packed, None)
        ss._unpack()
        got = [None] * world
        dist.all_gather_object(got, shard.admitted)
        log.extend(sum(got, []))

    def iteration(release=None):
        shard.admitted = []
        D.sharded_iteration(shard, comm, None, None if release is None else torch.tensor([release]))
        log.extend(shard.admitted[0])

    enqueue(qd["n_pre"])
    for op, n in qd["script"]:
        if op == "enq":
            enqueue(n)
        else:
            for _ in range(n):
                iteration(None if op == "iter" else 1)
    rows = [(shard._key(e), e["handle"], e["count"]) for e in shard.entries]
    got = [None] * world
    dist.all_gather_object(got, rows)
    if rank == 0:
        allrows = sorted(sum(got, []))
        q.put(dict(admitted=log, order=[r[1] for r in allrows], level=[r[0][0] for r in allrows],
                   count=[r[2] for r in allrows], running=int(shard.state.engine_running[0]),
                   iterations=int(shard.state.engine_iterations[0])))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name", ["q_basic", "q_promote", "q_complete"])
def test_sharded_queue_protocol_equals_single_queue(name):
    """Global admission over world_size 2 (gloo): relayed engine counters +
    all-gathered STJF candidates reproduce the golden single EngineSim."""
    qd = H.load_queue(name)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_queue_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(res["admitted"], qd["admitted"])
    np.testing.assert_array_equal(res["order"], qd["order"])
    np.testing.assert_array_equal(res["level"], qd["level"])
    np.testing.assert_array_equal(res["count"], qd["count"])
    assert res["running"] == qd["running"]
    assert res["iterations"] == qd["iterations"]
