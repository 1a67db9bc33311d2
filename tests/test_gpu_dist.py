"""ShardedScheduler.run_rows with the real kernels: two ranks (gloo, both on
cuda:0 -- the box has one GPU, and NCCL refuses two ranks per device) drive
GpuScheduler shards through dist.TorchComm, which runs the same packing /
folding kernels as the NCCL path (chm_inflight_pack / _fold / _local_sum /
_set_sum).

Checked against the oracle port:
  Mode B  each rank's decisions, priorities and estimated loads equal one
          serial schedule_request replay of the concatenated batch (rank 0's
          rows, then rank 1's); the tick-end in-flight sums are that replay's,
          bit for bit, on both ranks;
  Mode A  each rank's decisions equal an independent serial replay of its
          shard from the tick-start state; the tick-end sums equal the
          monitor after all dispatches in rank order (same state as Mode B);
  A vs B  the number of decisions Mode A changes (reported);
  completions  a second tick after each rank completes some of its own
          requests: the global in-flight sums equal the port's bit for bit
          (dyadic: exact int64 all-reduce; non-dyadic: the ranks' survivor
          lists merged in insertion order).
The expected values are computed inside the workers from the golden
scenarios (tests/golden/schedule_*.npz)."""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _port_replay(sc, rows_by_rank, mode, mon0_fn, pool):
    """Expected (model, priority, loads) per row and the tick-end monitor."""
    from oracle import hetsched_port as hp
    ids = sc["ids"]
    out = {}
    final = mon0_fn()
    engines = {m: hp.PortEngine(pool[m].max_batch_size) for m in ids}

    def run(rows, mon):
        for i in rows:
            r = _Req(sc, i)
            d = hp.port_schedule_request(
                r, _Rec(sc, i), pool, mon, engines,
                lambda rq, rc, i=i: {m: float(sc["q"][i, k]) for k, m in enumerate(ids)},
                lambda rq, rc, m, i=i: float(sc["yhat"][i, ids.index(m)]),
                sc["tau"], sc["margin"])
            out[i] = (ids.index(d.model), d.priority,
                      [d.estimated_loads[m] for m in ids] if d.estimated_loads else None)

    if mode == "B":
        for rows in rows_by_rank:
            run(rows, final)
    else:
        for rows in rows_by_rank:
            run(rows, mon0_fn())
        for rows in rows_by_rank:  # the canonical tick end: all dispatches in rank order
            for i in rows:
                m, y, _ = out[i]
                prior = final.assignment(f"p{int(sc['prog'][i]):06d}")
                if prior is None:
                    final.assign(f"p{int(sc['prog'][i]):06d}", ids[m])
                final.record_dispatch(ids[m], _Req(sc, i).request_id, y)
    return out, final


class _Req:
    def __init__(self, sc, i):
        self.program_id = f"p{int(sc['prog'][i]):06d}"
        self.stage_index = int(sc["stage"][i])
        self.arrival_time = 0.0  # one timestamp: rank order never moves a clock back
        self.request_id = f"{self.program_id}:{self.stage_index}"


class _Rec:
    def __init__(self, sc, i):
        self.sc, self.i = sc, i

    def out_tokens(self, stage, m):
        return int(self.sc["out_tok"][self.i, self.sc["ids"].index(m)])


def _worker(rank, port, name, q):
    import datetime
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD,
                            timeout=datetime.timedelta(seconds=90))
    torch.cuda.set_device(0)
    try:
        q.put((rank, _run_rank(rank, name)))
    except Exception as exc:  # noqa: BLE001 - reported to the parent
        import traceback
        q.put((rank, {"error": f"{exc!r}\n{traceback.format_exc()}"}))
        os._exit(0)  # the peer fails its next collective on the closed connection
    dist.barrier()
    dist.destroy_process_group()


def _run_rank(rank, name):
    from oracle import hetsched_port as hp
    from paper_2603_22206_b200 import dist as D
    from paper_2603_22206_b200.config import AgingConfig, BalancerConfig
    from paper_2603_22206_b200.predictor import PrecomputedPredictor
    from paper_2603_22206_b200.router import ScoreTableRouter
    from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch
    from paper_2603_22206_b200.state import request_key
    from tests import harness as H

    sc = H.load_schedule(name)
    ids, k = sc["ids"], sc["k"]
    pool = H.pool_of(sc)
    n = len(sc["prog"])
    # all stages of a program on one rank; rows keep their order within a rank
    rows_by_rank = [[i for i in range(n) if int(sc["prog"][i]) % WORLD == g]
                    for g in range(WORLD)]
    mine = rows_by_rank[rank]
    comm = D.TorchComm()
    report = {}

    def mon0():
        mon = hp.PortMonitor(ids)
        for j, (m, v) in enumerate(sc["p0"]):
            mon.record_dispatch(ids[int(m)], f"seed:{j}", float(v))
        for p, m in sc["pre"]:
            mon.assign(f"p{int(p):06d}", ids[int(m)])
        return mon

    def make():
        rt, pr = ScoreTableRouter(), PrecomputedPredictor()
        gs = GpuScheduler(pool, BalancerConfig(sc["tau"], sc["margin"]), AgingConfig(),
                          router=rt, predictor=pr, n_programs=sc["n_prog"],
                          max_rows=n, queue_capacity=10240)  # same on every rank
        per_model = {m: [] for m in ids}
        for m, v in sc["p0"]:
            per_model[ids[int(m)]].append(float(v))
        if rank == 0:  # the seeded entries live in rank 0's log ...
            gs.state.seed_inflight(per_model)
        else:          # ... while every rank starts from the global (s, c)
            from paper_2603_22206_b200.state import neumaier_state
            sc0 = [neumaier_state(per_model[m]) for m in ids]
            gs.state.inflight_sc.copy_(torch.tensor([a for a, _ in sc0] + [b for _, b in sc0],
                                                    dtype=torch.float64))
        if len(sc["pre"]):
            gs.state.preassign(sc["pre"][:, 0], sc["pre"][:, 1])
        rt.set(torch.as_tensor(sc["q"][mine], device="cuda"))
        pr.set(torch.as_tensor(sc["yhat"][mine], device="cuda"))
        batch = RowBatch.from_numpy("cuda", program=sc["prog"][mine], stage=sc["stage"][mine],
                                    arrival=np.zeros(len(mine)),
                                    out_tokens=sc["out_tok"][mine], handle=np.array(mine))
        return gs, batch

    models = {}
    for mode in ("A", "B"):
        gs, batch = make()
        ss = D.ShardedScheduler(gs, mode, comm=comm)
        stream = torch.cuda.current_stream()
        ss.run_rows(batch, n_iterations=0, stream=stream)
        torch.cuda.synchronize()
        gs.check_errors(f"mode {mode}")
        nr = len(mine)
        got_m = gs.buf.model[:nr].cpu().numpy()
        got_p = gs.buf.priority[:nr].cpu().numpy()
        got_l = gs.buf.loads[:nr * k].view(nr, k).cpu().numpy()
        fl = gs.buf.dflags[:nr].cpu().numpy()
        want, final = _port_replay(sc, rows_by_rank, mode, mon0, pool)
        for j, i in enumerate(mine):
            m, y, loads = want[i]
            assert got_m[j] == m, (mode, i, got_m[j], m)
            assert got_p[j] == y, (mode, i)
            if not fl[j] & 1:
                assert got_l[j].tolist() == loads, (mode, i)
        want_p = np.array([final.in_flight_sum(m) for m in ids])
        assert np.array(gs.state.in_flight_sums()).tobytes() == want_p.tobytes(), mode
        models[mode] = torch.as_tensor(got_m.astype(np.int64))
        report[f"mode_{mode}_rows"] = nr

        if mode == "B":
            # tick 2: every rank completes its own even rows, then re-sends
            # the odd programs' next stage
            done = [j for j in range(nr) if j % 2 == 0]
            c_model = torch.tensor(got_m[done].astype(np.int32), device="cuda")
            c_key = torch.tensor([request_key(int(sc["prog"][mine[j]]), int(sc["stage"][mine[j]]))
                                  for j in done], dtype=torch.int64, device="cuda")
            dyadic = np.all(np.asarray(sc["yhat"]) * 256 == np.floor(np.asarray(sc["yhat"]) * 256))
            dyadic = dyadic and all(float(v) * 256 == int(float(v) * 256) for _, v in sc["p0"])
            ss.run_rows(RowBatch.from_numpy("cuda", program=np.zeros(0), stage=np.zeros(0),
                                            arrival=np.zeros(0), out_tokens=np.zeros((0, k)),
                                            handle=np.zeros(0)),
                        n_iterations=0, completions=(c_model, c_key), stream=stream)
            torch.cuda.synchronize()
            gs.check_errors("completions")
            for g in range(WORLD):
                rows_g = rows_by_rank[g]
                for jj, i in enumerate(rows_g):
                    if jj % 2 == 0:
                        final.record_completion(ids[want[i][0]], _Req(sc, i).request_id)
            want_p = np.array([final.in_flight_sum(m) for m in ids])
            assert np.array(gs.state.in_flight_sums()).tobytes() == want_p.tobytes()
            report["completions"] = ("exact (dyadic all-reduce)" if dyadic
                                     else "exact (stamp-ordered merge)")
    report["a_vs_b_divergence"] = D.divergence(models["A"], models["B"], comm, None)
    return report


@pytest.mark.parametrize("name", ["k5_dyadic_p0", "k5_nondyadic_p0", "k8_mixed"])
def test_sharded_run_rows_vs_oracle(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, name, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = {}
    import queue as _queue
    for _ in range(WORLD):
        try:
            r, v = q.get(timeout=300)
        except _queue.Empty:
            break
        res[r] = v
        if "error" in v:
            break
    for p in procs:
        p.join(timeout=120)
        if p.exitcode is None:
            p.kill()
    for r, v in res.items():
        assert "error" not in v, f"rank {r}: {v['error']}"
    assert len(res) == WORLD, f"results from ranks {sorted(res)} only"
    print(json.dumps({"scenario": name, **res[0]}))
    assert all(p.exitcode == 0 for p in procs)
