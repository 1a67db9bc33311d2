"""Device trace store (csrc/trace.cu) against the reference's answers
(tests/golden/trace_small.*) and the numpy restatement (oracle/trace_ref.py),
bit-exact; large ragged traces through size-independent identities."""

import os

import numpy as np
import pytest
import torch

from oracle import trace_ref
from paper_2603_22206_b200 import errors
from paper_2603_22206_b200.trace import TraceColumns, TraceStore, load_ndjson

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def store():
    return TraceStore(load_ndjson(os.path.join(GOLD, "trace_small.ndjson")), "cuda")


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "trace_small.npz"))


def test_derive_matches_reference(store, gold):
    rem = store.remaining.cpu().numpy()
    want = gold["remaining"]
    live = want >= 0
    assert np.array_equal(rem[live], want[live])
    assert np.all(rem[~live] == 0)


def _all_completions(store):
    ns = store.cols.n_stages
    prog, comp, time, model = [], [], [], []
    for p in range(store.n_programs):
        for s in range(1, int(ns[p]) + 1):
            for k in range(store.K):
                prog.append(p), comp.append(s), time.append(1000.0 + p + 0.25 * s)
                model.append(k)
    return prog, comp, time, model


def test_next_stage_matches_reference(store, gold):
    prog, comp, time, model = _all_completions(store)
    d = "cuda"
    out = store.next_stage(torch.tensor(prog, dtype=torch.int32, device=d),
                           torch.tensor(comp, dtype=torch.int32, device=d),
                           torch.tensor(time, dtype=torch.float64, device=d),
                           torch.tensor(model, dtype=torch.int8, device=d))
    n = int(out["n"].item())
    want = trace_ref.ref_next_stage(store.cols.n_stages, store.cols.base_input, store.cols.carried,
                                    prog, comp, time, model)
    assert n == len(want)
    src = out["source_row"][:n].cpu().numpy()
    assert np.array_equal(src, [w[0] for w in want])  # completion order kept
    assert np.array_equal(out["program"][:n].cpu().numpy(), [w[1] for w in want])
    assert np.array_equal(out["stage"][:n].cpu().numpy(), [w[2] for w in want])
    assert np.array_equal(out["arrival"][:n].cpu().numpy(), [w[3] for w in want])
    got_in = out["input_tokens"][:n].cpu().numpy()
    assert np.array_equal(got_in, [w[4] for w in want])
    for j, i in enumerate(src):  # and the reference's own numbers
        assert got_in[j] == gold["next_input"][prog[i], comp[i] - 1, model[i]]


def test_first_stage_and_gather(store, gold):
    d = "cuda"
    NP = store.n_programs
    prog = torch.arange(NP, dtype=torch.int32, device=d)
    fs = store.first_stage(prog)
    assert np.array_equal(fs["input_tokens"].cpu().numpy(), gold["first_input"])
    assert np.array_equal(fs["arrival"].cpu().numpy(), gold["first_arrival"])
    # every (program, stage) row: out_tokens and the oracle prediction
    rows = [(p, s) for p in range(NP) for s in range(1, int(store.cols.n_stages[p]) + 1)]
    P = torch.tensor([r[0] for r in rows], dtype=torch.int32, device=d)
    S = torch.tensor([r[1] for r in rows], dtype=torch.int32, device=d)
    out_tok = torch.empty(len(rows), store.K, dtype=torch.int32, device=d)
    yhat = torch.empty(len(rows), store.K, dtype=torch.float64, device=d)
    nst = torch.empty(len(rows), dtype=torch.int32, device=d)
    store.gather_rows(P, S, out_tokens=out_tok, oracle=yhat, n_stages=nst)
    o, y = out_tok.cpu().numpy(), yhat.cpu().numpy()
    for i, (p, s) in enumerate(rows):
        assert np.array_equal(o[i], store.cols.out_tokens[p, s - 1])
        assert np.array_equal(y[i], gold["remaining"][p, s - 1].astype(np.float64))
    assert np.array_equal(nst.cpu().numpy(), [store.cols.n_stages[p] for p, _ in rows])


def test_unknown_stage_errors(store):
    d = "cuda"
    ns = int(store.cols.n_stages[3])
    P = torch.tensor([0, 3, 3], dtype=torch.int32, device=d)
    for bad in (0, ns + 1):
        S = torch.tensor([1, 1, bad], dtype=torch.int32, device=d)
        with pytest.raises(errors.UnknownStage):
            store.gather_rows(P, S, oracle=torch.empty(3, store.K, dtype=torch.float64,
                                                        device=d))
        with pytest.raises(errors.UnknownStage):
            store.next_stage(P, S, torch.zeros(3, dtype=torch.float64, device=d),
                             torch.zeros(3, dtype=torch.int8, device=d))


def _random_cols(NP, S, K, seed):
    rng = np.random.default_rng(seed)
    c = TraceColumns(NP, S, [f"m{k}" for k in range(K)])
    c.program_ids = [f"p{i}" for i in range(NP)]
    c.workflow_ids = ["wf"] * NP
    c.n_stages[:] = rng.integers(1, S + 1, NP)
    live = np.arange(S)[None, :] < c.n_stages[:, None]
    c.base_input[:] = np.where(live, rng.integers(1, 4000, (NP, S)), 0)
    c.out_tokens[:] = np.where(live[..., None], rng.integers(0, 20000, (NP, S, K)), 0)
    c.carried[:] = np.where(live[..., None], rng.integers(0, 20000, (NP, S, K)), 0)
    c.user_arrival[:] = rng.random(NP) * 1e6
    return c


@pytest.mark.parametrize("NP,S,K", [(1, 1, 1), (33, 4, 3), (100_003, 8, 5), (4096, 32, 8)])
def test_derive_random_vs_oracle(NP, S, K):
    c = _random_cols(NP, S, K, NP + S + K)
    st = TraceStore(c, "cuda")
    assert np.array_equal(st.remaining.cpu().numpy(), trace_ref.ref_remaining(c.n_stages,
                                                                              c.out_tokens))
    assert np.array_equal(st.carried_prefix.cpu().numpy(),
                          trace_ref.ref_carried_prefix(c.n_stages, c.carried))


def test_derive_large_identities():
    """4M programs (S=8, K=5: 1 GB of columns): remaining[:, 0] is each
    program's total output per model; remaining[s] - remaining[s+1] = out[s]."""
    NP, S, K = 4_000_000, 8, 5
    c = _random_cols(NP, S, K, 5)
    st = TraceStore(c, "cuda")
    out = st.out_tokens.long()
    total = out.sum(1)
    assert torch.equal(st.remaining[:, 0], total)
    diff = st.remaining[:, :-1] - st.remaining[:, 1:]
    live = (torch.arange(S - 1, device="cuda")[None, :] < st.n_stages[:, None] - 1)
    assert torch.equal(torch.where(live[..., None], diff, 0), torch.where(live[..., None],
                                                                          out[:, :-1], 0))


def test_derive_validation_errors():
    c = _random_cols(500, 4, 3, 9)
    c.out_tokens[321, 0, 1] = -1
    c.carried[457, 0, 2] = -5
    with pytest.raises(errors.ValidationError) as ei:
        TraceStore(c, "cuda")
    assert "row 321" in str(ei.value)  # the lowest offending program
    c = _random_cols(50, 4, 3, 10)
    c.n_stages[7] = 0
    with pytest.raises(errors.ValidationError):
        TraceStore(c, "cuda")


def test_two_tick_stage_chaining_vs_oracle_port(store):
    """Tick 1 schedules every program's first stage with the oracle predictor
    gathered from the store; next_stage turns the stage-1 completions into the
    tick-2 batch (cached branch, remaining tokens from stage 2). Both ticks
    against the oracle port of schedule_request fed the same scores."""
    from oracle import hetsched_port as hp
    from paper_2603_22206_b200.config import BalancerConfig, ModelProfile, Pool
    from paper_2603_22206_b200.predictor import GpuOraclePredictor
    from paper_2603_22206_b200.router import ScoreTableRouter
    from paper_2603_22206_b200.scheduler import GpuScheduler

    cols, ids, K, d = store.cols, store.model_ids, store.K, "cuda"
    pool = Pool(tuple(ModelProfile(m, 5.0 * (k + 1), max(1, 8 >> k)) for k, m in enumerate(ids)))
    rng = np.random.default_rng(3)
    NP = store.n_programs
    rt = ScoreTableRouter()
    gs = GpuScheduler(pool, BalancerConfig(0.5, 0.1), router=rt,
                      predictor=GpuOraclePredictor(trace=store), n_programs=NP, max_rows=NP)

    class _Rec:  # reference accessors over the columns
        def __init__(self, p):
            self.p = p

        def remaining_tokens(self, s, m):
            k = ids.index(m)
            return int(cols.out_tokens[self.p, s - 1:cols.n_stages[self.p], k].astype(np.int64).sum())

        def out_tokens(self, s, m):
            return int(cols.out_tokens[self.p, s - 1, ids.index(m)])

    class _Req:
        def __init__(self, p, s, t):
            self.program_id, self.stage_index, self.arrival_time = f"t{p}", s, t
            self.request_id = f"t{p}:{s}"
            self.workflow_id = "wf"

    mon = hp.PortMonitor(ids)
    engines = {m: hp.PortEngine(pool[m].max_batch_size) for m in ids}

    def run(program, stage, arrival):
        n = len(program)
        q = rng.random((n, K))  # fp64 scores (ConfidenceVector holds Python floats)
        rt.set(torch.as_tensor(q, device=d))
        P = torch.as_tensor(np.asarray(program, np.int32), device=d)
        batch = store.make_batch(P, torch.as_tensor(np.asarray(stage, np.int32), device=d),
                                 torch.as_tensor(np.asarray(arrival, np.float64), device=d))
        gs.run_rows(batch, n_iterations=0)
        torch.cuda.synchronize()
        gs.check_errors("trace tick")
        got_m = gs.buf.model[:n].cpu().numpy()
        got_p = gs.buf.priority[:n].cpu().numpy()
        for i in range(n):
            dec = hp.port_schedule_request(
                _Req(program[i], stage[i], arrival[i]), _Rec(program[i]), pool, mon, engines,
                lambda rq, rc, i=i: {m: float(q[i, k]) for k, m in enumerate(ids)},
                hp.port_oracle_predict, 0.5, 0.1)
            assert ids[got_m[i]] == dec.model, i
            assert got_p[i] == dec.priority, i
        return got_m

    prog = list(range(NP))
    m1 = run(prog, [1] * NP, [0.0] * NP)
    done = torch.arange(NP, dtype=torch.int32, device=d)
    nxt = store.next_stage(done, torch.ones(NP, dtype=torch.int32, device=d),
                           torch.full((NP,), 50.0, dtype=torch.float64, device=d),
                           torch.as_tensor(m1.astype(np.int8), device=d))
    n2 = int(nxt["n"].item())
    assert n2 == int(np.sum(cols.n_stages > 1))
    p2 = nxt["program"][:n2].cpu().tolist()
    run(p2, nxt["stage"][:n2].cpu().tolist(), nxt["arrival"][:n2].cpu().tolist())


@pytest.mark.parametrize("source", ["store", "columns"])
def test_predictor_error_stops_the_batch(store, source):
    """An UnknownStage raised by OraclePredictor.predict at row r (stage past
    the program's last) stops the batch there, as the reference's serial loop
    does: rows < r are scheduled, row r keeps only monitor.assign
    (balancer.py:113-115), later rows are untouched."""
    from oracle import hetsched_port as hp
    from paper_2603_22206_b200.config import BalancerConfig, ModelProfile, Pool
    from paper_2603_22206_b200.predictor import GpuOraclePredictor
    from paper_2603_22206_b200.router import ScoreTableRouter
    from paper_2603_22206_b200.scheduler import GpuScheduler, RowBatch

    cols, ids, K, d = store.cols, store.model_ids, store.K, "cuda"
    NP = store.n_programs
    n = min(NP, 40)
    r = 17
    pool = Pool(tuple(ModelProfile(m, 5.0 * (k + 1), max(1, 8 >> k)) for k, m in enumerate(ids)))
    rt = ScoreTableRouter()
    S = int(cols.n_stages.max())
    pred = GpuOraclePredictor(max_stages=S, trace=store if source == "store" else None)
    gs = GpuScheduler(pool, BalancerConfig(0.5, 0.1), router=rt, predictor=pred,
                      n_programs=NP, max_rows=n)
    prog = np.arange(n, dtype=np.int32)
    stage = np.ones(n, np.int32)
    stage[r] = int(cols.n_stages[r]) + 1  # UnknownStage at row r
    q = np.random.default_rng(5).random((n, K))
    rt.set(torch.as_tensor(q, device=d))
    extra = {}
    if source == "columns":
        extra = dict(n_stages=cols.n_stages[:n], stage_out=cols.out_tokens[:n, :S])
    batch = RowBatch.from_numpy(d, program=prog, stage=stage, arrival=np.zeros(n),
                                out_tokens=cols.out_tokens[prog, 0], handle=np.arange(n),
                                **extra)
    gs.run_rows(batch, n_iterations=0)
    torch.cuda.synchronize()
    with pytest.raises(errors.UnknownStage):
        gs.check_errors("predictor error")
    assert int(gs.buf.n_committed.item()) == r

    class _Rec:
        def __init__(self, p):
            self.p = p

        def remaining_tokens(self, s, m):
            if not 1 <= s <= cols.n_stages[self.p]:
                raise hp.PortError("UnknownStage", f"stage {s}")
            k = ids.index(m)
            return int(cols.out_tokens[self.p, s - 1:cols.n_stages[self.p], k].astype(np.int64).sum())

        def out_tokens(self, s, m):
            return int(cols.out_tokens[self.p, s - 1, ids.index(m)])

    class _Req:
        def __init__(self, p, s):
            self.program_id, self.stage_index, self.arrival_time = f"t{p}", s, 0.0
            self.request_id = f"t{p}:{s}"

    mon = hp.PortMonitor(ids)
    engines = {m: hp.PortEngine(pool[m].max_batch_size) for m in ids}
    got_m = gs.buf.model[:r].cpu().numpy()
    for i in range(n):
        try:
            dec = hp.port_schedule_request(
                _Req(prog[i], stage[i]), _Rec(prog[i]), pool, mon, engines,
                lambda rq, rc, i=i: {m: float(q[i, k]) for k, m in enumerate(ids)},
                hp.port_oracle_predict, 0.5, 0.1)
        except hp.PortError as exc:
            assert exc.kind == "UnknownStage" and i == r
            break
        assert ids[got_m[i]] == dec.model
    want_p = np.array([mon.in_flight_sum(m) for m in ids])
    assert np.array(gs.state.in_flight_sums()).tobytes() == want_p.tobytes()
    assign = gs.state.assignment[:n].cpu().numpy()
    for p in range(n):
        a = mon.assignment(f"t{p}")
        assert assign[p] == (-1 if a is None else ids.index(a)), p
    # decisions for the rows before the error ride on the exception
    with pytest.raises(errors.UnknownStage) as ei:
        gs.collect(batch)
    assert len(ei.value.decisions) == r
