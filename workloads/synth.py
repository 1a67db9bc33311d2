"""Synthetic workloads for BASELINE.json's configs, seeded.

Pool: model m_i has decode_ms_per_token = 5*(i+1), max_batch_size =
max(1, 32 >> i), prefill 0.02 (extends configs/pool_two_model.json, as
SPEC.md:134 allows). Length and success statistics interpolate linearly
between the paper's small and large model (APPS 447/1276 -> 649/534,
MATH 606/2587 -> 709/715; configs/synth_*.json). The predictor is
EmpiricalQuantilePredictor(q=0.5) trained on synthesize_trace(2000, seed=1),
which keeps predictions dyadic. A tick's batch is the first-stage requests of
B distinct programs from synthesize_trace(B, seed=100+tick), all arriving at
the same time; token ids are [CLS] + U[1000, 30522) (seed 1234+tick); router
weights are BERT-initialised from torch.manual_seed(0).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from paper_2603_22206_b200.config import AgingConfig, BalancerConfig, ModelProfile, Pool
from paper_2603_22206_b200.encoder import (BERT_BASE, SMALL, EncoderConfig, GpuEncoderRouter,
                                           synthetic_token_ids)
from paper_2603_22206_b200.predictor import GpuQuantilePredictor
from paper_2603_22206_b200.scheduler import RowBatch
from . import tracegen as W

APPS = ((447.0, 1276.0), (649.0, 534.0))
MATH = ((606.0, 2587.0), (709.0, 715.0))
CODE_SUCCESS = ({"easy": 0.45, "hard": 0.08}, {"easy": 0.85, "hard": 0.55})
MATH_SUCCESS = ({"easy": 0.55, "hard": 0.12}, {"easy": 0.9, "hard": 0.6})
CODE_3STAGE = W.workflow("code-3stage", "planner", "coder", "qa_agent")


@dataclass
class WorkloadSpec:
    name: str
    n_models: int
    batch: int
    encoder: EncoderConfig
    templates: tuple
    stats: tuple
    success: tuple
    description: str
    n_pre_queued: int = 0      # cfg4: entries pre-queued over the engines
    n_pre_inflight: int = 0    # cfg4: pre-existing in-flight entries
    bursts: int = 1


SPECS = {
    "cfg1": WorkloadSpec("cfg1", 3, 1000, SMALL, (CODE_3STAGE,), APPS, CODE_SUCCESS,
                         "reference CPU scheduler: 3-stage code-gen workflow, 3-model "
                         "heterogeneous cluster, 1k requests, small router"),
    "cfg2": WorkloadSpec("cfg2", 3, 4096, BERT_BASE, W.MATH_WORKFLOWS, MATH, MATH_SUCCESS,
                         "math-reasoning workflow, 3-model cluster, batch 4096 scheduling "
                         "tick on 1 B200"),
    "cfg3": WorkloadSpec("cfg3", 5, 4096, BERT_BASE, W.MATH_WORKFLOWS + W.CODE_WORKFLOWS,
                         MATH, MATH_SUCCESS,
                         "5-model heterogeneous cluster, BERT-base-size router, batch 4096"),
    "cfg4": WorkloadSpec("cfg4", 8, 4096, SMALL, W.MATH_WORKFLOWS, MATH, MATH_SUCCESS,
                         "bursty arrival trace, 64k in-flight requests, 8 engines, "
                         "STJF+aging sort stress", n_pre_queued=65536, n_pre_inflight=65536,
                         bursts=16),
    # cfg5 is quoted for 8 GPUs (16k requests/tick); per GPU that is 2048
    "cfg5": WorkloadSpec("cfg5", 5, 2048, EncoderConfig(seq_len=512), W.MATH_WORKFLOWS,
                         MATH, MATH_SUCCESS,
                         "long-prompt router inputs (seq 512), 2048 requests/tick per GPU "
                         "(16k over 8 B200), NCCL in-flight all-reduce"),
    "smoke": WorkloadSpec("smoke", 3, 64, SMALL, W.MATH_WORKFLOWS, MATH, MATH_SUCCESS,
                          "smoke: 64 requests, 3 models, small router"),
}


def make_pool(k: int) -> Pool:
    return Pool(tuple(ModelProfile(f"m{i}", 5.0 * (i + 1), max(1, 32 >> i), 0.02)
                      for i in range(k)))


def interp_stats(k: int, pair) -> dict:
    (m0, s0), (m1, s1) = pair
    out = {}
    for i in range(k):
        t = i / (k - 1) if k > 1 else 1.0
        out[f"m{i}"] = W.LengthStats(m0 + t * (m1 - m0), s0 + t * (s1 - s0))
    return out


def interp_success(k: int, pair) -> dict:
    lo, hi = pair
    out = {}
    for i in range(k):
        t = i / (k - 1) if k > 1 else 1.0
        out[f"m{i}"] = {d: lo[d] + t * (hi[d] - lo[d]) for d in lo}
    return out


@dataclass
class Workload:
    spec: WorkloadSpec
    pool: Pool
    balancer: BalancerConfig
    aging: AgingConfig
    router: GpuEncoderRouter | None
    predictor: GpuQuantilePredictor
    training: list
    device: torch.device
    n_programs: int
    host_batches: list = field(default_factory=list)
    dev_batches: list = field(default_factory=list)

    @property
    def batch_size(self) -> int:
        return self.spec.batch

    def host_columns(self, tick: int) -> dict:
        """Columnar numpy inputs of tick `tick` (what a caller hands the API)."""
        sp = self.spec
        k = len(self.pool)
        stats = interp_stats(k, sp.stats)
        succ = interp_success(k, sp.success)
        recs = W.synthesize_trace(sp.templates, stats, succ, sp.batch, 100 + tick)
        ids = self.pool.model_ids
        B = sp.batch
        out_tok = np.empty((B, k), np.int32)
        for i, rec in enumerate(recs):
            out_tok[i] = [rec.out_tokens(1, m) for m in ids]
        arrival = np.full(B, 1000.0 * (tick + 1))
        if sp.bursts > 1:  # bursts of B/bursts requests, each at one timestamp
            arrival = 1000.0 * (tick + 1) + np.repeat(np.arange(sp.bursts),
                                                      B // sp.bursts).astype(np.float64)
        return dict(
            program=(np.arange(B) + (tick % 4) * B).astype(np.int32),
            stage=np.ones(B, np.int32),
            arrival=arrival,
            out_tokens=out_tok,
            handle=(np.arange(B) + tick * B).astype(np.int64),
            workflow=self.predictor.workflow_column([r.workflow_id for r in recs]),
            input_tokens=np.array([r.stages[0].base_input_tokens for r in recs], np.int32),
            token_ids=synthetic_token_ids(B, sp.encoder.seq_len, 1234 + tick, sp.encoder.vocab),
            records=recs,
        )

    def batch(self, tick: int) -> RowBatch:
        cols = dict(self.host_columns(tick))
        cols.pop("records")
        return RowBatch.from_numpy(self.device, **cols)

    @property
    def queue_capacity(self) -> int:
        sp = self.spec
        if not sp.n_pre_queued:
            return 10240
        per = sp.n_pre_queued // sp.n_models
        return 1 << int(np.ceil(np.log2(per + sp.batch)))

    def seed_state(self, state, seed: int = 7) -> None:
        """cfg4: pre-existing in-flight predictions and pre-queued entries
        (integer lognormal predictions from the MATH stats), engines running
        full, so each tick exercises completions, admission and aging at scale."""
        sp = self.spec
        if not (sp.n_pre_queued or sp.n_pre_inflight):
            return
        rng = np.random.default_rng(seed)
        K = sp.n_models
        ids = self.pool.model_ids
        mu, sigma = np.log(650.0) - 0.5, 1.0
        if sp.n_pre_inflight:
            owner = rng.integers(0, K, sp.n_pre_inflight)
            vals = np.maximum(1, np.round(rng.lognormal(mu, sigma, sp.n_pre_inflight)))
            state.seed_inflight({ids[m]: vals[owner == m].tolist() for m in range(K)})
        per = sp.n_pre_queued // K
        for m in range(K):
            prio = np.maximum(1, np.round(rng.lognormal(mu, sigma, per)))
            arr = np.sort(rng.random(per) * 900.0)
            state.load_queue(m, prio, arr, np.arange(per), np.arange(per) + (m << 40),
                             out_tokens=rng.integers(1, 2000, per),
                             count=rng.integers(0, int(self.aging.starvation_threshold), per))
        state.set_engine_counters(
            running=[self.pool[i].max_batch_size for i in ids],
            seq=[per] * K, clock=[900.0] * K)

    def completions(self):
        """cfg4: every engine's running batch turns over once per tick: the
        b_m oldest in-flight requests of engine m finish (record_completion
        through chm_monitor_complete, then their slots free up). Returns
        (model int32[n], key int64[n]) device tensors; the pre-seeded
        entries of engine m have keys -1, -2, ... in insertion order."""
        if not self.spec.n_pre_queued:
            return None
        models, keys = [], []
        for k, mid in enumerate(self.pool.model_ids):
            b = self.pool[mid].max_batch_size
            models += [k] * b
            keys += list(range(-1, -b - 1, -1))
        return (torch.tensor(models, dtype=torch.int32, device=self.device),
                torch.tensor(keys, dtype=torch.int64, device=self.device))


def make_workload(name: str, device="cuda", with_router: bool = True) -> Workload:
    sp = SPECS[name]
    pool = make_pool(sp.n_models)
    stats = interp_stats(sp.n_models, sp.stats)
    succ = interp_success(sp.n_models, sp.success)
    training = W.synthesize_trace(sp.templates, stats, succ, 2000, 1)
    dev = torch.device(device)
    pred = GpuQuantilePredictor(training, pool.model_ids, 0.5, device=dev,
                                extra_workflows=[t.workflow_id for t in sp.templates])
    router = None
    if with_router:
        router = GpuEncoderRouter(sp.encoder, sp.n_models, max_rows=sp.batch, seed=0,
                                  device=dev)
    return Workload(sp, pool, BalancerConfig(0.5, 0.1), AgingConfig(8, 4), router, pred,
                    training, dev, n_programs=4 * sp.batch)
