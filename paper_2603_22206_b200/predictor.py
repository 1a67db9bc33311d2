"""Remaining-workflow-output predictors on the device (K5).

Each class keeps the reference's `predict(req, rec, model_id) -> float`
(hetsched/predictor.py:22-27) for single calls and adds
`predict_rows(batch, K, yhat_out, error, stream)`, which fills yhat[B, K]
for every model column in one kernel.

  GpuQuantilePredictor    EmpiricalQuantilePredictor (predictor.py:65-108)
  GpuOraclePredictor      OraclePredictor (predictor.py:30-36)
  GpuInputLengthPredictor InputLengthPredictor (predictor.py:39-45)

The quantile "training" (np.quantile over a training trace, predictor.py:95-98)
runs once on the host and is resolved -- fallback chain included -- into a
dense fp64 table [n_wf + 1, s_cap + 1, K] that stays resident on the device.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import EmptyTrainingSet, ValidationError


def _p(t):
    return None if t is None else t.data_ptr()


class GpuQuantilePredictor:
    name = "quantile"

    def __init__(self, training, model_ids, quantile: float = 0.5, device="cuda",
                 extra_workflows=()):
        if not 0.0 < quantile < 1.0:
            raise ValidationError(f"quantile must be in (0,1), got {quantile}")
        self.quantile = quantile
        self.model_ids = list(model_ids)
        by_key, by_sm, by_m, every = {}, {}, {}, []
        max_stage = 1
        for rec in training:
            for st in rec.stages:
                max_stage = max(max_stage, st.stage_index)
                for mid in sorted(st.models):
                    y = float(rec.remaining_tokens(st.stage_index, mid))
                    by_key.setdefault((rec.workflow_id, st.stage_index, mid), []).append(y)
                    by_sm.setdefault((st.stage_index, mid), []).append(y)
                    by_m.setdefault(mid, []).append(y)
                    every.append(y)
        if not every:
            raise EmptyTrainingSet("no training values at any fallback level")
        q = quantile
        self._by_key = {k: float(np.quantile(v, q)) for k, v in by_key.items()}
        self._by_sm = {k: float(np.quantile(v, q)) for k, v in by_sm.items()}
        self._by_m = {k: float(np.quantile(v, q)) for k, v in by_m.items()}
        self._global = float(np.quantile(every, q))
        wfs = sorted({k[0] for k in by_key} | set(extra_workflows))
        self.workflow_index = {w: i for i, w in enumerate(wfs)}
        self.s_cap = max_stage
        K = len(self.model_ids)
        table = np.empty((len(wfs) + 1, self.s_cap + 1, K), dtype=np.float64)
        for a, wf in enumerate(wfs + [None]):
            for st in range(self.s_cap + 1):
                for m, mid in enumerate(self.model_ids):
                    table[a, st, m] = self.lookup(wf, st if st else -1, mid)
        self.table_host = table
        self.table = torch.as_tensor(table.ravel(), device=device)
        self.n_wf = len(wfs)

    @classmethod
    def from_trace(cls, store, quantile: float = 0.5, extra_workflows=()):
        """Train on the device from a TraceStore (chm_quantile_train): the same
        table as the host build from the same trace, bit for bit."""
        if not 0.0 < quantile < 1.0:
            raise ValidationError(f"quantile must be in (0,1), got {quantile}")
        cols = store.cols
        n_entries = int(cols.n_stages.sum()) * store.K
        if n_entries == 0:
            raise EmptyTrainingSet("no training values at any fallback level")
        self = cls.__new__(cls)
        self.quantile = quantile
        self.model_ids = list(store.model_ids)
        wfs = sorted(set(cols.workflow_ids) | set(extra_workflows))
        self.workflow_index = {w: i for i, w in enumerate(wfs)}
        self.n_wf = len(wfs)
        self.s_cap = int(cols.n_stages.max())
        d = store.device
        wf = torch.as_tensor(np.array([self.workflow_index[w] for w in cols.workflow_ids],
                                      np.int32), device=d)
        lib = _lib.load()
        nbytes = int(lib.chm_quantile_train_scratch_bytes(n_entries, self.n_wf, self.s_cap,
                                                          store.K))
        scratch = torch.empty(nbytes, dtype=torch.uint8, device=d)
        self.table = torch.empty((self.n_wf + 1) * (self.s_cap + 1) * store.K,
                                 dtype=torch.float64, device=d)
        _lib.check(lib.chm_quantile_train(store.t, _p(wf), self.n_wf, self.s_cap, quantile,
                                          n_entries, _p(scratch), nbytes, _p(self.table),
                                          torch.cuda.current_stream(d).cuda_stream),
                   "chm_quantile_train")
        self.table_host = self.table.cpu().numpy().reshape(self.n_wf + 1, self.s_cap + 1, store.K)
        self._by_key = None  # lookups read the resolved table
        return self

    def lookup(self, workflow_id, stage_index, model_id) -> float:
        """The reference fallback chain (predictor.py:100-108)."""
        if self._by_key is None:  # device-trained: the table holds the resolved chain
            a = self.workflow_index.get(workflow_id, self.n_wf)
            st = stage_index if 1 <= stage_index <= self.s_cap else 0
            return float(self.table_host[a, st, self.model_ids.index(model_id)])
        v = self._by_key.get((workflow_id, stage_index, model_id))
        if v is None:
            v = self._by_sm.get((stage_index, model_id))
        if v is None:
            v = self._by_m.get(model_id)
        return self._global if v is None else v

    def predict(self, req, rec, model_id) -> float:
        return self.lookup(req.workflow_id, req.stage_index, model_id)

    def workflow_column(self, workflow_ids) -> np.ndarray:
        return np.array([self.workflow_index.get(w, self.n_wf) for w in workflow_ids],
                        dtype=np.int32)

    def columns_for(self, reqs, recs, model_ids):
        return {"workflow": self.workflow_column([r.workflow_id for r in reqs])}

    def predict_rows(self, batch, K, yhat, error, stream) -> None:
        _lib.check(_lib.load().chm_predict_quantile(
            _p(self.table), self.n_wf, self.s_cap, K, _p(batch.workflow), _p(batch.stage),
            batch.n_rows, _p(yhat), stream.cuda_stream), "chm_predict_quantile")


class GpuOraclePredictor:
    """With a TraceStore (trace.py) the prediction is gathered on the device
    from the derived suffix sums by (program, stage) alone; without one the
    batch carries per-row stage outputs (n_stages / stage_out columns)."""

    name = "oracle"

    def __init__(self, max_stages: int = 8, trace=None):
        self.max_stages = max_stages
        self.trace = trace

    def predict(self, req, rec, model_id) -> float:
        return float(rec.remaining_tokens(req.stage_index, model_id))

    def columns_for(self, reqs, recs, model_ids):
        B, K, S = len(reqs), len(model_ids), self.max_stages
        n_st = np.empty(B, np.int32)
        so = np.zeros((B, S, K), np.int32)
        for i, rec in enumerate(recs):
            n_st[i] = rec.n_stages
            if rec.n_stages > S:
                raise ValidationError(f"{rec.program_id}: more than {S} stages")
            for j, st in enumerate(rec.stages):
                so[i, j] = [st.models[m].out_tokens for m in model_ids]
        return {"n_stages": n_st, "stage_out": so}

    def predict_rows(self, batch, K, yhat, error, stream) -> None:
        if self.trace is not None:
            if K != self.trace.K:
                raise ValidationError(f"trace has {self.trace.K} models, pool has {K}")
            _lib.check(_lib.load().chm_trace_gather_rows(
                self.trace.t, _p(batch.program), _p(batch.stage), batch.n_rows, None, None, None,
                _p(yhat), _p(error), stream.cuda_stream), "chm_trace_gather_rows")
            return
        _lib.check(_lib.load().chm_predict_oracle(
            _p(batch.stage_out), _p(batch.n_stages), _p(batch.stage), self.max_stages, K,
            batch.n_rows, _p(yhat), _p(error), stream.cuda_stream), "chm_predict_oracle")


class GpuInputLengthPredictor:
    name = "input-length"

    def predict(self, req, rec, model_id) -> float:
        return float(req.input_tokens)

    def predict_rows(self, batch, K, yhat, error, stream) -> None:
        _lib.check(_lib.load().chm_predict_input_length(
            _p(batch.input_tokens), K, batch.n_rows, _p(yhat), stream.cuda_stream),
            "chm_predict_input_length")


class PrecomputedPredictor:
    """Predictions supplied per batch as a [B, K] tensor (parity harness)."""

    name = "precomputed"

    def __init__(self):
        self.values: torch.Tensor | None = None

    def set(self, values: torch.Tensor) -> None:
        self.values = values

    def predict_rows(self, batch, K, yhat, error, stream) -> None:
        n = batch.n_rows * K
        yhat[:n].copy_(self.values.reshape(-1)[:n], non_blocking=True)
