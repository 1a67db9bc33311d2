"""Predictor evaluation on the device.

`kendall_tau_distance`, `evaluate_predictor` and `arrival_order_distance` keep
the signatures and results of hetsched's (predictor.py:182-251): same
LengthMismatch errors, the same fp64 result bit for bit. The counting runs in
libchimera_sm100a.so (csrc/evaluate.cu). `evaluate_predictor` and
`arrival_order_distance` take a device TraceStore (trace.py) instead of a
record list, and rank every (program, stage) request of the trace, as the
reference does.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import SimError


class LengthMismatch(SimError):
    """Paired sequences differ in length (or are too short to rank)."""


def _p(t):
    return None if t is None else t.data_ptr()


def kendall_tau_distance(predicted, truth, device="cuda", return_counts: bool = False):
    """Fraction of discordant pairs between two rankings (predictor.py:182-214)."""
    p = torch.as_tensor(predicted, dtype=torch.float64, device=device).reshape(-1)
    t = torch.as_tensor(truth, dtype=torch.float64, device=device).reshape(-1)
    if p.numel() != t.numel():
        raise LengthMismatch(f"predicted has {p.numel()} values, truth has {t.numel()}")
    n = int(p.numel())
    if n < 2:
        raise LengthMismatch("need at least 2 values to compare rankings")
    lib = _lib.load()
    nbytes = int(lib.chm_kendall_tau_scratch_bytes(n))
    scratch = torch.empty(nbytes, dtype=torch.uint8, device=p.device)
    res = torch.empty(1, dtype=torch.float64, device=p.device)
    counts = torch.empty(4, dtype=torch.int64, device=p.device)
    _lib.check(lib.chm_kendall_tau_distance(
        _p(p), _p(t), n, _p(scratch), nbytes, _p(res), _p(counts),
        torch.cuda.current_stream(p.device).cuda_stream), "chm_kendall_tau_distance")
    if return_counts:
        return float(res.item()), [int(x) for x in counts.cpu().tolist()]
    return float(res.item())


def _request_rows(store):
    """(program, stage) of every request of the trace, in the reference's
    order (for rec in test: for st in rec.stages)."""
    ns = store.cols.n_stages
    prog = np.repeat(np.arange(len(ns), dtype=np.int32), ns)
    first = np.cumsum(ns) - ns
    stage = (np.arange(int(ns.sum()), dtype=np.int32) - np.repeat(first, ns) + 1).astype(np.int32)
    d = store.device
    return torch.as_tensor(prog, device=d), torch.as_tensor(stage, device=d)


def _truth(store, P, S, k):
    o = torch.empty(P.numel(), store.K, dtype=torch.float64, device=store.device)
    store.gather_rows(P, S, oracle=o)
    return o[:, k].contiguous()


def evaluate_predictor(predictor, store, model_id: str) -> float:
    """Kendall tau distance of `predictor` vs the ground truth on one model
    (predictor.py:230-251): every (program, stage) request of the trace, with
    the predictor's device kernel (`predict_rows`) producing the predictions."""
    from .scheduler import RowBatch
    k = store.model_ids.index(model_id)
    P, S = _request_rows(store)
    n = P.numel()
    wf = torch.empty(n, dtype=torch.int32, device=store.device)
    store.gather_rows(P, S, workflow=wf)
    inputs = None
    if getattr(predictor, "name", "") == "input-length":
        # input_tokens = base + carried context of the earlier stages under model_id
        # (predictor.py:240-246)
        base = torch.as_tensor(store.cols.base_input, device=store.device)[P.long(), S.long() - 1]
        carried = store.carried_prefix[P.long(), S.long() - 1, k]
        inputs = (base.long() + carried).to(torch.int32)
    batch = RowBatch(program=P, stage=S, arrival=torch.zeros(n, dtype=torch.float64,
                                                               device=store.device),
                     out_tokens=torch.zeros(n, store.K, dtype=torch.int32, device=store.device),
                     handle=torch.arange(n, dtype=torch.int64, device=store.device),
                     workflow=wf, input_tokens=inputs)
    yhat = torch.empty(n * store.K, dtype=torch.float64, device=store.device)
    err = torch.tensor([0, 2**31 - 1, -1, 0], dtype=torch.int32, device=store.device)
    predictor.predict_rows(batch, store.K, yhat, err, torch.cuda.current_stream(store.device))
    e = err.cpu().tolist()
    if e[0] != _lib.CHM_OK:
        _lib.raise_device_error(e, "evaluate_predictor")
    pred = yhat.view(n, store.K)[:, k].contiguous()
    return kendall_tau_distance(pred, _truth(store, P, S, k), store.device)


def arrival_order_distance(store, model_id: str) -> float:
    """First-come ordering vs the truth (predictor.py:254-261)."""
    k = store.model_ids.index(model_id)
    P, S = _request_rows(store)
    truth = _truth(store, P, S, k)
    pred = torch.arange(P.numel(), dtype=torch.float64, device=store.device)
    return kendall_tau_distance(pred, truth, store.device)
