"""Semantic router encoder on the device: config, weights, workspace, router.

BERT-style post-LN encoder (embedding + LN, L x [QKV -> attention -> out-proj
+ residual -> LN -> FFN(GELU) + residual -> LN]) and the paper's router head:
q[m] = sigmoid(Linear(h_[CLS]))[m]. Weights are bf16 in
nn.Linear layout [out, in]; LN/bias/head parameters fp32. The forward runs
entirely in libchimera_sm100a.so (chm_encoder_forward): tcgen05 GEMMs with
fused epilogues, tcgen05 attention, LayerNorms deferred into the consuming
GEMM's epilogue (weights folded once by chm_encoder_fold_weights).

FLOPs per routed request (S tokens):
  L * (8*S*H^2 + 4*S^2*H + 4*S*H*F) + 2*H*K
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


@dataclass(frozen=True)
class EncoderConfig:
    n_layers: int = 12
    hidden: int = 768
    n_heads: int = 12
    ffn: int = 3072
    vocab: int = 30522
    max_pos: int = 512
    seq_len: int = 128
    ln_eps: float = 1e-12

    def flops_per_request(self, n_models: int) -> int:
        """Nominal encoder FLOPs: every layer over all S tokens."""
        L, S, H, F = self.n_layers, self.seq_len, self.hidden, self.ffn
        return L * (8 * S * H * H + 4 * S * S * H + 4 * S * H * F) + 2 * H * n_models

    def flops_executed_per_request(self, n_models: int, cls_pool: bool = True) -> int:
        """Algorithmic FLOPs of what the device executes: the last layer serves
        the [CLS] query only (the head reads h_[CLS] alone). With the
        associative form (csrc/cls_pool.cu, the default) it projects Q_cls,
        forms u_h = W_k,h^T q_h (2 H^2), pools x twice (logits and
        xbar_h = sum_j p_hj x_j: 4 S H per head) and applies W_v,h (2 H^2);
        without it all S tokens feed the K|V projection (4 S H^2) and the CLS
        attention (4 S H). Out-projection / FFN run on the CLS row only."""
        L, S, H, F = self.n_layers, self.seq_len, self.hidden, self.ffn
        full = (L - 1) * (8 * S * H * H + 4 * S * S * H + 4 * S * H * F)
        if cls_pool:
            attn = 2 * H * H + 2 * H * H + 4 * S * H * self.n_heads + 2 * H * H
        else:
            attn = 4 * S * H * H + 2 * H * H + 4 * S * H
        last = attn + 2 * H * H + 4 * H * F
        return full + last + 2 * H * n_models


BERT_BASE = EncoderConfig()
SMALL = EncoderConfig(n_layers=4, hidden=256, n_heads=4, ffn=1024)


def init_weights(cfg: EncoderConfig, n_models: int, seed: int = 0, head_std: float = 0.02,
                 device="cuda") -> dict:
    """BERT initialisation: N(0, 0.02) matrices and embeddings, zero biases,
    LN gamma=1 beta=0; the head uses `head_std` (also report a
    spread variant 2/sqrt(H))."""
    g = torch.Generator().manual_seed(seed)
    H, F, L = cfg.hidden, cfg.ffn, cfg.n_layers

    def n(*shape, std=0.02):
        return torch.randn(*shape, generator=g) * std

    w = {
        "word_emb": n(cfg.vocab, H), "pos_emb": n(cfg.max_pos, H), "type_emb": n(H),
        "emb_ln_g": torch.ones(H), "emb_ln_b": torch.zeros(H),
        "head_w": n(n_models, H, std=head_std), "head_b": torch.zeros(n_models),
    }
    for i in range(L):
        w[f"w_qkv.{i}"] = n(3 * H, H)
        w[f"b_qkv.{i}"] = torch.zeros(3 * H)
        w[f"w_o.{i}"] = n(H, H)
        w[f"b_o.{i}"] = torch.zeros(H)
        w[f"ln1_g.{i}"] = torch.ones(H)
        w[f"ln1_b.{i}"] = torch.zeros(H)
        w[f"w_1.{i}"] = n(F, H)
        w[f"b_1.{i}"] = torch.zeros(F)
        w[f"w_2.{i}"] = n(H, F)
        w[f"b_2.{i}"] = torch.zeros(H)
        w[f"ln2_g.{i}"] = torch.ones(H)
        w[f"ln2_b.{i}"] = torch.zeros(H)
    # matrices/embeddings live in bf16 on the device; keep the bf16-rounded
    # values as the canonical weights so the fp32 restatement sees the same ones
    out = {}
    for k, v in w.items():
        if k.startswith(("w_", "word_emb", "pos_emb", "type_emb")):
            out[k] = v.to(torch.bfloat16).to(device)
        else:
            out[k] = v.float().to(device)
    return out


def synthetic_token_ids(n: int, seq_len: int, seed: int, vocab: int = 30522) -> np.ndarray:
    """[CLS]=101 at position 0, then U[1000, vocab)."""
    rng = np.random.default_rng(seed)
    ids = rng.integers(1000, vocab, size=(n, seq_len), dtype=np.int32)
    ids[:, 0] = 101
    return ids


class _PtrArray:
    def __init__(self, tensors):
        self.tensors = tensors
        self.arr = (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])

    @property
    def ptr(self):
        return ctypes.cast(self.arr, ctypes.c_void_p).value


PAD_ID = 0  # BERT [PAD]


def pack_tokens(seqs, seq_len: int, pad_id: int = PAD_ID) -> np.ndarray:
    """Token id sequences -> int32 [B, seq_len]: truncated to seq_len, shorter
    ones padded with `pad_id`. The encoder has no attention mask, so pad
    positions are attended like any token -- in the fp32 restatement too."""
    out = np.full((len(seqs), seq_len), pad_id, np.int32)
    for i, s in enumerate(seqs):
        a = np.asarray(s, dtype=np.int64)[:seq_len]
        out[i, :len(a)] = a
    return out


class GpuEncoderRouter:
    """Router backed by the sm_100a encoder (`score_rows` is the hot path).

    Drop-in for hetsched's `Router` (router.py:34-45): `score(req, rec, pool)`
    returns a ConfidenceVector over `pool.model_ids`, and `columns_for(reqs,
    recs)` supplies the token-id column `GpuScheduler.schedule_batch` batches.
    The token ids come from `tokens(req, rec) -> sequence of int` (the caller's
    tokenizer or token store; e.g. a dict lookup by request or program id),
    packed to `cfg.seq_len` by `pack_tokens`. Head row m scores the m-th
    model of `pool.model_ids` (sorted ids, the device's model order)."""

    name = "encoder"

    def __init__(self, cfg: EncoderConfig, n_models: int, weights: dict | None = None,
                 max_rows: int = 4096, seed: int = 0, head_std: float = 0.02, device="cuda",
                 tokens=None):
        self.lib = _lib.load()
        self.cfg = cfg
        self.K = n_models
        self.tokens = tokens
        self.device = torch.device(device)
        self.weights = weights if weights is not None else init_weights(
            cfg, n_models, seed, head_std, self.device)
        w, L = self.weights, cfg.n_layers
        self._arrays = {name: _PtrArray([w[f"{name}.{i}"] for i in range(L)])
                        for name in ("w_qkv", "b_qkv", "w_o", "b_o", "ln1_g", "ln1_b", "w_1",
                                     "b_1", "w_2", "b_2", "ln2_g", "ln2_b")}
        A = self._arrays
        self.w_c = _lib.EncoderWeights(
            w["word_emb"].data_ptr(), w["pos_emb"].data_ptr(), w["type_emb"].data_ptr(),
            w["emb_ln_g"].data_ptr(), w["emb_ln_b"].data_ptr(),
            A["w_qkv"].ptr, A["b_qkv"].ptr, A["w_o"].ptr, A["b_o"].ptr, A["ln1_g"].ptr,
            A["ln1_b"].ptr, A["w_1"].ptr, A["b_1"].ptr, A["w_2"].ptr, A["b_2"].ptr,
            A["ln2_g"].ptr, A["ln2_b"].ptr, w["head_w"].data_ptr(), w["head_b"].data_ptr())
        self.cfg_c = _lib.EncoderCfg(cfg.n_layers, cfg.hidden, cfg.n_heads, cfg.ffn, cfg.vocab,
                                     cfg.max_pos, n_models, cfg.ln_eps, 0)
        self.max_rows = max_rows
        T = max_rows * cfg.seq_len
        bf = torch.bfloat16
        H, F = cfg.hidden, cfg.ffn
        self.ws = {
            "x": torch.empty(T, H, dtype=bf, device=self.device),
            "qkv": torch.empty(T, 3 * H, dtype=bf, device=self.device),
            "ctx": torch.empty(T, H, dtype=bf, device=self.device),
            "tmp": torch.empty(T, H, dtype=bf, device=self.device),
            "ffn": torch.empty(T, F, dtype=bf, device=self.device),
        }
        # deferred-LayerNorm statistics and the LayerNorm-folded QKV / FFN1
        # weights (chm_encoder_fold_weights; recomputed by refold())
        self.ws["stats"] = torch.empty(
            int(self.lib.chm_encoder_stats_bytes(self.cfg_c, T)), dtype=torch.uint8,
            device=self.device)
        self.ws["folded"] = torch.empty(
            int(self.lib.chm_encoder_folded_bytes(self.cfg_c)), dtype=torch.uint8,
            device=self.device)
        self.ws_c = _lib.EncoderWorkspace(T, *(self.ws[k].data_ptr()
                                               for k in ("x", "qkv", "ctx", "tmp", "ffn",
                                                         "stats", "folded")))
        self.refold()

    def refold(self, stream=None) -> None:
        """Recompute the LayerNorm-folded weights after a weight change."""
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(self.lib.chm_encoder_fold_weights(self.cfg_c, self.w_c, self.ws_c,
                                                     s.cuda_stream), "chm_encoder_fold_weights")

    def forward(self, token_ids: torch.Tensor, q_out: torch.Tensor, rows=None, n_rows=None,
                n_seq: int | None = None, stream=None) -> None:
        """q_out[row*K + m] for the listed rows (all rows when `rows` is None)."""
        n_seq = token_ids.shape[0] if n_seq is None else n_seq
        if q_out.dtype != torch.float64:
            raise TypeError("q_out must be float64 (the scheduler's score buffer is fp64)")
        if n_seq > self.max_rows:
            raise ValueError(f"{n_seq} sequences exceed max_rows={self.max_rows}")
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _lib.check(self.lib.chm_encoder_forward(
            self.cfg_c, self.w_c, self.ws_c, token_ids.data_ptr(),
            None if rows is None else rows.data_ptr(),
            None if n_rows is None else n_rows.data_ptr(), n_seq, token_ids.shape[1],
            q_out.data_ptr(), s.cuda_stream), "chm_encoder_forward")

    # scheduler router protocol
    def score_rows(self, batch, route_rows, n_route, scores, stream) -> None:
        if batch.token_ids is None:
            raise ValueError("GpuEncoderRouter needs batch.token_ids")
        self.forward(batch.token_ids, scores, rows=route_rows, n_rows=n_route,
                     n_seq=batch.n_rows, stream=stream)

    def _token_ids(self, reqs, recs) -> np.ndarray:
        if self.tokens is None:
            raise ValueError("GpuEncoderRouter needs a token source: GpuEncoderRouter(..., "
                             "tokens=lambda req, rec: ids)")
        return pack_tokens([self.tokens(r, rc) for r, rc in zip(reqs, recs)], self.cfg.seq_len)

    def columns_for(self, reqs, recs) -> dict:
        """The router's batch column (GpuScheduler.rows_from_requests)."""
        return {"token_ids": self._token_ids(reqs, recs)}

    def score(self, req, rec, pool) -> "ConfidenceVector":
        """Router.score (router.py:39-42) for one request: one sequence through
        the same device encoder, fp64 scores keyed by pool.model_ids."""
        from .router import ConfidenceVector
        if len(pool.model_ids) != self.K:
            raise ValueError(f"router has {self.K} heads, pool has {len(pool.model_ids)} models")
        ids = torch.as_tensor(self._token_ids([req], [rec]), device=self.device)
        q = torch.empty(self.K, dtype=torch.float64, device=self.device)
        self.forward(ids, q)
        return ConfidenceVector(dict(zip(pool.model_ids, q.cpu().tolist())))
