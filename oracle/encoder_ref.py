"""torch fp32 restatement of the router encoder -- TEST INFRASTRUCTURE ONLY.

The reference has no neural router (router.py:34-45 pins only the contract:
one score in [0,1] per pool model). This is the checker for the device
encoder (paper_2603_22206_b200/encoder.py): the same weights (bf16 values
promoted to fp32), the same token ids, all arithmetic in fp32:

  x = LN(word_emb[id] + pos_emb[pos] + type_emb)
  per layer: x = LN(x + Attn(x) W_o^T + b_o);  x = LN(x + GELU(x W_1^T + b_1) W_2^T + b_2)
  (GELU in its tanh form, the router model's activation)
  q = sigmoid(x[CLS] head_w^T + head_b)

It runs on any device (CPU for the bench's cpu_baseline leg, which times it
with all host threads).
"""

from __future__ import annotations

import math

import torch
import torch.nn.functional as F


def encoder_forward_fp32(weights: dict, token_ids: torch.Tensor, n_layers: int, n_heads: int,
                         eps: float = 1e-12, device=None) -> torch.Tensor:
    dev = device or token_ids.device
    w = {k: v.to(device=dev, dtype=torch.float32) for k, v in weights.items()}
    ids = token_ids.to(dev).long()
    B, S = ids.shape
    H = w["word_emb"].shape[1]
    d = H // n_heads
    x = w["word_emb"][ids] + w["pos_emb"][:S][None] + w["type_emb"][None, None]
    x = F.layer_norm(x, (H,), w["emb_ln_g"], w["emb_ln_b"], eps)
    for i in range(n_layers):
        qkv = x @ w[f"w_qkv.{i}"].T + w[f"b_qkv.{i}"]
        q, k, v = qkv.split(H, dim=-1)
        q = q.view(B, S, n_heads, d).transpose(1, 2)
        k = k.view(B, S, n_heads, d).transpose(1, 2)
        v = v.view(B, S, n_heads, d).transpose(1, 2)
        att = torch.softmax((q @ k.transpose(-1, -2)) / math.sqrt(d), dim=-1)
        ctx = (att @ v).transpose(1, 2).reshape(B, S, H)
        x = F.layer_norm(x + ctx @ w[f"w_o.{i}"].T + w[f"b_o.{i}"], (H,), w[f"ln1_g.{i}"],
                         w[f"ln1_b.{i}"], eps)
        h = F.gelu(x @ w[f"w_1.{i}"].T + w[f"b_1.{i}"], approximate="tanh")
        x = F.layer_norm(x + h @ w[f"w_2.{i}"].T + w[f"b_2.{i}"], (H,), w[f"ln2_g.{i}"],
                         w[f"ln2_b.{i}"], eps)
    return torch.sigmoid(x[:, 0] @ w["head_w"].T + w["head_b"])
