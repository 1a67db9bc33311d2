"""GPU numerics for the encoder attention kernels against a torch fp32
reference of the same op (softmax(Q K^T) V per (sequence, head), no mask):

  chm_attention_bf16      S = 128 (4 CTA/SM kernel), S = 256/512 (persistent
                          ping-pong flash kernel), S = 384 (key-block loop)
  chm_qkv_attention_bf16  fused QKV projection + attention (S = 128)

Sizes are chosen so persistent CTAs process several items (Q double-buffer
and K/V ring wrap-around are exercised), plus single-item grids."""

import math

import numpy as np
import pytest
import torch

from paper_2603_22206_b200 import _lib
from paper_2603_22206_b200.encoder import SMALL, GpuEncoderRouter, synthetic_token_ids
from oracle.encoder_ref import encoder_forward_fp32  # test infrastructure

pytestmark = pytest.mark.gpu

# bf16 P and bf16 output: |err| well below 2e-2 for O(1) values; the mean
# error bounds systematic mistakes (a wrong tile would be O(1) off)
ATOL = 2e-2
MEAN_TOL = 2e-3


def _stream():
    return torch.cuda.current_stream().cuda_stream


def ref_attention(qkv: torch.Tensor, n_seq: int, S: int, H: int) -> torch.Tensor:
    NH = H // 64
    x = qkv.float().view(n_seq, S, 3, NH, 64)
    q = x[:, :, 0].permute(0, 2, 1, 3)
    k = x[:, :, 1].permute(0, 2, 1, 3)
    v = x[:, :, 2].permute(0, 2, 1, 3)
    p = torch.softmax(q @ k.transpose(-1, -2), dim=-1)
    return (p @ v).permute(0, 2, 1, 3).reshape(n_seq * S, H)


def _check(got, want):
    err = (got.float() - want).abs()
    assert err.max().item() <= ATOL, err.max().item()
    assert err.mean().item() <= MEAN_TOL, err.mean().item()


@pytest.mark.parametrize("S,n_seq,H", [(128, 3, 256), (128, 200, 768), (256, 2, 256),
                                       (256, 40, 768), (384, 5, 256), (512, 1, 256),
                                       (512, 64, 768)])
def test_attention_matches_fp32(S, n_seq, H):
    g = torch.Generator(device="cuda").manual_seed(S + n_seq + H)
    qkv = torch.randn(n_seq * S, 3 * H, device="cuda", generator=g)
    qkv[:, :H] *= 0.125 * 2.0  # pre-scaled Q with a peaky softmax
    qkv = qkv.to(torch.bfloat16)
    ctx = torch.full((n_seq * S, H), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.load().chm_attention_bf16(qkv.data_ptr(), ctx.data_ptr(), n_seq, S, H,
                                              _stream()), "attention")
    torch.cuda.synchronize()
    _check(ctx, ref_attention(qkv, n_seq, S, H))


def test_attention_rejects_bad_shapes():
    lib = _lib.load()
    assert lib.chm_attention_bf16(1, 1, 1, 100, 256, None) == _lib.CHM_ERR_UNSUPPORTED
    assert lib.chm_attention_bf16(1, 1, 1, 640, 256, None) == _lib.CHM_ERR_UNSUPPORTED
    assert lib.chm_attention_bf16(1, 1, 1, 128, 100, None) == _lib.CHM_ERR_INVALID_ARG


@pytest.mark.parametrize("n_seq,H", [(1, 256), (7, 768), (100, 256), (64, 768), (300, 768)])
def test_qkv_attention_matches_fp32(n_seq, H):
    """Fused kernel vs fp32: qkv = x W^T + b (Q x 1/8), rounded to bf16 as the
    unfused path stores it, then fp32 attention."""
    S = 128
    g = torch.Generator(device="cuda").manual_seed(n_seq * 31 + H)
    x = torch.randn(n_seq * S, H, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(3 * H, H, device="cuda", generator=g) / math.sqrt(H)).to(torch.bfloat16)
    b = torch.randn(3 * H, device="cuda", generator=g) * 0.5
    ctx = torch.full((n_seq * S, H), float("nan"), dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.load().chm_qkv_attention_bf16(x.data_ptr(), w.data_ptr(), b.data_ptr(),
                                                  ctx.data_ptr(), n_seq, H, _stream()),
               "qkv_attention")
    torch.cuda.synchronize()
    qkv = x.float() @ w.float().T + b
    qkv[:, :H] *= 0.125
    want = ref_attention(qkv.to(torch.bfloat16), n_seq, S, H)
    _check(ctx, want)
    # and against the unfused kernels on the same bf16 QKV
    ctx2 = torch.empty_like(ctx)
    _lib.check(_lib.load().chm_attention_bf16(qkv.to(torch.bfloat16).data_ptr(), ctx2.data_ptr(),
                                              n_seq, S, H, _stream()), "attention")
    torch.cuda.synchronize()
    assert (ctx.float() - ctx2.float()).abs().max().item() <= ATOL


def test_encoder_fused_equals_unfused():
    """The router with the fused QKV+attention kernel and with the two-kernel
    path give the same confidences (both within 1e-2 of the fp32 restatement)."""
    K, B = 5, 48
    r = GpuEncoderRouter(SMALL, K, max_rows=B, seed=11, head_std=2 / math.sqrt(256))
    ids = torch.as_tensor(synthetic_token_ids(B, 128, seed=3), device="cuda")
    q_f = torch.zeros(B * K, dtype=torch.float64, device="cuda")
    r.forward(ids, q_f)
    r.cfg_c.flags = _lib.ENC_UNFUSED_ATTENTION
    q_u = torch.zeros(B * K, dtype=torch.float64, device="cuda")
    r.forward(ids, q_u)
    r.cfg_c.flags = 0
    torch.cuda.synchronize()
    ref = encoder_forward_fp32(r.weights, ids, SMALL.n_layers, SMALL.n_heads,
                               SMALL.ln_eps).cpu().numpy()
    qf = q_f.view(B, K).cpu().numpy()
    qu = q_u.view(B, K).cpu().numpy()
    assert np.abs(qf - qu).max() <= 5e-3
    assert np.abs(qf - ref).max() <= 1e-2
    assert np.abs(qu - ref).max() <= 1e-2
