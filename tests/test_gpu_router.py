"""GPU numerics for the router: the tcgen05 GEMM against a torch fp32 matmul of
the same bf16 operands, and the full encoder against the fp32 restatement in
oracle/encoder_ref.py (north-star tolerance |dq| <= 1e-2)."""

import math

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from paper_2603_22206_b200 import _lib
from paper_2603_22206_b200.encoder import (SMALL, EncoderConfig, GpuEncoderRouter,
                                           synthetic_token_ids)

pytestmark = pytest.mark.gpu

# bf16 output of an fp32-accumulated GEMM: |err| <= 2^-8 relative + accumulation noise
GEMM_RTOL = 1e-2
GEMM_ATOL = 2e-2
Q_TOL = 1e-2


def gemm(A, B, bias=None, residual=None, epilogue=0):
    M, K = A.shape
    N = B.shape[0]
    C = torch.empty(M, N, dtype=torch.bfloat16, device=A.device)
    _lib.check(_lib.load().chm_gemm_bf16(
        A.data_ptr(), B.data_ptr(), C.data_ptr(), None if bias is None else bias.data_ptr(),
        None if residual is None else residual.data_ptr(), M, N, K, epilogue,
        torch.cuda.current_stream().cuda_stream), "gemm")
    return C


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 128), (1000, 768, 768),
                                   (4096, 2304, 768), (2048, 768, 3072), (300, 128, 192), (33000, 768, 768)])
@pytest.mark.parametrize("epilogue", [0, 1, 2, 3])
def test_gemm(M, N, K, epilogue):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K + epilogue)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda", generator=g)
    res = torch.randn(M, N, device="cuda", generator=g).to(torch.bfloat16)
    C = gemm(A, B, bias, res, epilogue)
    torch.cuda.synchronize()
    ref = A.float() @ B.float().T
    if epilogue >= 1:
        ref = ref + bias
    if epilogue == 2:
        ref = F.gelu(ref, approximate="tanh")
    if epilogue == 3:
        ref = ref + res.float()
    torch.testing.assert_close(C.float(), ref, rtol=GEMM_RTOL, atol=GEMM_ATOL)


@pytest.mark.parametrize("M,N,K", [(256, 256, 64), (1000, 768, 768), (4096, 768, 3072),
                                   (777, 512, 128), (2048, 1024, 256)])
@pytest.mark.parametrize("in_place", [False, True])
def test_gemm_residual_layernorm(M, N, K, in_place):
    """C = LN(A.B^T + bias + residual): fp32 statistics over the full row,
    rows spread over a 2N/256-CTA cluster (DSMEM exchange)."""
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    bias = 0.1 * torch.randn(N, device="cuda", generator=g)
    res = (torch.randn(M, N, device="cuda", generator=g) + 0.5).to(torch.bfloat16)
    gamma = 1 + 0.1 * torch.randn(N, device="cuda", generator=g)
    beta = 0.1 * torch.randn(N, device="cuda", generator=g)
    ref = F.layer_norm(A.float() @ B.float().T + bias + res.float(), (N,), gamma, beta, 1e-12)
    C = res if in_place else torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    _lib.check(_lib.load().chm_gemm_bf16_ln(
        A.data_ptr(), B.data_ptr(), C.data_ptr(), bias.data_ptr(), res.data_ptr(),
        gamma.data_ptr(), beta.data_ptr(), 1e-12, M, N, K,
        torch.cuda.current_stream().cuda_stream), "gemm_ln")
    torch.cuda.synchronize()
    torch.testing.assert_close(C.float(), ref, rtol=GEMM_RTOL, atol=GEMM_ATOL)


def _ref_q(router, ids):
    from oracle.encoder_ref import encoder_forward_fp32
    return encoder_forward_fp32(router.weights, ids, router.cfg.n_layers, router.cfg.n_heads,
                                router.cfg.ln_eps).cpu().numpy()


@pytest.mark.parametrize("cfg,head_std", [(SMALL, 0.02), (SMALL, 2 / math.sqrt(256)),
                                          (EncoderConfig(n_layers=2), 2 / math.sqrt(768))])
def test_encoder_matches_fp32(cfg, head_std):
    K, B = 5, 24
    r = GpuEncoderRouter(cfg, K, max_rows=B, seed=3, head_std=head_std)
    ids = torch.as_tensor(synthetic_token_ids(B, cfg.seq_len, seed=11), device="cuda")
    q = torch.zeros(B * K, dtype=torch.float32, device="cuda")
    r.forward(ids, q)
    torch.cuda.synchronize()
    got = q.view(B, K).cpu().numpy()
    want = _ref_q(r, ids)
    err = np.abs(got - want).max()
    assert err <= Q_TOL, err
    assert np.all((got >= 0) & (got <= 1))


@pytest.mark.parametrize("S", [256, 512])
def test_encoder_long_prompts(S):
    """S > 128: flash-style key-block loop with online softmax (cfg5 S=512)."""
    from dataclasses import replace
    cfg = replace(SMALL, seq_len=S)
    K, B = 5, 6
    r = GpuEncoderRouter(cfg, K, max_rows=B, seed=8, head_std=2 / math.sqrt(256))
    ids = torch.as_tensor(synthetic_token_ids(B, S, seed=21), device="cuda")
    q = torch.zeros(B * K, dtype=torch.float32, device="cuda")
    r.forward(ids, q)
    torch.cuda.synchronize()
    err = np.abs(q.view(B, K).cpu().numpy() - _ref_q(r, ids)).max()
    assert err <= Q_TOL, err


def test_encoder_routed_rows_only():
    """Only rows listed in route_rows[:n_route] are written (balancer.py:104-114)."""
    K, B = 3, 16
    r = GpuEncoderRouter(SMALL, K, max_rows=B, seed=4, head_std=0.2)
    ids = torch.as_tensor(synthetic_token_ids(B, 128, seed=5), device="cuda")
    rows = torch.tensor([3, 7, 8, 15, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0], dtype=torch.int32,
                        device="cuda")
    n = torch.tensor([4], dtype=torch.int32, device="cuda")
    q = torch.full((B * K,), -1.0, device="cuda")
    r.forward(ids, q, rows=rows, n_rows=n, n_seq=B)
    torch.cuda.synchronize()
    got = q.view(B, K).cpu().numpy()
    want = _ref_q(r, ids)
    for i in range(B):
        if i in (3, 7, 8, 15):
            assert np.abs(got[i] - want[i]).max() <= Q_TOL
        else:
            assert np.all(got[i] == -1.0)
