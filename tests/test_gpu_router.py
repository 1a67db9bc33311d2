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
                                          (EncoderConfig(n_layers=2), 2 / math.sqrt(768)),
                                          (EncoderConfig(n_layers=2, hidden=512, n_heads=8,
                                                         ffn=2048), 2 / math.sqrt(512)),
                                          (EncoderConfig(n_layers=2, hidden=1024, n_heads=16,
                                                         ffn=4096), 2 / math.sqrt(1024))])
def test_encoder_matches_fp32(cfg, head_std):
    K, B = 5, 24
    r = GpuEncoderRouter(cfg, K, max_rows=B, seed=3, head_std=head_std)
    ids = torch.as_tensor(synthetic_token_ids(B, cfg.seq_len, seed=11), device="cuda")
    q = torch.zeros(B * K, dtype=torch.float64, device="cuda")
    r.forward(ids, q)
    torch.cuda.synchronize()
    got = q.view(B, K).cpu().numpy()
    want = _ref_q(r, ids)
    err = np.abs(got - want).max()
    assert err <= Q_TOL, err
    assert np.all((got >= 0) & (got <= 1))


@pytest.mark.parametrize("S,B", [(128, 64), (256, 48), (384, 40), (512, 40)])
def test_encoder_cls_pool_bert_base(S, B):
    """Enough rows for the associative last layer (cls_pool.cu) at H = 768:
    U = Q_cls Wk_bd^T, xbar = pool(x, U), ctx = xbar Wv_bd^T + b_v."""
    from dataclasses import replace
    cfg = replace(EncoderConfig(n_layers=2), seq_len=S)
    K = 5
    r = GpuEncoderRouter(cfg, K, max_rows=B, seed=6, head_std=2 / math.sqrt(768))
    ids = torch.as_tensor(synthetic_token_ids(B, S, seed=17), device="cuda")
    q = torch.zeros(B * K, dtype=torch.float64, device="cuda")
    r.forward(ids, q)
    torch.cuda.synchronize()
    err = np.abs(q.view(B, K).cpu().numpy() - _ref_q(r, ids)).max()
    print(f"cls_pool S={S} B={B}: max|dq| = {err:.2e}")
    assert err <= Q_TOL, err


@pytest.mark.parametrize("S", [256, 512])
def test_encoder_long_prompts(S):
    """S > 128: flash-style key-block loop with online softmax (cfg5 S=512)."""
    from dataclasses import replace
    cfg = replace(SMALL, seq_len=S)
    K, B = 5, 6
    r = GpuEncoderRouter(cfg, K, max_rows=B, seed=8, head_std=2 / math.sqrt(256))
    ids = torch.as_tensor(synthetic_token_ids(B, S, seed=21), device="cuda")
    q = torch.zeros(B * K, dtype=torch.float64, device="cuda")
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
    q = torch.full((B * K,), -1.0, dtype=torch.float64, device="cuda")
    r.forward(ids, q, rows=rows, n_rows=n, n_seq=B)
    torch.cuda.synchronize()
    got = q.view(B, K).cpu().numpy()
    want = _ref_q(r, ids)
    for i in range(B):
        if i in (3, 7, 8, 15):
            assert np.abs(got[i] - want[i]).max() <= Q_TOL
        else:
            assert np.all(got[i] == -1.0)


def _partials(x):
    """(mean, M2) per 128-column chunk of every row, fp32 (deferred_ln.cuh)."""
    M, N = x.shape
    c = x.float().view(M, N // 128, 128)
    mean = c.mean(-1)
    m2 = ((c - mean[..., None]) ** 2).sum(-1)
    return torch.stack([mean, m2], -1).contiguous()


def _deferred(A, B, bias, epilogue, residual=None, gamma=None, beta=None, stats_in=None,
              colsum=None, eps=1e-12):
    M, K = A.shape
    N = B.shape[0]
    C = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    st_out = torch.full((M, N // 128, 2), float("nan"), device="cuda")
    n_part = 0 if stats_in is None else stats_in.shape[1]
    ptr = lambda t: None if t is None else t.data_ptr()  # noqa: E731
    _lib.check(_lib.load().chm_gemm_bf16_deferred_ln(
        A.data_ptr(), B.data_ptr(), C.data_ptr(), bias.data_ptr(), epilogue, ptr(residual),
        ptr(gamma), ptr(beta), ptr(stats_in), n_part, ptr(colsum), st_out.data_ptr(), eps,
        M, N, K, torch.cuda.current_stream().cuda_stream), "deferred_ln")
    torch.cuda.synchronize()
    return C, st_out


@pytest.mark.parametrize("M,N,K", [(256, 768, 768), (1000, 768, 3072), (777, 256, 128),
                                   (2048, 1024, 256)])
@pytest.mark.parametrize("with_ln", [False, True])
def test_gemm_resln_stats(M, N, K, with_ln):
    """Epilogue 6: C = A.B^T + bias + LN(residual) (statistics of the residual
    from its own partials) and the (mean, M2) partials of C per 128 columns."""
    g = torch.Generator(device="cuda").manual_seed(M + 3 * N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    bias = 0.1 * torch.randn(N, device="cuda", generator=g)
    res = (2 * torch.randn(M, N, device="cuda", generator=g) + 0.7).to(torch.bfloat16)
    gamma = 1 + 0.2 * torch.randn(N, device="cuda", generator=g)
    beta = 0.1 * torch.randn(N, device="cuda", generator=g)
    if with_ln:
        st = _partials(res)
        C, st_out = _deferred(A, B, bias, 6, res, gamma, beta, st)
        r = F.layer_norm(res.float(), (N,), gamma, beta, 1e-12)
    else:
        C, st_out = _deferred(A, B, bias, 6, res)
        r = res.float()
    ref = A.float() @ B.float().T + bias + r
    torch.testing.assert_close(C.float(), ref, rtol=GEMM_RTOL, atol=GEMM_ATOL)
    want = _partials(ref)
    torch.testing.assert_close(st_out[..., 0], want[..., 0], rtol=1e-3, atol=2e-3)
    torch.testing.assert_close(st_out[..., 1], want[..., 1], rtol=1e-2, atol=1e-1)


@pytest.mark.parametrize("M,N,K", [(256, 3072, 768), (1000, 2304, 768), (300, 512, 256)])
@pytest.mark.parametrize("epilogue", [1, 2])
def test_gemm_folded_layernorm(M, N, K, epilogue):
    """Epilogues 1/2 with stats_in: the LayerNorm of A's rows folded into the
    epilogue with chm_encoder_fold_weights' rule equals GEMM(LN(A))."""
    g = torch.Generator(device="cuda").manual_seed(M + N + 5 * K + epilogue)
    A = (torch.randn(M, K, device="cuda", generator=g) * 1.5 + 0.3).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    b = 0.1 * torch.randn(N, device="cuda", generator=g)
    gamma = 1 + 0.2 * torch.randn(K, device="cuda", generator=g)
    beta = 0.1 * torch.randn(K, device="cuda", generator=g)
    Wf = (W.float() * gamma).to(torch.bfloat16)
    colsum = Wf.float().sum(1)
    bf = b + W.float() @ beta
    C, _ = _deferred(A, Wf, bf, epilogue, stats_in=_partials(A), colsum=colsum)
    ref = F.layer_norm(A.float(), (K,), gamma, beta, 1e-12) @ W.float().T + b
    if epilogue == 2:
        ref = F.gelu(ref, approximate="tanh")
    torch.testing.assert_close(C.float(), ref, rtol=GEMM_RTOL, atol=3e-2)


@pytest.mark.parametrize("cfg,S,flags", [(SMALL, 128, 0), (SMALL, 128, _lib.ENC_DEFERRED_LN),
                                         (EncoderConfig(n_layers=3), 128, 0),
                                         (EncoderConfig(n_layers=3), 128, _lib.ENC_CLUSTER_LN),
                                         (SMALL, 256, _lib.ENC_DEFERRED_LN)])
def test_encoder_random_layernorm_params(cfg, S, flags):
    """Non-trivial LayerNorm gamma/beta (BERT init has 1/0): exercises the
    folded weights and the residual-side LayerNorm of the deferred path, and
    the cluster-LayerNorm path, on both hidden sizes."""
    from dataclasses import replace
    cfg = replace(cfg, seq_len=S)
    K, B = 5, 8
    r = GpuEncoderRouter(cfg, K, max_rows=B, seed=6, head_std=2 / math.sqrt(cfg.hidden))
    r.cfg_c.flags |= flags
    gen = torch.Generator(device="cuda").manual_seed(17)
    for name, t in r.weights.items():
        if name.startswith(("ln1_", "ln2_", "emb_ln_")):
            if "_g" in name:
                t.copy_(1 + 0.3 * torch.randn(t.shape, device="cuda", generator=gen))
            else:
                t.copy_(0.2 * torch.randn(t.shape, device="cuda", generator=gen))
    r.refold()
    ids = torch.as_tensor(synthetic_token_ids(B, S, seed=31), device="cuda")
    q = torch.zeros(B * K, dtype=torch.float64, device="cuda")
    r.forward(ids, q)
    torch.cuda.synchronize()
    err = np.abs(q.view(B, K).cpu().numpy() - _ref_q(r, ids)).max()
    assert err <= Q_TOL, err


@pytest.mark.parametrize("M,Fd", [(256, 1024), (1000, 1024), (131072, 1024), (777, 512),
                                  (300, 128), (5000, 2048)])
def test_ffn_fused_matches_two_gemms(M, Fd):
    """Fused H = 256 FFN sublayer (ffn_fused.cu) vs fp32 and vs the unfused
    FFN1 (bias + GELU) + FFN2 (bias + residual + LayerNorm) GEMMs on the same
    bf16 operands."""
    H = 256
    g = torch.Generator(device="cuda").manual_seed(M + Fd)
    x = (torch.randn(M, H, device="cuda", generator=g) + 0.3).to(torch.bfloat16)
    w1 = (torch.randn(Fd, H, device="cuda", generator=g) / math.sqrt(H)).to(torch.bfloat16)
    w2 = (torch.randn(H, Fd, device="cuda", generator=g) / math.sqrt(Fd)).to(torch.bfloat16)
    b1 = 0.1 * torch.randn(Fd, device="cuda", generator=g)
    b2 = 0.1 * torch.randn(H, device="cuda", generator=g)
    gamma = 1 + 0.1 * torch.randn(H, device="cuda", generator=g)
    beta = 0.1 * torch.randn(H, device="cuda", generator=g)
    st = torch.cuda.current_stream().cuda_stream
    h = F.gelu(x.float() @ w1.float().T + b1, approximate="tanh").to(torch.bfloat16)
    ref = F.layer_norm(h.float() @ w2.float().T + b2 + x.float(), (H,), gamma, beta, 1e-12)
    # unfused path
    hu = gemm(x, w1, b1, None, 2)
    yu = torch.empty_like(x)
    _lib.check(_lib.load().chm_gemm_bf16_ln(
        hu.data_ptr(), w2.data_ptr(), yu.data_ptr(), b2.data_ptr(), x.data_ptr(),
        gamma.data_ptr(), beta.data_ptr(), 1e-12, M, H, Fd, st), "gemm_ln")
    # fused, in place
    y = x.clone()
    _lib.check(_lib.load().chm_ffn_fused_bf16(
        y.data_ptr(), w1.data_ptr(), b1.data_ptr(), w2.data_ptr(), b2.data_ptr(),
        gamma.data_ptr(), beta.data_ptr(), 1e-12, M, H, Fd, st), "ffn_fused")
    torch.cuda.synchronize()
    torch.testing.assert_close(y.float(), ref, rtol=GEMM_RTOL, atol=GEMM_ATOL)
    assert (y.float() - yu.float()).abs().max().item() <= 2e-2


def test_ffn_fused_rejects_shapes():
    lib = _lib.load()
    assert lib.chm_ffn_fused_bf16(1, 1, 1, 1, 1, 1, 1, 1e-12, 10, 768, 1024, None) == \
        _lib.CHM_ERR_UNSUPPORTED
    assert lib.chm_ffn_fused_bf16(1, 1, 1, 1, 1, 1, 1, 1e-12, 10, 256, 1000, None) == \
        _lib.CHM_ERR_UNSUPPORTED
