// K2+K3 fused on CTA PAIRS (tcgen05 cta_group::2): QKV projection + attention
// for S = 128, two sequences per pair, one head per item.
//
// Why pairs: the cta_group::1 kernel (qkv_attn.cu) streams 40 KB of operands
// per 384 tensor cycles into each SM's shared memory and reads as much back
// into the tensor core; that traffic caps its projection near 50 % of the
// tensor pipe (profiles/r1c_gemm_cycles.md). A pair MMA (M = 256: CTA x holds
// sequence x's 128 token rows) splits the head's 192 W rows 96 / 96 between
// the two SMs, so each SM moves 28 KB per 384 cycles.
//
// All tcgen05 ops of a kernel share one cta_group, so attention is pair MMAs
// too, with block-structured operands instead of per-sequence MMAs:
//   S = [Q_A; Q_B] [K_A; K_B]^T   (M 256, N 256, K 64): CTA x keeps columns
//       [128x, 128x + 128) -- its own keys; the cross block is never read.
//   O = P' V'                     (M 256, N 128, K 256): CTA 0's P' rows are
//       [P_A | 0], CTA 1's [0 | P_B]; B rows [0, 64) (CTA 0's half) hold V_A
//       for keys [0, 128) and zeros after, rows [64, 128) (CTA 1's half) zeros
//       then V_B. CTA x's O columns [64x, 64x + 64) = P_x V_x. The zero halves
//       are written once; the attention MMAs cost 2x (~18 % of the item).
// TMEM (512 columns per CTA): projection accumulator [0, 192) (single
// buffer), S [256, 512), O over S after the softmax read it.
//
// Roles per CTA (320 threads): warp 0 TMA producer (both CTAs, 3-stage ring,
// loads signal the leader's barrier), warp 1 MMA issuer (leader CTA), warps
// 2-9 epilogue (both CTAs, 2 threads per token row). Per item the leader
// issues the projection, and after the epilogues of both CTAs drained the
// accumulator (bf16 Q / K / V tiles in smem), S of that item, then the next
// item's projection k-blocks with O slotted in as soon as both CTAs' P is
// written.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <stdlib.h>
#include "common.cuh"
#include "deferred_ln.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace gemm {
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, uint64_t ld);
}
namespace qap {

constexpr int kS = 128;
constexpr int kStages = 3;
constexpr int kThreads = 320;
constexpr uint32_t kXTile = kS * 64 * 2;        // x [128][64] bf16, 16 KB
constexpr uint32_t kWHalf = 96 * 64 * 2;        // this CTA's 96 W rows, 12 KB
constexpr uint32_t kStageBytes = kXTile + kWHalf;
constexpr uint32_t kTile = kS * 64 * 2;         // 16 KB: Q, K, one P chunk, half V'
constexpr uint32_t kAccCols = 192;
constexpr uint32_t kSCol = 256;

struct __align__(1024) Smem {
  uint8_t stages[kStages][kStageBytes];
  uint8_t q[kTile];
  uint8_t k[kTile];
  uint8_t p[4][kTile];   // P' chunks (64 keys each): live 2x, 2x+1 in CTA x, zeros else
  uint8_t v[2][kTile];   // V' (MN-major, 128 keys x 64 dims): live [x] in CTA x, zero else
  float red_max[2][kS];
  float red_sum[2][kS];
  uint64_t full[kStages], empty[kStages], kdone[kStages];
  uint64_t acc_full, drained, s_full, p_ready, o_full;
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// Waits on barriers the partner CTA arrives on with release.cluster.
__device__ __forceinline__ void mbar_wait_acq(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITA_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITA_%=;\n\t}" ::"r"(sm100::smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ bool mbar_test_acq(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(sm100::smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__global__ void __launch_bounds__(kThreads, 1)
    qkv_attention_pair_kernel(const __grid_constant__ CUtensorMap tm_x,
                              const __grid_constant__ CUtensorMap tm_w,
                              const float* __restrict__ b_qkv, const float* __restrict__ c_qkv,
                              const float2* __restrict__ stats_in, int n_part, float eps,
                              int n_seq, int n_heads, int hidden,
                              __nv_bfloat16* __restrict__ ctx, int lag, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = sm100::align_smem_1024<Smem>(smem_raw);
  const int warp = sm100::warp_id(), lane = threadIdx.x & 31;
  const int k_blocks = hidden / 64;
  const uint32_t px = sm100::cluster_ctarank() & 1;
  const bool leader = px == 0;
  const int cl = (int)sm100::cluster_id_x(), n_cl = (int)sm100::n_clusters_x();
  const int n_items = ((n_seq + 1) / 2) * n_heads;
  const int per = (n_items + n_cl - 1) / n_cl;
  const int c_lo = cl * per;
  const int n_my = c_lo < n_items ? min(per, n_items - c_lo) : 0;
  auto item_of = [&](int it, int& seq, int& h) {
    const int c = c_lo + it;
    const int sp = c / n_heads;
    h = c - sp * n_heads;
    seq = 2 * sp + (int)px;
  };

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_x);
    sm100::tma_prefetch(&tm_w);
    for (int i = 0; i < kStages; ++i) {
      sm100::mbar_init(&s.full[i], 1);
      sm100::mbar_init(&s.empty[i], 1);
      sm100::mbar_init(&s.kdone[i], 1);
    }
    sm100::mbar_init(&s.acc_full, 1);
    sm100::mbar_init(&s.drained, 2 * 256);
    sm100::mbar_init(&s.s_full, 1);
    sm100::mbar_init(&s.p_ready, 2 * 256);
    sm100::mbar_init(&s.o_full, 1);
    sm100::fence_barrier_init();
  }
  // permanent zero halves of P' and V'
  {
    const int zc0 = px ? 0 : 2;  // P' chunks of the partner's keys
    uint4 z = make_uint4(0, 0, 0, 0);
    for (int i = threadIdx.x; i < 2 * (int)kTile / 16; i += kThreads) {
      const int c = zc0 + i / ((int)kTile / 16);
      reinterpret_cast<uint4*>(s.p[c])[i % (kTile / 16)] = z;
    }
    for (int i = threadIdx.x; i < (int)kTile / 16; i += kThreads)
      reinterpret_cast<uint4*>(s.v[px ^ 1])[i] = z;
    sm100::fence_proxy_async_smem();
  }
  if (warp == 1) sm100::tmem_alloc_cg2<512>(&s.tmem_base);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem = sm100::uniform(s.tmem_base);

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; warp-uniform loop) ----------------
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0; it < n_my; ++it) {
        int seq, h;
        item_of(it, seq, h);
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&s.empty[stage], phase ^ 1);
          const uint32_t full_leader = sm100::mapa(sm100::smem_u32(&s.full[stage]), 0);
          if (sm100::elect_one()) {
          if (leader) sm100::mbar_arrive_expect_tx(&s.full[stage], 2 * kStageBytes);
          uint8_t* st = s.stages[stage];
          sm100::tma_load_2d_cg2(st, &tm_x, full_leader, kb * 64, seq * kS);
#pragma unroll
          for (int bb = 0; bb < 3; ++bb) {
            const int b = (int)px * 3 + bb;  // box of the head's 6: part b/2, half b%2
            sm100::tma_load_2d_cg2(st + kXTile + bb * 32 * 128, &tm_w, full_leader, kb * 64,
                                   (b >> 1) * hidden + h * 64 + (b & 1) * 32);
          }
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader; warp-uniform loop, elected lane issues) ----------------
    if (leader) {
      constexpr uint32_t idesc_g = sm100::umma_idesc_bf16(256, kAccCols);
      constexpr uint32_t idesc_s = sm100::umma_idesc_bf16(256, 256);
      constexpr uint32_t idesc_o = sm100::umma_idesc_bf16(256, 128) | (1u << 16);  // V' MN-major
      const uint32_t q_addr = sm100::smem_u32(s.q), k_addr = sm100::smem_u32(s.k);
      const uint32_t p_addr = sm100::smem_u32(s.p[0]), v_addr = sm100::smem_u32(s.v[0]);
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;  // projection k-blocks issued so far
      // With O of the previous item pending, keep at most `lag` projection
      // k-blocks queued on the tensor pipe so O starts soon after P is ready.
      auto gemm_kb = [&](int kb, bool throttle) {
        if (throttle && lag > 0 && g >= lag) {
          const int d = g - lag;
          sm100::mbar_wait(&s.kdone[d % kStages], (d / kStages) & 1);
        }
        sm100::mbar_wait(&s.full[stage], phase);
        sm100::tc_fence_after();
        const uint32_t a = sm100::smem_u32(s.stages[stage]);
        const uint32_t b = a + kXTile;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sm100::mma_bf16_cg2_w(tmem, sm100::umma_desc_sw128(a + k * 32),
                                sm100::umma_desc_sw128(b + k * 32), idesc_g, (kb | k) != 0);
        sm100::mma_commit_cg2_mc_w(&s.empty[stage], 0x3);
        sm100::mma_commit_cg2_mc_w(&s.kdone[stage], 0x1);
        if (kb == k_blocks - 1) sm100::mma_commit_cg2_mc_w(&s.acc_full, 0x3);
        ++g;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      };
      auto issue_s = [&]() {
        sm100::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sm100::mma_bf16_cg2_w(tmem + kSCol, sm100::umma_desc_sw128(q_addr + k * 32),
                                sm100::umma_desc_sw128(k_addr + k * 32), idesc_s, k);
        sm100::mma_commit_cg2_mc_w(&s.s_full, 0x3);
      };
      auto issue_o = [&]() {
        sm100::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk)
          sm100::mma_bf16_cg2_w(tmem + kSCol,
                                sm100::umma_desc_sw128(p_addr + (kk >> 2) * kTile + (kk & 3) * 32),
                                sm100::umma_desc_sw128(v_addr + kk * 2048), idesc_o, kk);
        sm100::mma_commit_cg2_mc_w(&s.o_full, 0x3);
      };
      if (n_my > 0)
        for (int kb = 0; kb < k_blocks; ++kb) gemm_kb(kb, false);
      for (int it = 0; it < n_my; ++it) {
        const uint32_t par = it & 1;
        // both CTAs drained item it: accumulator free, Q / K / V' staged
        mbar_wait_acq(&s.drained, par);
        if (dbg) {  // measurement: projections only
          if (it + 1 < n_my)
            for (int kb = 0; kb < k_blocks; ++kb) gemm_kb(kb, false);
          continue;
        }
        issue_s();
        bool o_done = false;
        if (it + 1 < n_my) {
          for (int kb = 0; kb < k_blocks; ++kb) {
            if (!o_done && __shfl_sync(0xffffffffu, mbar_test_acq(&s.p_ready, par), 0)) {
              issue_o();
              o_done = true;
            }
            gemm_kb(kb, !o_done);
            if (!o_done && __shfl_sync(0xffffffffu, mbar_test_acq(&s.p_ready, par), 0)) {
              issue_o();
              o_done = true;
            }
          }
        }
        if (!o_done) {
          mbar_wait_acq(&s.p_ready, par);
          issue_o();
        }
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue / softmax (warps 2-9, both CTAs) ----------------
    const int quarter = warp & 3;
    const int hf = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t drained_l = sm100::mapa(sm100::smem_u32(&s.drained), 0);
    const uint32_t p_ready_l = sm100::mapa(sm100::smem_u32(&s.p_ready), 0);
    constexpr float kLog2e = 1.4426950408889634f;
    int aff_seq = -1;
    float rs_a = 1.f, rs_b = 0.f;
    for (int it = 0; it < n_my; ++it) {
      int seq, h;
      item_of(it, seq, h);
      const uint32_t par = it & 1;
      if (stats_in != nullptr && seq != aff_seq && seq < n_seq) {
        row_affine(stats_in + ((size_t)seq * kS + r) * n_part, n_part, eps, rs_a, rs_b);
        aff_seq = seq;
      }
      // (1) accumulator + bias (+ folded LayerNorm) -> bf16 Q (x 1/8), K, V'
      sm100::mbar_wait(&s.acc_full, par);
      sm100::tc_fence_after();
      if (dbg) {
        sm100::tc_fence_before();
        sm100::mbar_arrive_cluster(drained_l);
        continue;
      }
#pragma unroll 1
      for (int cc = 0; cc < 3; ++cc) {
        const int c = hf * 3 + cc;
        const int t = c >> 1, c32 = c & 1;
        uint32_t raw[32];
        sm100::tmem_ld_32x32b_x32(lane_base + c * 32, raw);
        sm100::tmem_ld_wait();
        const float* bp = b_qkv + t * hidden + h * 64 + c32 * 32;
        const float* cp = c_qkv + t * hidden + h * 64 + c32 * 32;
        const float scale = t == 0 ? 0.125f : 1.0f;
        uint8_t* rowp = (t == 0 ? s.q : t == 1 ? s.k : s.v[px]) + r * 128;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 b0 = __ldg(reinterpret_cast<const float4*>(bp + q4 * 8));
          const float4 b1 = __ldg(reinterpret_cast<const float4*>(bp + q4 * 8 + 4));
          float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          if (stats_in != nullptr) {
            const float4 c0 = __ldg(reinterpret_cast<const float4*>(cp + q4 * 8));
            const float4 c1 = __ldg(reinterpret_cast<const float4*>(cp + q4 * 8 + 4));
            const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) bb[e] = fmaf(rs_b, cv[e], bb[e]);
          }
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            v[e] = fmaf(rs_a, __uint_as_float(raw[q4 * 8 + e]), bb[e]) * scale;
          uint4 u;
          u.x = pack_bf16(v[0], v[1]);
          u.y = pack_bf16(v[2], v[3]);
          u.z = pack_bf16(v[4], v[5]);
          u.w = pack_bf16(v[6], v[7]);
          const int piece = c32 * 4 + q4;
          *reinterpret_cast<uint4*>(rowp + ((piece ^ (r & 7)) << 4)) = u;
        }
      }
      sm100::tc_fence_before();
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive_cluster(drained_l);
      // (2) softmax over this thread's 64 of its own sequence's 128 keys
      sm100::mbar_wait(&s.s_full, par);
      sm100::tc_fence_after();
      uint32_t sv[2][32];
      const uint32_t scol = kSCol + px * 128 + hf * 64;
      sm100::tmem_ld_32x32b_x32(lane_base + scol, sv[0]);
      sm100::tmem_ld_32x32b_x32(lane_base + scol + 32, sv[1]);
      sm100::tmem_ld_wait();
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 32; ++e)
        mx = fmaxf(mx, fmaxf(__uint_as_float(sv[0][e]), __uint_as_float(sv[1][e])));
      s.red_max[hf][r] = mx;
      epi_sync();
      mx = fmaxf(mx, s.red_max[hf ^ 1][r]);
      const float mxl = mx * kLog2e;
      float sum = 0.f;
      uint8_t* prow = s.p[px * 2 + hf] + r * 128;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        __align__(16) __nv_bfloat162 pv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float p0 =
              sm100::ex2_approx(fmaf(__uint_as_float(sv[q >> 2][(q & 3) * 8 + 2 * e]), kLog2e, -mxl));
          const float p1 =
              sm100::ex2_approx(fmaf(__uint_as_float(sv[q >> 2][(q & 3) * 8 + 2 * e + 1]), kLog2e, -mxl));
          pv[e] = __floats2bfloat162_rn(p0, p1);
          const float2 back = __bfloat1622float2(pv[e]);
          sum += back.x + back.y;
        }
        *reinterpret_cast<uint4*>(prow + ((q ^ (r & 7)) << 4)) = *reinterpret_cast<uint4*>(pv);
      }
      s.red_sum[hf][r] = sum;
      sm100::tc_fence_before();
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive_cluster(p_ready_l);
      // (3) O / rowsum -> ctx: this CTA's 64 output features, 32 per thread
      sm100::mbar_wait(&s.o_full, par);
      sm100::tc_fence_after();
      uint32_t ov[32];
      sm100::tmem_ld_32x32b_x32(lane_base + kSCol + px * 64 + hf * 32, ov);
      sm100::tmem_ld_wait();
      epi_sync();
      const float inv = 1.0f / (sum + s.red_sum[hf ^ 1][r]);
      if (seq < n_seq) {
        __nv_bfloat16* dst = ctx + ((size_t)seq * kS + r) * hidden + h * 64 + hf * 32;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(ov[q4 * 8 + 0]) * inv, __uint_as_float(ov[q4 * 8 + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(ov[q4 * 8 + 2]) * inv, __uint_as_float(ov[q4 * 8 + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(ov[q4 * 8 + 4]) * inv, __uint_as_float(ov[q4 * 8 + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(ov[q4 * 8 + 6]) * inv, __uint_as_float(ov[q4 * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + q4 * 8) = u;
        }
      }
      // the softmax exchange buffers are reused by the next item
      epi_sync();
    }
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_cg2<512>(tmem);
  }
}

static int n_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

}  // namespace qap

chm_status qkv_attention_pair(const void* x, const void* w_qkv, const float* b_qkv,
                              const float* c_qkv, const float2* stats_in, int n_part, float eps,
                              void* ctx, int n_seq, int hidden, cudaStream_t st) {
  const int n_heads = hidden / 64;
  const long long T = (long long)n_seq * qap::kS;
  CUtensorMap tm_x, tm_w;
  if (!gemm::make_tmap_bf16(&tm_x, x, (uint64_t)T, (uint64_t)hidden, qap::kS, 64, 0))
    return CHM_ERR_CUDA;
  if (!gemm::make_tmap_bf16(&tm_w, w_qkv, (uint64_t)3 * hidden, (uint64_t)hidden, 32, 64, 0))
    return CHM_ERR_CUDA;
  auto kern = qap::qkv_attention_pair_kernel;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(qap::kThreads, 1, 1);
  cfg.dynamicSmemBytes = qap::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_clusters = 0;
  if (!max_clusters) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qap::kSmemBytes);
    cfg.gridDim = dim3(2 * (qap::n_sms() / 2), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1)
      n = qap::n_sms() / 2;
    max_clusters = n;
  }
  const int items = ((n_seq + 1) / 2) * n_heads;
  const int n_cl = items < max_clusters ? items : max_clusters;
  cfg.gridDim = dim3(2 * n_cl, 1, 1);
  prof::begin(prof::K_QKV_ATTENTION, st);
  static const int lag = getenv("CHM_QAP_LAG") ? atoi(getenv("CHM_QAP_LAG")) : 0;
  static const int dbg = getenv("CHM_QA_DEBUG") ? atoi(getenv("CHM_QA_DEBUG")) : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm_x, tm_w, b_qkv, c_qkv, stats_in, n_part, eps,
                                     n_seq, n_heads, hidden,
                                     reinterpret_cast<__nv_bfloat16*>(ctx), lag, dbg);
  prof::end(prof::K_QKV_ATTENTION, st,
            2.0 * T * 3.0 * hidden * hidden + 4.0 * qap::kS * qap::kS * 64.0 * n_seq * n_heads);
  if (e != cudaSuccess) return CHM_ERR_CUDA;
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace chm
