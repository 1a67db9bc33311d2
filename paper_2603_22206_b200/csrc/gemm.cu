// K2 -- tcgen05 / TMEM / TMA GEMM for the router encoder.
//
//   C[M, N] = A[M, K] . B[N, K]^T  (+ bias[N]) (GELU) (+ residual[M, N]) (LayerNorm)
//   A: activations, B: nn.Linear weight [out, in]; both K-major bf16,
//   fp32 accumulation in tensor memory, bf16 output.
//
// Structure: persistent clusters of CTA PAIRS (one CTA per SM, 384 threads).
// A pair owns a 256 x 256 output tile; CTA x of the pair stages rows
// [128x, 128x+128) of the A tile and rows [128x, 128x+128) of the B tile
// (N half), so the pair MMA (tcgen05.mma.cta_group::2, M=256 N=256 K=16)
// reads half of each operand from each SM's shared memory.
//   warp 0      TMA producer (both CTAs): 4-stage ring of A 128x64 + B 128x64
//               tiles (128B swizzle); completion counted on the pair leader's
//               mbarrier (cta_group::2 TMA)
//   warp 1      TMEM (512 cols, cta_group::2) alloc/dealloc in both CTAs; in
//               the leader one elected thread issues the MMAs into a
//               double-buffered accumulator; tcgen05.commit multicasts
//               "stage free" / "accumulator full" to both CTAs of the pair
//   warps 4-11  epilogue (both CTAs): tcgen05.ld 32 lanes x 64 columns, bias
//               / tanh-GELU / residual / QKV split in fp32, bf16 into a
//               128B-swizzled smem box, TMA store (bulk group); residual
//               boxes arrive by TMA into the same staging buffers.
//
// EPI_RESIDUAL_LN (post-LN sublayer output, N = 256 g, g <= 4): the cluster is
// g pairs (2g CTAs; 6 for H = 768) covering one 256 x N row block, so every
// output row lives in g CTAs. Each epilogue thread owns (row, 128 columns): pass 1 forms
// v = acc + bias + residual and its (mean, M2); the partials are pushed to
// the three CTAs of the row group through distributed shared memory and an
// mbarrier; pass 2 re-reads TMEM and writes LayerNorm(v) in bf16. The sum
// never round-trips through HBM (no separate LayerNorm kernel, no bf16
// rounding of the pre-LN sum), and x is updated in place.
//
// FLOPs per launch: 2*M*N*K.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "deferred_ln.cuh"
#include "gemm.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace gemm {

constexpr int BM = 256, BN = 256, BK = 64;  // pair tile
constexpr int CM = 128, CN = 128;           // per-CTA operand rows (A half, B half)
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr uint32_t kTileABytes = CM * BK * 2;  // 16 KB
constexpr uint32_t kTileBBytes = CN * BK * 2;  // 16 KB
constexpr uint32_t kStageBytes = kTileABytes + kTileBBytes;
constexpr uint32_t kBoxBytes = 32 * 128;       // 32 rows x 64 bf16, one epilogue box
constexpr int kMaxLnGroups = 4;                // pairs per cluster in LN mode (N <= 1024)

enum Epilogue : int {
  EPI_NONE = 0,
  EPI_BIAS = 1,
  EPI_BIAS_GELU = 2,
  EPI_BIAS_RESIDUAL = 3,
  // QKV projection: bias, and columns [0, H) (Q) pre-scaled by 1/sqrt(64)
  // (exact in bf16) so attention needs no score scaling.
  EPI_QKV = 4,
  // C = LayerNorm(A.B^T + bias + residual) * gamma + beta, N = 256 g.
  EPI_RESIDUAL_LN = 5,
  // Deferred LayerNorm (post-LN sublayer without whole-row ownership):
  //   C = A.B^T + bias + LN(residual)   (LN(residual) = residual when no
  //   statistics are given), plus per-row partial statistics (mean, M2) of C
  //   over every 128-column chunk -> stats_out[M][N/128]. The consumer
  //   applies the LayerNorm: the next GEMM folds it into its epilogue
  //   (EPI_BIAS / EPI_BIAS_GELU / EPI_QKV with stats_in + colsum, weights
  //   pre-scaled by gamma: LN(x).W^T = rstd (x.W'^T) - rstd mean c + W.beta),
  //   the next residual sublayer normalises its residual box here.
  EPI_RESLN_STATS = 6,
};

struct EpiParams {
  int hidden;          // QKV: H
  const float* gamma;  // LN
  const float* beta;   // LN
  float eps;           // LN
  long long res_ld;    // residual row pitch in elements (0 = N)
  const float2* stats_in;  // deferred LN of the A rows (fold) / residual rows (EPI 6):
  int n_part;              //   [M][n_part] partial (mean, M2) over 128 columns each
  const float* colsum;     // fold: c_n = sum_k B'[n][k]
  float2* stats_out;       // EPI 6: [M][N/128]
  const int32_t* live_rows;  // rows computed: min(M, *live_rows * live_mult) (nullptr: M)
  int live_mult;
  int work_div;        // measurement only (prof): algorithmic FLOPs = 2 M N K / work_div
  int dbg;             // measurement only: 1 = epilogue drains TMEM without math/stores,
                       // 2 = also no operand loads (MMAs on stale shared memory)
};

// STAGES-deep operand ring; NBOX epilogue staging boxes per warp (2 lets a
// warp fill one box while the TMA store of the other drains); the LN
// statistics exchange exists only in the LN variant.
template <int STAGES, int NBOX, bool LN>
struct __align__(1024) SmemT {
  uint8_t tiles[STAGES][kStageBytes];                // A (16 KB) then B (16 KB) per stage
  uint8_t stage_out[kEpiWarps][NBOX][kBoxBytes];     // epilogue boxes (SW128)
  float2 stats[LN ? 2 : 1][LN ? kMaxLnGroups : 1][LN ? 2 : 1][LN ? CM : 1];  // [buf][pair][half][row]
  float ln_vec[LN ? 3 : 1][LN ? BN : 1];             // LN: bias, gamma, beta of this CTA's columns
  uint64_t full[STAGES];
  uint64_t empty[STAGES];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t res_bar[kEpiWarps][2];
  uint64_t stats_bar[2];
  uint32_t tmem_base;
};
template <int STAGES, int NBOX, bool LN>
constexpr size_t smem_bytes() { return sizeof(SmemT<STAGES, NBOX, LN>) + 1024; }  // + alignment slack

// GELU, tanh form: 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))), with the
// hardware tanh (MUFU). oracle/encoder_ref.py uses the same definition.
__device__ __forceinline__ float gelu_tanh(float x) {
  const float u = x * x;
  const float inner = x * fmaf(0.0356774081f, u, 0.7978845608f);
  const float hx = 0.5f * x;
  return fmaf(hx, sm100::tanh_approx(inner), hx);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ void st_async_f2(uint32_t addr, float2 v, uint32_t bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
          addr),
      "f"(v.x), "f"(v.y), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(sm100::smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void ld8(const float* p, float (&v)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p + 4));
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// v[0..63] = acc + bias + residual for this thread's row and a 64-column chunk.
// `bias_s` points at the chunk's first column in the staged shared-memory copy.
__device__ __forceinline__ void load_chunk_ln(const uint32_t (&r0)[32], const uint32_t (&r1)[32],
                                              const float* bias_s, const uint8_t* rowp, int lane,
                                              float (&v)[64]) {
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float4 b0 = *reinterpret_cast<const float4*>(bias_s + j * 8);
    const float4 b1 = *reinterpret_cast<const float4*>(bias_s + j * 8 + 4);
    const uint4 u = *reinterpret_cast<const uint4*>(rowp + ((j ^ (lane & 7)) << 4));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float acc = __uint_as_float(j < 4 ? r0[j * 8 + e] : r1[(j - 4) * 8 + e]);
      const float2 f = __bfloat1622float2(h[e >> 1]);
      v[j * 8 + e] = acc + bb[e] + ((e & 1) ? f.y : f.x);
    }
  }
}

template <int EPI, int kStages, bool FOLD>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                const __grid_constant__ CUtensorMap tmap_b,
                const __grid_constant__ CUtensorMap tmap_c,
                const __grid_constant__ CUtensorMap tmap_r, const float* __restrict__ bias,
                int M, int N, int K, EpiParams ep) {
  constexpr bool kLN = EPI == EPI_RESIDUAL_LN;
  constexpr int kBoxes = kStages > 4 ? 1 : 2;
  using Smem = SmemT<kStages, kBoxes, kLN>;
  const int ln_groups = kLN ? N / BN : 1;
  extern __shared__ uint8_t smem_raw[];
  Smem& s = sm100::align_smem_1024<Smem>(smem_raw);
  const int warp = sm100::warp_id(), lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const uint32_t px = rank & 1;          // position in the pair (M half)
  const uint32_t pair = rank >> 1;       // pair index in the cluster (LN: N tile)
  const uint32_t leader_rank = rank & ~1u;
  const bool leader = px == 0;
  const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pair));
  const int cluster = (int)sm100::cluster_id_x();
  const int n_cl = (int)sm100::n_clusters_x();
  // LN: a cluster tile is one 256-row block (all three N tiles); otherwise a
  // pair tile (256 x 256), row-block major.
  const int n_tiles_n = kLN ? 1 : (N + BN - 1) / BN;
  // only the live rows' tiles run (the routed sequences of the tick)
  if (ep.live_rows) M = min(M, __ldg(ep.live_rows) * ep.live_mult);
  const int n_tiles = ((M + BM - 1) / BM) * n_tiles_n;
  const int k_blocks = K / BK;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmap_a);
    sm100::tma_prefetch(&tmap_b);
    sm100::tma_prefetch(&tmap_c);
    if (EPI == EPI_BIAS_RESIDUAL || EPI == EPI_RESLN_STATS || kLN) sm100::tma_prefetch(&tmap_r);
    for (int i = 0; i < kStages; ++i) {
      sm100::mbar_init(&s.full[i], 1);
      sm100::mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s.tmem_full[i], 1);
      sm100::mbar_init(&s.tmem_empty[i], 2 * kEpiWarps);  // epilogues of both CTAs
      sm100::mbar_init(&s.stats_bar[i], 1);  // local arm; pushes complete tx bytes
    }
    for (int w = 0; w < kEpiWarps; ++w)
      for (int b = 0; b < 2; ++b) sm100::mbar_init(&s.res_bar[w][b], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc_cg2<512>(&s.tmem_base);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = sm100::uniform(s.tmem_base);

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    // warp-uniform loop, one elected lane issues (see sm100::elect_one)
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < n_tiles; t += n_cl) {
        const int m0 = (t / n_tiles_n) * BM + (int)px * CM;
        const int n0 = (kLN ? (int)pair : (t % n_tiles_n)) * BN + (int)px * CN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&s.empty[stage], phase ^ 1);
          const uint32_t full_leader =
              sm100::mapa(sm100::smem_u32(&s.full[stage]), leader_rank);
          if (!kLN && ep.dbg == 2) {
            if (leader && lane == 0) sm100::mbar_arrive(&s.full[stage]);
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          if (sm100::elect_one()) {
            if (leader) sm100::mbar_arrive_expect_tx(&s.full[stage], 2 * kStageBytes);
            uint8_t* base = s.tiles[stage];
            sm100::tma_load_2d_cg2(base, &tmap_a, full_leader, kb * BK, m0);
            sm100::tma_load_2d_cg2(base + kTileABytes, &tmap_b, full_leader, kb * BK, n0);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (pair leader) ----------------
    if (leader) {
      constexpr uint32_t idesc = sm100::umma_idesc_bf16(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = cluster; t < n_tiles; t += n_cl) {
        sm100::mbar_wait(&s.tmem_empty[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&s.full[stage], phase);
          sm100::tc_fence_after();
          {
            const uint32_t a_addr = sm100::smem_u32(s.tiles[stage]);
            const uint32_t b_addr = a_addr + kTileABytes;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = sm100::umma_desc_sw128(a_addr + k * 32);
              const uint64_t bd = sm100::umma_desc_sw128(b_addr + k * 32);
              sm100::mma_bf16_cg2_w(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
            sm100::mma_commit_cg2_mc_w(&s.empty[stage], pair_mask);
            if (kb == k_blocks - 1) sm100::mma_commit_cg2_mc_w(&s.tmem_full[acc], pair_mask);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs) ----------------
    const int ew = warp - 4;       // 0..7
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int half = ew >> 2;      // which 128 of the 256 columns
    const uint32_t empty_leader0 = sm100::mapa(sm100::smem_u32(&s.tmem_empty[0]), leader_rank);
    const uint32_t empty_leader1 = sm100::mapa(sm100::smem_u32(&s.tmem_empty[1]), leader_rank);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t res_phase = 0;  // bit b = phase of res_bar[ew][b]
    int box = 0;             // alternates the two staging boxes
    int it = 0;              // tiles processed by this CTA (LN stats buffer parity)
    if constexpr (kLN) {
      // this CTA's 256 columns are fixed for the whole launch: stage the
      // per-column vectors once (epilogue warps only: named barrier 1)
      const int et = threadIdx.x - 4 * 32;
      const int nb = (int)pair * BN;
      s.ln_vec[0][et] = bias[nb + et];
      s.ln_vec[1][et] = ep.gamma[nb + et];
      s.ln_vec[2][et] = ep.beta[nb + et];
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    }
    for (int t = cluster; t < n_tiles; t += n_cl, ++it) {
      const int mrow0 = (t / n_tiles_n) * BM + (int)px * CM + quarter * 32;
      const int n_tile0 = (kLN ? (int)pair : (t % n_tiles_n)) * BN + half * 128;
      const uint32_t lane_base = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN +
                                 half * 128;
      if (!kLN && ep.dbg != 0) {  // (not in the LN variant: keeps it spill-free)
        sm100::mbar_wait(&s.tmem_full[acc], acc_phase);
        sm100::tc_fence_after();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_remote(acc ? empty_leader1 : empty_leader0);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      if constexpr (kLN) {
        // ---- residual + LayerNorm epilogue ----
        if (lane == 0) {
          sm100::bulk_wait_read<0>();
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            sm100::mbar_arrive_expect_tx(&s.res_bar[ew][c], kBoxBytes);
            sm100::tma_load_2d(s.stage_out[ew][c], &tmap_r, &s.res_bar[ew][c], n_tile0 + c * 64,
                               mrow0);
          }
          // the next tile's residual rows into L2 now, so its loads do not wait
          // on HBM when the epilogue is the critical path (out-proj: tensor
          // pipe 48 -> 52 % per cycle, tools/experiments/res_prefetch_l2.sh)
          const int tn = t + n_cl;
          if (tn < n_tiles) {
            const int mrow_n = (tn / n_tiles_n) * BM + (int)px * CM + quarter * 32;
#pragma unroll
            for (int c = 0; c < 2; ++c) sm100::tma_prefetch_2d(&tmap_r, n_tile0 + c * 64, mrow_n);
          }
        }
        __syncwarp();
        sm100::mbar_wait(&s.tmem_full[acc], acc_phase);
        sm100::tc_fence_after();
        // pass 1: per-thread (mean, M2) over its 128 columns
        float mean = 0.f, m2 = 0.f;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t r0[32], r1[32];
          sm100::tmem_ld_32x32b_x32(lane_base + c * 64, r0);
          sm100::tmem_ld_32x32b_x32(lane_base + c * 64 + 32, r1);
          sm100::tmem_ld_wait();
          sm100::mbar_wait(&s.res_bar[ew][c], (res_phase >> c) & 1);
          float v[64];
          load_chunk_ln(r0, r1, &s.ln_vec[0][half * 128 + c * 64], s.stage_out[ew][c] + lane * 128,
                        lane, v);
          float cs = 0.f;
#pragma unroll
          for (int j = 0; j < 64; ++j) cs += v[j];
          const float cm = cs * (1.0f / 64.0f);
          float cm2 = 0.f;
#pragma unroll
          for (int j = 0; j < 64; ++j) cm2 = fmaf(v[j] - cm, v[j] - cm, cm2);
          if (c == 0) {
            mean = cm;
            m2 = cm2;
          } else {  // Chan merge of two equal-size groups
            const float d = cm - mean;
            mean = 0.5f * (mean + cm);
            m2 = m2 + cm2 + d * d * 32.0f;
          }
        }
        res_phase ^= 3u;
        // push (mean, M2) to the CTAs holding this row (same pair position)
        const int buf = it & 1;
        const int row_local = quarter * 32 + lane;
        // st.async: each 8-byte push completes bytes on the destination's
        // barrier (armed locally for ln_groups x 256 pushes), no fences
        if (ew == 0 && lane == 0)
          sm100::mbar_arrive_expect_tx(&s.stats_bar[buf], ln_groups * kEpiWarps * 32 * 8);
        for (int g = 0; g < ln_groups; ++g) {
          const uint32_t dst_rank = px + 2 * g;
          st_async_f2(sm100::mapa(sm100::smem_u32(&s.stats[buf][pair][half][row_local]), dst_rank),
                      make_float2(mean, m2),
                      sm100::mapa(sm100::smem_u32(&s.stats_bar[buf]), dst_rank));
        }
        mbar_wait_cluster(&s.stats_bar[buf], (it >> 1) & 1);
        float gm = 0.f;
        for (int g = 0; g < ln_groups; ++g)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) gm += s.stats[buf][g][hh][row_local].x;
        gm *= 1.0f / (2 * ln_groups);
        float gm2 = 0.f;
        for (int g = 0; g < ln_groups; ++g)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const float2 p = s.stats[buf][g][hh][row_local];
            gm2 += p.y + 128.0f * (p.x - gm) * (p.x - gm);
          }
        const float rstd = rsqrtf(gm2 / (float)(2 * ln_groups * 128) + ep.eps);
        // pass 2: normalise, write bf16 in place of the residual box, TMA store
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t r0[32], r1[32];
          sm100::tmem_ld_32x32b_x32(lane_base + c * 64, r0);
          sm100::tmem_ld_32x32b_x32(lane_base + c * 64 + 32, r1);
          sm100::tmem_ld_wait();
          if (c == 1) {
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive_remote(acc ? empty_leader1 : empty_leader0);
          }
          const int col0 = n_tile0 + c * 64;
          uint8_t* rowp = s.stage_out[ew][c] + lane * 128;
          float v[64];
          const int lc = half * 128 + c * 64;
          load_chunk_ln(r0, r1, &s.ln_vec[0][lc], rowp, lane, v);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 g0 = *reinterpret_cast<const float4*>(&s.ln_vec[1][lc + j * 8]);
            const float4 g1 = *reinterpret_cast<const float4*>(&s.ln_vec[1][lc + j * 8 + 4]);
            const float4 b0 = *reinterpret_cast<const float4*>(&s.ln_vec[2][lc + j * 8]);
            const float4 b1 = *reinterpret_cast<const float4*>(&s.ln_vec[2][lc + j * 8 + 4]);
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            float o[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o[e] = (v[j * 8 + e] - gm) * rstd * gg[e] + bb[e];
            uint4 u;
            u.x = pack_bf16(o[0], o[1]);
            u.y = pack_bf16(o[2], o[3]);
            u.z = pack_bf16(o[4], o[5]);
            u.w = pack_bf16(o[6], o[7]);
            *reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4)) = u;
          }
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sm100::tma_store_2d(&tmap_c, s.stage_out[ew][c], col0, mrow0);
            sm100::bulk_commit();
          }
        }
      } else {
        // ---- pointwise epilogues ----
        constexpr bool kRes = EPI == EPI_BIAS_RESIDUAL || EPI == EPI_RESLN_STATS;
        // FOLD instantiations carry the folded-LayerNorm arithmetic; the plain
        // ones compile without it
        constexpr bool kFold = FOLD && (EPI == EPI_BIAS || EPI == EPI_BIAS_GELU || EPI == EPI_QKV);
        const int row = mrow0 + lane;
        // Deferred LayerNorm of this thread's row (statistics from the producer
        // GEMM's partials; loaded before the accumulator wait so the L2
        // latency overlaps the MMAs). fold: v = rs_a acc + (rs_b c_n + b_n);
        // EPI_RESLN_STATS: LN(r) = (rs_a r + rs_b) gamma_n + beta_n.
        float rs_a = 1.f, rs_b = 0.f;
        const bool have_stats = (kFold || EPI == EPI_RESLN_STATS) && ep.stats_in != nullptr;
        if (have_stats && row < M) row_affine(ep.stats_in + (size_t)row * ep.n_part, ep.n_part,
                                              ep.eps, rs_a, rs_b);
        float sh = 0.f, s1 = 0.f, s2 = 0.f;  // EPI_RESLN_STATS: shifted sums of the output row
        if constexpr (kRes) {
          // residual boxes of both chunks requested before the accumulator
          // wait: their HBM latency overlaps the MMAs instead of the epilogue
          // (box c <- chunk c; both boxes are free once the previous tile's
          // stores have read them)
          static_assert(kBoxes == 2, "residual epilogues stage both chunks");
          if (lane == 0) {
            sm100::bulk_wait_read<0>();
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              if (n_tile0 + c * 64 < N) {
                sm100::mbar_arrive_expect_tx(&s.res_bar[ew][c], kBoxBytes);
                sm100::tma_load_2d(s.stage_out[ew][c], &tmap_r, &s.res_bar[ew][c],
                                   n_tile0 + c * 64, mrow0);
              }
            }
            // the next tile's residual boxes into L2 (see the LN epilogue)
            const int tn = t + n_cl;
            if (tn < n_tiles) {
              const int mrow_n = (tn / n_tiles_n) * BM + (int)px * CM + quarter * 32;
              const int ncol_n = (tn % n_tiles_n) * BN + half * 128;
#pragma unroll
              for (int c = 0; c < 2; ++c)
                if (ncol_n + c * 64 < N) sm100::tma_prefetch_2d(&tmap_r, ncol_n + c * 64, mrow_n);
            }
          }
          __syncwarp();
        }
        sm100::mbar_wait(&s.tmem_full[acc], acc_phase);
        sm100::tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          const int col0 = n_tile0 + c * 64;
          if (kRes) box = c;
          uint8_t* sb = s.stage_out[ew][box];
          // the box is free once the TMA store issued from it two chunks ago
          // has finished reading shared memory
          if (!kRes) {
            if (lane == 0) sm100::bulk_wait_read<kBoxes - 1>();
            __syncwarp();
          }
          uint32_t r0[32], r1[32];
          sm100::tmem_ld_32x32b_x32(lane_base + c * 64, r0);
          sm100::tmem_ld_32x32b_x32(lane_base + c * 64 + 32, r1);
          sm100::tmem_ld_wait();
          if (c == 1) {
            // accumulator fully read: hand it back to the leader's MMA warp
            sm100::tc_fence_before();
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive_remote(acc ? empty_leader1 : empty_leader0);
          }
          if (col0 >= N) continue;
          if (kRes) {
            sm100::mbar_wait(&s.res_bar[ew][box], (res_phase >> box) & 1);
            res_phase ^= 1u << box;
          }
          const float qscale = (EPI == EPI_QKV && col0 < ep.hidden) ? 0.125f : 1.0f;
          uint8_t* rowp = sb + lane * 128;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float v[8];
#pragma unroll
            for (int e = 0; e < 8; ++e)
              v[e] = __uint_as_float(j < 4 ? r0[j * 8 + e] : r1[(j - 4) * 8 + e]);
            if (EPI != EPI_NONE) {
              float bb[8];
              ld8(bias + col0 + j * 8, bb);
              if (kFold && have_stats) {
                float cc[8];
                ld8(ep.colsum + col0 + j * 8, cc);
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = fmaf(rs_a, v[e], fmaf(rs_b, cc[e], bb[e]));
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] += bb[e];
              }
            }
            uint4* slot = reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4));
            if (kRes) {
              const uint4 u = *slot;
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
              float r[8];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                r[2 * e] = f.x;
                r[2 * e + 1] = f.y;
              }
              if (EPI == EPI_RESLN_STATS && have_stats) {
                float gg[8], be[8];
                ld8(ep.gamma + col0 + j * 8, gg);
                ld8(ep.beta + col0 + j * 8, be);
#pragma unroll
                for (int e = 0; e < 8; ++e) r[e] = fmaf(fmaf(rs_a, r[e], rs_b), gg[e], be[e]);
              }
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] += r[e];
            }
            if (EPI == EPI_BIAS_GELU) {
#pragma unroll
              for (int e = 0; e < 8; ++e) v[e] = gelu_tanh(v[e]);
            }
            if (EPI == EPI_RESLN_STATS) {
              if (c == 0 && j == 0) sh = v[0];
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float d = v[e] - sh;
                s1 += d;
                s2 = fmaf(d, d, s2);
              }
            }
            uint4 o;
            o.x = pack_bf16(v[0] * qscale, v[1] * qscale);
            o.y = pack_bf16(v[2] * qscale, v[3] * qscale);
            o.z = pack_bf16(v[4] * qscale, v[5] * qscale);
            o.w = pack_bf16(v[6] * qscale, v[7] * qscale);
            *slot = o;
          }
          sm100::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            sm100::tma_store_2d(&tmap_c, sb, col0, mrow0);
            sm100::bulk_commit();
          }
          if (kBoxes == 2 && !kRes) box ^= 1;
        }
        if (EPI == EPI_RESLN_STATS && row < M) {
          // (mean, M2) of the fp32 (pre-rounding) output over this thread's
          // 128 columns: partial n_tile0 / 128 of the row
          const float mean = sh + s1 * (1.0f / 128.0f);
          const float m2 = fmaxf(fmaf(-s1, s1 * (1.0f / 128.0f), s2), 0.0f);
          ep.stats_out[(size_t)row * (N / 128) + n_tile0 / 128] = make_float2(mean, m2);
        }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0) sm100::bulk_wait_all();
    __syncwarp();
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc_cg2<512>(tmem_base);
  }
}

// ---- host: tensor maps -------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Row-major bf16 matrix [rows, cols] with row pitch `ld` elements as a 2D
// tensor map with a (box_cols x box_rows) box and 128-byte swizzle.
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, uint64_t ld) {
  auto fn = encode_fn();
  if (!fn) return false;
  if (ld == 0) ld = cols;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// W_qkv [3 * H, H] viewed as [3 parts][H rows][H cols]: one box = `box_rows`
// rows of each of the 3 parts (Q, K, V of a head), 64 columns, 128B swizzle;
// the box lands in shared memory as 3 * box_rows contiguous 128-byte rows.
bool make_tmap_qkv3(CUtensorMap* map, const void* ptr, uint64_t hidden, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {hidden, hidden, 3};
  cuuint64_t strides[2] = {hidden * 2, hidden * hidden * 2};
  cuuint32_t box[3] = {64, box_rows, 3};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int EPI, int kStages, bool FOLD = false>
static chm_status launch(const void* A, const void* B, void* C, const float* bias,
                         const void* residual, int M, int N, int K, EpiParams ep,
                         cudaStream_t s) {
  CUtensorMap ta, tb, tc, tr;
  if (!make_tmap_bf16(&ta, A, (uint64_t)M, (uint64_t)K, CM, BK, 0)) return CHM_ERR_CUDA;
  if (!make_tmap_bf16(&tb, B, (uint64_t)N, (uint64_t)K, CN, BK, 0)) return CHM_ERR_CUDA;
  if (!make_tmap_bf16(&tc, C, (uint64_t)M, (uint64_t)N, 32, 64, 0)) return CHM_ERR_CUDA;
  if (EPI == EPI_BIAS_RESIDUAL || EPI == EPI_RESIDUAL_LN || EPI == EPI_RESLN_STATS) {
    if (!make_tmap_bf16(&tr, residual, (uint64_t)M, (uint64_t)N, 32, 64, (uint64_t)ep.res_ld))
      return CHM_ERR_CUDA;
  } else {
    tr = tc;
  }
  constexpr size_t kSmemBytes =
      smem_bytes<kStages, (kStages > 4 ? 1 : 2), EPI == EPI_RESIDUAL_LN>();
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_kernel<EPI, kStages, FOLD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemBytes);
    attr_set = true;
  }
  const int cluster = (EPI == EPI_RESIDUAL_LN) ? 2 * (N / BN) : 2;
  const int tiles = (EPI == EPI_RESIDUAL_LN) ? (M + BM - 1) / BM
                                             : ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // Persistent grid: only as many clusters as can be co-resident (clusters
  // must fit inside a GPC, so e.g. 6-CTA clusters cannot use every SM); a
  // second partial wave would double the kernel time.
  static int max_active[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // per template instance
  if (!max_active[cluster - 1]) {
    cfg.gridDim = dim3(cluster * (num_sms() / cluster), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_kernel<EPI, kStages, FOLD>, &cfg) != cudaSuccess || n < 1)
      n = num_sms() / cluster;
    max_active[cluster - 1] = n;
  }
  const int max_clusters = max_active[cluster - 1];
  const int n_clusters = tiles < max_clusters ? tiles : max_clusters;
  cfg.gridDim = dim3(cluster * n_clusters, 1, 1);
  prof::begin(prof::K_GEMM, s);
  cudaError_t e = cudaLaunchKernelEx(&cfg, gemm_kernel<EPI, kStages, FOLD>, ta, tb, tc, tr, bias, M, N, K, ep);
  prof::end(prof::K_GEMM, s, 2.0 * M * N * K / (ep.work_div > 0 ? ep.work_div : 1));
  if (e != cudaSuccess) return CHM_ERR_CUDA;
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace gemm

// Internal entry (gemm.cuh), used by the encoder and the C-ABI wrappers.
chm_status gemm_run(const void* A, const void* B, void* C, int M, int N, int K,
                    const GemmArgs& g, cudaStream_t s) {
  const int epilogue = g.epilogue;
  if (M <= 0 || N <= 0 || K <= 0) return M == 0 ? CHM_OK : CHM_ERR_INVALID_ARG;
  if (K % gemm::BK != 0 || N % 64 != 0) return CHM_ERR_INVALID_ARG;
  if (epilogue != gemm::EPI_NONE && !g.bias) return CHM_ERR_INVALID_ARG;
  const bool res = epilogue == gemm::EPI_BIAS_RESIDUAL || epilogue == gemm::EPI_RESIDUAL_LN ||
                   epilogue == gemm::EPI_RESLN_STATS;
  if (res && !g.residual) return CHM_ERR_INVALID_ARG;
  if (g.res_ld != 0 && g.res_ld < N) return CHM_ERR_INVALID_ARG;
  if (epilogue == gemm::EPI_QKV && (g.hidden % 64 != 0 || N != 3 * g.hidden))
    return CHM_ERR_INVALID_ARG;
  if (epilogue == gemm::EPI_RESIDUAL_LN &&
      (N % gemm::BN != 0 || N / gemm::BN > gemm::kMaxLnGroups || !g.gamma || !g.beta))
    return CHM_ERR_UNSUPPORTED;
  if (g.stats_in && (g.n_part < 1 || g.n_part > kLnMaxParts)) return CHM_ERR_INVALID_ARG;
  if (g.stats_in && (epilogue == gemm::EPI_BIAS || epilogue == gemm::EPI_BIAS_GELU ||
                     epilogue == gemm::EPI_QKV) && !g.colsum)
    return CHM_ERR_INVALID_ARG;
  if (epilogue == gemm::EPI_RESLN_STATS &&
      (N % kLnPartCols != 0 || !g.stats_out || (g.stats_in && (!g.gamma || !g.beta))))
    return CHM_ERR_INVALID_ARG;
  gemm::EpiParams ep{};
  ep.hidden = g.hidden;
  ep.gamma = g.gamma;
  ep.beta = g.beta;
  ep.eps = g.eps;
  ep.res_ld = g.res_ld;
  ep.stats_in = g.stats_in;
  ep.n_part = g.n_part;
  ep.colsum = g.colsum;
  ep.stats_out = g.stats_out;
  ep.live_rows = g.live_rows;
  ep.live_mult = g.live_mult;
  ep.work_div = g.work_div;
  const float* bias = g.bias;
  const void* residual = g.residual;
  // measurement overrides: CHM_GEMM_STAGES (4 or 6 operand stages for the
  // pointwise epilogues), CHM_GEMM_DEBUG (EpiParams::dbg)
  static const int stages = getenv("CHM_GEMM_STAGES") ? atoi(getenv("CHM_GEMM_STAGES")) : 4;
  static const int dbg = getenv("CHM_GEMM_DEBUG") ? atoi(getenv("CHM_GEMM_DEBUG")) : 0;
  ep.dbg = dbg;
#define CHM_GEMM_CASE(E)                                                                    \
  case E:                                                                                    \
    if (g.stats_in)                                                                          \
      return gemm::launch<E, 4, true>(A, B, C, bias, residual, M, N, K, ep, s);              \
    return stages == 6 ? gemm::launch<E, 6>(A, B, C, bias, residual, M, N, K, ep, s)         \
                       : gemm::launch<E, 4>(A, B, C, bias, residual, M, N, K, ep, s);
  switch (epilogue) {
    case gemm::EPI_NONE:
      return stages == 6 ? gemm::launch<gemm::EPI_NONE, 6>(A, B, C, bias, residual, M, N, K, ep, s)
                         : gemm::launch<gemm::EPI_NONE, 4>(A, B, C, bias, residual, M, N, K, ep, s);
    CHM_GEMM_CASE(gemm::EPI_BIAS)
    CHM_GEMM_CASE(gemm::EPI_BIAS_GELU)
    CHM_GEMM_CASE(gemm::EPI_QKV)
    case gemm::EPI_BIAS_RESIDUAL:
      return gemm::launch<gemm::EPI_BIAS_RESIDUAL, 4>(A, B, C, bias, residual, M, N, K, ep, s);
    case gemm::EPI_RESLN_STATS:
      return gemm::launch<gemm::EPI_RESLN_STATS, 4>(A, B, C, bias, residual, M, N, K, ep, s);
    case gemm::EPI_RESIDUAL_LN:
      return gemm::launch<gemm::EPI_RESIDUAL_LN, 4>(A, B, C, bias, residual, M, N, K, ep, s);
    default: return CHM_ERR_INVALID_ARG;
  }
#undef CHM_GEMM_CASE
}

}  // namespace chm

extern "C" chm_status chm_gemm_bf16(const void* A, const void* B, void* C, const float* bias,
                                    const void* residual, int32_t M, int32_t N, int32_t K,
                                    int32_t epilogue, void* stream) {
  if (epilogue < chm::gemm::EPI_NONE || epilogue > chm::gemm::EPI_BIAS_RESIDUAL)
    return CHM_ERR_INVALID_ARG;
  chm::GemmArgs g;
  g.epilogue = epilogue;
  g.bias = bias;
  g.residual = residual;
  return chm::gemm_run(A, B, C, M, N, K, g, (cudaStream_t)stream);
}

extern "C" chm_status chm_gemm_bf16_ln(const void* A, const void* B, void* C, const float* bias,
                                       const void* residual, const float* gamma,
                                       const float* beta, float eps, int32_t M, int32_t N,
                                       int32_t K, void* stream) {
  chm::GemmArgs g;
  g.epilogue = chm::gemm::EPI_RESIDUAL_LN;
  g.bias = bias;
  g.residual = residual;
  g.gamma = gamma;
  g.beta = beta;
  g.eps = eps;
  return chm::gemm_run(A, B, C, M, N, K, g, (cudaStream_t)stream);
}

extern "C" chm_status chm_gemm_bf16_deferred_ln(const void* A, const void* B, void* C,
                                                const float* bias, int32_t epilogue,
                                                const void* residual, const float* gamma,
                                                const float* beta, const void* stats_in,
                                                int32_t n_part, const float* colsum,
                                                void* stats_out, float eps, int32_t M,
                                                int32_t N, int32_t K, void* stream) {
  if (epilogue != chm::gemm::EPI_BIAS && epilogue != chm::gemm::EPI_BIAS_GELU &&
      epilogue != chm::gemm::EPI_RESLN_STATS)
    return CHM_ERR_INVALID_ARG;
  chm::GemmArgs g;
  g.epilogue = epilogue;
  g.bias = bias;
  g.residual = residual;
  g.gamma = gamma;
  g.beta = beta;
  g.eps = eps;
  g.stats_in = reinterpret_cast<const float2*>(stats_in);
  g.n_part = n_part;
  g.colsum = colsum;
  g.stats_out = reinterpret_cast<float2*>(stats_out);
  return chm::gemm_run(A, B, C, M, N, K, g, (cudaStream_t)stream);
}
