// Fused feed-forward sublayer for H = 256 routers (the small router of
// cfg1 / cfg4):
//
//   x <- LayerNorm(x + GELU(x W1^T + b1) W2^T + b2) * gamma + beta
//
// in one kernel, the [T, F] intermediate never leaving the SM. The unfused
// pair (FFN1 with a GELU epilogue, FFN2 with the cluster-LN epilogue) moves
// 2 x T x F x 2 bytes through HBM (2.1 GB per layer at cfg4) and is
// memory-bound at H = 256 (FFN1 0.31 ms, FFN2 0.27 ms per layer).
//
// Persistent clusters of CTA pairs; a pair owns 256 rows (each CTA 128), and
// because H = 256 = one pair N-tile, every output row lives in one CTA, so the
// LayerNorm needs no cross-CTA exchange. Per 256-row tile, F is processed in
// chunks of 128 hidden units:
//   G1(c): acc_h[c & 1] = x . W1[128 c, +128)^T   pair MMA M 256 N 128 K 256
//   E1(c): acc_h -> + b1 -> GELU -> bf16 H[c & 1] (shared memory, the A
//          operand of G2 in the UMMA K-major 128B-swizzled layout)
//   G2(c): acc_y += H[c & 1] . W2[:, 128 c, +128)^T  pair MMA M 256 N 256 K 128
// TMEM: acc_h double-buffered [0, 128) / [128, 256), acc_y [256, 512). H is
// double-buffered in shared memory, so E1(c) overlaps G2(c - 1) and G1(c + 1).
// After the last chunk the epilogue adds b2 and the residual (x, re-read from
// L2) and applies the LayerNorm (two passes over acc_y), writing x in place.
//
//   warp 0      TMA: the tile's x (4 x [128 x 64] boxes), then W1 / W2
//               k-blocks through two rings (W1: 4 x 8 KB, W2: 2 x 16 KB)
//   warp 1      G1 issuer, warp 18 G2 issuer (the pair leader issues for both CTAs)
//   warps 2-17  epilogue: warp w owns TMEM lanes 32 (w % 4) (token rows) and
//               column group (w - 2) / 4: 32 of a chunk's 128 columns in E1,
//               64 of the 256 output columns in the LayerNorm
// Numerics equal the unfused path: fp32 accumulation in the same K order,
// bf16 GELU output, v = (acc + b2) + residual, LayerNorm in fp32 from
// (mean, M2) partials merged by Chan's formula.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace gemm {
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, uint64_t ld);
}  // namespace gemm
namespace ffn {

constexpr int kH = 256;                       // hidden size this kernel serves
constexpr int kRows = 128;                    // rows per CTA (pair tile: 256)
constexpr int kChunk = 128;                   // hidden units per chunk
// Two operand rings: W1 k-blocks (8 KB, 4 slots) and W2 k-blocks (16 KB, 2
// stages). One ring for both stalled the W1 prefetch behind W2 blocks whose
// G2 waits for the epilogue (head-of-line blocking): a chunk then took a full
// TMA round trip.
constexpr int kSlots1 = 4, kSlots2 = 2;
constexpr int kEpiWarps = 16;
constexpr int kThreads = 64 + kEpiWarps * 32 + 32;  // 608: + the G2 issuer (warp 18)
constexpr int kMaxF = 4096;
constexpr uint32_t kBox = kRows * 64 * 2;      // [128 rows][64 cols] bf16, 16 KB
constexpr uint32_t kW1Bytes = 64 * 64 * 2;     // W1 k-block half: [64 rows][64] = 8 KB
constexpr uint32_t kW2Bytes = 128 * 64 * 2;    // W2 k-block half: [128 rows][64] = 16 KB

struct __align__(1024) Smem {
  uint8_t xt[4][kBox];          // x tile, K = 256 in four 64-column boxes
  uint8_t hb[2][2][kBox];       // H chunks (double-buffered), K = 128 in two boxes
  uint8_t ring1[kSlots1][kW1Bytes];  // W1 k-blocks [64 rows][64]
  uint8_t ring2[kSlots2][kW2Bytes];  // W2 k-blocks [128 rows][64]
  float b1[kMaxF];
  float b2[kH], gamma[kH], beta[kH];
  float2 red[2][4][kRows];      // [tile parity][column group][row] (mean, M2)
  uint64_t full1[kSlots1], empty1[kSlots1], full2[kSlots2], empty2[kSlots2];
  uint64_t x_full, x_empty;
  uint64_t hacc_full[2], hacc_empty[2], h_full[2], h_empty[2];
  uint64_t y_full, y_empty;
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;
static_assert(kSmemBytes <= 227 * 1024, "shared memory");

// dbg (CHM_FFN_TL=1, measurement): CTA 0's timeline for its first tiles into x
// as int64 [32 chunks][8] = {E1 acc ready, E1 acc released, E1 H free, E1 done,
// G1 issued, G2 issued, -, -} and [32 + tile][8] = {Y ready, Y done}; x is not
// written then.
__device__ __forceinline__ void stamp(int dbg, void* x, int i, int k) {
  if ((dbg & 1) && blockIdx.x == 0 && i < 48) reinterpret_cast<long long*>(x)[i * 8 + k] = clock64();
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
// GELU, tanh form, as the unfused FFN1 epilogue (gemm.cu gelu_tanh)
__device__ __forceinline__ float gelu_tanh(float x) {
  const float u = x * x;
  const float inner = x * fmaf(0.0356774081f, u, 0.7978845608f);
  const float hx = 0.5f * x;
  return fmaf(hx, sm100::tanh_approx(inner), hx);
}

__global__ void __maxnreg__(96)
    ffn_fused_kernel(const __grid_constant__ CUtensorMap tm_x,
                     const __grid_constant__ CUtensorMap tm_w1,
                     const __grid_constant__ CUtensorMap tm_w2, const float* __restrict__ b1,
                     const float* __restrict__ b2, const float* __restrict__ gamma,
                     const float* __restrict__ beta, float eps, int M, int F,
                     __nv_bfloat16* __restrict__ x, const int32_t* __restrict__ live_rows,
                     int live_mult, int dbg) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = sm100::align_smem_1024<Smem>(smem_raw);
  const int warp = sm100::warp_id(), lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const bool leader = rank == 0;
  if (live_rows) M = min(M, __ldg(live_rows) * live_mult);
  for (int i = threadIdx.x; i < F; i += blockDim.x) s.b1[i] = b1[i];
  const int n_chunks = F / kChunk;
  const int n_tiles = (M + 2 * kRows - 1) / (2 * kRows);
  const int cl = (int)sm100::cluster_id_x(), n_cl = (int)sm100::n_clusters_x();
  const int n_my = cl < n_tiles ? (n_tiles - 1 - cl) / n_cl + 1 : 0;

  for (int i = threadIdx.x; i < kH; i += blockDim.x) {
    s.b2[i] = b2[i];
    s.gamma[i] = gamma[i];
    s.beta[i] = beta[i];
  }
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_x);
    sm100::tma_prefetch(&tm_w1);
    sm100::tma_prefetch(&tm_w2);
    for (int i = 0; i < kSlots1; ++i) {
      sm100::mbar_init(&s.full1[i], 1);
      sm100::mbar_init(&s.empty1[i], 1);
    }
    for (int i = 0; i < kSlots2; ++i) {
      sm100::mbar_init(&s.full2[i], 1);
      sm100::mbar_init(&s.empty2[i], 1);
    }
    sm100::mbar_init(&s.x_full, 1);
    // the tile's last G1 (commit) and the LayerNorm's residual reads (warps)
    sm100::mbar_init(&s.x_empty, 1 + kEpiWarps);
    for (int b = 0; b < 2; ++b) {
      sm100::mbar_init(&s.hacc_full[b], 1);
      sm100::mbar_init(&s.hacc_empty[b], 2 * kEpiWarps);  // both CTAs' epilogue warps
      sm100::mbar_init(&s.h_full[b], 2 * kEpiWarps);
      sm100::mbar_init(&s.h_empty[b], 1);
    }
    sm100::mbar_init(&s.y_full, 1);
    sm100::mbar_init(&s.y_empty, 2 * kEpiWarps);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc_cg2<512>(&s.tmem_base);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem = sm100::uniform(s.tmem_base);

  if (warp == 0) {
    // ---------------- TMA producer: two independent streams, polled ----------------
    // stream 1: per tile the x tile, then W1 k-blocks of chunks 0..n-1;
    // stream 2: W2 k-blocks of chunks 0..n-1 per tile. Each issues its next
    // load as soon as that slot is free, so neither blocks the other.
    const uint32_t full_x = sm100::mapa(sm100::smem_u32(&s.x_full), 0);
    int it1 = 0, c1 = -1, kb1 = 0, slot1 = 0;  // c1 = -1: the tile's x is next
    uint32_t ph1 = 0;
    int it2 = 0, c2 = 0, kb2 = 0, slot2 = 0;
    uint32_t ph2 = 0;
    while (it1 < n_my || it2 < n_my) {
      bool progressed = false;
      if (it1 < n_my) {
        if (c1 < 0) {
          if (__shfl_sync(0xffffffffu, sm100::mbar_test(&s.x_empty, (it1 & 1) ^ 1), 0)) {
            const int tile = cl + it1 * n_cl;
            if (sm100::elect_one()) {
              if (leader) sm100::mbar_arrive_expect_tx(&s.x_full, 2 * 4 * kBox);
#pragma unroll
              for (int kb = 0; kb < 4; ++kb)
                sm100::tma_load_2d_cg2(s.xt[kb], &tm_x, full_x, kb * 64,
                                       tile * 2 * kRows + (int)rank * kRows);
            }
            __syncwarp();
            c1 = 0;
            progressed = true;
          }
        } else if (__shfl_sync(0xffffffffu, sm100::mbar_test(&s.empty1[slot1], ph1 ^ 1), 0)) {
          if (sm100::elect_one()) {
            if (leader) sm100::mbar_arrive_expect_tx(&s.full1[slot1], 2 * kW1Bytes);
            // rows [128 c + 64 rank, +64) of W1, columns [64 kb, +64)
            sm100::tma_load_2d_cg2(s.ring1[slot1], &tm_w1,
                                   sm100::mapa(sm100::smem_u32(&s.full1[slot1]), 0), kb1 * 64,
                                   c1 * kChunk + 64 * (int)rank);
          }
          __syncwarp();
          if (++slot1 == kSlots1) { slot1 = 0; ph1 ^= 1; }
          if (++kb1 == 4) {
            kb1 = 0;
            if (++c1 == n_chunks) { c1 = -1; ++it1; }
          }
          progressed = true;
        }
      }
      if (it2 < n_my && __shfl_sync(0xffffffffu, sm100::mbar_test(&s.empty2[slot2], ph2 ^ 1), 0)) {
        if (sm100::elect_one()) {
          if (leader) sm100::mbar_arrive_expect_tx(&s.full2[slot2], 2 * kW2Bytes);
          // rows [128 rank, +128) of W2, columns [128 c + 64 kb, +64)
          sm100::tma_load_2d_cg2(s.ring2[slot2], &tm_w2,
                                 sm100::mapa(sm100::smem_u32(&s.full2[slot2]), 0),
                                 c2 * kChunk + kb2 * 64, 128 * (int)rank);
        }
        __syncwarp();
        if (++slot2 == kSlots2) { slot2 = 0; ph2 ^= 1; }
        if (++kb2 == 2) {
          kb2 = 0;
          if (++c2 == n_chunks) { c2 = 0; ++it2; }
        }
        progressed = true;
      }
      if (!progressed) __nanosleep(20);
    }
  } else if (warp == 1 || warp == 2 + kEpiWarps) {
    // ---------------- MMA issuers (the leader issues for both CTAs) ----------------
    // Warp 1 issues the G1 stream, warp 18 the G2 stream. Each waits only for
    // its own operands (W1 / W2 ring, acc_h / H buffers), so a G2 whose W2
    // k-blocks are still in flight no longer holds back the next G1 and vice
    // versa (one issuer serialised both behind each ring's reload).
    constexpr uint32_t idesc1 = sm100::umma_idesc_bf16(256, kChunk);
    constexpr uint32_t idesc2 = sm100::umma_idesc_bf16(256, kH);
    int slot1 = 0, slot2 = 0;
    uint32_t ph1 = 0, ph2 = 0;
    int gc1 = 0, gc2 = 0;  // global chunk counters of G1 / G2 (buffer = gc & 1)
    auto g1 = [&](int c) {
      const int b = gc1 & 1;
      sm100::mbar_wait(&s.hacc_empty[b], ((gc1 >> 1) & 1) ^ 1);  // E1(gc1 - 2) drained it
      sm100::tc_fence_after();
      for (int kb = 0; kb < 4; ++kb) {
        sm100::mbar_wait(&s.full1[slot1], ph1);
        sm100::tc_fence_after();
        const uint32_t a = sm100::smem_u32(s.xt[kb]);
        const uint32_t w = sm100::smem_u32(s.ring1[slot1]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sm100::mma_bf16_cg2_w(tmem + b * kChunk, sm100::umma_desc_sw128(a + k * 32),
                                sm100::umma_desc_sw128(w + k * 32), idesc1, (kb | k) != 0);
        sm100::mma_commit_cg2_mc_w(&s.empty1[slot1], 0x3);
        if (++slot1 == kSlots1) { slot1 = 0; ph1 ^= 1; }
      }
      sm100::mma_commit_cg2_mc_w(&s.hacc_full[b], 0x3);
      if (lane == 0 && gc1 < 32) stamp(dbg, x, gc1, 4);
      ++gc1;
      (void)c;
    };
    auto g2 = [&](int c) {
      const int b = gc2 & 1;
      sm100::mbar_wait(&s.h_full[b], (gc2 >> 1) & 1);  // E1(gc2) wrote H[b] in both CTAs
      sm100::tc_fence_after();
      for (int kb = 0; kb < 2; ++kb) {
        sm100::mbar_wait(&s.full2[slot2], ph2);
        sm100::tc_fence_after();
        const uint32_t a = sm100::smem_u32(s.hb[b][kb]);
        const uint32_t w = sm100::smem_u32(s.ring2[slot2]);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sm100::mma_bf16_cg2_w(tmem + 2 * kChunk, sm100::umma_desc_sw128(a + k * 32),
                                sm100::umma_desc_sw128(w + k * 32), idesc2, (c | kb | k) != 0);
        sm100::mma_commit_cg2_mc_w(&s.empty2[slot2], 0x3);
        if (++slot2 == kSlots2) { slot2 = 0; ph2 ^= 1; }
      }
      sm100::mma_commit_cg2_mc_w(&s.h_empty[b], 0x3);
      if (lane == 0 && gc2 < 32) stamp(dbg, x, gc2, 5);
      ++gc2;
    };
    if (warp == 1) {
      for (int it = 0; it < (leader ? n_my : 0); ++it) {
        sm100::mbar_wait(&s.x_full, it & 1);
        sm100::tc_fence_after();
        for (int c = 0; c < n_chunks; ++c) {
          g1(c);
          if (c == n_chunks - 1) sm100::mma_commit_cg2_mc_w(&s.x_empty, 0x3);
        }
      }
    } else {
      for (int it = 0; it < (leader ? n_my : 0); ++it) {
        for (int c = 0; c < n_chunks; ++c) {
          if (c == 0) {  // acc_y free: the previous tile's LayerNorm has read it
            sm100::mbar_wait(&s.y_empty, (it & 1) ^ 1);
            sm100::tc_fence_after();
          }
          g2(c);
        }
        sm100::mma_commit_cg2_mc_w(&s.y_full, 0x3);
      }
    }
    __syncwarp();
  } else if (warp >= 2 && warp < 2 + kEpiWarps) {
    // ---------------- epilogue ----------------
    const int quarter = warp & 3;
    const int grp = (warp - 2) >> 2;         // column group 0..3
    const int r = quarter * 32 + lane;       // row within the CTA's 128
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    const uint32_t hacc_empty0 = sm100::mapa(sm100::smem_u32(&s.hacc_empty[0]), 0);
    const uint32_t hacc_empty1 = sm100::mapa(sm100::smem_u32(&s.hacc_empty[1]), 0);
    const uint32_t h_full0 = sm100::mapa(sm100::smem_u32(&s.h_full[0]), 0);
    const uint32_t h_full1 = sm100::mapa(sm100::smem_u32(&s.h_full[1]), 0);
    const uint32_t y_empty_l = sm100::mapa(sm100::smem_u32(&s.y_empty), 0);
    int gc = 0;
    for (int it = 0; it < n_my; ++it) {
      const int tile = cl + it * n_cl;
      const int row = tile * 2 * kRows + (int)rank * kRows + r;
      for (int c = 0; c < n_chunks; ++c, ++gc) {
        // (E1) acc_h -> + b1 -> GELU -> bf16 H[b], columns [32 grp, +32) of the chunk
        const int b = gc & 1;
        const uint32_t par = (gc >> 1) & 1;
        sm100::mbar_wait(&s.hacc_full[b], par);
        sm100::tc_fence_after();
        const bool tl = warp == 2 && lane == 0 && gc < 32;
        if (tl) stamp(dbg, x, gc, 0);
        uint32_t raw[32];
        sm100::tmem_ld_32x32b_x32(lane_base + b * kChunk + grp * 32, raw);
        sm100::tmem_ld_wait();
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_remote(b ? hacc_empty1 : hacc_empty0);
        if (tl) stamp(dbg, x, gc, 1);
        // H[b] free: G2(gc - 2) has read it
        sm100::mbar_wait(&s.h_empty[b], par ^ 1);
        if (tl) stamp(dbg, x, gc, 2);
        uint8_t* rowp = s.hb[b][grp >> 1] + r * 128;
        const float* bp = s.b1 + c * kChunk + grp * 32;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = gelu_tanh(__uint_as_float(raw[j * 8 + e]) + bp[j * 8 + e]);
          uint4 u;
          u.x = pack_bf16(v[0], v[1]);
          u.y = pack_bf16(v[2], v[3]);
          u.z = pack_bf16(v[4], v[5]);
          u.w = pack_bf16(v[6], v[7]);
          const int piece = (grp & 1) * 4 + j;
          *reinterpret_cast<uint4*>(rowp + ((piece ^ (r & 7)) << 4)) = u;
        }
        sm100::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_remote(b ? h_full1 : h_full0);
        if (tl) stamp(dbg, x, gc, 3);
      }
      // (LN) v = (acc_y + b2) + x, LayerNorm over the row's 256 columns; this
      // thread: columns [64 grp, +64) in two halves of 32
      sm100::mbar_wait(&s.y_full, it & 1);
      sm100::tc_fence_after();
      if (warp == 2 && lane == 0) stamp(dbg, x, 32 + it, 0);
      const bool live = row < M && !(dbg & 1);
      // pass 1: v = (acc + b2) + residual, the residual from the x tile still
      // in shared memory (box grp, row r); v goes back into acc_y
      float mean = 0.f, m2 = 0.f;
      const uint8_t* xrow = s.xt[grp] + r * 128;
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t raw[32];
        const uint32_t ta = lane_base + 2 * kChunk + grp * 64 + hh * 32;
        sm100::tmem_ld_32x32b_x32(ta, raw);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int piece = hh * 4 + j;
          const uint4 u = *reinterpret_cast<const uint4*>(xrow + ((piece ^ (r & 7)) << 4));
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float2 f = __bfloat1622float2(h2[e >> 1]);
            const float v = (__uint_as_float(raw[j * 8 + e]) + s.b2[grp * 64 + piece * 8 + e]) +
                            ((e & 1) ? f.y : f.x);
            raw[j * 8 + e] = __float_as_uint(v);
          }
        }
        sm100::tmem_st_32x32b_x32(ta, raw);
        float cs = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) cs += __uint_as_float(raw[j]);
        const float cm = cs * (1.0f / 32.0f);
        float cm2 = 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float d = __uint_as_float(raw[j]) - cm;
          cm2 = fmaf(d, d, cm2);
        }
        if (hh == 0) {
          mean = cm;
          m2 = cm2;
        } else {  // Chan merge of two equal-size groups
          const float d = cm - mean;
          mean = 0.5f * (mean + cm);
          m2 = m2 + cm2 + d * d * 16.0f;
        }
      }
      sm100::tmem_st_wait();
      // the x tile has served as the residual: the next tile's x may load
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&s.x_empty);
      const int rp = it & 1;
      s.red[rp][grp][r] = make_float2(mean, m2);
      asm volatile("bar.sync 1, 512;" ::: "memory");
      float gm = 0.f;
#pragma unroll
      for (int g = 0; g < 4; ++g) gm += s.red[rp][g][r].x;
      gm *= 0.25f;
      float gm2 = 0.f;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const float2 p = s.red[rp][g][r];
        gm2 += p.y + 64.0f * (p.x - gm) * (p.x - gm);
      }
      const float rstd = rsqrtf(gm2 / (float)kH + eps);
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t raw[32];
        sm100::tmem_ld_32x32b_x32(lane_base + 2 * kChunk + grp * 64 + hh * 32, raw);
        sm100::tmem_ld_wait();
        if (hh == 1) {  // acc_y read completely: the next tile's G2 may start
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive_remote(y_empty_l);
        }
        uint4 out[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float o[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int col = grp * 64 + hh * 32 + j * 8 + e;
            o[e] = (__uint_as_float(raw[j * 8 + e]) - gm) * rstd * s.gamma[col] + s.beta[col];
          }
          out[j].x = pack_bf16(o[0], o[1]);
          out[j].y = pack_bf16(o[2], o[3]);
          out[j].z = pack_bf16(o[4], o[5]);
          out[j].w = pack_bf16(o[6], o[7]);
        }
        // every thread of the row has read its residual before any writes:
        // the row's four column groups are disjoint, so in-place is safe
        if (hh == 1 && warp == 2 && lane == 0) stamp(dbg, x, 32 + it, 1);
        if (live) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint4*>(x + (size_t)row * kH + grp * 64 + hh * 32 + j * 8) = out[j];
        }
      }
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

}  // namespace ffn

// x[M, 256] <- LN(x + GELU(x W1^T + b1) W2^T + b2) (gamma, beta), in place.
// W1 [F, 256], W2 [256, F] bf16 (nn.Linear layout), F a multiple of 128 up to
// 4096. live_rows (device, nullable): rows computed = min(M, *live_rows * live_mult).
chm_status ffn_fused(const void* x, const void* w1, const float* b1, const void* w2,
                     const float* b2, const float* gamma, const float* beta, float eps, int M,
                     int H, int F, const int32_t* live_rows, int live_mult, cudaStream_t st) {
  if (H != ffn::kH || F % ffn::kChunk != 0 || F > ffn::kMaxF || F < ffn::kChunk || M < 0)
    return CHM_ERR_UNSUPPORTED;
  if (M == 0) return CHM_OK;
  CUtensorMap tm_x, tm_w1, tm_w2;
  if (!gemm::make_tmap_bf16(&tm_x, x, (uint64_t)M, (uint64_t)H, ffn::kRows, 64, 0) ||
      !gemm::make_tmap_bf16(&tm_w1, w1, (uint64_t)F, (uint64_t)H, 64, 64, 0) ||
      !gemm::make_tmap_bf16(&tm_w2, w2, (uint64_t)H, (uint64_t)F, 128, 64, 0))
    return CHM_ERR_CUDA;
  auto kern = ffn::ffn_fused_kernel;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(ffn::kThreads, 1, 1);
  cfg.dynamicSmemBytes = ffn::kSmemBytes;
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
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ffn::kSmemBytes);
    cfg.gridDim = dim3(2 * (ffn::n_sms() / 2), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1)
      n = ffn::n_sms() / 2;
    max_clusters = n;
  }
  const int tiles = (M + 2 * ffn::kRows - 1) / (2 * ffn::kRows);
  const int n_cl = tiles < max_clusters ? tiles : max_clusters;
  cfg.gridDim = dim3(2 * n_cl, 1, 1);
  static const int dbg = getenv("CHM_FFN_TL") ? atoi(getenv("CHM_FFN_TL")) : 0;
  prof::begin(prof::K_GEMM, st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm_x, tm_w1, tm_w2, b1, b2, gamma, beta, eps, M,
                                     F, reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(x)),
                                     live_rows, live_mult, dbg);
  prof::end(prof::K_GEMM, st, 2.0 * 2.0 * M * (double)H * F);
  if (e != cudaSuccess) return CHM_ERR_CUDA;
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace chm

extern "C" chm_status chm_ffn_fused_bf16(void* x, const void* w1, const float* b1, const void* w2,
                                         const float* b2, const float* gamma, const float* beta,
                                         float eps, int32_t M, int32_t hidden, int32_t ffn,
                                         void* stream) {
  if (!x || !w1 || !b1 || !w2 || !b2 || !gamma || !beta || M < 0) return CHM_ERR_INVALID_ARG;
  return chm::ffn_fused(x, w1, b1, w2, b2, gamma, beta, eps, M, hidden, ffn, nullptr, 1,
                        (cudaStream_t)stream);
}
