// K2+K3 fused QKV projection + attention, S = 128, two epilogue groups
// ("duo"). Same item and projection as the PAIR kernel in
// qkv_attn.cu -- one item = (sequence, head); a cluster of two CTAs projects
// two sequences of one head with one cta_group::2 MMA per k-block (M = 256,
// N = 192 = the head's Q | K | V rows, split 96 / 96) -- but the per-item
// attention epilogue is no longer on the critical path.
//
// Measured on the PAIR kernel (tools/experiments/r2_qa_modes.sh, H = 768):
// the projection alone runs at 1.14 ms per layer (~98 % of the tensor peak),
// the full kernel at 1.73 ms: one epilogue group works through drain -> wait
// S -> softmax -> wait O -> store per item (~5.7k cycles of dependent
// latency), longer than the next item's projection (~4.7k cycles), and the
// accumulator double buffer cannot run further ahead. Here items alternate
// between two epilogue groups (warps 2-9: even items, warps 10-17: odd
// items), each owning half of tensor memory and its own Q / K / V tiles:
//
//   TMEM buffer e = columns [256 e, 256 e + 256):
//     [0, 192)   projection accumulator of the group's current item
//     [0, 128)   S = Q K^T, after the accumulator has been drained
//     [192, 256) O = P V
//   A buffer is released (projection of item i + 2 may start) once item i's O
//   has been read, so two items' latency chains overlap the projections.
//
//   warp 0      TMA producer: 4-stage ring of x[128 x 64] + the CTA's half
//               of the head's W rows [96 x 64] (28 KB), cta_group::2 loads
//   warp 1      MMA issuer: the leader CTA issues the pair projection; both
//               CTAs slot their own items' S(i) / O(i) (cta_group::1) into the
//               tensor pipe between k-blocks as soon as each is ready
//   warps 2-17  epilogue group e = (warp - 2) / 8, 2 threads per token row:
//               (1) acc + bias -> bf16 Q (x 1/8), K, V in shared memory
//               (2) softmax of S (row max / sum exchanged through shared
//                   memory), P bf16 over the Q | K tiles
//               (3) O / row sum -> ctx (bf16, HBM), buffer released
// Numerics equal the PAIR kernel and the unfused path: fp32 accumulation,
// fp32 bias, bf16 Q/K/V, exp2-based softmax normalised by the sum of the
// bf16-rounded P.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "deferred_ln.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace gemm {
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, uint64_t ld);
bool make_tmap_qkv3(CUtensorMap* map, const void* ptr, uint64_t hidden, uint32_t box_rows);
}  // namespace gemm
namespace qa_duo {

constexpr int kS = 128;                      // tokens per sequence = MMA M per CTA
constexpr int kStages = 4;                   // operand ring depth
constexpr int kGroups = 2;                   // epilogue groups
constexpr int kEpiWarps = 8;                 // warps per group (2 threads per row)
constexpr int kThreads = 64 + kGroups * kEpiWarps * 32;  // 576
constexpr uint32_t kATile = kS * 64 * 2;     // x [128][64] bf16, 16 KB
constexpr uint32_t kBHalf = 96 * 64 * 2;     // this CTA's W rows [96][64], 12 KB
constexpr uint32_t kStageBytes = kATile + kBHalf;
constexpr uint32_t kHeadTile = kS * 64 * 2;  // Q / K / V [128][64] bf16, 16 KB
constexpr uint32_t kBufCols = 256;           // TMEM columns per group
constexpr uint32_t kOCol = 192;              // O within a group's buffer

struct __align__(1024) Smem {
  uint8_t stages[kStages][kStageBytes];
  alignas(1024) uint8_t qkv[kGroups][3][kHeadTile];  // per group: Q, K, V (P over Q | K)
  float red_max[kGroups][2][kS];
  float red_sum[kGroups][2][kS];
  uint64_t full[kStages], empty[kStages];
  uint64_t acc_full[kGroups], buf_free[kGroups];
  uint64_t qkv_ready[kGroups], s_full[kGroups], p_ready[kGroups], o_full[kGroups];
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;
static_assert(kSmemBytes <= 227 * 1024, "shared memory");

// dbg (CHM_QA_DUO_TL=1, measurement): CTA 0's per-item timeline into ctx as
// int64 [32 items][12] (clock64); ctx is not written then.
__device__ __forceinline__ void stamp(int dbg, void* ctx, int it, int k) {
  if (dbg && blockIdx.x == 0 && it < 32) reinterpret_cast<long long*>(ctx)[it * 12 + k] = clock64();
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <bool FOLD>
__global__ void __maxnreg__(96)
    qkv_attention_duo_kernel(const __grid_constant__ CUtensorMap tm_x,
                             const __grid_constant__ CUtensorMap tm_w,
                             const float* __restrict__ b_qkv, const float* __restrict__ c_qkv,
                             const float2* __restrict__ stats_in, int n_part, float eps,
                             int n_seq, int n_heads, int hidden,
                             __nv_bfloat16* __restrict__ ctx, const int32_t* __restrict__ n_live,
                             int dbg) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = sm100::align_smem_1024<Smem>(smem_raw);
  const int warp = sm100::warp_id(), lane = threadIdx.x & 31;
  const int k_blocks = hidden / 64;
  const uint32_t rank = sm100::cluster_ctarank();  // sequence within the pair
  const bool leader = rank == 0;
  if (n_live) n_seq = min(n_seq, __ldg(n_live));  // only the routed sequences
  const int n_citems = ((n_seq + 1) / 2) * n_heads;
  const int cl = (int)sm100::cluster_id_x(), n_cl = (int)sm100::n_clusters_x();
  const int n_my = cl < n_citems ? (n_citems - 1 - cl) / n_cl + 1 : 0;
  auto item_of = [&](int it, int& seq, int& h) {
    const int c = cl + it * n_cl;
    const int sg = c / n_heads;
    h = c - sg * n_heads;
    seq = sg * 2 + (int)rank;
  };

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_x);
    sm100::tma_prefetch(&tm_w);
    for (int i = 0; i < kStages; ++i) {
      sm100::mbar_init(&s.full[i], 1);
      sm100::mbar_init(&s.empty[i], 1);
    }
    for (int e = 0; e < kGroups; ++e) {
      sm100::mbar_init(&s.acc_full[e], 1);
      sm100::mbar_init(&s.buf_free[e], 2 * kEpiWarps);  // the group's warps of both CTAs
      sm100::mbar_init(&s.qkv_ready[e], kEpiWarps * 32);
      sm100::mbar_init(&s.s_full[e], 1);
      sm100::mbar_init(&s.p_ready[e], kEpiWarps * 32);
      sm100::mbar_init(&s.o_full[e], 1);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc_cg2<512>(&s.tmem_base);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem = sm100::uniform(s.tmem_base);

  if (warp == 0) {
    // ---------------- TMA producer: own x tile + own half of the head's W ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; it < n_my; ++it) {
      int seq, h;
      item_of(it, seq, h);
      for (int kb = 0; kb < k_blocks; ++kb) {
        sm100::mbar_wait(&s.empty[stage], phase ^ 1);
        if (sm100::elect_one()) {
          if (leader) sm100::mbar_arrive_expect_tx(&s.full[stage], 2 * kStageBytes);
          const uint32_t full_leader = sm100::mapa(sm100::smem_u32(&s.full[stage]), 0);
          uint8_t* st = s.stages[stage];
          sm100::tma_load_2d_cg2(st, &tm_x, full_leader, kb * 64, seq * kS);
          // rows [32 rank, +32) of the head's Q, K and V parts (3-part view)
          sm100::tma_load_3d_cg2(st + kATile, &tm_w, full_leader, kb * 64, h * 64 + rank * 32, 0);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-uniform; *_w helpers elect the lane) ----------------
    constexpr uint32_t idesc_p = sm100::umma_idesc_bf16(256, 192);
    constexpr uint32_t idesc_s = sm100::umma_idesc_bf16(128, 128);
    constexpr uint32_t idesc_o = sm100::umma_idesc_bf16(128, 64) | (1u << 16);  // V MN-major
    int stage = 0;
    uint32_t phase = 0;
    int ns = 0, no = 0;  // next item whose S / O is to be issued (this CTA)
    // S(j) once Q/K/V(j) are staged, O(j) once P(j) is; S in issue order,
    // O(j) after S(j). Polled between projection k-blocks; never blocks.
    auto try_events = [&]() {
      if (ns < n_my) {
        const int e = ns & 1;
        if (__shfl_sync(0xffffffffu, sm100::mbar_test(&s.qkv_ready[e], (ns >> 1) & 1), 0)) {
          sm100::tc_fence_after();
          const uint32_t q_addr = sm100::smem_u32(s.qkv[e][0]);
          const uint32_t k_addr = sm100::smem_u32(s.qkv[e][1]);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            sm100::mma_bf16_w(tmem + e * kBufCols, sm100::umma_desc_sw128(q_addr + k * 32),
                              sm100::umma_desc_sw128(k_addr + k * 32), idesc_s, k);
          sm100::mma_commit_w(&s.s_full[e]);
          if (lane == 0) stamp(dbg, ctx, ns, 6);
          ++ns;
        }
      }
      if (no < ns) {
        const int e = no & 1;
        if (__shfl_sync(0xffffffffu, sm100::mbar_test(&s.p_ready[e], (no >> 1) & 1), 0)) {
          sm100::tc_fence_after();
          const uint32_t q_addr = sm100::smem_u32(s.qkv[e][0]);
          const uint32_t k_addr = sm100::smem_u32(s.qkv[e][1]);
          const uint32_t v_addr = sm100::smem_u32(s.qkv[e][2]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t pa = ((kk >> 2) ? k_addr : q_addr) + (kk & 3) * 32;
            sm100::mma_bf16_w(tmem + e * kBufCols + kOCol, sm100::umma_desc_sw128(pa),
                              sm100::umma_desc_sw128(v_addr + kk * 2048), idesc_o, kk);
          }
          sm100::mma_commit_w(&s.o_full[e]);
          if (lane == 0) stamp(dbg, ctx, no, 7);
          ++no;
        }
      }
    };
    for (int it = 0; it < (leader ? n_my : 0); ++it) {  // the leader projects for both
      const int e = it & 1;
      // buffer e free: item it - 2 finished in both CTAs
      while (!__shfl_sync(0xffffffffu, sm100::mbar_test(&s.buf_free[e], ((it >> 1) & 1) ^ 1), 0))
        try_events();
      sm100::tc_fence_after();
      if (lane == 0) stamp(dbg, ctx, it, 8);
      const uint32_t d = tmem + e * kBufCols;
      for (int kb = 0; kb < k_blocks; ++kb) {
        sm100::mbar_wait(&s.full[stage], phase);
        sm100::tc_fence_after();
        const uint32_t a = sm100::smem_u32(s.stages[stage]);
        const uint32_t b = a + kATile;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sm100::mma_bf16_cg2_w(d, sm100::umma_desc_sw128(a + k * 32),
                                sm100::umma_desc_sw128(b + k * 32), idesc_p, (kb | k) != 0);
        sm100::mma_commit_cg2_mc_w(&s.empty[stage], 0x3);
        if (kb == k_blocks - 1) sm100::mma_commit_cg2_mc_w(&s.acc_full[e], 0x3);
        if (lane == 0 && (kb == 0 || kb == k_blocks - 1)) stamp(dbg, ctx, it, kb == 0 ? 9 : 10);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
        try_events();
      }
    }
    while (no < n_my) try_events();
    __syncwarp();
  } else {
    // ---------------- epilogue group e: items e, e + 2, ... ----------------
    const int e = (warp - 2) / kEpiWarps;
    const int we = (warp - 2) % kEpiWarps;
    const int quarter = warp & 3;       // TMEM lane quarter this warp may access
    const int hf = we >> 2;             // column half
    const int r = quarter * 32 + lane;  // token row of the item
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16) + e * kBufCols;
    const uint32_t bar_id = 1 + e;
    auto epi_sync = [&]() { asm volatile("bar.sync %0, 256;" ::"r"(bar_id) : "memory"); };
    constexpr float kLog2e = 1.4426950408889634f;
    int aff_seq = -1;
    float rs_a = 1.f, rs_b = 0.f;
    for (int it = e; it < n_my; it += kGroups) {
      int seq, h;
      item_of(it, seq, h);
      const uint32_t par = (it >> 1) & 1;
      if (FOLD && seq != aff_seq && seq < n_seq) {
        row_affine(stats_in + ((size_t)seq * kS + r) * n_part, n_part, eps, rs_a, rs_b);
        aff_seq = seq;
      }
      // (1) acc + bias -> bf16 Q/K/V. Chunk c (32 columns) of the 192:
      // half c / 3 of the pair, part t = c % 3 (Q, K, V)
      sm100::mbar_wait(&s.acc_full[e], par);
      sm100::tc_fence_after();
      const bool tl = we == 0 && lane == 0;
      if (tl) stamp(dbg, ctx, it, 0);
      {
#pragma unroll 1
        for (int cc = 0; cc < 3; ++cc) {
          const int c = hf * 3 + cc;
          uint32_t raw[1][32];
          sm100::tmem_ld_32x32b_x32(lane_base + c * 32, raw[0]);
          sm100::tmem_ld_wait();
          const int t = c % 3, c32 = c / 3;
          const float* bp = b_qkv + t * hidden + h * 64 + c32 * 32;
          const float* cp = c_qkv + t * hidden + h * 64 + c32 * 32;
          const float scale = t == 0 ? 0.125f : 1.0f;
          uint8_t* rowp = s.qkv[e][t] + r * 128;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            const float4 b0 = __ldg(reinterpret_cast<const float4*>(bp + q4 * 8));
            const float4 b1 = __ldg(reinterpret_cast<const float4*>(bp + q4 * 8 + 4));
            float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
            if (FOLD) {
              const float4 c0 = __ldg(reinterpret_cast<const float4*>(cp + q4 * 8));
              const float4 c1 = __ldg(reinterpret_cast<const float4*>(cp + q4 * 8 + 4));
              const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
              for (int x = 0; x < 8; ++x) bb[x] = fmaf(rs_b, cv[x], bb[x]);
            }
            float v[8];
#pragma unroll
            for (int x = 0; x < 8; ++x)
              v[x] = fmaf(rs_a, __uint_as_float(raw[0][q4 * 8 + x]), bb[x]) * scale;
            uint4 u;
            u.x = pack_bf16(v[0], v[1]);
            u.y = pack_bf16(v[2], v[3]);
            u.z = pack_bf16(v[4], v[5]);
            u.w = pack_bf16(v[6], v[7]);
            const int piece = c32 * 4 + q4;
            *reinterpret_cast<uint4*>(rowp + ((piece ^ (r & 7)) << 4)) = u;
          }
        }
      }
      sm100::tc_fence_before();
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive(&s.qkv_ready[e]);
      if (tl) stamp(dbg, ctx, it, 1);
      // (2) softmax over this thread's 64 keys [64 hf, 64 hf + 64)
      sm100::mbar_wait(&s.s_full[e], par);
      sm100::tc_fence_after();
      if (tl) stamp(dbg, ctx, it, 2);
      uint32_t sv[2][32];
      sm100::tmem_ld_32x32b_x32(lane_base + hf * 64, sv[0]);
      sm100::tmem_ld_32x32b_x32(lane_base + hf * 64 + 32, sv[1]);
      sm100::tmem_ld_wait();
      float mq[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) mq[t] = -INFINITY;
#pragma unroll
      for (int x = 0; x < 32; ++x)
        mq[x & 3] = fmaxf(mq[x & 3], fmaxf(__uint_as_float(sv[0][x]), __uint_as_float(sv[1][x])));
      float mx = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
      s.red_max[e][hf][r] = mx;
      epi_sync();
      mx = fmaxf(mx, s.red_max[e][hf ^ 1][r]);
      const float mxl = mx * kLog2e;
      float sum = 0.f;
      uint8_t* prow = s.qkv[e][hf] + r * 128;  // P keys [64 hf, +64) over the Q (hf 0) / K tile
      const uint64_t l2e2 = sm100::f2_pack(kLog2e, kLog2e), negm2 = sm100::f2_pack(-mxl, -mxl);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        __align__(16) __nv_bfloat162 pv[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const uint32_t* src = &sv[q >> 2][(q & 3) * 8 + 2 * x];
          const uint64_t xx = sm100::f2_fma(
              sm100::f2_pack(__uint_as_float(src[0]), __uint_as_float(src[1])), l2e2, negm2);
          float x0, x1;
          sm100::f2_unpack(xx, x0, x1);
          pv[x] = __floats2bfloat162_rn(sm100::ex2_approx(x0), sm100::ex2_approx(x1));
          const float2 back = __bfloat1622float2(pv[x]);
          sum += back.x + back.y;
        }
        *reinterpret_cast<uint4*>(prow + ((q ^ (r & 7)) << 4)) = *reinterpret_cast<uint4*>(pv);
      }
      s.red_sum[e][hf][r] = sum;
      sm100::tc_fence_before();
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive(&s.p_ready[e]);
      if (tl) stamp(dbg, ctx, it, 3);
      // (3) O / rowsum -> ctx, this thread's 32 of the head's 64 features
      sm100::mbar_wait(&s.o_full[e], par);
      sm100::tc_fence_after();
      if (tl) stamp(dbg, ctx, it, 4);
      uint32_t ov[32];
      sm100::tmem_ld_32x32b_x32(lane_base + kOCol + hf * 32, ov);
      sm100::tmem_ld_wait();
      // buffer e (accumulator, S, O) no longer needed by this warp: the
      // projection of item it + 2 may start once both CTAs' warps are here
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive_remote(sm100::mapa(sm100::smem_u32(&s.buf_free[e]), 0));
      epi_sync();
      const float inv = 1.0f / (sum + s.red_sum[e][hf ^ 1][r]);
      if (tl) stamp(dbg, ctx, it, 5);
      if (seq < n_seq && !dbg) {  // the last sequence pair may be padded
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
    }
  }
  sm100::tc_fence_before();
  // no CTA may leave while its peer can still write into it or arrive on its barriers
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

template <bool FOLD>
static chm_status launch(const void* x, const void* w_qkv, const float* b_qkv,
                         const float* c_qkv, const float2* stats_in, int n_part, float eps,
                         void* ctx, int n_seq, int hidden, cudaStream_t st,
                         const int32_t* n_live) {
  const int n_heads = hidden / 64;
  const long long T = (long long)n_seq * kS;
  CUtensorMap tm_x, tm_w;
  if (!gemm::make_tmap_bf16(&tm_x, x, (uint64_t)T, (uint64_t)hidden, kS, 64, 0)) return CHM_ERR_CUDA;
  if (!gemm::make_tmap_qkv3(&tm_w, w_qkv, (uint64_t)hidden, 32)) return CHM_ERR_CUDA;
  auto kern = qkv_attention_duo_kernel<FOLD>;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_clusters[2] = {0, 0};
  int& mc = max_clusters[FOLD ? 1 : 0];
  if (!mc) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBytes);
    cfg.gridDim = dim3(2 * (n_sms() / 2), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) n = n_sms() / 2;
    mc = n;
  }
  const int citems = ((n_seq + 1) / 2) * n_heads;
  const int n_cl = citems < mc ? citems : mc;
  static const int dbg = getenv("CHM_QA_DUO_TL") ? atoi(getenv("CHM_QA_DUO_TL")) : 0;
  cfg.gridDim = dim3(2 * n_cl, 1, 1);
  prof::begin(prof::K_QKV_ATTENTION, st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm_x, tm_w, b_qkv, c_qkv, stats_in, n_part, eps,
                                     n_seq, n_heads, hidden,
                                     reinterpret_cast<__nv_bfloat16*>(ctx), n_live, dbg);
  prof::end(prof::K_QKV_ATTENTION, st,
            2.0 * T * 3.0 * hidden * hidden + 4.0 * kS * kS * 64.0 * n_seq * n_heads);
  if (e != cudaSuccess) return CHM_ERR_CUDA;
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace qa_duo

chm_status qkv_attention_duo(const void* x, const void* w_qkv, const float* b_qkv,
                             const float* c_qkv, const float2* stats_in, int n_part, float eps,
                             void* ctx, int n_seq, int hidden, cudaStream_t st,
                             const int32_t* n_live) {
  return stats_in ? qa_duo::launch<true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx,
                                         n_seq, hidden, st, n_live)
                  : qa_duo::launch<false>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx,
                                          n_seq, hidden, st, n_live);
}

}  // namespace chm
