// K3' -- the router's last layer for the [CLS] query by associativity.
//
// After the last layer only h_[CLS] reaches the router head, so per
// (sequence, head) the attention has ONE query q_h (64 dims). Its logits and
// output are linear in the token states x_j (post-LN, [S, H]):
//   logit_hj = q_h . (W_k,h x_j + b_k,h) / 8 = u_h . x_j + c_h,   u_h = W_k,h^T q_h / 8
//   ctx_h    = sum_j p_hj (W_v,h x_j + b_v,h) = W_v,h xbar_h + b_v,h,  xbar_h = sum_j p_hj x_j
// (c_h is constant over j and cancels in the softmax; sum_j p_hj = 1). So the
// [T, 2H] K|V projection of every token (2 T H^2 MACs) becomes
//   U = Q_cls . Wk_bd^T      [n_seq, NH*H]   (block-diagonal weights, a GEMM)
//   xbar = pool(x, U)        [n_seq, NH*H]   (this kernel: one pass pair over x)
//   ctx_cls = xbar . Wv_bd^T + b_v [n_seq, H] (a GEMM)
// with Wk_bd[h H + c][k] = Wk[k][c] / 8 for k in head h's 64 rows (else 0) and
// Wv_bd[h 64 + d][h' H + c] = Wv[h 64 + d][c] for h' = h (else 0).
//
// cls_pool_kernel, persistent, sequences in turn per CTA, pass 1 of sequence
// i + 1 issued before pass 2 of i (the tensor pipe works while the softmax of
// i runs; 0.30 -> 0.25 ms at cfg3):
//   warp 0      TMA: U_seq (16 x H, K-major), then x_seq twice as 128-token x
//               128-feature slots (two 64-feature SW128 boxes), 4-slot ring
//   warp 1      MMA issuer:
//                 pass 1  L_t [128 tokens x 16 heads] = X_t . U^T   (A = x K-major)
//                 pass 2  xbar^T_f [128 features x 16 heads] += X_t^T . P_t^T
//                         (A = the same slot read MN-major: features contiguous)
//   warps 2-5   softmax over the S tokens of every head column (cross-lane
//               max / sum through shared memory), P_t^T to shared memory in
//               bf16, then the xbar^T epilogue to global (bf16)
// TMEM: L_t at 16 t (t < S / 128 <= 4), xbar^T_f at 64 + 16 f (f < H / 128 <= 8).
// Algorithmic bytes: 2 S H reads of x per sequence (pass 2 mostly from L2).
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "gemm.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace gemm {
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, uint64_t ld);
}
namespace clsp {

constexpr int kStages = 4;
constexpr int kThreads = 192;
constexpr int kMaxBoxes = 16;  // H <= 1024
constexpr uint32_t kBox = 128 * 128;  // 128 rows x 64 bf16

struct __align__(1024) Smem {
  uint8_t ring[kStages][2][kBox];      // [slot][feature half] x [128 tokens][64 features]
  uint8_t u[kMaxBoxes][16 * 128];      // U_seq [16 heads][64 features] per box
  uint8_t p[4][2][16 * 128];           // P_t^T [16 heads][64 tokens] per (tile, half)
  float red[2][4][16];                 // [max | sum][warp][head]
  uint64_t full[kStages], empty[kStages];
  uint64_t u_full, u_empty, l_full, l_free, p_full, x_full, x_free;
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;

// UMMA descriptor for an MN-major SW128 operand: 64-element atoms along M/N
// (128 B rows), 8-row groups along K at 1024 B (SBO), atoms along M/N at LBO.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t smem_addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr & 0x3FFFFu) >> 4);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__global__ void __launch_bounds__(kThreads, 1)
    cls_pool_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_u,
                    int n_seq, int S, int H, int NH, const int32_t* __restrict__ n_live,
                    __nv_bfloat16* __restrict__ xbar) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = sm100::align_smem_1024<Smem>(smem_raw);
  const int warp = sm100::warp_id(), lane = threadIdx.x & 31;
  const int TT = S / 128, KB = H / 64, FT = H / 128;
  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_x);
    sm100::tma_prefetch(&tm_u);
    for (int i = 0; i < kStages; ++i) {
      sm100::mbar_init(&s.full[i], 1);
      sm100::mbar_init(&s.empty[i], 1);
    }
    sm100::mbar_init(&s.u_full, 1);
    sm100::mbar_init(&s.u_empty, 1);
    sm100::mbar_init(&s.l_full, 1);
    sm100::mbar_init(&s.l_free, 128);
    sm100::mbar_init(&s.p_full, 128);
    sm100::mbar_init(&s.x_full, 1);
    sm100::mbar_init(&s.x_free, 128);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc<256>(&s.tmem_base);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = sm100::uniform(s.tmem_base);
  const int n = n_live ? min(n_seq, *n_live) : n_seq;
  const int n_my = (int)blockIdx.x < n ? (n - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

  if (warp == 0) {
    if (lane == 0) {
      int slot = 0;
      uint32_t ph = 0;
      auto load_u = [&](int it) {
        const int seq = (int)blockIdx.x + it * (int)gridDim.x;
        sm100::mbar_wait(&s.u_empty, (it & 1) ^ 1);
        sm100::mbar_arrive_expect_tx(&s.u_full, (uint32_t)KB * 16 * 128);
        for (int kb = 0; kb < KB; ++kb)
          sm100::tma_load_2d(s.u[kb], &tm_u, &s.u_full, kb * 64, seq * NH);
      };
      auto load_x = [&](int it) {  // one pass over x_seq in (t, f) slot order
        const int seq = (int)blockIdx.x + it * (int)gridDim.x;
        for (int t = 0; t < TT; ++t)
          for (int f = 0; f < FT; ++f) {
            sm100::mbar_wait(&s.empty[slot], ph ^ 1);
            sm100::mbar_arrive_expect_tx(&s.full[slot], 2 * kBox);
            sm100::tma_load_2d(s.ring[slot][0], &tm_x, &s.full[slot], 128 * f, seq * S + 128 * t);
            sm100::tma_load_2d(s.ring[slot][1], &tm_x, &s.full[slot], 128 * f + 64,
                               seq * S + 128 * t);
            if (++slot == kStages) { slot = 0; ph ^= 1; }
          }
      };
      // pass 1 of sequence it + 1 is loaded (and issued) before pass 2 of it,
      // so the tensor pipe has work while the softmax of it runs
      if (n_my > 0) { load_u(0); load_x(0); }
      for (int it = 0; it < n_my; ++it) {
        if (it + 1 < n_my) { load_u(it + 1); load_x(it + 1); }
        load_x(it);
      }
    }
  } else if (warp == 1) {
    // MMA issuer (warp-uniform)
    constexpr uint32_t idesc1 = sm100::umma_idesc_bf16(128, 16);
    constexpr uint32_t idesc2 = sm100::umma_idesc_bf16(128, 16) | (1u << 15);  // A MN-major
    int slot = 0;
    uint32_t ph = 0;
    auto pass1 = [&](int it) {
      sm100::mbar_wait(&s.u_full, it & 1);
      if (it > 0) sm100::mbar_wait(&s.l_free, (it - 1) & 1);  // softmax read L of it - 1
      sm100::tc_fence_after();
      for (int t = 0; t < TT; ++t)
        for (int f = 0; f < FT; ++f) {
          sm100::mbar_wait(&s.full[slot], ph);
          sm100::tc_fence_after();
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const uint32_t xa = sm100::smem_u32(s.ring[slot][b]);
            const uint32_t ua = sm100::smem_u32(s.u[2 * f + b]);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              sm100::mma_bf16_w(tmem + 16 * t, sm100::umma_desc_sw128(xa + k * 32),
                                sm100::umma_desc_sw128(ua + k * 32), idesc1, (f | b | k) != 0);
          }
          sm100::mma_commit_w(&s.empty[slot]);
          if (++slot == kStages) { slot = 0; ph ^= 1; }
        }
      sm100::mma_commit_w(&s.l_full);
      sm100::mma_commit_w(&s.u_empty);
    };
    auto pass2 = [&](int it) {
      sm100::mbar_wait(&s.p_full, it & 1);
      if (it > 0) sm100::mbar_wait(&s.x_free, (it - 1) & 1);  // epilogue read xbar of it - 1
      sm100::tc_fence_after();
      for (int t = 0; t < TT; ++t)
        for (int f = 0; f < FT; ++f) {
          sm100::mbar_wait(&s.full[slot], ph);
          sm100::tc_fence_after();
          const uint32_t xa = sm100::smem_u32(s.ring[slot][0]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {  // 16 tokens per step
            const uint32_t pa = sm100::smem_u32(s.p[t][kk >> 2]) + (kk & 3) * 32;
            sm100::mma_bf16_w(tmem + 64 + 16 * f, desc_mn_sw128(xa + kk * 2048, kBox),
                              sm100::umma_desc_sw128(pa), idesc2, (t | kk) != 0);
          }
          sm100::mma_commit_w(&s.empty[slot]);
          if (++slot == kStages) { slot = 0; ph ^= 1; }
        }
      sm100::mma_commit_w(&s.x_full);
    };
    if (n_my > 0) pass1(0);
    for (int it = 0; it < n_my; ++it) {
      if (it + 1 < n_my) pass1(it + 1);
      pass2(it);
    }
    __syncwarp();
  } else {
    // softmax + epilogue; thread = TMEM lane (token row in pass 1, feature row in pass 2)
    const int quarter = warp & 3, wi = warp - 2;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    constexpr float kLog2e = 1.4426950408889634f;
    for (int it = 0; it < n_my; ++it) {
      const int seq = (int)blockIdx.x + it * (int)gridDim.x;
      sm100::mbar_wait(&s.l_full, it & 1);
      sm100::tc_fence_after();
      uint32_t lv[2][32];
      sm100::tmem_ld_32x32b_x32(lane_base, lv[0]);
      if (TT > 2) sm100::tmem_ld_32x32b_x32(lane_base + 32, lv[1]);
      sm100::tmem_ld_wait();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&s.l_free);
      // per head: max over the S tokens (this thread's TT values, then lanes, then warps)
      float m[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        float v = __uint_as_float(lv[0][h]);
#pragma unroll
        for (int t = 1; t < 4; ++t)
          if (t < TT) v = fmaxf(v, __uint_as_float(lv[t >> 1][16 * (t & 1) + h]));
#pragma unroll
        for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        m[h] = v;
      }
      if (lane < 16) {
        float mine = m[0];
#pragma unroll
        for (int h = 1; h < 16; ++h) mine = lane == h ? m[h] : mine;
        s.red[0][wi][lane] = mine;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
#pragma unroll
      for (int h = 0; h < 16; ++h)
        m[h] = fmaxf(fmaxf(s.red[0][0][h], s.red[0][1][h]), fmaxf(s.red[0][2][h], s.red[0][3][h])) *
               kLog2e;
      float l[16];
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        float sum = 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (t < TT) {
            uint32_t& e = lv[t >> 1][16 * (t & 1) + h];
            const float p = sm100::ex2_approx(fmaf(__uint_as_float(e), kLog2e, -m[h]));
            e = __float_as_uint(p);
            sum += p;
          }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        l[h] = sum;
      }
      if (lane < 16) {
        float mine = l[0];
#pragma unroll
        for (int h = 1; h < 16; ++h) mine = lane == h ? l[h] : mine;
        s.red[1][wi][lane] = mine;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      // P_t^T [head][token] in bf16, normalised; heads >= NH are 0 (U's pad rows)
#pragma unroll
      for (int h = 0; h < 16; ++h) {
        const float inv =
            h < NH ? 1.0f / ((s.red[1][0][h] + s.red[1][1][h]) + (s.red[1][2][h] + s.red[1][3][h]))
                   : 0.f;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (t < TT) {
            const float p = __uint_as_float(lv[t >> 1][16 * (t & 1) + h]) * inv;
            const int half = r >> 6, c = r & 63;
            uint8_t* row = s.p[t][half] + h * 128;
            const int chunk = (c >> 3) ^ (h & 7);
            *reinterpret_cast<__nv_bfloat16*>(row + (chunk << 4) + (c & 7) * 2) =
                __float2bfloat16_rn(p);
          }
      }
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive(&s.p_full);
      // xbar^T_f -> xbar[seq * NH + h][128 f + r]
      sm100::mbar_wait(&s.x_full, it & 1);
      sm100::tc_fence_after();
      for (int f = 0; f < FT; f += 2) {
        uint32_t xv[32];
        sm100::tmem_ld_32x32b_x32(lane_base + 64 + 16 * f, xv);
        sm100::tmem_ld_wait();
#pragma unroll
        for (int ff = 0; ff < 2; ++ff)
#pragma unroll
          for (int h = 0; h < 16; ++h)
            if (h < NH)
              xbar[((size_t)seq * NH + h) * H + 128 * (f + ff) + r] =
                  __float2bfloat16_rn(__uint_as_float(xv[16 * ff + h]));
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(&s.x_free);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<256>(tmem);
  }
}

// Block-diagonal weights of the associative form (see the header).
__global__ void build_bd_kernel(const __nv_bfloat16* __restrict__ wqkv, int H, int NH,
                                __nv_bfloat16* __restrict__ wk_bd, __nv_bfloat16* __restrict__ wv_bd) {
  const __nv_bfloat16* wk = wqkv + (size_t)H * H;
  const __nv_bfloat16* wv = wqkv + (size_t)2 * H * H;
  const size_t total = (size_t)NH * H * H;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    // wk_bd [NH H][H]: row (h, c), column k
    {
      const size_t row = i / H, k = i - row * H;
      const int h = (int)(row / H), c = (int)(row - (size_t)h * H);
      wk_bd[i] = ((int)k >> 6) == h
                     ? __float2bfloat16_rn(__bfloat162float(wk[k * H + c]) * 0.125f)
                     : __float2bfloat16_rn(0.f);
    }
    // wv_bd [H][NH H]: row (h 64 + d), column (h', c)
    {
      const size_t row = i / ((size_t)NH * H), col = i - row * ((size_t)NH * H);
      const int h = (int)row >> 6, hp = (int)(col / H), c = (int)(col - (size_t)hp * H);
      wv_bd[i] = hp == h ? wv[row * H + c] : __float2bfloat16_rn(0.f);
    }
  }
}

}  // namespace clsp

chm_status cls_pool_build_bd(const void* wqkv, int H, void* wk_bd, void* wv_bd, cudaStream_t st) {
  const int NH = H / 64;
  const size_t total = (size_t)NH * H * H;
  const unsigned grid = (unsigned)((total + 255) / 256 < 4096 ? (total + 255) / 256 : 4096);
  clsp::build_bd_kernel<<<grid, 256, 0, st>>>(reinterpret_cast<const __nv_bfloat16*>(wqkv), H,
                                              NH, reinterpret_cast<__nv_bfloat16*>(wk_bd),
                                              reinterpret_cast<__nv_bfloat16*>(wv_bd));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

chm_status cls_pool(const void* x, const void* u, void* xbar, int n_seq, int S, int H,
                    const int32_t* n_live, cudaStream_t st) {
  const int NH = H / 64;
  if (S % 128 || S > 512 || H % 256 || H > 1024 || NH > 16) return CHM_ERR_UNSUPPORTED;
  CUtensorMap tm_x, tm_u;
  if (!gemm::make_tmap_bf16(&tm_x, x, (uint64_t)n_seq * S, (uint64_t)H, 128, 64, 0) ||
      !gemm::make_tmap_bf16(&tm_u, u, (uint64_t)n_seq * NH, (uint64_t)H, 16, 64, 0))
    return CHM_ERR_CUDA;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(clsp::cls_pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)clsp::kSmemBytes);
    attr = true;
  }
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = (unsigned)(n_seq < sms ? n_seq : sms);
  prof::begin(prof::K_ATTENTION, st);
  clsp::cls_pool_kernel<<<grid, clsp::kThreads, clsp::kSmemBytes, st>>>(
      tm_x, tm_u, n_seq, S, H, NH, n_live, reinterpret_cast<__nv_bfloat16*>(xbar));
  prof::end(prof::K_ATTENTION, st, 4.0 * S * H * NH * n_seq);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace chm
