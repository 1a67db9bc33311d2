// K2 -- tcgen05 / TMEM / TMA GEMM for the router encoder.
//
//   C[M, N] = A[M, K] . B[N, K]^T  (+ bias[N]) (GELU) (+ residual[M, N])
//   A: activations, B: nn.Linear weight [out, in]; both K-major bf16,
//   fp32 accumulation in tensor memory, bf16 output.
//
// Structure: persistent CTA PAIRS (cluster 2x1, one CTA per SM, 384 threads).
// A cluster owns a 256 x 256 output tile; CTA r of the pair stages rows
// [128r, 128r+128) of the A tile and rows [128r, 128r+128) of the B tile
// (N half), so the pair MMA (tcgen05.mma.cta_group::2, M=256 N=256 K=16)
// reads half of each operand from each SM's shared memory.
//   warp 0      TMA producer (both CTAs): 4-stage ring of A 128x64 + B 128x64
//               tiles (128B swizzle); completion counted on the leader's
//               mbarrier (cta_group::2 TMA)
//   warp 1      TMEM (512 cols, cta_group::2) alloc/dealloc in both CTAs; in
//               the leader one elected thread issues the MMAs into a
//               double-buffered accumulator; tcgen05.commit multicasts
//               "stage free" / "accumulator full" to both CTAs
//   warps 4-11  epilogue (both CTAs): tcgen05.ld 32 lanes x 64 columns, bias
//               / tanh-GELU / residual / QKV split in fp32, bf16 into a
//               128B-swizzled smem box, TMA store (bulk group); residual
//               boxes arrive by TMA into the same staging buffers. Two
//               buffers per warp overlap the store of one chunk with the next.
// Tiles go row-block-major over clusters so the A block is read from HBM once
// and the weights stay L2 resident.
//
// FLOPs per launch: 2*M*N*K.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace gemm {

constexpr int BM = 256, BN = 256, BK = 64;  // cluster tile
constexpr int CM = 128, CN = 128;           // per-CTA operand rows (A half, B half)
constexpr int kStages = 4;
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr uint32_t kTileABytes = CM * BK * 2;  // 16 KB
constexpr uint32_t kTileBBytes = CN * BK * 2;  // 16 KB
constexpr uint32_t kStageBytes = kTileABytes + kTileBBytes;
constexpr uint32_t kBoxBytes = 32 * 128;       // 32 rows x 64 bf16, one epilogue box

enum Epilogue : int {
  EPI_NONE = 0,
  EPI_BIAS = 1,
  EPI_BIAS_GELU = 2,
  EPI_BIAS_RESIDUAL = 3,
  // QKV projection: columns [0, H) are Q (pre-scaled by 1/sqrt(64), exact in
  // bf16), [H, 2H) are K -> C with row stride 2H; columns [2H, 3H) are V,
  // written transposed per (sequence, head) as vt[seq][head][d][s] so the
  // attention kernel's P.V MMA reads V^T K-major. A 32-lane TMEM quarter holds
  // 32 consecutive tokens of one sequence, so each transposed store is one
  // coalesced 64-byte segment.
  EPI_QKV = 4,
};

struct QkvParams {
  __nv_bfloat16* vt;  // [n_seq, n_heads, 64, seq_len]
  int hidden;         // H
  int seq_len;        // S (multiple of 128)
};

struct __align__(1024) Smem {
  uint8_t tiles[kStages][kStageBytes];          // A (16 KB) then B (16 KB) per stage
  uint8_t stage_out[kEpiWarps][2][kBoxBytes];   // epilogue boxes (SW128)
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t res_bar[kEpiWarps][2];
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;  // + alignment slack

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

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                const __grid_constant__ CUtensorMap tmap_b,
                const __grid_constant__ CUtensorMap tmap_c,
                const __grid_constant__ CUtensorMap tmap_r, const float* __restrict__ bias,
                int M, int N, int K, QkvParams qkv) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                     ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = sm100::cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = (int)sm100::cluster_id_x();
  const int n_cl = (int)sm100::n_clusters_x();
  const int n_tiles_n = (N + BN - 1) / BN;
  const int n_tiles = ((M + BM - 1) / BM) * n_tiles_n;
  const int k_blocks = K / BK;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmap_a);
    sm100::tma_prefetch(&tmap_b);
    sm100::tma_prefetch(&tmap_c);
    if (EPI == EPI_BIAS_RESIDUAL) sm100::tma_prefetch(&tmap_r);
    for (int i = 0; i < kStages; ++i) {
      sm100::mbar_init(&s.full[i], 1);
      sm100::mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s.tmem_full[i], 1);
      sm100::mbar_init(&s.tmem_empty[i], 2 * kEpiWarps);  // epilogues of both CTAs
    }
    for (int w = 0; w < kEpiWarps; ++w)
      for (int b = 0; b < 2; ++b) sm100::mbar_init(&s.res_bar[w][b], 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc_cg2<512>(&s.tmem_base);
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem_base = s.tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cluster; t < n_tiles; t += n_cl) {
        const int m0 = (t / n_tiles_n) * BM + (int)rank * CM;
        const int n0 = (t % n_tiles_n) * BN + (int)rank * CN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&s.empty[stage], phase ^ 1);
          const uint32_t full_leader = sm100::mapa(sm100::smem_u32(&s.full[stage]), 0);
          if (leader) sm100::mbar_arrive_expect_tx(&s.full[stage], 2 * kStageBytes);
          uint8_t* base = s.tiles[stage];
          sm100::tma_load_2d_cg2(base, &tmap_a, full_leader, kb * BK, m0);
          sm100::tma_load_2d_cg2(base + kTileABytes, &tmap_b, full_leader, kb * BK, n0);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
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
          if (lane == 0) {
            const uint32_t a_addr = sm100::smem_u32(s.tiles[stage]);
            const uint32_t b_addr = a_addr + kTileABytes;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = sm100::umma_desc_sw128(a_addr + k * 32);
              const uint64_t bd = sm100::umma_desc_sw128(b_addr + k * 32);
              sm100::mma_bf16_cg2(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
            sm100::mma_commit_cg2_mc(&s.empty[stage], 0x3);
            if (kb == k_blocks - 1) sm100::mma_commit_cg2_mc(&s.tmem_full[acc], 0x3);
          }
          __syncwarp();
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
    const uint32_t empty_leader0 = sm100::mapa(sm100::smem_u32(&s.tmem_empty[0]), 0);
    const uint32_t empty_leader1 = sm100::mapa(sm100::smem_u32(&s.tmem_empty[1]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t res_phase = 0;  // bit b = phase of res_bar[ew][b]
    int box = 0;             // alternates the two staging boxes
    for (int t = cluster; t < n_tiles; t += n_cl) {
      const int mrow0 = (t / n_tiles_n) * BM + (int)rank * CM + quarter * 32;
      const int n_tile0 = (t % n_tiles_n) * BN + half * 128;
      sm100::mbar_wait(&s.tmem_full[acc], acc_phase);
      sm100::tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 2; ++c) {
        const int col0 = n_tile0 + c * 64;
        uint8_t* sb = s.stage_out[ew][box];
        // the box is free once the TMA store issued from it two chunks ago has
        // finished reading shared memory
        if (lane == 0) sm100::bulk_wait_read<1>();
        __syncwarp();
        if (EPI == EPI_BIAS_RESIDUAL && lane == 0 && col0 < N) {
          sm100::mbar_arrive_expect_tx(&s.res_bar[ew][box], kBoxBytes);
          sm100::tma_load_2d(sb, &tmap_r, &s.res_bar[ew][box], col0, mrow0);
        }
        uint32_t r0[32], r1[32];
        const uint32_t taddr =
            tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + half * 128 + c * 64;
        sm100::tmem_ld_32x32b_x32(taddr, r0);
        sm100::tmem_ld_32x32b_x32(taddr + 32, r1);
        sm100::tmem_ld_wait();
        if (c == 1) {
          // accumulator fully read: hand it back to the leader's MMA warp
          sm100::tc_fence_before();
          __syncwarp();
          if (lane == 0) sm100::mbar_arrive_cluster(acc ? empty_leader1 : empty_leader0);
        }
        if (col0 >= N) continue;
        if (EPI == EPI_BIAS_RESIDUAL) {
          sm100::mbar_wait(&s.res_bar[ew][box], (res_phase >> box) & 1);
          res_phase ^= 1u << box;
        }
        const int row = mrow0 + lane;
        if (EPI == EPI_QKV && col0 >= 2 * qkv.hidden) {
          // V: transposed direct stores, one coalesced 64 B segment per column
          if (row < M) {
            const int hn = col0 - 2 * qkv.hidden, h = hn >> 6;
            const int seq = row / qkv.seq_len, sp = row - seq * qkv.seq_len;
            __nv_bfloat16* vp =
                qkv.vt + ((size_t)(seq * (qkv.hidden >> 6) + h) * 64) * qkv.seq_len + sp;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              vp[(size_t)j * qkv.seq_len] =
                  __float2bfloat16_rn(__uint_as_float(r0[j]) + __ldg(bias + col0 + j));
              vp[(size_t)(j + 32) * qkv.seq_len] =
                  __float2bfloat16_rn(__uint_as_float(r1[j]) + __ldg(bias + col0 + 32 + j));
            }
          }
          continue;
        }
        const float qscale = (EPI == EPI_QKV && col0 < qkv.hidden) ? 0.125f : 1.0f;
        uint8_t* rowp = sb + lane * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            v[e] = __uint_as_float(j < 4 ? r0[j * 8 + e] : r1[(j - 4) * 8 + e]);
          if (EPI != EPI_NONE) {
            const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + col0 + j * 8));
            const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + col0 + j * 8 + 4));
            v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
            v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
          }
          uint4* slot = reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4));
          if (EPI == EPI_BIAS_RESIDUAL) {
            const uint4 u = *slot;
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(h[e]);
              v[2 * e] += f.x;
              v[2 * e + 1] += f.y;
            }
          }
          if (EPI == EPI_BIAS_GELU) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = gelu_tanh(v[e]);
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
        box ^= 1;
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

static int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <int EPI>
static chm_status launch(const void* A, const void* B, void* C, const float* bias,
                         const void* residual, int M, int N, int K, QkvParams qkv,
                         cudaStream_t s) {
  CUtensorMap ta, tb, tc, tr;
  if (!make_tmap_bf16(&ta, A, (uint64_t)M, (uint64_t)K, CM, BK, 0)) return CHM_ERR_CUDA;
  if (!make_tmap_bf16(&tb, B, (uint64_t)N, (uint64_t)K, CN, BK, 0)) return CHM_ERR_CUDA;
  const uint64_t c_cols = (EPI == EPI_QKV) ? (uint64_t)2 * qkv.hidden : (uint64_t)N;
  if (!make_tmap_bf16(&tc, C, (uint64_t)M, c_cols, 32, 64, 0)) return CHM_ERR_CUDA;
  if (EPI == EPI_BIAS_RESIDUAL) {
    if (!make_tmap_bf16(&tr, residual, (uint64_t)M, (uint64_t)N, 32, 64, 0)) return CHM_ERR_CUDA;
  } else {
    tr = tc;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemBytes);
    attr_set = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int pairs = num_sms() / 2;
  const int grid = 2 * (tiles < pairs ? tiles : pairs);
  prof::begin(prof::K_GEMM, s);
  gemm_kernel<EPI><<<grid, kThreads, kSmemBytes, s>>>(ta, tb, tc, tr, bias, M, N, K, qkv);
  prof::end(prof::K_GEMM, s, 2.0 * M * N * K);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace gemm

// Internal entry (also used by the encoder): epilogue 4 = QKV split with V^T.
chm_status gemm_bf16(const void* A, const void* B, void* C, const float* bias,
                     const void* residual, int M, int N, int K, int epilogue, cudaStream_t s,
                     void* vt, int hidden, int seq_len) {
  if (M <= 0 || N <= 0 || K <= 0) return M == 0 ? CHM_OK : CHM_ERR_INVALID_ARG;
  if (K % gemm::BK != 0 || N % 64 != 0) return CHM_ERR_INVALID_ARG;
  if (epilogue != gemm::EPI_NONE && !bias) return CHM_ERR_INVALID_ARG;
  if (epilogue == gemm::EPI_BIAS_RESIDUAL && !residual) return CHM_ERR_INVALID_ARG;
  gemm::QkvParams qkv{reinterpret_cast<__nv_bfloat16*>(vt), hidden, seq_len};
  if (epilogue == gemm::EPI_QKV &&
      (!vt || hidden % 64 != 0 || N != 3 * hidden || seq_len % 128 != 0 || M % seq_len != 0))
    return CHM_ERR_INVALID_ARG;
  switch (epilogue) {
    case gemm::EPI_NONE:
      return gemm::launch<gemm::EPI_NONE>(A, B, C, bias, residual, M, N, K, qkv, s);
    case gemm::EPI_BIAS:
      return gemm::launch<gemm::EPI_BIAS>(A, B, C, bias, residual, M, N, K, qkv, s);
    case gemm::EPI_BIAS_GELU:
      return gemm::launch<gemm::EPI_BIAS_GELU>(A, B, C, bias, residual, M, N, K, qkv, s);
    case gemm::EPI_BIAS_RESIDUAL:
      return gemm::launch<gemm::EPI_BIAS_RESIDUAL>(A, B, C, bias, residual, M, N, K, qkv, s);
    case gemm::EPI_QKV:
      return gemm::launch<gemm::EPI_QKV>(A, B, C, bias, residual, M, N, K, qkv, s);
    default: return CHM_ERR_INVALID_ARG;
  }
}

}  // namespace chm

extern "C" chm_status chm_gemm_bf16(const void* A, const void* B, void* C, const float* bias,
                                    const void* residual, int32_t M, int32_t N, int32_t K,
                                    int32_t epilogue, void* stream) {
  if (epilogue == chm::gemm::EPI_QKV) return CHM_ERR_INVALID_ARG;
  return chm::gemm_bf16(A, B, C, bias, residual, M, N, K, epilogue, (cudaStream_t)stream,
                        nullptr, 0, 0);
}
