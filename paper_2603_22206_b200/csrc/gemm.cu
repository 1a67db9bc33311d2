// K2 -- tcgen05 / TMEM / TMA GEMM for the router encoder.
//
//   C[M, N] = A[M, K] . B[N, K]^T  (+ bias[N]) (GELU) (+ residual[M, N])
//   A: activations, B: nn.Linear weight [out, in]; both K-major bf16,
//   fp32 accumulation in tensor memory, bf16 output.
//
// Structure (one persistent CTA per SM, 384 threads):
//   warp 0      TMA producer: A 128x64 and B 256x64 tiles (128B swizzle) into a
//               4-stage shared-memory ring, completion via mbarrier tx-count
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma 128x256x16
//               (4 per 64-wide k-block) into a double-buffered TMEM accumulator
//               (2 x 256 fp32 columns = all 512 columns), tcgen05.commit frees
//               the smem stage / publishes the accumulator
//   warp 2      TMEM allocator
//   warps 4-11  epilogue: tcgen05.ld 32 lanes x 32 columns, bias / erf-GELU /
//               residual in fp32, bf16 stores; two warps per TMEM lane quarter
//               split the 256 columns
// Tiles are scheduled row-block-major (all N tiles of a 128-row block on
// consecutive CTAs) so the A block is read from HBM once and the weight
// matrix stays L2 resident.
//
// FLOPs per launch: 2*M*N*K (algorithmic; reported against the measured bf16
// peak in bench.py).
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "sm100.cuh"
#include "prof.cuh"

namespace chm {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64;
constexpr int kStages = 4;
constexpr int kThreads = 384;
constexpr int kEpiWarps = 8;
constexpr uint32_t kTileABytes = BM * BK * 2;  // 16 KB
constexpr uint32_t kTileBBytes = BN * BK * 2;  // 32 KB
constexpr uint32_t kStageBytes = kTileABytes + kTileBBytes;

enum Epilogue : int {
  EPI_NONE = 0,
  EPI_BIAS = 1,
  EPI_BIAS_GELU = 2,
  EPI_BIAS_RESIDUAL = 3,
  // QKV projection: columns [0, H) are Q (pre-scaled by 1/sqrt(64), exact in
  // bf16), [H, 2H) are K -> written to C with row stride 2H; columns [2H, 3H)
  // are V, written transposed per (sequence, head) as vt[seq][head][d][s] so
  // the attention kernel's P.V MMA reads V^T K-major. A 32-lane TMEM quarter
  // holds 32 consecutive tokens of one sequence, so each transposed store is
  // one coalesced 64-byte segment.
  EPI_QKV = 4,
};

struct QkvParams {
  __nv_bfloat16* vt;  // [n_seq, n_heads, 64, seq_len]
  int hidden;         // H
  int seq_len;        // S (multiple of 128)
};

struct Smem {
  uint8_t tiles[kStages][kStageBytes];  // each stage: A (16 KB) then B (32 KB)
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;  // + alignment slack

__device__ __forceinline__ float gelu_erf(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                const __grid_constant__ CUtensorMap tmap_b, __nv_bfloat16* __restrict__ C,
                const float* __restrict__ bias, const __nv_bfloat16* __restrict__ residual,
                int M, int N, int K, QkvParams qkv) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                     ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_n = (N + BN - 1) / BN;
  const int n_tiles = ((M + BM - 1) / BM) * n_tiles_n;
  const int k_blocks = K / BK;

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tmap_a);
    sm100::tma_prefetch(&tmap_b);
    for (int i = 0; i < kStages; ++i) {
      sm100::mbar_init(&s.full[i], 1);
      sm100::mbar_init(&s.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s.tmem_full[i], 1);
      sm100::mbar_init(&s.tmem_empty[i], kEpiWarps);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc<512>(&s.tmem_base);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = s.tmem_base;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int m0 = (t / n_tiles_n) * BM, n0 = (t % n_tiles_n) * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&s.empty[stage], phase ^ 1);
          uint8_t* base = s.tiles[stage];
          sm100::mbar_arrive_expect_tx(&s.full[stage], kStageBytes);
          sm100::tma_load_2d(base, &tmap_a, &s.full[stage], kb * BK, m0);
          sm100::tma_load_2d(base + kTileABytes, &tmap_b, &s.full[stage], kb * BK, n0);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = sm100::umma_idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
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
            // advance 16 bf16 (32 B) inside the 128 B swizzle row
            const uint64_t ad = sm100::umma_desc_sw128(a_addr + k * 32);
            const uint64_t bd = sm100::umma_desc_sw128(b_addr + k * 32);
            sm100::mma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          sm100::mma_commit(&s.empty[stage]);
          if (kb == k_blocks - 1) sm100::mma_commit(&s.tmem_full[acc]);
        }
        __syncwarp();
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int ew = warp - 4;            // 0..7
    const int quarter = warp & 3;       // TMEM lane quarter this warp may access
    const int col_half = ew >> 2;       // which 128 of the 256 columns
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int m0 = (t / n_tiles_n) * BM, n0 = (t % n_tiles_n) * BN;
      sm100::mbar_wait(&s.tmem_full[acc], acc_phase);
      sm100::tc_fence_after();
      const int row = m0 + quarter * 32 + lane;
#pragma unroll 1
      for (int cc = 0; cc < 4; ++cc) {
        const int c0 = col_half * 128 + cc * 32;
        uint32_t r[32];
        sm100::tmem_ld_32x32b_x32(
            tmem_base + ((uint32_t)(quarter * 32) << 16) + acc * BN + c0, r);
        sm100::tmem_ld_wait();
        const int n = n0 + c0;
        if (row < M && n < N) {
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
          if (EPI != EPI_NONE) {
            const float4* b4 = reinterpret_cast<const float4*>(bias + n);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 bb = __ldg(b4 + j);
              v[4 * j] += bb.x; v[4 * j + 1] += bb.y; v[4 * j + 2] += bb.z; v[4 * j + 3] += bb.w;
            }
          }
          if (EPI == EPI_BIAS_GELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
          }
          if (EPI == EPI_BIAS_RESIDUAL) {
            const uint4* rp = reinterpret_cast<const uint4*>(residual + (size_t)row * N + n);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              uint4 u = __ldg(rp + j);
              const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                float2 f = __bfloat1622float2(h[e]);
                v[8 * j + 2 * e] += f.x;
                v[8 * j + 2 * e + 1] += f.y;
              }
            }
          }
          int ldc = N;
          if (EPI == EPI_QKV) {
            ldc = 2 * qkv.hidden;
            if (n >= ldc) {
              const int hn = n - ldc, h = hn >> 6, d0 = hn & 63;
              const int seq = row / qkv.seq_len, sp = row - seq * qkv.seq_len;
              __nv_bfloat16* vp =
                  qkv.vt + ((size_t)(seq * (qkv.hidden >> 6) + h) * 64 + d0) * qkv.seq_len + sp;
#pragma unroll
              for (int j = 0; j < 32; ++j) vp[(size_t)j * qkv.seq_len] = __float2bfloat16_rn(v[j]);
              continue;
            }
            if (n < qkv.hidden) {
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] *= 0.125f;
            }
          }
          uint4* cp = reinterpret_cast<uint4*>(C + (size_t)row * ldc + n);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 o;
            o.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
            o.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
            o.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
            o.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
            cp[j] = o;
          }
        }
      }
      sm100::tc_fence_before();
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&s.tmem_empty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<512>(tmem_base);
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

// Row-major bf16 matrix [rows, cols] as a 2D tensor map with a
// (box_cols x box_rows) box and 128-byte swizzle.
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * 2};
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
  CUtensorMap ta, tb;
  if (!make_tmap_bf16(&ta, A, (uint64_t)M, (uint64_t)K, BM, BK)) return CHM_ERR_CUDA;
  if (!make_tmap_bf16(&tb, B, (uint64_t)N, (uint64_t)K, BN, BK)) return CHM_ERR_CUDA;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_kernel<EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSmemBytes);
    attr_set = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  prof::begin(prof::K_GEMM, s);
  gemm_kernel<EPI><<<grid, kThreads, kSmemBytes, s>>>(
      ta, tb, reinterpret_cast<__nv_bfloat16*>(C), bias,
      reinterpret_cast<const __nv_bfloat16*>(residual), M, N, K, qkv);
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
  if (K % gemm::BK != 0 || N % 32 != 0) return CHM_ERR_INVALID_ARG;
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
