// Microbenchmark: cycles per tcgen05.mma (kind::f16, SS operands) on one SM
// for several shapes and issue patterns, to find what paces the fused QKV +
// attention projection (profiles/r1c_gemm_cycles.md).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../include \
//        -o mma_probe mma_probe.cu && ./mma_probe
//
// One CTA (128 threads), operands are whatever shared memory holds (values do
// not matter), accumulator in TMEM; cycles from issue of the first MMA to the
// completion of the last (commit + wait). Patterns:
//   burst   n MMAs back to back, one commit at the end
//   commit  a commit (mbarrier arrive) after every 4 MMAs, no waits
//   wait4   after every 4 MMAs: commit, then wait for the commit of the group
//           issued 4 groups earlier (a 4-stage pipeline's release pacing),
//           2: mbarrier.try_wait loop, 3: mbarrier.test_wait spin
// probe_warp: the same with a warp-uniform loop (elect.sync issues).
// probe_contend: the warp-uniform loop while other warps write shared memory
// (1: cp.async.bulk global->shared ring, 2: st.shared.v4 from two warps), on
// one CTA or one CTA per SM -- does operand staging traffic slow the MMAs?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2603_22206_b200/csrc/sm100.cuh"

using namespace chm::sm100;

// Completion-timed variant: issue n MMAs then commit and wait; total cycles.
template <int M, int N>
__global__ void probe_total(int n_mma, int pattern, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bars[9];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0)
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(M, N);
    const uint32_t a = smem_u32(smem), b = a + 32768;
    uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 3;
      mma_bf16(tmem, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), idesc, i != 0);
      if (pattern >= 1 && k == 3) {
        const int g = (i >> 2) & 7;
        mma_commit(&bars[g]);
        if (pattern >= 2 && (i >> 2) >= 4) {
          const int w = ((i >> 2) - 4) & 7;
          if (pattern == 2) {
            mbar_wait(&bars[w], phase[w]);  // try_wait loop
          } else {
            while (!mbar_test(&bars[w], phase[w])) {  // test_wait spin
            }
          }
          phase[w] ^= 1;
        }
      }
    }
    mma_commit(&bars[8]);
    mbar_wait(&bars[8], 0);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}


// Whole-warp issue loop: descriptors are warp-uniform (uniform datapath), one
// elected lane issues each tcgen05 instruction. wait: as pattern 2/3 (0 = burst).
template <int M, int N>
__global__ void probe_warp(int n_mma, int wait, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bars[9];
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0)
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(M, N);
    const uint32_t a = smem_u32(smem), b = a + 32768;
    uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 3;
      if (elect_one())
        mma_bf16(tmem, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), idesc, i != 0);
      __syncwarp();
      if (k == 3) {
        const int g = (i >> 2) & 7;
        if (elect_one()) mma_commit(&bars[g]);
        __syncwarp();
        if (wait && (i >> 2) >= 4) {
          const int w = ((i >> 2) - 4) & 7;
          mbar_wait(&bars[w], phase[w]);
          phase[w] ^= 1;
        }
      }
    }
    if (elect_one()) mma_commit(&bars[8]);
    __syncwarp();
    mbar_wait(&bars[8], 0);
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

constexpr uint32_t kRing = 65536;         // write region offset
constexpr uint32_t kChunk = 16384;        // bulk copy size
constexpr int kRingSlots = 6;             // 96 KB ring

template <int M, int N>
__global__ void probe_contend(int n_mma, int mode, const uint8_t* __restrict__ src,
                              unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bars[9];
  __shared__ __align__(8) uint64_t ring_bar[kRingSlots];
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < kRingSlots; ++i) mbar_init(&ring_bar[i], 1);
    done = 0;
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  unsigned long long written = 0, w0 = 0, w1 = 0;
  if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(M, N);
    const uint32_t a = smem_u32(smem), b = a + 32768;
    uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 3;
      if (elect_one())
        mma_bf16(tmem, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), idesc, i != 0);
      __syncwarp();
      if (k == 3) {
        const int g = (i >> 2) & 7;
        if (elect_one()) mma_commit(&bars[g]);
        __syncwarp();
        if ((i >> 2) >= 4) {
          const int w = ((i >> 2) - 4) & 7;
          mbar_wait(&bars[w], phase[w]);
          phase[w] ^= 1;
        }
      }
    }
    if (elect_one()) mma_commit(&bars[8]);
    __syncwarp();
    mbar_wait(&bars[8], 0);
    unsigned long long t1 = clock64();
    if (lane == 0) {
      out[blockIdx.x * 3] = t1 - t0;
      done = 1;
    }
  } else if (warp == 0 && mode == 1) {
    uint32_t ph[kRingSlots] = {0, 0, 0, 0, 0, 0};
    w0 = clock64();
    int i = 0;
    for (; !done; ++i) {
      const int sl = i % kRingSlots;
      if (i >= kRingSlots) {
        mbar_wait(&ring_bar[sl], ph[sl]);
        ph[sl] ^= 1;
      }
      if (elect_one()) {
        mbar_arrive_expect_tx(&ring_bar[sl], kChunk);
        bulk_load_1d(smem + kRing + sl * kChunk, src + (size_t)(i & 63) * kChunk, kChunk, &ring_bar[sl]);
      }
      __syncwarp();
    }
    for (int j = (i > kRingSlots ? i - kRingSlots : 0); j < i; ++j) {
      const int sl = j % kRingSlots;
      mbar_wait(&ring_bar[sl], ph[sl]);
      ph[sl] ^= 1;
    }
    w1 = clock64();
    written = (unsigned long long)i * kChunk;
  } else if ((warp == 2 || warp == 3) && mode == 2) {
    const uint32_t base = smem_u32(smem) + kRing + (uint32_t)(threadIdx.x - 64) * 16;
    const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    w0 = clock64();
    unsigned long long n = 0;
    while (!done) {
#pragma unroll
      for (int j = 0; j < 64; ++j) st_shared_v4(base + (uint32_t)(j % 96) * 1024, v);
      n += 64;
    }
    w1 = clock64();
    written = n * 16 * 64;  // both warps
  }
  if (lane == 0 && written && (warp == 0 || warp == 2)) {
    out[blockIdx.x * 3 + 1] = written;
    out[blockIdx.x * 3 + 2] = w1 - w0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int M, int N>
void run_contend(const char* name, int mode, int grid) {
  unsigned long long* d;
  uint8_t* src;
  cudaMalloc(&d, 3 * 8 * grid);
  cudaMemset(d, 0, 3 * 8 * grid);
  cudaMalloc(&src, 64 * kChunk);
  cudaMemset(src, 1, 64 * kChunk);
  const int n = 16384;
  auto k = probe_contend<M, N>;
  const int smem = kRing + kRingSlots * kChunk;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int rep = 0; rep < 2; ++rep) k<<<grid, 128, smem>>>(n, mode, src, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long* h = new unsigned long long[3 * grid];
  cudaMemcpy(h, d, 3 * 8 * grid, cudaMemcpyDeviceToHost);
  double mx = 0, sum = 0, bpc = 0;
  for (int i = 0; i < grid; ++i) {
    mx = h[3 * i] > mx ? h[3 * i] : mx;
    sum += h[3 * i];
    if (h[3 * i + 2]) bpc += (double)h[3 * i + 1] / h[3 * i + 2];
  }
  const double ideal = (double)M * N / 256.0;
  printf("%-12s mode %d grid %3d: %7.1f cycles/MMA mean (max %7.1f; ideal %5.1f, %5.1f %%), "
         "writes %6.1f B/clk/SM %s\n",
         name, mode, grid, sum / grid / n, mx / n, ideal, 100.0 * ideal / (sum / grid / n), bpc / grid,
         cudaGetErrorString(e));
  delete[] h;
  cudaFree(d);
  cudaFree(src);
}

// Operand layout: A at stage base, B at + b_off; `stages` stage buffers of
// `stride` bytes rotated per group of 4 MMAs (the fused kernel: b_off 16 KB,
// stride 40 KB, 4 stages).
__device__ __forceinline__ void mma_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// VAR 0: warp = threadIdx.x / 32; 1: warp index made provably uniform with
// __shfl_sync (CUTLASS canonical_warp_idx_sync); 2: as 0 with elect + mma in
// one predicated asm block (no branch); 3: 1 and 2.
template <int M, int N, int VAR>
__global__ void probe_layout(int n_mma, uint32_t b_off, uint32_t stride, int stages,
                             unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bars[9];
  const int warp = (VAR & 1) ? __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0) : (int)(threadIdx.x >> 5);
  if (threadIdx.x == 0)
    for (int i = 0; i < 9; ++i) mbar_init(&bars[i], 1);
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base;
  if (warp == 1) {
    constexpr uint32_t idesc = umma_idesc_bf16(M, N);
    const uint32_t base = (smem_u32(smem) + 1023) & ~1023u;
    uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int stage = 0;
    unsigned long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 3;
      const uint32_t a = base + (uint32_t)stage * stride, b = a + b_off;
      if (VAR & 2) {
        mma_elect(tmem, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), idesc, i != 0);
      } else {
        if (elect_one())
          mma_bf16(tmem, umma_desc_sw128(a + k * 32), umma_desc_sw128(b + k * 32), idesc, i != 0);
        __syncwarp();
      }
      if (k == 3) {
        const int g = (i >> 2) & 7;
        if (elect_one()) mma_commit(&bars[g]);
        __syncwarp();
        if ((i >> 2) >= 4) {
          const int w = ((i >> 2) - 4) & 7;
          mbar_wait(&bars[w], phase[w]);
          phase[w] ^= 1;
        }
        if (++stage == stages) stage = 0;
      }
    }
    if (elect_one()) mma_commit(&bars[8]);
    __syncwarp();
    mbar_wait(&bars[8], 0);
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int M, int N, int VAR>
void run_layout(const char* name, uint32_t b_off, uint32_t stride, int stages) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int n = 4096;
  auto k = probe_layout<M, N, VAR>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 128, 200 * 1024>>>(n, b_off, stride, stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double ideal = (double)M * N / 256.0;
  printf("var %d %-10s b_off %6u stride %6u stages %d: %7.1f cycles/MMA (ideal %5.1f, %5.1f %%) %s\n", VAR, name,
         b_off, stride, stages, (double)h / n, ideal, 100.0 * ideal / ((double)h / n),
         cudaGetErrorString(e));
  cudaFree(d);
}

template <int M, int N>
void run_warp(const char* name, int wait) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int n = 4096;
  auto k = probe_warp<M, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 128, 100 * 1024>>>(n, wait, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double ideal = (double)M * N / 256.0;
  printf("%-28s warp-uniform wait %d: %7.1f cycles/MMA (ideal %5.1f, %5.1f %%) %s\n", name, wait,
         (double)h / n, ideal, 100.0 * ideal / ((double)h / n), cudaGetErrorString(e));
  cudaFree(d);
}

template <int M, int N>
void run(const char* name, int pattern) {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int n = 4096;
  auto k = probe_total<M, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int rep = 0; rep < 2; ++rep) k<<<1, 128, 100 * 1024>>>(n, pattern, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double ideal = (double)M * N / 256.0;  // cycles per K=16 MMA at 8192 FLOP/clk/SM
  printf("%-28s pattern %d: %7.1f cycles/MMA (ideal %5.1f, %5.1f %%) %s\n", name, pattern,
         (double)h / n, ideal, 100.0 * ideal / ((double)h / n), cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1) {  // layout probe only
    run_layout<128, 192, 0>("M128 N192", 16384, 40960, 4);
    run_layout<128, 192, 1>("M128 N192", 16384, 40960, 4);
    run_layout<128, 192, 2>("M128 N192", 16384, 40960, 4);
    run_layout<128, 192, 3>("M128 N192", 16384, 40960, 4);
    run_layout<128, 192, 1>("M128 N192", 16384, 0, 1);
    run_layout<128, 256, 1>("M128 N256", 16384, 32768, 4);
    run_layout<128, 128, 1>("M128 N128", 16384, 32768, 4);
    run_layout<128, 128, 3>("M128 N128", 16384, 32768, 4);
    return 0;
  }
  for (int p = 0; p < 4; ++p) {
    run<128, 64>("M128 N64", p);
    run<128, 128>("M128 N128", p);
    run<128, 192>("M128 N192", p);
    run<128, 256>("M128 N256", p);
  }
  for (int g : {1, 148})
    for (int m = 0; m < 3; ++m) {
      run_contend<128, 128>("M128 N128", m, g);
      run_contend<128, 192>("M128 N192", m, g);
      run_contend<128, 256>("M128 N256", m, g);
    }
  for (int w = 0; w < 2; ++w) {
    run_warp<128, 64>("M128 N64", w);
    run_warp<128, 128>("M128 N128", w);
    run_warp<128, 192>("M128 N192", w);
    run_warp<128, 256>("M128 N256", w);
  }
  return 0;
}
