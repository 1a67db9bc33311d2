// Probe: may one kernel issue both tcgen05.mma.cta_group::2 (pair MMA from the
// leader CTA) and tcgen05.mma.cta_group::1 (each CTA on its own TMEM), on a
// cta_group::2 TMEM allocation? If yes, a fused QKV+attention kernel can run
// its projection as a pair MMA (28 KB of operands per SM per k-block instead
// of 40 KB) and its per-sequence attention as cta_group::1 MMAs.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../include \
//        -o cta_group_mix_probe cta_group_mix_probe.cu && ./cta_group_mix_probe
//
// Operands are constant (all elements equal), so the swizzled layout does not
// matter: pair MMA (A = B = 1) -> D = 16 per element (K = 16), then each CTA's
// own MMA (A = B = 2) into other columns -> 64 per element.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include "../paper_2603_22206_b200/csrc/sm100.cuh"

using namespace chm::sm100;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(float* out, int mode) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = &align_smem_1024<uint8_t>(smem_raw);
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar_pair, bar_own;
  const int warp = warp_id(), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  // tiles: [0] pair A (128 x 64 bf16 of 1.0), [1] pair B half (32 rows used),
  // [2] own A (2.0), [3] own B (2.0)
  __nv_bfloat16* t = reinterpret_cast<__nv_bfloat16*>(smem);
  for (int i = threadIdx.x; i < 4 * 8192; i += blockDim.x)
    t[i] = __float2bfloat16(i < 2 * 8192 ? 1.0f : 2.0f);
  if (threadIdx.x == 0) {
    mbar_init(&bar_pair, 1);
    mbar_init(&bar_own, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc_cg2<256>(&tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = uniform(tmem_base);
  const uint32_t a = smem_u32(smem);
  if (warp == 1) {
    if (rank == 0 && (mode & 1)) {  // pair MMA M = 256, N = 64, K = 16 -> columns [0, 64)
      mma_bf16_cg2_w(tmem, umma_desc_sw128(a), umma_desc_sw128(a + 16384),
                     umma_idesc_bf16(256, 64), 0);
      mma_commit_cg2_mc_w(&bar_pair, 0x3);
    }
    if (mode & 2) {  // own MMA M = 128, N = 64, K = 16 -> columns [128, 192)
      if (mode & 1) mbar_wait(&bar_pair, 0);  // after the pair result landed here
      tc_fence_after();
      mma_bf16_w(tmem + 128, umma_desc_sw128(a + 2 * 16384), umma_desc_sw128(a + 3 * 16384),
                 umma_idesc_bf16(128, 64), 0);
      mma_commit_w(&bar_own);
    }
  }
  __syncthreads();
  if (warp < 4) {
    uint32_t r[32];
    const uint32_t lb = tmem + ((uint32_t)(warp * 32) << 16);
    if (mode & 1) {
      mbar_wait(&bar_pair, 0);
      tc_fence_after();
      tmem_ld_32x32b_x32(lb, r);
      tmem_ld_wait();
      out[(rank * 128 + warp * 32 + lane) * 2 + 0] = __uint_as_float(r[lane & 31]);
    }
    if (mode & 2) {
      mbar_wait(&bar_own, 0);
      tc_fence_after();
      tmem_ld_32x32b_x32(lb + 128, r);
      tmem_ld_wait();
      out[(rank * 128 + warp * 32 + lane) * 2 + 1] = __uint_as_float(r[lane & 31]);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc_cg2<256>(tmem);
}

int main() {
  float* d;
  cudaMalloc(&d, 256 * 2 * sizeof(float));
  for (int mode = 1; mode <= 3; ++mode) {
    cudaMemset(d, 0, 256 * 2 * sizeof(float));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 16384);
    probe<<<2, 128, 5 * 16384>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    float h[512];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int bad_pair = 0, bad_own = 0;
    for (int i = 0; i < 256; ++i) {
      if ((mode & 1) && h[2 * i] != 16.0f) ++bad_pair;
      if ((mode & 2) && h[2 * i + 1] != 64.0f) ++bad_own;
    }
    printf("mode %d (%s): %s; pair rows wrong %d, own rows wrong %d (sample %g %g)\n", mode,
           mode == 1 ? "pair only" : mode == 2 ? "own only" : "pair then own",
           cudaGetErrorString(e), bad_pair, bad_own, h[0], h[1]);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
