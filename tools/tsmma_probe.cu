// tcgen05.mma throughput for the flash-attention MMA shapes (one CTA, one SM):
// M = 128, N = 16 / 64 / 128 / 256, K = 16 per instruction, A from shared
// memory (SS) or tensor memory (TS), B K-major or MN-major (V), issued by a
// warp-uniform loop (elect.sync inside the asm) with one commit at the end.
// Prints cycles per MMA against the floor 128 N / 256.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2603_22206_b200/csrc -o tools/tsmma_probe tools/tsmma_probe.cu
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"

using namespace chm::sm100;

struct __align__(1024) Smem {
  uint8_t a[128 * 64 * 2];   // 16 KB
  uint8_t b[256 * 64 * 2];   // 32 KB
  uint64_t done;
  uint32_t tbase;
};

// mix: 0 = single shape; 1 = the flash v5 block mix (per tile: S N64 x4 TS,
// O N64 MN-major x4 TS + l N16 x4 TS)
__global__ void probe(int n, int N, int ts, int mn, int mix, unsigned long long* out) {
  extern __shared__ uint8_t raw[];
  Smem& s = align_smem_1024<Smem>(raw);
  const int warp = warp_id();
  if (threadIdx.x == 0) {
    mbar_init(&s.done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&s.tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = uniform(s.tbase);
  if (warp == 1) {
    const uint32_t a = smem_u32(s.a), b = smem_u32(s.b);
    const uint32_t idesc = umma_idesc_bf16(128, N) | (mn ? (1u << 16) : 0u);
    constexpr uint32_t id64 = umma_idesc_bf16(128, 64), id64mn = umma_idesc_bf16(128, 64) | (1u << 16),
                       id16 = umma_idesc_bf16(128, 16);
    const unsigned long long t0 = clock64();
    if (!mix) {
      for (int i = 0; i < n; ++i) {
        const uint32_t d = tmem + (uint32_t)((i & 1) * 256 % (512 - N + 1));
        if (ts)
          mma_bf16_ts_w(tmem + 256 * ((i >> 3) & 1), tmem + 448 + (i & 3) * 8,
                        umma_desc_sw128(b + (i & 3) * 32), idesc, i & 3);
        else
          mma_bf16_w(d, umma_desc_sw128(a + (i & 3) * 32), umma_desc_sw128(b + (i & 3) * 32),
                     idesc, i & 3);
      }
    } else {
      for (int i = 0; i < n; ++i) {  // one block of one tile per iteration
        const int g = i & 1;
        for (int k = 0; k < 4; ++k)
          mma_bf16_ts_w(tmem + 128 * g, tmem + 256 + 32 * g + k * 8, umma_desc_sw128(b + k * 32),
                        id64, k);
        for (int k = 0; k < 4; ++k) {
          mma_bf16_ts_w(tmem + 320 + 64 * g, tmem + 128 * g + 64 + k * 8,
                        umma_desc_sw128(b + k * 2048), id64mn, k);
          mma_bf16_ts_w(tmem + 448 + 16 * g, tmem + 128 * g + 64 + k * 8,
                        umma_desc_sw128(a + k * 32), id16, k);
        }
      }
    }
    mma_commit_w(&s.done);
    mbar_wait(&s.done, 0);
    const unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int n = 4096;
  for (int ts = 0; ts <= 1; ++ts)
    for (int mn = 0; mn <= 1; ++mn)
      for (int N : {16, 32, 64, 128, 256}) {
        if (ts && N > 64) continue;
        probe<<<1, 128, smem>>>(n, N, ts, mn, 0, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long c;
        cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
        const double floor = 128.0 * N / 256.0;
        printf("%s B %s N %3d: %6.1f cycles/MMA (floor %5.1f, %5.1f %%)\n", ts ? "TS" : "SS",
               mn ? "MN-major" : "K-major ", N, (double)c / n, floor, 100.0 * floor * n / c);
      }
  probe<<<1, 128, smem>>>(2048, 64, 1, 0, 1, d);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  // floor per tile-block: S 4 x 32 + O 4 x 32 + l 4 x 8 = 288 cycles
  printf("flash v5 block mix: %6.1f cycles per tile-block (floor 288, %5.1f %%)\n", (double)c / 2048,
         100.0 * 288 * 2048 / c);
  return 0;
}
