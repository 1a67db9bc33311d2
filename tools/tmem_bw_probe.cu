// tcgen05.ld (TMEM -> registers) throughput probe: W warps of one CTA each
// issue N loads of 32 lanes x 32 columns (4 KB) from their lane quarter, with
// a wait after every 1 or 2 loads; prints bytes per cycle per SM. Also the
// same with a cta_group::1 MMA stream running (TS and SS) to see whether
// MMAs and tcgen05.ld share a port.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2603_22206_b200/csrc \
//      -o tools/tmem_bw_probe tools/tmem_bw_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"

constexpr int N = 2048;

template <int PER_WAIT>
__global__ void probe(long long* cyc, uint32_t* sink, int warps_active) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) chm::sm100::tmem_alloc<512>(&tbase);
  chm::sm100::tc_fence_before();
  __syncthreads();
  chm::sm100::tc_fence_after();
  const uint32_t tmem = chm::sm100::uniform(tbase);
  uint32_t acc = 0;
  long long t0 = 0, t1 = 0;
  if (warp < warps_active) {
    const uint32_t base = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
    t0 = clock64();
    for (int i = 0; i < N; i += PER_WAIT) {
      uint32_t r[PER_WAIT][32];
#pragma unroll
      for (int p = 0; p < PER_WAIT; ++p) chm::sm100::tmem_ld_32x32b_x32(base + (uint32_t)(((i + p) & 7) * 32) % 256, r[p]);
      chm::sm100::tmem_ld_wait();
#pragma unroll
      for (int p = 0; p < PER_WAIT; ++p)
#pragma unroll
        for (int e = 0; e < 32; ++e) acc ^= r[p][e];
    }
    t1 = clock64();
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && warp < warps_active) cyc[warp] = t1 - t0;
  if (acc == 0x12345678u) sink[threadIdx.x] = acc;
  chm::sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    chm::sm100::tc_fence_after();
    chm::sm100::tmem_dealloc<512>(tmem);
  }
}

int main() {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 64 * sizeof(long long));
  cudaMalloc(&sink, 1024 * 4);
  for (int per = 1; per <= 2; ++per) {
    for (int w : {1, 2, 4, 8, 16}) {
      cudaMemset(cyc, 0, 64 * 8);
      if (per == 1)
        probe<1><<<1, 512>>>(cyc, sink, w);
      else
        probe<2><<<1, 512>>>(cyc, sink, w);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long h[64];
      cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
      long long mx = 0;
      for (int i = 0; i < w; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bytes = (double)w * N * 4096;
      printf("loads/wait %d warps %2d: %lld cycles, %.1f B/cycle/SM, %.1f cycles per x32 load per warp\n",
             per, w, mx, bytes / mx, (double)mx / N);
    }
  }
  return 0;
}
