// MUFU exp2 throughput per SM: ex2.approx.ftz.f32 vs ex2.approx.f16x2 vs
// ex2.approx.ftz.bf16x2 (two results per lane), 16 warps x 8 independent
// chains per thread. Prints exponentials per cycle per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mufu_probe tools/mufu_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

constexpr int N = 4096;

template <int KIND>
__global__ void probe(long long* cyc, uint32_t* sink, float seed) {
  uint32_t v[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float f = -0.001f * (threadIdx.x + i) + seed;
    if (KIND == 0 || KIND == 3) v[i] = __float_as_uint(f);
    else if (KIND == 1) { __half2 h = __floats2half2_rn(f, f * 0.5f); v[i] = *reinterpret_cast<uint32_t*>(&h); }
    else { v[i] = (__float_as_uint(f) >> 16) | (__float_as_uint(f * 0.5f) & 0xffff0000u); }
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int n = 0; n < N; ++n) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+r"(v[i]));
      else if (KIND == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v[i]));
      else if (KIND == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v[i]));
      else asm volatile("tanh.approx.f32 %0, %0;" : "+r"(v[i]));
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x ^= v[i];
  sink[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 4096);
  const char* names[4] = {"ex2.approx.ftz.f32", "ex2.approx.f16x2", "ex2.approx.ftz.bf16x2",
                          "tanh.approx.f32"};
  for (int k = 0; k < 4; ++k) {
    for (int threads : {128, 512}) {
      if (k == 0) probe<0><<<1, threads>>>(cyc, sink, 0.3f);
      if (k == 1) probe<1><<<1, threads>>>(cyc, sink, 0.3f);
      if (k == 2) probe<2><<<1, threads>>>(cyc, sink, 0.3f);
      if (k == 3) probe<3><<<1, threads>>>(cyc, sink, 0.3f);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      long long c;
      cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double instrs = (double)threads * N * 8;  // thread-level MUFU ops
      const double results = instrs * (k == 0 || k == 3 ? 1 : 2);
      printf("%-22s threads %3d: %.2f thread-ops/cycle/SM, %.2f exp2 results/cycle/SM\n", names[k],
             threads, instrs / c, results / c);
    }
  }
  return 0;
}
