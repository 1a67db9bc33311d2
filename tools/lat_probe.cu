// Dependent-chain latency probe for the instructions on K6's serial path
// (fp64 add / mul, 64-bit integer compare + select, FLO, shared-memory load).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_probe tools/lat_probe.cu
#include <cstdio>
#include <cstdint>

constexpr int N = 4096;

__global__ void probe(double* out, long long* cyc, double a, double b, unsigned long long u) {
  __shared__ unsigned long long sm[64];
  if (threadIdx.x < 64) sm[threadIdx.x] = (threadIdx.x + 1) & 63;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double x = a;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x = __dadd_rn(x, b);
  long long t1 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) x = __dmul_rn(x, b);
  long long t2 = clock64();
  unsigned long long v = u, w = u ^ 0x5555;
#pragma unroll 8
  for (int i = 0; i < N; ++i) {  // 64-bit compare + select chain
    const bool lt = v < w;
    v = lt ? w : v + 1;
  }
  long long t3 = clock64();
  unsigned int f = (unsigned int)u | 1u;
#pragma unroll 8
  for (int i = 0; i < N; ++i) f = (unsigned)(31 - __clz(f)) | 0x100u;
  long long t4 = clock64();
  unsigned long long p = 0;
#pragma unroll 8
  for (int i = 0; i < N; ++i) p = sm[p & 63];
  long long t5 = clock64();
  int q = (int)u & 7;
#pragma unroll 8
  for (int i = 0; i < N; ++i) q = (q == 3) ? (q + 2) & 7 : (q + 1) & 7;  // ISETP + SEL int chain
  long long t6 = clock64();
  out[0] = x + (double)v + f + p + q;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  cyc[5] = t6 - t5;
}

// warp-collective latencies (whole warp 0 runs the chain)
__global__ void probe_warp(double* out, long long* cyc, unsigned u) {
  if (threadIdx.x >= 32) return;
  const unsigned lane = threadIdx.x;
  unsigned a = u + lane;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) a = __reduce_or_sync(0xffffffffu, a) ^ lane;
  long long t1 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) a = __reduce_min_sync(0xffffffffu, a) + lane;
  long long t2 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) a = __shfl_sync(0xffffffffu, a, (a & 7)) + 1;
  long long t3 = clock64();
#pragma unroll 8
  for (int i = 0; i < N; ++i) a = __ballot_sync(0xffffffffu, (a >> lane) & 1) + lane;
  long long t4 = clock64();
  double d = (double)a;
#pragma unroll 8
  for (int i = 0; i < N; ++i) d = __shfl_sync(0xffffffffu, d, (int)lane ^ 1);
  long long t5 = clock64();
  out[1 + lane] = a + d;
  if (lane == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
  }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8 * 8);
  for (int r = 0; r < 3; ++r) probe<<<1, 64>>>(out, cyc, 1.0, 1.0000001, 12345);
  cudaDeviceSynchronize();
  long long h[8];
  cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
  const char* names[] = {"dadd", "dmul", "u64 cmp+sel", "clz", "lds chain", "int cmp+sel"};
  for (int i = 0; i < 6; ++i) printf("%-12s %.2f cycles/iter (8x unrolled)\n", names[i], (double)h[i] / N);
  double* out2;
  cudaMalloc(&out2, 64 * 8);
  for (int r = 0; r < 3; ++r) probe_warp<<<1, 32>>>(out2, cyc, 7);
  cudaDeviceSynchronize();
  cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
  const char* wn[] = {"redux.or", "redux.min", "shfl idx", "ballot", "shfl f64"};
  for (int i = 0; i < 5; ++i) printf("%-12s %.2f cycles/iter (8x unrolled)\n", wn[i], (double)h[i] / N);
  return 0;
}
