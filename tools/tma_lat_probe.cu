// TMA load latency: one thread per CTA issues a 2D tensor load of a
// [rows x 64] bf16 box (128B swizzle) from an L2-resident buffer and waits on
// the mbarrier; cycles per load (issue -> complete_tx observed), serial, for
// box sizes 4 / 8 / 16 / 28 KB, on 1 CTA and on every SM at once (each CTA
// loading different boxes of the same 4 MB buffer, like the router kernels'
// weight tiles). Also `depth` loads in flight per CTA (pipelined throughput).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2603_22206_b200/csrc -o tools/tma_lat_probe tools/tma_lat_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cudaTypedefs.h>
#include <cuda.h>
#include "sm100.cuh"

using namespace chm::sm100;

constexpr int kIters = 64;

struct __align__(1024) Smem {
  uint8_t buf[8][28 * 1024];
  uint64_t bar[8];
};

// csize > 1: cluster of csize CTAs; each loads rows / csize of every box and
// multicasts it to all, so each CTA still receives whole boxes while L2 reads
// each byte once per cluster
__global__ void probe(const __grid_constant__ CUtensorMap tm, int rows, int depth,
                      unsigned long long* out, int csize) {
  extern __shared__ uint8_t raw[];
  Smem& s = align_smem_1024<Smem>(raw);
  const uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) mbar_init(&s.bar[i], 1);
    fence_barrier_init();
  }
  cluster_sync();
  // the whole warp runs the loop (cluster barriers need every thread); lane 0 issues
  const bool issuer = threadIdx.x == 0;
  const uint32_t bytes = rows * 128;
  uint32_t phase = 0;
  const unsigned long long t0 = clock64();
  for (int it = 0; it < kIters; ++it) {
    if (issuer) {
      for (int d = 0; d < depth; ++d) {
        mbar_arrive_expect_tx(&s.bar[d], bytes);
        const int row = (((blockIdx.x / csize) * 7 + it * depth + d) * rows) % (16384 - rows);
        if (csize == 1) {
          tma_load_2d(s.buf[d], &tm, &s.bar[d], (it & 3) * 64, row);
        } else {
          const int sub = rows / csize;  // this CTA's slice, multicast to the cluster
          tma_load_2d_mc(s.buf[d] + rank * sub * 128, &tm, &s.bar[d], (it & 3) * 64,
                         row + (int)rank * sub, (uint16_t)((1u << csize) - 1));
        }
      }
    }
    __syncwarp();
    for (int d = 0; d < depth; ++d) mbar_wait(&s.bar[d], phase);
    phase ^= 1;
    // every CTA has consumed the round before anyone overwrites it
    if (csize > 1) cluster_sync();
  }
  const unsigned long long t1 = clock64();
  if (issuer) out[blockIdx.x] = t1 - t0;
  cluster_sync();
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

int main() {
  const int R = 16384, C = 256;  // 8 MB bf16
  void* buf;
  cudaMalloc(&buf, (size_t)R * C * 2);
  cudaMemset(buf, 1, (size_t)R * C * 2);
  unsigned long long* out;
  cudaMalloc(&out, 1024 * 8);
  const size_t smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int rows : {128, 224}) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)rows};
    cuuint32_t estr[2] = {1, 1};
    if (encode()(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, estr,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    for (int csize : {1, 2, 4}) {
    for (int grid : {sms}) {
      for (int depth : {4, 8}) {
        grid = (grid / csize) * csize;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(32);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = csize;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, probe, tm, rows, depth, out, csize);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        unsigned long long h[1024];
        cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
        double mean = 0;
        unsigned long long mx = 0;
        for (int i = 0; i < grid; ++i) { mean += h[i]; mx = h[i] > mx ? h[i] : mx; }
        mean /= grid;
        const double per = mean / kIters;  // cycles per round of `depth` loads
        printf("box %3d rows (%5.1f KB) cluster %d grid %3d depth %d: %7.0f cycles per round, %6.1f B/cycle/SM delivered\n",
               rows, rows * 0.125, csize, grid, depth, per, depth * rows * 128.0 / per);
        fflush(stdout);
      }
    }
    }
  }
  return 0;
}
