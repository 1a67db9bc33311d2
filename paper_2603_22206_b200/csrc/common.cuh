// Shared helpers for the sm_100a kernels of libchimera_sm100a.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include "../../include/chimera_b200.h"

#define CHM_LAUNCH_CHECK()                                     \
  do {                                                         \
    cudaError_t e__ = cudaGetLastError();                      \
    if (e__ != cudaSuccess) return CHM_ERR_CUDA;               \
  } while (0)

namespace chm {

// Error word layout (int32[4], 8-byte aligned): {code, row, model, aux}.
// The host initialises it to {0, INT32_MAX, -1, 0}. Words 0..1 are updated as
// one little-endian uint64 (row << 32 | code) with atomicMin, so among
// parallel detectors the lowest row wins -- the error the reference's serial
// loop would have raised first.
__device__ __forceinline__ void report_error(int32_t* err, int32_t code, int32_t row,
                                             int32_t model, int32_t aux) {
  if (err == nullptr) return;
  unsigned long long packed = ((unsigned long long)(uint32_t)row << 32) | (uint32_t)code;
  unsigned long long old =
      atomicMin(reinterpret_cast<unsigned long long*>(err), packed);
  if (packed < old) {
    err[2] = model;
    err[3] = aux;
  }
}

__device__ __forceinline__ bool is_nan64(double x) { return x != x; }

}  // namespace chm
