// Launch accounting and optional CUDA-event profiling of every kernel the
// library launches (used by bench.py to time the dominant kernel live, on the
// stream it is launched on, inside the timed region).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace chm {
namespace prof {

enum Kind : int {
  K_GEMM = 0,
  K_ATTENTION = 1,
  K_ROWWISE = 2,   // embedding+LN, LayerNorm, CLS head
  K_PREDICT = 3,
  K_PREPARE = 4,
  K_SELECT = 5,
  K_QUEUE = 6,
  K_QKV_ATTENTION = 7,  // fused QKV projection + attention (qkv_attn.cu)
  K_TRACE = 8,          // columnar trace store derivation (trace.cu)
  K_EVAL = 9,           // predictor evaluation (evaluate.cu)
  K_NUM = 10
};

// Call around one kernel launch on `s`. `work` is the algorithmic FLOPs
// (GEMM/attention) or bytes (memory-bound kernels) of the launch.
void begin(int kind, cudaStream_t s);
void end(int kind, cudaStream_t s, double work);

}  // namespace prof
}  // namespace chm
