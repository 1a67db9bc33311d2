// Internal interface of the tcgen05 GEMM (gemm.cu) for the encoder kernels.
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace chm {

// Epilogue selector and operands (see gemm.cu's Epilogue enum):
//  0 none, 1 bias, 2 bias+GELU, 3 bias+residual, 4 QKV (bias, Q x 1/8),
//  5 residual+LayerNorm (cluster rows), 6 bias + LN(residual) + row statistics.
struct GemmArgs {
  int epilogue = 0;
  const float* bias = nullptr;
  const void* residual = nullptr;
  long long res_ld = 0;          // residual row pitch in elements (0 = N)
  const float* gamma = nullptr;  // 5: LN of the output; 6: LN of the residual
  const float* beta = nullptr;
  float eps = 0.f;
  int hidden = 0;                // 4: H (Q columns [0, H))
  const float2* stats_in = nullptr;  // fold (1/2/4) or residual LN (6): [M][n_part]
  int n_part = 0;
  const float* colsum = nullptr;     // fold: per output column sum of the folded weights
  float2* stats_out = nullptr;       // 6: [M][N/128]
  // rows actually computed: min(M, *live_rows * live_mult) read on the device
  // (the routed sequences of a tick; nullptr = all M rows)
  const int32_t* live_rows = nullptr;
  int live_mult = 1;
  // measurement only: algorithmic FLOPs = 2 M N K / work_div (block-diagonal
  // weights: the zero blocks are executed but are not work)
  int work_div = 1;
};

chm_status gemm_run(const void* A, const void* B, void* C, int M, int N, int K,
                    const GemmArgs& g, cudaStream_t s);

}  // namespace chm
