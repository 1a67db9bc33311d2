// Deferred LayerNorm helpers shared by the router kernels.
//
// The post-LN encoder's LayerNorms are not applied where their input is
// produced (that needs every column of a row in one cluster). The producer
// GEMM (EPI_RESLN_STATS) writes the pre-LN row plus partial statistics, one
// (mean, M2) pair per 128 columns; consumers turn the P = H/128 partials of a
// row into its affine map LN(x)_n = (a x_n + b) gamma_n + beta_n.
#pragma once
#include <cuda_runtime.h>

namespace chm {

constexpr int kLnPartCols = 128;  // columns per partial statistic
constexpr int kLnMaxParts = 8;    // H <= 1024

// a = rstd, b = -mean * rstd of a row from its P partials (Chan's merge of
// equal-size groups: M2 = sum M2_j + 128 sum (mean_j - mean)^2).
__device__ __forceinline__ void row_affine(const float2* __restrict__ st, int P, float eps,
                                           float& a, float& b) {
  float2 v[kLnMaxParts];
#pragma unroll
  for (int j = 0; j < kLnMaxParts; ++j) v[j] = j < P ? st[j] : make_float2(0.f, 0.f);
  float mean = 0.f;
#pragma unroll
  for (int j = 0; j < kLnMaxParts; ++j) mean += v[j].x;
  mean /= (float)P;
  float m2 = 0.f;
#pragma unroll
  for (int j = 0; j < kLnMaxParts; ++j) {
    if (j < P) {
      const float d = v[j].x - mean;
      m2 += fmaf(d * d, (float)kLnPartCols, v[j].y);
    }
  }
  a = rsqrtf(m2 / (float)(kLnPartCols * P) + eps);
  b = -mean * a;
}

}  // namespace chm
