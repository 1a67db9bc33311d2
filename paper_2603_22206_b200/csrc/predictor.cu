// K5 -- remaining-workflow-output predictors.
//
// The reference evaluates Predictor.predict(req, rec, model) for the chosen
// model only (balancer.py:115). The predictors are pure functions, so the GPU
// evaluates every model column of every row in one coalesced pass and the
// selection kernel (K6) gathers the chosen column. Output layout: yhat[B, K]
// row-major fp64 (Python floats are IEEE doubles).
//
// HBM bytes per row (algorithmic): quantile 8 (wf, stage) + 8K (out);
// oracle 8 + 4*max_stages*K + 8K; input-length 4 + 8K.
#include "common.cuh"
#include "prof.cuh"

namespace chm {

// EmpiricalQuantilePredictor.predict (predictor.py:100-108). The fallback
// chain (workflow,stage,model) -> (stage,model) -> (model) -> global is
// resolved into the dense table when it is built on the host (the
// np.quantile "training" at predictor.py:95-98 is not on the per-tick path),
// so the device does a bounds-clamped gather: unseen workflows map to row
// n_wf and stages outside [1, s_cap] to column 0.
__global__ void __launch_bounds__(256) predict_quantile_kernel_dyn(
    const double* __restrict__ table, int n_wf, int s_cap, int K,
    const int32_t* __restrict__ workflow, const int32_t* __restrict__ stage, int n_rows,
    double* __restrict__ yhat) {
  extern __shared__ double s_table[];
  const int n_tab = (n_wf + 1) * (s_cap + 1) * K;
  for (int i = threadIdx.x; i < n_tab; i += blockDim.x) s_table[i] = table[i];
  __syncthreads();
  // One thread per output element: fully coalesced stores.
  const long long total = (long long)n_rows * K;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int row = (int)(e / K), m = (int)(e - (long long)row * K);
    int wf = __ldg(workflow + row);
    int st = __ldg(stage + row);
    wf = (wf < 0 || wf >= n_wf) ? n_wf : wf;
    st = (st < 1 || st > s_cap) ? 0 : st;
    yhat[e] = s_table[(wf * (s_cap + 1) + st) * K + m];
  }
}

// Same gather straight from global memory, for tables larger than the
// shared-memory budget (the reference has no size limit): the table stays
// L2-resident (126 MB) across the grid.
__global__ void __launch_bounds__(256) predict_quantile_kernel_l2(
    const double* __restrict__ table, int n_wf, int s_cap, int K,
    const int32_t* __restrict__ workflow, const int32_t* __restrict__ stage, int n_rows,
    double* __restrict__ yhat) {
  const long long total = (long long)n_rows * K;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int row = (int)(e / K), m = (int)(e - (long long)row * K);
    int wf = __ldg(workflow + row);
    int st = __ldg(stage + row);
    wf = (wf < 0 || wf >= n_wf) ? n_wf : wf;
    st = (st < 1 || st > s_cap) ? 0 : st;
    yhat[e] = __ldg(table + ((size_t)wf * (s_cap + 1) + st) * K + m);
  }
}

// OraclePredictor.predict = rec.remaining_tokens(stage, model)
// (predictor.py:30-36, workload.py:160-165): integer suffix sum, exact.
__global__ void __launch_bounds__(256) predict_oracle_kernel(
    const int32_t* __restrict__ stage_out, const int32_t* __restrict__ n_stages,
    const int32_t* __restrict__ stage, int max_stages, int K, int n_rows,
    double* __restrict__ yhat, int32_t* err) {
  const long long total = (long long)n_rows * K;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int row = (int)(e / K), m = (int)(e - (long long)row * K);
    int st = stage[row], ns = n_stages[row];
    if (st < 1 || st > ns || ns > max_stages) {
      // TraceRecord._stage raises UnknownStage (workload.py:143-147).
      if (m == 0) report_error(err, CHM_ERR_UNKNOWN_STAGE, row, -1, st);
      yhat[e] = 0.0;
      continue;
    }
    long long acc = 0;
    const int32_t* base = stage_out + (size_t)row * max_stages * K + m;
    for (int j = st - 1; j < ns; ++j) acc += base[(size_t)j * K];
    yhat[e] = (double)acc;
  }
}

// InputLengthPredictor.predict = float(req.input_tokens) (predictor.py:39-45).
__global__ void __launch_bounds__(256) predict_input_length_kernel(
    const int32_t* __restrict__ input_tokens, int K, int n_rows, double* __restrict__ yhat) {
  const long long total = (long long)n_rows * K;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    int row = (int)(e / K);
    yhat[e] = (double)__ldg(input_tokens + row);
  }
}

static int grid_for(long long work, int block) {
  long long g = (work + block - 1) / block;
  // 148 SMs x 8 resident 256-thread CTAs is one full wave; never launch more
  // than 4 waves of a grid-stride kernel.
  const long long cap = 148LL * 8 * 4;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace chm

extern "C" chm_status chm_predict_quantile(const double* table, int32_t n_wf, int32_t s_cap,
                                           int32_t n_models, const int32_t* workflow,
                                           const int32_t* stage, int32_t n_rows,
                                           double* yhat, void* stream) {
  if (n_rows < 0 || n_models < 1 || n_models > CHM_MAX_MODELS || n_wf < 0 || s_cap < 0)
    return CHM_ERR_INVALID_ARG;
  if (n_rows == 0) return CHM_OK;
  if (!table || !workflow || !stage || !yhat) return CHM_ERR_INVALID_ARG;
  size_t smem = (size_t)(n_wf + 1) * (s_cap + 1) * n_models * sizeof(double);
  cudaStream_t s = (cudaStream_t)stream;
  if (smem > 160 * 1024) {
    chm::prof::begin(chm::prof::K_PREDICT, s);
    chm::predict_quantile_kernel_l2<<<chm::grid_for((long long)n_rows * n_models, 256), 256, 0,
                                      s>>>(table, n_wf, s_cap, n_models, workflow, stage,
                                           n_rows, yhat);
    chm::prof::end(chm::prof::K_PREDICT, s, (double)n_rows * (8.0 + 8.0 * n_models));
    CHM_LAUNCH_CHECK();
    return CHM_OK;
  }
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(chm::predict_quantile_kernel_dyn,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  chm::prof::begin(chm::prof::K_PREDICT, s);
  chm::predict_quantile_kernel_dyn<<<chm::grid_for((long long)n_rows * n_models, 256), 256,
                                     smem, s>>>(table, n_wf, s_cap, n_models, workflow,
                                                stage, n_rows, yhat);
  chm::prof::end(chm::prof::K_PREDICT, s, (double)n_rows * (8.0 + 8.0 * n_models));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_predict_oracle(const int32_t* stage_out, const int32_t* n_stages,
                                         const int32_t* stage, int32_t max_stages,
                                         int32_t n_models, int32_t n_rows, double* yhat,
                                         int32_t* error, void* stream) {
  if (n_rows < 0 || n_models < 1 || n_models > CHM_MAX_MODELS || max_stages < 1)
    return CHM_ERR_INVALID_ARG;
  if (n_rows == 0) return CHM_OK;
  if (!stage_out || !n_stages || !stage || !yhat) return CHM_ERR_INVALID_ARG;
  chm::prof::begin(chm::prof::K_PREDICT, (cudaStream_t)stream);
  chm::predict_oracle_kernel<<<chm::grid_for((long long)n_rows * n_models, 256), 256, 0,
                               (cudaStream_t)stream>>>(stage_out, n_stages, stage,
                                                       max_stages, n_models, n_rows, yhat,
                                                       error);
  chm::prof::end(chm::prof::K_PREDICT, (cudaStream_t)stream,
                 (double)n_rows * (8.0 + 4.0 * max_stages * n_models + 8.0 * n_models));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_predict_input_length(const int32_t* input_tokens, int32_t n_models,
                                               int32_t n_rows, double* yhat, void* stream) {
  if (n_rows < 0 || n_models < 1 || n_models > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  if (n_rows == 0) return CHM_OK;
  if (!input_tokens || !yhat) return CHM_ERR_INVALID_ARG;
  chm::prof::begin(chm::prof::K_PREDICT, (cudaStream_t)stream);
  chm::predict_input_length_kernel<<<chm::grid_for((long long)n_rows * n_models, 256), 256,
                                     0, (cudaStream_t)stream>>>(input_tokens, n_models,
                                                                n_rows, yhat);
  chm::prof::end(chm::prof::K_PREDICT, (cudaStream_t)stream, (double)n_rows * (4.0 + 8.0 * n_models));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}
