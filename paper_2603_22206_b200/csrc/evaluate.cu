// Predictor evaluation on the device:
// kendall_tau_distance (hetsched predictor.py:182-214) -- the fraction of
// discordant pairs between a predicted and a true ranking, pairs tied in
// exactly one sequence counting one half -- and its building blocks
// _count_inversions (132-160), _tie_pairs (163-173), _pair_run_lengths
// (217-227).
//
// The reference sorts by (predicted, truth), counts strict inversions of the
// truth column by a bottom-up merge sort, and counts tied pairs in three
// sorted sequences. Here every step is a sort/merge over order-preserving
// 64-bit keys (fp64 -> uint64 with -0.0 folded into +0.0, so Python's
// equality is key equality):
//   1. bottom-up merge sort of the (predicted, truth) key pairs: one launch
//      per level, every element finds its output slot by binary search in the
//      partner run (left elements go before equal right elements: stable);
//   2. the truth column in that order is merge-sorted again, and every right
//      run element adds (left run length - #left elements <= it) = the left
//      elements strictly greater than it: the strict inversion count;
//   3. tied pairs of a sorted sequence = sum_i (i - first index of v_i), one
//      binary search per element (no scan).
// All counts are exact int64; the distance is formed exactly as the
// reference does: (discordant + 0.5 * half) / total in fp64.
//
// The same merge machinery trains EmpiricalQuantilePredictor's tables
// (chm_quantile_train, below).
//
// Work: O(n log^2 n) key reads (binary searches hit L2), O(n log n) key
// writes. Scratch: 6 * 8 bytes per element (chm_kendall_tau_scratch_bytes).
#include <utility>
#include "common.cuh"
#include "prof.cuh"

namespace chm {
namespace eval {

__device__ __forceinline__ uint64_t okey(double x) {
  if (x == 0.0) x = 0.0;  // -0.0 == 0.0 in Python: same key
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

template <bool PAIR>
struct Key {
  uint64_t a, b;
  __device__ __forceinline__ bool operator<(const Key& o) const {
    return PAIR ? (a < o.a || (a == o.a && b < o.b)) : a < o.a;
  }
  __device__ __forceinline__ bool operator<=(const Key& o) const { return !(o < *this); }
};

template <bool PAIR>
__device__ __forceinline__ Key<PAIR> load(const uint64_t* a, const uint64_t* b, int64_t i) {
  Key<PAIR> k;
  k.a = a[i];
  k.b = PAIR ? b[i] : 0;
  return k;
}

__global__ void keys_kernel(const double* __restrict__ p, const double* __restrict__ t, int64_t n,
                            uint64_t* __restrict__ kp, uint64_t* __restrict__ kt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  kp[i] = okey(p[i]);
  kt[i] = okey(t[i]);
}

// One bottom-up merge level of width w: runs [lo, lo+w) and [lo+w, lo+2w).
// COUNT: accumulate, for every right-run element, the left-run elements
// strictly greater than it (strict inversions across the two runs).
template <bool PAIR, bool COUNT>
__global__ void __launch_bounds__(256) merge_level(const uint64_t* __restrict__ a1,
                                                   const uint64_t* __restrict__ a2,
                                                   uint64_t* __restrict__ b1,
                                                   uint64_t* __restrict__ b2, int64_t n, int64_t w,
                                                   unsigned long long* __restrict__ inv) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (i < n) {
    const int64_t lo = (i / (2 * w)) * (2 * w);
    const int64_t mid = min(lo + w, n), hi = min(lo + 2 * w, n);
    const Key<PAIR> x = load<PAIR>(a1, a2, i);
    int64_t pos;
    if (i < mid) {
      // right elements strictly less than x come first
      int64_t l = mid, h = hi;
      while (l < h) {
        const int64_t m = (l + h) >> 1;
        if (load<PAIR>(a1, a2, m) < x) l = m + 1; else h = m;
      }
      pos = i + (l - mid);
    } else {
      // left elements <= x come first
      int64_t l = lo, h = mid;
      while (l < h) {
        const int64_t m = (l + h) >> 1;
        if (load<PAIR>(a1, a2, m) <= x) l = m + 1; else h = m;
      }
      pos = lo + (i - mid) + (l - lo);
      if (COUNT) c = (unsigned long long)(mid - l);
    }
    b1[pos] = x.a;
    if (PAIR) b2[pos] = x.b;
  }
  if (COUNT) {
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(inv, c);
  }
}

// _tie_pairs of a sorted sequence: sum over elements of (i - first index of
// an equal element). PAIR: equality of both keys (_pair_run_lengths).
template <bool PAIR>
__global__ void __launch_bounds__(256) tie_pairs_kernel(const uint64_t* __restrict__ a1,
                                                        const uint64_t* __restrict__ a2,
                                                        int64_t n,
                                                        unsigned long long* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long c = 0;
  if (i < n) {
    const Key<PAIR> x = load<PAIR>(a1, a2, i);
    int64_t l = 0, h = i;
    while (l < h) {
      const int64_t m = (l + h) >> 1;
      if (load<PAIR>(a1, a2, m) < x) l = m + 1; else h = m;
    }
    c = (unsigned long long)(i - l);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// counts = {discordant, ties_p, ties_t, ties_both}; result = distance.
__global__ void finish_kernel(const unsigned long long* __restrict__ counts, int64_t n,
                              double* __restrict__ result) {
  const long long disc = (long long)counts[0], tp = (long long)counts[1];
  const long long tt = (long long)counts[2], tb = (long long)counts[3];
  const long long half = (tp - tb) + (tt - tb);
  const long long total = n * (n - 1) / 2;
  // Python: (discordant + 0.5 * half) / total -- int + float, then float / int
  *result = __ddiv_rn(__dadd_rn((double)disc, __dmul_rn(0.5, (double)half)), (double)total);
}

static unsigned grid_of(int64_t n) { return (unsigned)((n + 255) / 256); }

// ---------------------------------------------------------------------------
// EmpiricalQuantilePredictor training (predictor.py:78-98): per group the
// np.quantile(values, q) of the remaining-token values y = remaining[p, s, m]
// of every training (program, stage, model), at four levels:
//   L0 (workflow, stage, model), L1 (stage, model), L2 (model), L3 global.
// Each level: one sort of (group id, value key) pairs (the merge levels
// above), then per group id its [start, end) by binary search and numpy's
// 'linear' quantile (method 7) with numpy's exact arithmetic:
//   v = (n - 1) * q; v >= n - 1 -> last; else i = floor(v), g = v - i,
//   d = x[i+1] - x[i]; g >= 0.5 ? x[i+1] - d * (1 - g) : x[i] + d * g   (_lerp)
// The table [n_wf + 1, s_cap + 1, K] resolves the fallback chain
// (predictor.py:100-108) exactly like the host build.
__device__ __forceinline__ double okey_inv(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}

// level ids: L0 (wf * (s_cap+1) + st) * K + m, L1 st * K + m, L2 m, L3 0
__global__ void train_entries_kernel(chm_trace t, const int32_t* __restrict__ workflow,
                                     int s_cap, int level, uint64_t* __restrict__ id,
                                     uint64_t* __restrict__ val,
                                     unsigned long long* __restrict__ cursor) {
  const int S = t.max_stages, K = t.n_models;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)t.n_programs * S * K) return;
  const long long p = idx / ((long long)S * K);
  const int r = (int)(idx - p * S * K), s = r / K, m = r - s * K;
  if (s >= t.n_stages[p]) return;
  const int st = s + 1, wf = workflow[p];
  uint64_t g;
  switch (level) {
    case 0: g = ((uint64_t)wf * (s_cap + 1) + st) * K + m; break;
    case 1: g = (uint64_t)st * K + m; break;
    case 2: g = (uint64_t)m; break;
    default: g = 0; break;
  }
  const unsigned long long at = atomicAdd(cursor, 1ull);
  id[at] = g;
  val[at] = okey((double)t.remaining[idx]);
}

__device__ __forceinline__ int64_t lower_id(const uint64_t* id, int64_t n, uint64_t g) {
  int64_t l = 0, h = n;
  while (l < h) {
    const int64_t m = (l + h) >> 1;
    if (id[m] < g) l = m + 1; else h = m;
  }
  return l;
}

// One thread per group id of the level: quantile of its sorted values.
__global__ void group_quantile_kernel(const uint64_t* __restrict__ id,
                                      const uint64_t* __restrict__ val, int64_t n, int n_groups,
                                      double q, double* __restrict__ out,
                                      uint8_t* __restrict__ present) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n_groups) return;
  const int64_t a = lower_id(id, n, (uint64_t)g), b = lower_id(id, n, (uint64_t)g + 1);
  const int64_t cnt = b - a;
  present[g] = cnt > 0;
  if (cnt <= 0) return;
  const double v = __dmul_rn((double)(cnt - 1), q);  // (n - 1) * quantiles
  double r;
  if (v >= (double)(cnt - 1)) {
    r = okey_inv(val[b - 1]);
  } else if (v < 0.0) {
    r = okey_inv(val[a]);
  } else {
    const double fl = floor(v);
    const int64_t i = (int64_t)fl;
    const double gam = __dsub_rn(v, fl);
    const double x0 = okey_inv(val[a + i]), x1 = okey_inv(val[a + i + 1]);
    const double d = __dsub_rn(x1, x0);
    r = gam >= 0.5 ? __dsub_rn(x1, __dmul_rn(d, __dsub_rn(1.0, gam)))
                   : __dadd_rn(x0, __dmul_rn(d, gam));
  }
  out[g] = r;
}

// table[a, st, m] with the fallback chain; a == n_wf: unknown workflow,
// st == 0: stage outside 1..s_cap (no L0 / L1 entry can match).
__global__ void table_kernel(const double* __restrict__ q0, const uint8_t* __restrict__ h0,
                             const double* __restrict__ q1, const uint8_t* __restrict__ h1,
                             const double* __restrict__ q2, const uint8_t* __restrict__ h2,
                             const double* __restrict__ q3, int n_wf, int s_cap, int K,
                             double* __restrict__ table) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (n_wf + 1) * (s_cap + 1) * K) return;
  const int m = e % K, st = (e / K) % (s_cap + 1), a = e / (K * (s_cap + 1));
  double v = q3[0];
  if (h2[m]) v = q2[m];
  if (st >= 1 && h1[st * K + m]) v = q1[st * K + m];
  if (a < n_wf && st >= 1 && h0[(a * (s_cap + 1) + st) * K + m]) v = q0[(a * (s_cap + 1) + st) * K + m];
  table[e] = v;
}

}  // namespace eval
}  // namespace chm

extern "C" uint64_t chm_quantile_train_scratch_bytes(int64_t n_entries, int32_t n_wf,
                                                     int32_t s_cap, int32_t n_models) {
  if (n_entries < 0 || n_wf < 0 || s_cap < 1 || n_models < 1) return 0;
  const uint64_t groups = (uint64_t)(n_wf * (s_cap + 1) + (s_cap + 1) + 2) * n_models + 1;
  return (uint64_t)n_entries * 4 * 8 + groups * 9 + 256;
}

extern "C" chm_status chm_quantile_train(const chm_trace* t, const int32_t* workflow,
                                         int32_t n_wf, int32_t s_cap, double quantile,
                                         int64_t n_entries, void* scratch,
                                         uint64_t scratch_bytes, double* table, void* stream) {
  using namespace chm::eval;
  if (!t || !workflow || !t->remaining || !t->n_stages || !scratch || !table || n_wf < 1 ||
      s_cap < 1 || n_entries < 1 || !(quantile > 0.0 && quantile < 1.0))
    return CHM_ERR_INVALID_ARG;
  if (scratch_bytes < chm_quantile_train_scratch_bytes(n_entries, n_wf, s_cap, t->n_models))
    return CHM_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int K = t->n_models;
  const int64_t n = n_entries;
  char* sp = reinterpret_cast<char*>(scratch);
  unsigned long long* cursor = reinterpret_cast<unsigned long long*>(sp);
  uint64_t* id0 = reinterpret_cast<uint64_t*>(sp + 256);
  uint64_t *v0 = id0 + n, *id1 = id0 + 2 * n, *v1 = id0 + 3 * n;
  const int ng[4] = {n_wf * (s_cap + 1) * K, (s_cap + 1) * K, K, 1};
  double* qv = reinterpret_cast<double*>(id0 + 4 * n);
  double* qs[4] = {qv, qv + ng[0], qv + ng[0] + ng[1], qv + ng[0] + ng[1] + ng[2]};
  uint8_t* hv = reinterpret_cast<uint8_t*>(qv + ng[0] + ng[1] + ng[2] + ng[3]);
  uint8_t* hs[4] = {hv, hv + ng[0], hv + ng[0] + ng[1], hv + ng[0] + ng[1] + ng[2]};
  const long long cells = (long long)t->n_programs * t->max_stages * K;
  chm::prof::begin(chm::prof::K_EVAL, st);
  for (int level = 0; level < 4; ++level) {
    if (cudaMemsetAsync(cursor, 0, 8, st) != cudaSuccess) return CHM_ERR_CUDA;
    train_entries_kernel<<<grid_of(cells), 256, 0, st>>>(*t, workflow, s_cap, level, id0, v0,
                                                           cursor);
    uint64_t *a1 = id0, *a2 = v0, *b1 = id1, *b2 = v1;
    for (int64_t w = 1; w < n; w *= 2) {
      merge_level<true, false><<<grid_of(n), 256, 0, st>>>(a1, a2, b1, b2, n, w, nullptr);
      std::swap(a1, b1);
      std::swap(a2, b2);
    }
    group_quantile_kernel<<<(unsigned)((ng[level] + 255) / 256), 256, 0, st>>>(
        a1, a2, n, ng[level], quantile, qs[level], hs[level]);
  }
  const int cells_t = (n_wf + 1) * (s_cap + 1) * K;
  table_kernel<<<(unsigned)((cells_t + 255) / 256), 256, 0, st>>>(
      qs[0], hs[0], qs[1], hs[1], qs[2], hs[2], qs[3], n_wf, s_cap, K, table);
  chm::prof::end(chm::prof::K_EVAL, st, (double)n * 4 * 16.0);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" uint64_t chm_kendall_tau_scratch_bytes(int64_t n) {
  if (n < 0) return 0;
  return (uint64_t)n * 6 * 8 + 64;
}

extern "C" chm_status chm_kendall_tau_distance(const double* predicted, const double* truth,
                                               int64_t n, void* scratch, uint64_t scratch_bytes,
                                               double* result, int64_t* counts_out,
                                               void* stream) {
  using namespace chm::eval;
  if (!predicted || !truth || !scratch || !result || n < 2) return CHM_ERR_INVALID_ARG;
  if (scratch_bytes < chm_kendall_tau_scratch_bytes(n)) return CHM_ERR_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long* counts = reinterpret_cast<unsigned long long*>(scratch);  // 4 (+pad)
  uint64_t* buf = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(scratch) + 64);
  uint64_t *p0 = buf, *t0 = buf + n, *p1 = buf + 2 * n, *t1 = buf + 3 * n;
  uint64_t *c0 = buf + 4 * n, *c1 = buf + 5 * n;
  if (cudaMemsetAsync(counts, 0, 64, st) != cudaSuccess) return CHM_ERR_CUDA;
  chm::prof::begin(chm::prof::K_EVAL, st);
  keys_kernel<<<grid_of(n), 256, 0, st>>>(predicted, truth, n, p0, t0);
  // 1. sort by (predicted, truth)
  for (int64_t w = 1; w < n; w *= 2) {
    merge_level<true, false><<<grid_of(n), 256, 0, st>>>(p0, t0, p1, t1, n, w, nullptr);
    std::swap(p0, p1);
    std::swap(t0, t1);
  }
  // ties in predicted, and in (predicted, truth) jointly
  tie_pairs_kernel<false><<<grid_of(n), 256, 0, st>>>(p0, nullptr, n, counts + 1);
  tie_pairs_kernel<true><<<grid_of(n), 256, 0, st>>>(p0, t0, n, counts + 3);
  // 2. strict inversions of the truth column in that order (merge sort)
  if (cudaMemcpyAsync(c0, t0, (size_t)n * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return CHM_ERR_CUDA;
  for (int64_t w = 1; w < n; w *= 2) {
    merge_level<false, true><<<grid_of(n), 256, 0, st>>>(c0, nullptr, c1, nullptr, n, w,
                                                          counts + 0);
    std::swap(c0, c1);
  }
  // 3. ties in sorted(truth)
  tie_pairs_kernel<false><<<grid_of(n), 256, 0, st>>>(c0, nullptr, n, counts + 2);
  finish_kernel<<<1, 1, 0, st>>>(counts, n, result);
  int levels = 0;
  for (int64_t w = 1; w < n; w *= 2) ++levels;
  // bytes: keys 16 B/element/level (pair sort) + 8 B/element/level (inversions), writes alike
  chm::prof::end(chm::prof::K_EVAL, st, (double)n * levels * 48.0);
  if (counts_out &&
      cudaMemcpyAsync(counts_out, counts, 4 * 8, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
    return CHM_ERR_CUDA;
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}
