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

}  // namespace eval
}  // namespace chm

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
