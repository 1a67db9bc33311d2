// Completion path of the activity monitor:
// ActivityMonitor.record_completion (monitor.py:98-106) removes a finished
// request's prediction from the model's in-flight set, and the next
// in_flight_sum (monitor.py:122-129) is the builtin sum() -- Neumaier
// compensated on CPython 3.12 -- over the remaining entries in insertion
// order.
//
// Device form: one CTA per model. The batch's completion keys for the model
// are sorted in shared memory (bitonic), every live log entry binary-searches
// its key among them (found -> dead), the log is compacted in place (stable,
// so insertion order is kept), and (sum, comp) are recomputed over the
// survivors:
//   * exact fast path: if every live value is a multiple of 2^-8 below 2^36
//     and the total stays below 2^44, every partial sum of any order is exact
//     in fp64, so Neumaier returns the exact sum with zero compensation --
//     computed as a parallel int64 reduction (dyadic predictor tables, the
//     synthetic workloads);
//   * otherwise one thread replays the serial Neumaier recurrence in insertion
//     order (bit-identical to the reference for any values).
// A completion naming a request that is not in flight on that model is
// errors.UnknownRequest (monitor.py:104-105). The (program, stage) in-flight
// bit is cleared, so the same request id may be dispatched again.
#include <climits>
#include "common.cuh"
#include "prof.cuh"

namespace chm {
namespace mon {

constexpr int kThreads = 1024;
constexpr int kMaxPerModel = 8192;  // completions per model per call

__device__ __forceinline__ void neumaier_add(double& s, double& c, double x) {
  const double t = __dadd_rn(s, x);
  if (fabs(s) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
  else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
  s = t;
}

struct Smem {
  long long key[kMaxPerModel];
  int idx[kMaxPerModel];
  int found[kMaxPerModel];
  int scan[kThreads / 32];
  int misc[4];
  unsigned long long red[kThreads / 32];
  int dy[kThreads / 32];
};

__global__ void __launch_bounds__(kThreads) complete_kernel(chm_monitor_state mon,
                                                            const int32_t* __restrict__ model,
                                                            const int64_t* __restrict__ key, int n,
                                                            int32_t* n_complete, int32_t* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int m = blockIdx.x, K = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- this model's completions, in call order ----
  if (tid == 0) s.misc[0] = 0;
  __syncthreads();
  for (int b0 = 0; b0 < n; b0 += kThreads) {
    const int j = b0 + tid;
    const int mj = j < n ? model[j] : -1;
    if (j < n && (mj < 0 || mj >= K) && m == 0)
      report_error(err, CHM_ERR_VALIDATION, j, mj, 0);  // errors.UnknownModel
    const bool mine = j < n && mj == m;
    const unsigned bal = __ballot_sync(0xffffffffu, mine);
    if (lane == 0) s.scan[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = s.scan[lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      s.scan[lane] = incl - v;
      if (lane == 31) s.misc[1] = incl;
    }
    __syncthreads();
    if (mine) {
      const int pos = s.misc[0] + s.scan[warp] + __popc(bal & ((1u << lane) - 1u));
      if (pos < kMaxPerModel) {
        s.key[pos] = key[j];
        s.idx[pos] = j;
      }
    }
    __syncthreads();
    if (tid == 0) s.misc[0] += s.misc[1];
    __syncthreads();
  }
  const int nm = s.misc[0];
  if (nm > kMaxPerModel) {
    if (tid == 0) report_error(err, CHM_ERR_UNSUPPORTED, 0, m, nm);
    return;
  }
  if (n_complete && tid == 0) n_complete[m] = nm;
  if (nm == 0) return;
  // ---- bitonic sort of (key, idx) by key over the next power of two ----
  int np2 = 1;
  while (np2 < nm) np2 <<= 1;
  for (int i = nm + tid; i < np2; i += kThreads) {
    s.key[i] = LLONG_MAX;
    s.idx[i] = -1;
  }
  for (int i = tid; i < np2; i += kThreads) s.found[i] = 0;
  __syncthreads();
  for (int size = 2; size <= np2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < np2; i += kThreads) {
        const int pr = i ^ stride;
        if (pr > i) {
          const bool up = (i & size) == 0;
          const long long a = s.key[i], b = s.key[pr];
          if ((a > b) == up) {
            s.key[i] = b;
            s.key[pr] = a;
            const int t = s.idx[i];
            s.idx[i] = s.idx[pr];
            s.idx[pr] = t;
          }
        }
      }
      __syncthreads();
    }
  }
  // duplicate completions of one request: the second is unknown by then
  for (int i = tid + 1; i < nm; i += kThreads)
    if (s.key[i] == s.key[i - 1]) report_error(err, CHM_ERR_UNKNOWN_REQUEST, s.idx[i], m, 0);
  // ---- mark, then stable in-place compaction of the live log ----
  const size_t base = (size_t)m * mon.inflight_capacity;
  const int live = (int)mon.inflight_count[m];
  int out = 0;
  bool dyadic = true;
  unsigned long long fixed = 0;  // exact sum in units of 2^-8 (fast path)
  for (int b0 = 0; b0 < live; b0 += kThreads) {
    const int i = b0 + tid;
    long long kk = 0;
    double y = 0.0;
    bool keep = false;
    if (i < live) {
      kk = mon.inflight_key[base + i];
      y = mon.inflight_yhat[base + i];
      int lo = 0, hi = nm - 1, hit = -1;
      while (lo <= hi) {
        const int mid = (lo + hi) >> 1;
        const long long v = s.key[mid];
        if (v == kk) { hit = mid; break; }
        if (v < kk) lo = mid + 1; else hi = mid - 1;
      }
      if (hit >= 0) {
        // first occurrence among duplicates
        while (hit > 0 && s.key[hit - 1] == kk) --hit;
        s.found[hit] = 1;
        if (kk >= 0 && kk / 32 < mon.n_programs)
          atomicAnd(mon.stage_bits + kk / 32, ~(1u << (int)(kk & 31)));
      } else {
        keep = true;
        const double sc = y * 256.0;
        if (!(y >= 0.0 && y < 68719476736.0 && sc == floor(sc))) dyadic = false;
        else fixed += (unsigned long long)sc;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s.scan[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = s.scan[lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      s.scan[lane] = incl - v;
      if (lane == 31) s.misc[1] = incl;
    }
    __syncthreads();
    if (keep) {
      const size_t pos = base + out + s.scan[warp] + __popc(bal & ((1u << lane) - 1u));
      mon.inflight_key[pos] = kk;
      mon.inflight_yhat[pos] = y;
    }
    out += s.misc[1];
    __syncthreads();
  }
  // completions that matched nothing
  for (int i = tid; i < nm; i += kThreads)
    if (!s.found[i] && (i == 0 || s.key[i] != s.key[i - 1]))
      report_error(err, CHM_ERR_UNKNOWN_REQUEST, s.idx[i], m, 0);
  // ---- recompute (sum, comp) over the survivors ----
  for (int o = 16; o; o >>= 1) fixed += __shfl_xor_sync(0xffffffffu, fixed, o);
  const int dy_all = __all_sync(0xffffffffu, dyadic);
  if (lane == 0) {
    s.red[warp] = fixed;
    s.dy[warp] = dy_all;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long tot = 0;
    int ok = 1;
    for (int w = 0; w < kThreads / 32; ++w) {
      tot += s.red[w];
      ok &= s.dy[w];
    }
    double sum, comp = 0.0;
    if (ok && tot < (1ull << 52)) {  // total < 2^44 in units of 2^-8
      sum = (double)tot * (1.0 / 256.0);
    } else {
      sum = 0.0;
      for (int i = 0; i < out; ++i) neumaier_add(sum, comp, mon.inflight_yhat[base + i]);
    }
    mon.inflight_sum[m] = sum;
    mon.inflight_comp[m] = comp;
    mon.inflight_count[m] = out;
  }
}

}  // namespace mon
}  // namespace chm

extern "C" chm_status chm_monitor_complete(const chm_pool* pool, const chm_monitor_state* mon,
                                           const int32_t* model, const int64_t* key, int32_t n,
                                           int32_t* n_complete, int32_t* error, void* stream) {
  if (!pool || !mon || n < 0 || (n > 0 && (!model || !key))) return CHM_ERR_INVALID_ARG;
  if (!mon->inflight_key || !mon->inflight_yhat || mon->inflight_capacity < 1)
    return CHM_ERR_UNSUPPORTED;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = sizeof(chm::mon::Smem);
  cudaFuncSetAttribute(chm::mon::complete_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  chm::prof::begin(chm::prof::K_PREPARE, s);
  chm::mon::complete_kernel<<<K, chm::mon::kThreads, smem, s>>>(*mon, model, key, n, n_complete,
                                                                 error);
  // bytes: the completion list per model + live log read + survivors written
  chm::prof::end(chm::prof::K_PREPARE, s, (double)n * 12.0 * K);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}
