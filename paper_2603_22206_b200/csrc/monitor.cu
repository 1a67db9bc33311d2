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
// With decay_in_flight (monitor.inflight_progress != NULL) the recomputed sum
// is over max(yhat - progress, 0) (monitor.py:122-129), and
// chm_monitor_note_progress sets the progress column (monitor.py:108-111).
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

// The term one live entry contributes to in_flight_sum (monitor.py:122-129):
// y, or with decay Python's max(y - progress, 0.0) (first argument unless 0.0
// is strictly greater).
__device__ __forceinline__ double live_term(double y, const double* prog, size_t at) {
  if (!prog) return y;
  const double d = __dsub_rn(y, prog[at]);
  return (0.0 > d) ? 0.0 : d;
}

// (sum, comp) of model m's n_live entries in insertion order, as CPython 3.12
// sum() leaves them (Neumaier):
//   * exact fast path: every term a multiple of 2^-8 below 2^36 and the total
//     below 2^44 -> every partial sum is exact in fp64 in any order and the
//     compensation is exactly 0: a parallel int64 reduction;
//   * otherwise one thread replays the recurrence in insertion order.
// Block-wide (all threads call it); writes sum / comp / count of model m.
__device__ void recompute_sum(const chm_monitor_state& mon, int m, int n_live,
                              unsigned long long* red, int* dy) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t base = (size_t)m * mon.inflight_capacity;
  bool dyadic = true;
  unsigned long long fixed = 0;  // exact sum in units of 2^-8
  for (int i = tid; i < n_live; i += blockDim.x) {
    const double y = live_term(mon.inflight_yhat[base + i], mon.inflight_progress, base + i);
    const double sc = y * 256.0;
    if (!(y >= 0.0 && y < 68719476736.0 && sc == floor(sc))) dyadic = false;
    else fixed += (unsigned long long)sc;
  }
  for (int o = 16; o; o >>= 1) fixed += __shfl_xor_sync(0xffffffffu, fixed, o);
  const int dy_all = __all_sync(0xffffffffu, dyadic);
  if (lane == 0) {
    red[warp] = fixed;
    dy[warp] = dy_all;
  }
  __syncthreads();
  if (tid == 0) {
    unsigned long long tot = 0;
    int ok = 1;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      tot += red[w];
      ok &= dy[w];
    }
    double sum, comp = 0.0;
    if (ok && tot < (1ull << 52)) {  // total < 2^44 in units of 2^-8
      sum = (double)tot * (1.0 / 256.0);
    } else {
      sum = 0.0;
      for (int i = 0; i < n_live; ++i)
        neumaier_add(sum, comp,
                     live_term(mon.inflight_yhat[base + i], mon.inflight_progress, base + i));
    }
    mon.inflight_sum[m] = sum;
    mon.inflight_comp[m] = comp;
    mon.inflight_count[m] = n_live;
  }
}

// This model's entries of the call's (model, key) list, sorted by (key, call
// index) in shared memory (bitonic over the next power of two). Returns the
// count, or -1 when it exceeds kMaxPerModel (reported).
__device__ int gather_sorted(Smem& s, int m, int K, const int32_t* __restrict__ model,
                             const int64_t* __restrict__ key, int n, int32_t* err,
                             bool unknown_model_is_error) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s.misc[0] = 0;
  __syncthreads();
  for (int b0 = 0; b0 < n; b0 += kThreads) {
    const int j = b0 + tid;
    const int mj = j < n ? model[j] : -1;
    if (unknown_model_is_error && j < n && (mj < 0 || mj >= K) && m == 0)
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
    return -1;
  }
  if (nm == 0) return 0;
  int np2 = 1;
  while (np2 < nm) np2 <<= 1;
  for (int i = nm + tid; i < np2; i += kThreads) {
    s.key[i] = LLONG_MAX;
    s.idx[i] = INT_MAX;
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
          const bool gt = a > b || (a == b && s.idx[i] > s.idx[pr]);  // (key, call order)
          if (gt == up) {
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
  return nm;
}

__device__ __forceinline__ int find_key(const Smem& s, int nm, long long kk) {
  int lo = 0, hi = nm - 1;
  while (lo <= hi) {
    const int mid = (lo + hi) >> 1;
    const long long v = s.key[mid];
    if (v == kk) return mid;
    if (v < kk) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

__global__ void __launch_bounds__(kThreads) complete_kernel(chm_monitor_state mon,
                                                            const int32_t* __restrict__ model,
                                                            const int64_t* __restrict__ key, int n,
                                                            int32_t* n_complete, int32_t* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int m = blockIdx.x, K = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nm = gather_sorted(s, m, K, model, key, n, err, true);
  if (nm < 0) return;
  if (n_complete && tid == 0) n_complete[m] = nm;
  if (nm == 0) return;
  // duplicate completions of one request: the second is unknown by then
  for (int i = tid + 1; i < nm; i += kThreads)
    if (s.key[i] == s.key[i - 1]) report_error(err, CHM_ERR_UNKNOWN_REQUEST, s.idx[i], m, 0);
  // ---- mark, then stable in-place compaction of the live log ----
  const size_t base = (size_t)m * mon.inflight_capacity;
  const int live = (int)mon.inflight_count[m];
  int out = 0;
  double* prog = mon.inflight_progress;
  for (int b0 = 0; b0 < live; b0 += kThreads) {
    const int i = b0 + tid;
    long long kk = 0, sp = 0;
    double y = 0.0, pg = 0.0;
    bool keep = false;
    if (i < live) {
      kk = mon.inflight_key[base + i];
      y = mon.inflight_yhat[base + i];
      if (prog) pg = prog[base + i];
      if (mon.inflight_stamp) sp = mon.inflight_stamp[base + i];
      int hit = find_key(s, nm, kk);
      if (hit >= 0) {
        // first occurrence among duplicates
        while (hit > 0 && s.key[hit - 1] == kk) --hit;
        s.found[hit] = 1;
        if (kk >= 0 && kk / 32 < mon.n_programs)
          atomicAnd(mon.stage_bits + kk / 32, ~(1u << (int)(kk & 31)));
      } else {
        keep = true;
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
    // (all reads of this block of entries precede the writes: the barrier
    // above; writes go to positions <= the read positions, stable order)
    if (keep) {
      const size_t pos = base + out + s.scan[warp] + __popc(bal & ((1u << lane) - 1u));
      mon.inflight_key[pos] = kk;
      mon.inflight_yhat[pos] = y;
      if (prog) prog[pos] = pg;
      if (mon.inflight_stamp) mon.inflight_stamp[pos] = sp;
    }
    out += s.misc[1];
    __syncthreads();
  }
  // completions that matched nothing
  for (int i = tid; i < nm; i += kThreads)
    if (!s.found[i] && (i == 0 || s.key[i] != s.key[i - 1]))
      report_error(err, CHM_ERR_UNKNOWN_REQUEST, s.idx[i], m, 0);
  __syncthreads();
  recompute_sum(mon, m, out, s.red, s.dy);
}

// ActivityMonitor.note_progress for this model's updates, then the decayed sum.
__global__ void __launch_bounds__(kThreads) progress_kernel(chm_monitor_state mon,
                                                            const int32_t* __restrict__ model,
                                                            const int64_t* __restrict__ key,
                                                            const double* __restrict__ emitted,
                                                            int n, int32_t* err) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem& s = *reinterpret_cast<Smem*>(smem_raw);
  const int m = blockIdx.x, K = gridDim.x;
  // note_progress ignores unknown models and requests not in flight
  const int nm = gather_sorted(s, m, K, model, key, n, err, false);
  if (nm < 0) return;
  const size_t base = (size_t)m * mon.inflight_capacity;
  const int live = (int)mon.inflight_count[m];
  if (nm > 0) {
    for (int i = threadIdx.x; i < live; i += kThreads) {
      const long long kk = mon.inflight_key[base + i];
      int hit = find_key(s, nm, kk);
      if (hit >= 0) {
        while (hit + 1 < nm && s.key[hit + 1] == kk) ++hit;  // the last call wins
        mon.inflight_progress[base + i] = emitted[s.idx[hit]];
      }
    }
  }
  __syncthreads();
  recompute_sum(mon, m, live, s.red, s.dy);
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

extern "C" chm_status chm_monitor_note_progress(const chm_pool* pool,
                                                const chm_monitor_state* mon,
                                                const int32_t* model, const int64_t* key,
                                                const double* emitted, int32_t n,
                                                int32_t* error, void* stream) {
  if (!pool || !mon || n < 0 || (n > 0 && (!model || !key || !emitted)))
    return CHM_ERR_INVALID_ARG;
  if (!mon->inflight_key || !mon->inflight_yhat || !mon->inflight_progress ||
      mon->inflight_capacity < 1)
    return CHM_ERR_UNSUPPORTED;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t smem = sizeof(chm::mon::Smem);
  cudaFuncSetAttribute(chm::mon::progress_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  chm::prof::begin(chm::prof::K_PREPARE, s);
  chm::mon::progress_kernel<<<K, chm::mon::kThreads, smem, s>>>(*mon, model, key, emitted, n,
                                                                 error);
  chm::prof::end(chm::prof::K_PREPARE, s, (double)n * 20.0 * K);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}
