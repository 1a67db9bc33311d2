// Multi-GPU exchange of the activity monitor: request batches
// shard across GPUs by program, so the only cross-GPU state is the
// per-engine in-flight predicted-token vector P (K doubles, CPython's
// Neumaier (sum, comp) pair per engine, monitor.py:122-129).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2 -- in a PyTorch process
// the one torch already mapped), so the library keeps no link-time NCCL
// dependency; nccl.h supplies only the types.
//
// Canonical tick-end state (both modes): P_prev folded with rank 0's
// dispatches in row order, then rank 1's, ... -- exactly the monitor of ONE
// serial schedule_request loop over the concatenated batch.
//   Mode A (chm_allreduce_inflight): every rank's chain starts from the
//     tick-start P; afterwards each rank packs its committed (model, yhat)
//     rows, one ncclAllGather moves them, and every rank folds them in rank
//     order on the device. When every value is a multiple of 2^-8 and the
//     totals stay below 2^45 the fold is an int64 sum (every partial sum of
//     any order is exact in fp64, compensation 0); otherwise K threads replay
//     the Neumaier recurrence over the gathered rows.
//   Mode B (chm_inflight_relay_recv / _send): rank g receives (s, c) from
//     g-1 right before its selection kernel, sends it on after, and the last
//     rank broadcasts the tick-end state. The routers and predictors run
//     before the receive, so they overlap the predecessors' chains.
// Sharded completions: every rank's in-flight log holds only its own
// dispatches, so after record_completion each rank reduces its survivors
// exactly (int64 units of 2^-8, chm_inflight_local_sum), the sums are
// all-reduced, and chm_inflight_set_sum installs the global exact sum (the
// builtin sum() of the survivors in any order, compensation 0). Non-dyadic
// survivors have no order-free exact sum: set_sum reports UNSUPPORTED and the
// host takes the merge path -- every rank packs its survivors with their
// global insertion stamps (chm_inflight_pack_live), the lists are
// all-gathered, and chm_inflight_merge_sum replays the Neumaier recurrence in
// the merged insertion order on every rank.
#include <dlfcn.h>
#include <nccl.h>
#include <climits>
#include <cstring>
#include <mutex>
#include "common.cuh"

namespace chm {
namespace comm {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  bool ok = false;
};

static Nccl g_nccl;
static std::once_flag g_once;

static void load_nccl() {
  const char* names[] = {getenv("CHM_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names)
    if (n && (h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
  if (!h) return;
  Nccl& f = g_nccl;
#define CHM_SYM(field, name) f.field = reinterpret_cast<decltype(f.field)>(dlsym(h, name))
  CHM_SYM(GetUniqueId, "ncclGetUniqueId");
  CHM_SYM(CommInitRank, "ncclCommInitRank");
  CHM_SYM(CommDestroy, "ncclCommDestroy");
  CHM_SYM(AllGather, "ncclAllGather");
  CHM_SYM(AllReduce, "ncclAllReduce");
  CHM_SYM(Broadcast, "ncclBroadcast");
  CHM_SYM(Send, "ncclSend");
  CHM_SYM(Recv, "ncclRecv");
  CHM_SYM(GroupStart, "ncclGroupStart");
  CHM_SYM(GroupEnd, "ncclGroupEnd");
#undef CHM_SYM
  f.ok = f.GetUniqueId && f.CommInitRank && f.CommDestroy && f.AllGather && f.AllReduce &&
         f.Broadcast && f.Send && f.Recv && f.GroupStart && f.GroupEnd;
}

static const Nccl* nccl() {
  std::call_once(g_once, load_nccl);
  return g_nccl.ok ? &g_nccl : nullptr;
}

// ---- Mode A record (one per rank, all-gathered) ---------------------------
// int64 words: [0] committed rows n, [1] dyadic flag, [2, 2+K) sum of the
// rank's dispatched values per engine in units of 2^-8 (valid when dyadic),
// then max_rows x {int64 model, double yhat} in row order.
constexpr int kHdr = 2;
constexpr double kScale = 256.0;            // units of 2^-8
constexpr double kMaxTerm = 536870912.0;    // 2^29 per value
constexpr long long kMaxUnits = 1ll << 53;  // totals exact below 2^45

__host__ __device__ inline size_t record_words(int K, int max_rows) {
  return (size_t)kHdr + CHM_MAX_MODELS + 2 * (size_t)max_rows;
}

__device__ __forceinline__ bool dyadic_term(double y) {
  const double sc = y * kScale;
  return y >= 0.0 && y < kMaxTerm && sc == trunc(sc);
}

__device__ __forceinline__ void neumaier_add(double& s, double& c, double x) {
  const double t = __dadd_rn(s, x);
  if (fabs(s) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
  else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
  s = t;
}

__global__ void __launch_bounds__(256) pack_kernel(int K, chm_decisions dec, int max_rows,
                                                  long long* __restrict__ rec) {
  const int n = *dec.n_committed;
  __shared__ unsigned long long s_units[CHM_MAX_MODELS];
  __shared__ int s_dy;
  if (threadIdx.x < CHM_MAX_MODELS) s_units[threadIdx.x] = 0;
  if (threadIdx.x == 0) s_dy = 1;
  __syncthreads();
  int dy = 1;
  double* rows = reinterpret_cast<double*>(rec + kHdr + CHM_MAX_MODELS);
  for (int i = threadIdx.x; i < max_rows; i += blockDim.x) {
    if (i < n) {
      const int m = dec.model[i];
      const double y = dec.priority[i];  // Decision.priority = the dispatched yhat
      reinterpret_cast<long long*>(rows)[2 * i] = m;
      rows[2 * i + 1] = y;
      if (dyadic_term(y)) atomicAdd(&s_units[m], (unsigned long long)(y * kScale));
      else dy = 0;
    } else {
      reinterpret_cast<long long*>(rows)[2 * i] = -1;
      rows[2 * i + 1] = 0.0;
    }
  }
  if (!dy) atomicAnd(&s_dy, 0);
  __syncthreads();
  if (threadIdx.x == 0) {
    rec[0] = n;
    rec[1] = s_dy;
  }
  if (threadIdx.x < CHM_MAX_MODELS)
    rec[kHdr + threadIdx.x] = threadIdx.x < K ? (long long)s_units[threadIdx.x] : 0;
}

// Fold the gathered records into (s, c) = the canonical tick-end state,
// starting from the tick-start (s0, c0). One thread per engine.
__global__ void __launch_bounds__(32) fold_kernel(int K, chm_monitor_state mon,
                                                  const double* __restrict__ s0,
                                                  const double* __restrict__ c0,
                                                  const long long* __restrict__ gathered,
                                                  int world, int max_rows, int32_t* err) {
  const int m = threadIdx.x;
  if (m >= K) return;
  const size_t words = record_words(K, max_rows);
  bool dy = c0[m] == 0.0 && s0[m] >= 0.0 && s0[m] * kScale == trunc(s0[m] * kScale) &&
            s0[m] < 35184372088832.0;  // 2^45
  long long units = dy ? (long long)(s0[m] * kScale) : 0;
  for (int g = 0; g < world && dy; ++g) {
    const long long* r = gathered + (size_t)g * words;
    dy = r[1] != 0;
    units += r[kHdr + m];
    dy = dy && units < kMaxUnits;
  }
  double s, c;
  if (dy) {
    s = (double)units / kScale;
    c = 0.0;
  } else {
    s = s0[m];
    c = c0[m];
    for (int g = 0; g < world; ++g) {
      const long long* r = gathered + (size_t)g * words;
      const int n = (int)r[0];
      const long long* rows = r + kHdr + CHM_MAX_MODELS;
      for (int i = 0; i < n; ++i)
        if (rows[2 * i] == m) neumaier_add(s, c, __longlong_as_double(rows[2 * i + 1]));
    }
  }
  mon.inflight_sum[m] = s;
  mon.inflight_comp[m] = c;
  (void)err;
}

// Exact per-engine sum of this rank's live log entries (units of 2^-8) and a
// flag word (1 = some entry is not dyadic): out[0..K), out[K].
__global__ void __launch_bounds__(1024) local_sum_kernel(chm_monitor_state mon,
                                                        long long* __restrict__ out, int K) {
  const int m = blockIdx.x;
  const int n = (int)mon.inflight_count[m];
  const size_t base = (size_t)m * mon.inflight_capacity;
  unsigned long long u = 0;
  int bad = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double y = mon.inflight_yhat[base + i];
    if (mon.inflight_progress) {  // decay_in_flight: max(y - progress, 0) (monitor.py:122-129)
      const double d = __dsub_rn(y, mon.inflight_progress[base + i]);
      y = (0.0 > d) ? 0.0 : d;
    }
    if (dyadic_term(y)) u += (unsigned long long)(y * kScale);
    else bad = 1;
  }
  __shared__ unsigned long long s_u;
  __shared__ int s_bad;
  if (threadIdx.x == 0) {
    s_u = 0;
    s_bad = 0;
  }
  __syncthreads();
  for (int o = 16; o; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
  bad = __any_sync(0xffffffffu, bad);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_u, u);
    if (bad) atomicOr(&s_bad, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[m] = (long long)s_u;
    if (s_bad) atomicAdd(reinterpret_cast<unsigned long long*>(out + K), 1ull);
  }
}

__global__ void zero_flag_kernel(long long* out, int K) { out[K] = 0; }

// (stamp, live term) of this rank's log, per engine, padded to cap.
__global__ void __launch_bounds__(1024) pack_live_kernel(chm_monitor_state mon, int cap,
                                                        long long* __restrict__ rec) {
  const int m = blockIdx.x;
  const int n = (int)mon.inflight_count[m];
  const size_t base = (size_t)m * mon.inflight_capacity;
  long long* out = rec + (size_t)m * cap * 2;
  for (int i = threadIdx.x; i < cap; i += blockDim.x) {
    long long st = LLONG_MAX;
    double y = 0.0;
    if (i < n) {
      st = mon.inflight_stamp[base + i];
      y = mon.inflight_yhat[base + i];
      if (mon.inflight_progress) {  // decay_in_flight (monitor.py:122-129)
        const double d = __dsub_rn(y, mon.inflight_progress[base + i]);
        y = (0.0 > d) ? 0.0 : d;
      }
    }
    out[2 * i] = st;
    out[2 * i + 1] = __double_as_longlong(y);
  }
}

// Per engine (one thread): merge the G stamp-ordered survivor lists and
// replay builtin sum()'s Neumaier recurrence in that order.
__global__ void merge_sum_kernel(chm_monitor_state mon, const long long* __restrict__ gathered,
                                 const long long* __restrict__ counts, int G, int K, int cap) {
  const int m = threadIdx.x;
  if (m >= K) return;
  int pos[64];
  for (int g = 0; g < G; ++g) pos[g] = 0;
  double s = 0.0, c = 0.0;
  while (true) {
    int best = -1;
    long long bs = LLONG_MAX;
    for (int g = 0; g < G; ++g) {
      if (pos[g] >= (int)counts[(size_t)g * K + m]) continue;
      const long long st = gathered[(((size_t)g * K + m) * cap + pos[g]) * 2];
      if (st < bs) {
        bs = st;
        best = g;
      }
    }
    if (best < 0) break;
    const double y =
        __longlong_as_double(gathered[(((size_t)best * K + m) * cap + pos[best]) * 2 + 1]);
    neumaier_add(s, c, y);
    ++pos[best];
  }
  mon.inflight_sum[m] = s;
  mon.inflight_comp[m] = c;
}

__global__ void set_sum_kernel(chm_monitor_state mon, const long long* __restrict__ summed, int K,
                               int32_t* err) {
  const int m = threadIdx.x;
  if (m >= K) return;
  bool exact = summed[K] == 0;
  for (int k = 0; k < K; ++k) exact = exact && summed[k] < kMaxUnits;
  if (!exact) {  // no order-free exact sum: the merge path (or the error) follows
    if (m == 0 && err) report_error(err, CHM_ERR_UNSUPPORTED, 0, -1, 2);
    return;
  }
  mon.inflight_sum[m] = (double)summed[m] / kScale;
  mon.inflight_comp[m] = 0.0;
}

}  // namespace comm
}  // namespace chm

struct chm_comm {
  ncclComm_t nc = nullptr;
  int rank = 0, world = 1;
};

using chm::comm::nccl;

#define CHM_NCCL(call)                                \
  do {                                                \
    if ((call) != ncclSuccess) return CHM_ERR_NCCL;   \
  } while (0)

extern "C" chm_status chm_comm_available(void) {
  return nccl() ? CHM_OK : CHM_ERR_NCCL;
}

extern "C" chm_status chm_comm_unique_id(uint8_t* id_out) {
  if (!id_out) return CHM_ERR_INVALID_ARG;
  const auto* f = nccl();
  if (!f) return CHM_ERR_NCCL;
  ncclUniqueId id;
  CHM_NCCL(f->GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == CHM_COMM_ID_BYTES, "ncclUniqueId size");
  memcpy(id_out, &id, sizeof(id));
  return CHM_OK;
}

extern "C" chm_status chm_comm_init(const uint8_t* id, int32_t rank, int32_t world,
                                    int32_t device, chm_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return CHM_ERR_INVALID_ARG;
  const auto* f = nccl();
  if (!f) return CHM_ERR_NCCL;
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return CHM_ERR_CUDA;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  chm_comm* c = new chm_comm();
  c->rank = rank;
  c->world = world;
  if (f->CommInitRank(&c->nc, world, uid, rank) != ncclSuccess) {
    delete c;
    return CHM_ERR_NCCL;
  }
  *out = c;
  return CHM_OK;
}

extern "C" chm_status chm_comm_destroy(chm_comm* c) {
  if (!c) return CHM_ERR_INVALID_ARG;
  const auto* f = nccl();
  if (f && c->nc) f->CommDestroy(c->nc);
  delete c;
  return CHM_OK;
}

extern "C" chm_status chm_comm_allgather(chm_comm* c, const void* send, void* recv,
                                         uint64_t bytes, void* stream) {
  if (!c || !send || !recv) return CHM_ERR_INVALID_ARG;
  const auto* f = nccl();
  if (!f) return CHM_ERR_NCCL;
  CHM_NCCL(f->AllGather(send, recv, bytes, ncclUint8, c->nc, (cudaStream_t)stream));
  return CHM_OK;
}

extern "C" chm_status chm_comm_allreduce_i64(chm_comm* c, int64_t* buf, int32_t n,
                                             void* stream) {
  if (!c || !buf || n < 0) return CHM_ERR_INVALID_ARG;
  const auto* f = nccl();
  if (!f) return CHM_ERR_NCCL;
  CHM_NCCL(f->AllReduce(buf, buf, (size_t)n, ncclInt64, ncclSum, c->nc, (cudaStream_t)stream));
  return CHM_OK;
}

extern "C" uint64_t chm_inflight_record_bytes(int32_t n_models, int32_t max_rows) {
  if (n_models < 1 || n_models > CHM_MAX_MODELS || max_rows < 0) return 0;
  return 8ull * chm::comm::record_words(n_models, max_rows);
}

extern "C" chm_status chm_inflight_pack(const chm_pool* pool, const chm_decisions* dec,
                                        int32_t max_rows, void* record, void* stream) {
  if (!pool || !dec || !record || !dec->model || !dec->priority || !dec->n_committed ||
      max_rows < 0)
    return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  chm::comm::pack_kernel<<<1, 256, 0, (cudaStream_t)stream>>>(
      K, *dec, max_rows, reinterpret_cast<long long*>(record));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_inflight_fold(const chm_pool* pool, const chm_monitor_state* mon,
                                        const double* s0, const double* c0,
                                        const void* gathered, int32_t world, int32_t max_rows,
                                        int32_t* error, void* stream) {
  if (!pool || !mon || !s0 || !c0 || !gathered || world < 1 || max_rows < 0)
    return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  chm::comm::fold_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
      K, *mon, s0, c0, reinterpret_cast<const long long*>(gathered), world, max_rows, error);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_allreduce_inflight(chm_comm* c, const chm_pool* pool,
                                             const chm_monitor_state* mon, const double* s0,
                                             const double* c0, const chm_decisions* dec,
                                             int32_t max_rows, void* workspace,
                                             int32_t* error, void* stream) {
  if (!c || !workspace) return CHM_ERR_INVALID_ARG;
  const uint64_t rb = chm_inflight_record_bytes(pool ? pool->n_models : 0, max_rows);
  if (!rb) return CHM_ERR_INVALID_ARG;
  uint8_t* own = reinterpret_cast<uint8_t*>(workspace);
  uint8_t* all = own + rb;
  chm_status st = chm_inflight_pack(pool, dec, max_rows, own, stream);
  if (st != CHM_OK) return st;
  st = chm_comm_allgather(c, own, all, rb, stream);
  if (st != CHM_OK) return st;
  return chm_inflight_fold(pool, mon, s0, c0, all, c->world, max_rows, error, stream);
}

extern "C" chm_status chm_inflight_relay_recv(chm_comm* c, double* state, int32_t n,
                                              void* stream) {
  if (!c || !state || n < 0) return CHM_ERR_INVALID_ARG;
  const auto* f = nccl();
  if (!f) return CHM_ERR_NCCL;
  if (c->rank > 0)
    CHM_NCCL(f->Recv(state, (size_t)n, ncclFloat64, c->rank - 1, c->nc, (cudaStream_t)stream));
  return CHM_OK;
}

extern "C" chm_status chm_inflight_relay_send(chm_comm* c, double* state, int32_t n,
                                              void* stream) {
  if (!c || !state || n < 0) return CHM_ERR_INVALID_ARG;
  const auto* f = nccl();
  if (!f) return CHM_ERR_NCCL;
  cudaStream_t s = (cudaStream_t)stream;
  if (c->rank + 1 < c->world)
    CHM_NCCL(f->Send(state, (size_t)n, ncclFloat64, c->rank + 1, c->nc, s));
  CHM_NCCL(f->Broadcast(state, state, (size_t)n, ncclFloat64, c->world - 1, c->nc, s));
  return CHM_OK;
}

extern "C" chm_status chm_inflight_local_sum(const chm_pool* pool, const chm_monitor_state* mon,
                                             int64_t* out, void* stream) {
  if (!pool || !mon || !out || !mon->inflight_key) return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  chm::comm::zero_flag_kernel<<<1, 1, 0, s>>>(reinterpret_cast<long long*>(out), K);
  chm::comm::local_sum_kernel<<<K, 1024, 0, s>>>(*mon, reinterpret_cast<long long*>(out), K);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_inflight_set_sum(const chm_pool* pool, const chm_monitor_state* mon,
                                           const int64_t* summed, int32_t* error, void* stream) {
  if (!pool || !mon || !summed) return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  chm::comm::set_sum_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
      *mon, reinterpret_cast<const long long*>(summed), K, error);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_inflight_pack_live(const chm_pool* pool, const chm_monitor_state* mon,
                                             int32_t cap, void* records, void* stream) {
  if (!pool || !mon || !records || cap < 0 || !mon->inflight_stamp) return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  if (cap == 0) return CHM_OK;
  chm::comm::pack_live_kernel<<<K, 1024, 0, (cudaStream_t)stream>>>(
      *mon, cap, reinterpret_cast<long long*>(records));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_inflight_merge_sum(const chm_pool* pool, const chm_monitor_state* mon,
                                             const void* gathered, const int64_t* counts,
                                             int32_t world, int32_t cap, void* stream) {
  if (!pool || !mon || !gathered || !counts || world < 1 || world > 64 || cap < 0)
    return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  chm::comm::merge_sum_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(
      *mon, reinterpret_cast<const long long*>(gathered),
      reinterpret_cast<const long long*>(counts), world, K, cap);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}
