// Columnar trace store on the device: the fields of
// hetsched's TraceRecord that the scheduling path reads, as dense SoA columns,
// plus the two derived columns the path needs every tick:
//
//   remaining[p, s, m]      = sum_{j >= s} out_tokens[p, j, m]
//                             TraceRecord.remaining_tokens (workload.py:160-165),
//                             the OraclePredictor feature (predictor.py:30-36)
//   carried_prefix[p, s, m] = sum_{j < s} carried_context[p, j, m]
//                             next_stage_request's carried context
//                             (workload.py:467-495: input = base + carried)
//
// Layout (s 0-based, padded to max_stages S, m in pool order):
//   n_stages i32[NP], workflow i32[NP], user_arrival f64[NP], base i32[NP*S],
//   out_tokens / carried i32[NP*S*K], remaining / carried_prefix i64[NP*S*K].
// Program p's S*K block is contiguous, so a chunk of programs is one
// contiguous span: chm_trace_derive moves whole chunks between HBM and shared
// memory with 1D TMA bulk copies, pipelined (HBM bound: 8 bytes read + 16
// written per entry, + 4 per (program, stage) and per program for validation).
//
// Per-row consumers: chm_trace_gather_rows (out_tokens for EngineSim.enqueue,
// oracle predictions, workflow index), chm_trace_next_stage (stage chaining
// for completions, order-preserving compaction), chm_trace_first_stage.
#include <stdlib.h>
#include "common.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace trace {

constexpr int kDeriveThreads = 256;
constexpr int kInStages = 4;    // input chunks in flight per CTA (bulk loads)
constexpr int kOutStages = 2;   // output chunks being stored per CTA (bulk stores)
constexpr int kChunkEntries = 1024;  // target (program, stage, model) entries per chunk

// Programs per chunk: a multiple of 4 (every span is then a multiple of 16
// bytes) holding about `entries` entries.
__host__ __device__ inline int chunk_programs(int S, int K, int entries) {
  int p = entries / (S * K);
  p &= ~3;
  return p < 4 ? 4 : p;
}

// Shared-memory layout of one CTA (offsets in bytes, all 16-aligned).
struct DeriveSmem {
  int P, span;  // programs / entries per chunk
  size_t in_stage, out_stage, in_off, out_off, bar_off, total;
  __host__ __device__ DeriveSmem(int S, int K, int entries) {
    P = chunk_programs(S, K, entries);
    span = P * S * K;
    // per input stage: out_tokens + carried (4 B each per entry), base_input
    // (4 B per program-stage), n_stages (4 B per program)
    in_stage = (size_t)span * 8 + (size_t)P * S * 4 + (size_t)P * 4;
    in_stage = (in_stage + 15) & ~size_t(15);
    out_stage = (size_t)span * 16;  // remaining + carried_prefix (8 B each)
    in_off = 0;
    out_off = in_off + kInStages * in_stage;
    bar_off = out_off + kOutStages * out_stage;
    total = bar_off + kInStages * sizeof(uint64_t);
  }
};

// Derive one chunk from staged inputs into staged outputs (shared memory).
__device__ __forceinline__ void derive_chunk(const int* s_out, const int* s_car, const int* s_base,
                                             const int* s_ns, long long* s_rem, long long* s_pre,
                                             long long p0, int np, int S, int K, int32_t* err) {
  for (int pk = threadIdx.x; pk < np * K; pk += blockDim.x) {
    const int lp = pk / K, k = pk - lp * K;
    const long long p = p0 + lp;
    const int ns = s_ns[lp];
    if (ns < 1 || ns > S) {
      report_error(err, CHM_ERR_VALIDATION, (int32_t)p, -1, ns);
      for (int j = 0; j < S; ++j) {
        s_rem[(lp * S + j) * K + k] = 0;
        s_pre[(lp * S + j) * K + k] = 0;
      }
      continue;
    }
    // TraceRecord.validate (workload.py:185-200): non-negative token counts,
    // base_input_tokens >= 1 (checked once per program, by k == 0)
    long long pre = 0;
    for (int j = 0; j < S; ++j) {
      const int at = (lp * S + j) * K + k;
      s_pre[at] = j < ns ? pre : 0;
      if (j < ns) {
        const int cv = s_car[at], ov = s_out[at];
        if (cv < 0 || ov < 0) report_error(err, CHM_ERR_VALIDATION, (int32_t)p, k, j + 1);
        if (k == 0 && s_base[lp * S + j] < 1)
          report_error(err, CHM_ERR_VALIDATION, (int32_t)p, -1, j + 1);
        pre += cv;
      }
    }
    long long rem = 0;
    for (int j = S - 1; j >= 0; --j) {
      const int at = (lp * S + j) * K + k;
      if (j < ns) rem += s_out[at];
      s_rem[at] = j < ns ? rem : 0;
    }
  }
}

// Persistent CTAs over full chunks. Inputs arrive by 1D TMA bulk copies into
// a kInStages ring (mbarrier completion), outputs leave by TMA bulk stores
// from a kOutStages ring, so HBM reads of the next chunks, the integer scans
// of this one and the stores of the previous ones overlap. The final partial
// chunk (fewer than P programs) goes through plain loads and stores.
__global__ void __launch_bounds__(kDeriveThreads) derive_kernel(chm_trace t, int entries,
                                                                int32_t* err) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = t.max_stages, K = t.n_models;
  const DeriveSmem L(S, K, entries);
  const int P = L.P, span = L.span;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  const long long n_full = (long long)t.n_programs / P;
  const long long n_mine = blockIdx.x < n_full ? (n_full - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  auto in_ptr = [&](int st) { return smem + L.in_off + st * L.in_stage; };
  auto issue = [&](long long it) {  // thread 0: bulk loads of my it-th chunk
    const int st = (int)(it % kInStages);
    const long long p0 = (blockIdx.x + it * gridDim.x) * (long long)P;
    unsigned char* b = in_ptr(st);
    sm100::mbar_arrive_expect_tx(&bars[st], (uint32_t)(span * 8 + P * S * 4 + P * 4));
    sm100::bulk_load_1d(b, t.out_tokens + p0 * S * K, span * 4, &bars[st]);
    sm100::bulk_load_1d(b + span * 4, t.carried + p0 * S * K, span * 4, &bars[st]);
    sm100::bulk_load_1d(b + span * 8, t.base_input + p0 * S, P * S * 4, &bars[st]);
    sm100::bulk_load_1d(b + span * 8 + P * S * 4, t.n_stages + p0, P * 4, &bars[st]);
  };
  if (threadIdx.x == 0) {
    for (int i = 0; i < kInStages; ++i) sm100::mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (long long it = 0; it < n_mine && it < kInStages; ++it) issue(it);
  }
  __syncthreads();
  for (long long it = 0; it < n_mine; ++it) {
    const int st = (int)(it % kInStages), ob = (int)(it % kOutStages);
    const long long p0 = (blockIdx.x + it * gridDim.x) * (long long)P;
    sm100::mbar_wait(&bars[st], (uint32_t)((it / kInStages) & 1));
    if (threadIdx.x == 0) sm100::bulk_wait_read<kOutStages - 1>();  // output buffer ob free
    __syncthreads();
    const unsigned char* b = in_ptr(st);
    long long* o_rem = reinterpret_cast<long long*>(smem + L.out_off + ob * L.out_stage);
    long long* o_pre = o_rem + span;
    derive_chunk(reinterpret_cast<const int*>(b), reinterpret_cast<const int*>(b + span * 4),
                 reinterpret_cast<const int*>(b + span * 8),
                 reinterpret_cast<const int*>(b + span * 8 + P * S * 4), o_rem, o_pre, p0, P, S,
                 K, err);
    sm100::fence_proxy_async_smem();  // this thread's outputs -> visible to the bulk store
    __syncthreads();  // input stage consumed, output stage complete
    if (threadIdx.x == 0) {
      sm100::bulk_store_1d(t.remaining + p0 * S * K, o_rem, span * 8);
      sm100::bulk_store_1d(t.carried_prefix + p0 * S * K, o_pre, span * 8);
      sm100::bulk_commit();
      if (it + kInStages < n_mine) issue(it + kInStages);
    }
  }
  // partial tail chunk: the CTA that would own chunk n_full
  const int tail = (int)((long long)t.n_programs - n_full * P);
  if (tail > 0 && blockIdx.x == (int)(n_full % gridDim.x)) {
    const long long p0 = n_full * P;
    if (threadIdx.x == 0) sm100::bulk_wait_all();
    __syncthreads();
    unsigned char* b = in_ptr(0);
    int* s_out = reinterpret_cast<int*>(b);
    int* s_car = s_out + span;
    int* s_base = s_car + span;
    int* s_ns = s_base + P * S;
    const int n = tail * S * K;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      s_out[i] = t.out_tokens[p0 * S * K + i];
      s_car[i] = t.carried[p0 * S * K + i];
    }
    for (int i = threadIdx.x; i < tail * S; i += blockDim.x) s_base[i] = t.base_input[p0 * S + i];
    for (int i = threadIdx.x; i < tail; i += blockDim.x) s_ns[i] = t.n_stages[p0 + i];
    __syncthreads();
    long long* o_rem = reinterpret_cast<long long*>(smem + L.out_off);
    long long* o_pre = o_rem + span;
    derive_chunk(s_out, s_car, s_base, s_ns, o_rem, o_pre, p0, tail, S, K, err);
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      t.remaining[p0 * S * K + i] = o_rem[i];
      t.carried_prefix[p0 * S * K + i] = o_pre[i];
    }
  }
  if (threadIdx.x == 0) sm100::bulk_wait_all();
}

// Per (row, model): rows carry (program, 1-based stage).
__global__ void __launch_bounds__(256) gather_kernel(chm_trace t, const int32_t* __restrict__ program,
                                                     const int32_t* __restrict__ stage, int n_rows,
                                                     int32_t* __restrict__ out_tokens,
                                                     int32_t* __restrict__ workflow,
                                                     int32_t* __restrict__ n_stages_out,
                                                     double* __restrict__ oracle, int32_t* err) {
  const int S = t.max_stages, K = t.n_models;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)n_rows * K) return;
  const int i = (int)(idx / K), k = (int)(idx - (long long)i * K);
  const int p = program[i], s = stage[i];
  if (p < 0 || p >= t.n_programs) {
    if (k == 0) report_error(err, CHM_ERR_INVALID_ARG, i, -1, p);
    return;
  }
  const int ns = t.n_stages[p];
  if (k == 0) {
    if (workflow) workflow[i] = t.workflow[p];
    if (n_stages_out) n_stages_out[i] = ns;
  }
  // TraceRecord._stage (workload.py:143-147)
  if (s < 1 || s > ns) {
    if (k == 0) report_error(err, CHM_ERR_UNKNOWN_STAGE, i, -1, s);
    return;
  }
  const size_t at = ((size_t)p * S + (s - 1)) * K + k;
  if (out_tokens) out_tokens[idx] = t.out_tokens[at];
  if (oracle) oracle[idx] = (double)t.remaining[at];  // exact below 2^53
}

// next_stage_request for n completions, order-preserving compaction of the
// requests that have a next stage. One CTA (completions per tick << 10^6).
__global__ void __launch_bounds__(1024) next_stage_kernel(
    chm_trace t, const int32_t* __restrict__ program, const int32_t* __restrict__ completed,
    const double* __restrict__ time, const int8_t* __restrict__ model, int n,
    int32_t* __restrict__ next_program, int32_t* __restrict__ next_stage,
    double* __restrict__ next_arrival, int32_t* __restrict__ next_input,
    int32_t* __restrict__ next_workflow, int32_t* __restrict__ source_row,
    int32_t* __restrict__ n_next, int32_t* err) {
  const int S = t.max_stages, K = t.n_models;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, n_warps = blockDim.x >> 5;
  __shared__ int s_warp[32];
  __shared__ int s_total;
  int out_base = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + tid;
    bool emit = false;
    int p = 0, s = 0, m = 0;
    long long input = 0;
    if (i < n) {
      p = program[i];
      s = completed[i];
      m = model[i];
      if (p < 0 || p >= t.n_programs || m < 0 || m >= K) {
        report_error(err, CHM_ERR_INVALID_ARG, i, m, p);
      } else {
        const int ns = t.n_stages[p];
        if (s < 1 || s > ns) {
          report_error(err, CHM_ERR_UNKNOWN_STAGE, i, m, s);
        } else if (s < ns) {
          // stage s+1 (0-based index s): base + sum_{j=1..s} carried(j, m)
          input = (long long)t.base_input[(size_t)p * S + s] +
                  t.carried_prefix[((size_t)p * S + s) * K + m];
          if (input > 0x7fffffffLL) report_error(err, CHM_ERR_CAPACITY, i, m, 0);
          else emit = true;
        }
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, emit);
    const int wprefix = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = lane < n_warps ? s_warp[lane] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (lane < n_warps) s_warp[lane] = incl - v;
      if (lane == 31) s_total = incl;
    }
    __syncthreads();
    if (emit) {
      const int o = out_base + s_warp[warp] + wprefix;
      next_program[o] = p;
      next_stage[o] = s + 1;
      next_arrival[o] = time[i];  // arrival_time = completion_time
      next_input[o] = (int32_t)input;
      if (next_workflow) next_workflow[o] = t.workflow[p];
      if (source_row) source_row[o] = i;
    }
    out_base += s_total;
    __syncthreads();
  }
  if (tid == 0) *n_next = out_base;
}

// first_stage_request (workload.py:454-464)
__global__ void __launch_bounds__(256) first_stage_kernel(chm_trace t,
                                                          const int32_t* __restrict__ program,
                                                          const double* __restrict__ arrival_in,
                                                          int n, int32_t* __restrict__ input,
                                                          double* __restrict__ arrival,
                                                          int32_t* __restrict__ workflow,
                                                          int32_t* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int p = program[i];
  if (p < 0 || p >= t.n_programs) {
    report_error(err, CHM_ERR_INVALID_ARG, i, -1, p);
    return;
  }
  input[i] = t.base_input[(size_t)p * t.max_stages];
  arrival[i] = arrival_in ? arrival_in[i] : t.user_arrival[p];
  if (workflow) workflow[i] = t.workflow[p];
}

static int n_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

static bool valid(const chm_trace* t) {
  return t && t->n_programs >= 0 && t->max_stages >= 1 && t->max_stages <= CHM_MAX_STAGES &&
         t->n_models >= 1 && t->n_models <= CHM_MAX_MODELS;
}

}  // namespace trace
}  // namespace chm

extern "C" chm_status chm_trace_derive(const chm_trace* t, int32_t* error, void* stream) {
  using namespace chm::trace;
  if (!valid(t) || !t->n_stages || !t->base_input || !t->out_tokens || !t->carried ||
      !t->remaining || !t->carried_prefix)
    return CHM_ERR_INVALID_ARG;
  // 1D bulk copies need 16-byte aligned column bases
  const uintptr_t al = reinterpret_cast<uintptr_t>(t->n_stages) |
                       reinterpret_cast<uintptr_t>(t->base_input) |
                       reinterpret_cast<uintptr_t>(t->out_tokens) |
                       reinterpret_cast<uintptr_t>(t->carried) |
                       reinterpret_cast<uintptr_t>(t->remaining) |
                       reinterpret_cast<uintptr_t>(t->carried_prefix);
  if (al & 15) return CHM_ERR_INVALID_ARG;
  if (t->n_programs == 0) return CHM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  // CHM_TRACE_CHUNK: measurement override of the chunk size (entries)
  static const int entries =
      getenv("CHM_TRACE_CHUNK") ? atoi(getenv("CHM_TRACE_CHUNK")) : kChunkEntries;
  const DeriveSmem L(t->max_stages, t->n_models, entries);
  if (L.total > 200 * 1024) return CHM_ERR_UNSUPPORTED;
  cudaFuncSetAttribute(derive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)L.total);
  const long long n_chunks = ((long long)t->n_programs + L.P - 1) / L.P;
  int per_sm = (int)(220 * 1024 / (L.total + 1024));
  if (per_sm < 1) per_sm = 1;
  const long long cap = (long long)n_sms() * per_sm;
  const long long grid = n_chunks < cap ? n_chunks : cap;
  chm::prof::begin(chm::prof::K_TRACE, st);
  derive_kernel<<<(unsigned)grid, kDeriveThreads, L.total, st>>>(*t, entries, error);
  chm::prof::end(chm::prof::K_TRACE, st,
                 (double)t->n_programs * (t->max_stages * (t->n_models * 24.0 + 4.0) + 4.0));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_trace_gather_rows(const chm_trace* t, const int32_t* program,
                                            const int32_t* stage, int32_t n_rows,
                                            int32_t* out_tokens, int32_t* workflow,
                                            int32_t* n_stages, double* oracle_yhat,
                                            int32_t* error, void* stream) {
  if (!chm::trace::valid(t) || !program || !stage || n_rows < 0) return CHM_ERR_INVALID_ARG;
  if (oracle_yhat && !t->remaining) return CHM_ERR_INVALID_ARG;
  if (n_rows == 0) return CHM_OK;
  const long long n = (long long)n_rows * t->n_models;
  chm::trace::gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      *t, program, stage, n_rows, out_tokens, workflow, n_stages, oracle_yhat, error);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_trace_next_stage(const chm_trace* t, const int32_t* program,
                                           const int32_t* completed_stage,
                                           const double* completion_time, const int8_t* model,
                                           int32_t n, int32_t* next_program, int32_t* next_stage,
                                           double* next_arrival, int32_t* next_input_tokens,
                                           int32_t* next_workflow, int32_t* source_row,
                                           int32_t* n_next, int32_t* error, void* stream) {
  if (!chm::trace::valid(t) || !t->carried_prefix || !program || !completed_stage ||
      !completion_time || !model || n < 0 || !next_program || !next_stage || !next_arrival ||
      !next_input_tokens || !n_next)
    return CHM_ERR_INVALID_ARG;
  chm::trace::next_stage_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
      *t, program, completed_stage, completion_time, model, n, next_program, next_stage,
      next_arrival, next_input_tokens, next_workflow, source_row, n_next, error);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_trace_first_stage(const chm_trace* t, const int32_t* program,
                                            const double* arrival_in, int32_t n,
                                            int32_t* input_tokens, double* arrival,
                                            int32_t* workflow, int32_t* error, void* stream) {
  if (!chm::trace::valid(t) || !program || !input_tokens || !arrival || n < 0)
    return CHM_ERR_INVALID_ARG;
  if (n == 0) return CHM_OK;
  chm::trace::first_stage_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      *t, program, arrival_in, n, input_tokens, arrival, workflow, error);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}
