// K6 -- fused activity monitor + load estimate + confidence-gated slack
// selection + dispatch, serial-exact.
//
// Reference semantics (hetsched, /root/reference/pkg/src/hetsched):
//   schedule_request      balancer.py:89-129  (Algorithm 1)
//   estimate_load         balancer.py:49-60   L[m] = (P_m * d_m) / b_m, fp64
//   select_model          balancer.py:63-77   argmin (L, id); limit = (1+tau)*L_fast;
//                                             first by (-q, id) with L<=limit and
//                                             q >= q_fast + margin; else m_fast
//   ActivityMonitor       monitor.py:52-63, 86-96, 122-129
//                         P_m = sum(entries.values()) -- CPython >= 3.12 sums
//                         floats with Neumaier compensation in insertion order,
//                         so a running (s, c) pair per model reproduces every
//                         intermediate P_m bit for bit.
//   EngineSim.enqueue     engine.py:145-158, 135-143, 283-293 (clock, seq, admit)
//
// Decision i depends on P after decisions 0..i-1 (record_dispatch happens
// inside schedule_request), so the recurrence is serial. Everything that does
// not depend on P is precomputed in parallel: per-row rank of every model in
// descending-q order and, per candidate m_fast, the mask of models that clear
// the confidence margin. The serial step then needs only K fp64 compares for
// argmin, one multiply for the limit, K compares for the slack mask, a few
// integer ops, one Neumaier update and one mul+div for the changed model.
//
// Layout: one CTA of 256 threads. Lane 0 of warp 0 runs the chain with the K
// (s, c, L) triples in registers; per-engine counters that do not feed back
// into the selection live in shared memory. The other 7 warps stream the
// next chunk of per-row inputs into a shared-memory double buffer while the
// chain consumes the current one.
#include "common.cuh"
#include "prof.cuh"

namespace chm {

enum : uint32_t {
  RF_CACHED_PRE = 1u,    // program already assigned before the batch
  RF_REPEAT = 2u,        // an earlier row of this batch has the same program
  RF_BAD_SCORE = 4u,     // routed row has a score outside [0,1] (or NaN)
  RF_DUP_PRE = 8u,       // (program, stage) already in flight before the batch
  RF_BAD_STAGE = 16u,    // stage outside [1, 32]
  RF_BAD_PROGRAM = 32u,  // program index outside [0, n_programs)
  RF_ROUTE = 64u,        // row takes the routing branch
};

enum : uint8_t { DF_CACHED = 1u, DF_ADMITTED = 2u, DF_QUEUED = 4u };

// ---------------------------------------------------------------------------
// chm_prepare_rows: assignment lookup + in-batch repeat detection + compaction
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) prepare_rows_kernel(chm_monitor_state mon,
                                                            chm_rows rows,
                                                            chm_row_scratch sc,
                                                            uint32_t* epoch_counter) {
  const int B = rows.n_rows;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_warps = blockDim.x >> 5;
  const uint32_t epoch = *epoch_counter + 1u;
  const unsigned long long hi = (unsigned long long)(~epoch) << 32;
  // Newer epochs have smaller high words, so atomicMin keeps the first row of
  // the current batch and overwrites any stale stamp.
  for (int i = tid; i < B; i += blockDim.x) {
    int p = rows.program[i];
    if (p >= 0 && p < mon.n_programs)
      atomicMin(reinterpret_cast<unsigned long long*>(mon.batch_stamp) + p,
                hi | (unsigned long long)(uint32_t)i);
  }
  __syncthreads();
  __shared__ int s_warp[32];
  __shared__ int s_total;
  int base_out = 0;
  for (int base = 0; base < B; base += blockDim.x) {
    const int i = base + tid;
    bool route = false;
    if (i < B) {
      const int p = rows.program[i];
      int first = i;
      int8_t pre = -1;
      if (p >= 0 && p < mon.n_programs) {
        unsigned long long st =
            __ldcg(reinterpret_cast<const unsigned long long*>(mon.batch_stamp) + p);
        first = (int)(uint32_t)(st & 0xffffffffull);
        pre = *(volatile int8_t*)(mon.assignment + p);
        route = (first == i) && pre < 0;
      }
      sc.first_row[i] = first;
      sc.pre_model[i] = pre;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, route);
    const int wprefix = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) s_warp[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      int v = lane < n_warps ? s_warp[lane] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane < n_warps) s_warp[lane] = incl - v;
      if (lane == 31) s_total = incl;
    }
    __syncthreads();
    if (route) sc.route_rows[base_out + s_warp[warp] + wprefix] = i;
    base_out += s_total;
    __syncthreads();
  }
  if (tid == 0) {
    *sc.n_route = base_out;
    *epoch_counter = epoch;
  }
}

// ---------------------------------------------------------------------------
// chm_schedule_rows
// ---------------------------------------------------------------------------
struct SelectParams {
  double d[CHM_MAX_MODELS];       // decode_ms_per_token
  double b[CHM_MAX_MODELS];       // float(max_batch_size)
  double inv_b[CHM_MAX_MODELS];   // 1/b, used only when b is a power of two (exact)
  int32_t b_int[CHM_MAX_MODELS];
  uint32_t b_pow2_mask;
  double one_plus_slack;          // (1.0 + cfg.latency_slack), balancer.py:72
  double margin;                  // cfg.confidence_margin
  double tie_tol;                 // tie band of the router tolerance (north star)
};

constexpr int kChunk = 256;
constexpr bool warp_chain_smem = true;  // the warp chain's prefix-sum rebuild of the loads
constexpr int kThreads = 256;

// record_dispatch's insertion into _in_flight[model] (monitor.py:95): the
// live log keeps insertion order, position = live count at dispatch.
__device__ __forceinline__ void log_append(const chm_monitor_state& mon, int m, long long pos,
                                           int program, int stage, double y, int32_t* err,
                                           int row) {
  if (!mon.inflight_key) return;
  if (pos >= mon.inflight_capacity) {
    report_error(err, CHM_ERR_CAPACITY, row, m, (int)mon.inflight_capacity);
    return;
  }
  const size_t at = (size_t)m * mon.inflight_capacity + pos;
  mon.inflight_key[at] = (long long)program * 32 + (stage - 1);
  mon.inflight_yhat[at] = y;
  if (mon.inflight_stamp) mon.inflight_stamp[at] = *mon.stamp_base + row;
  if (mon.inflight_progress) mon.inflight_progress[at] = 0.0;  // nothing emitted yet
}

template <int K>
struct ChunkBuf {
  uint64_t qual[kChunk];   // byte f: models clearing the gate of m_fast = f, rank space
  uint64_t qualm[kChunk];  // byte f: the same set in model space (bit k = model k)
  uint64_t rbits[kChunk];  // byte k: rank-space bit of model k
  uint32_t rank[kChunk];   // nibble k: descending-q rank of model k
  double yhat[kChunk * K];
  double arrival[kChunk];
  uint32_t perm[kChunk];   // nibble (7 - r): the model of rank r
  uint32_t flags[kChunk];
  int32_t out_tokens[kChunk * K];
  int32_t first_row[kChunk];
  int32_t pre_model[kChunk];
};

__device__ __forceinline__ double load_of(double P, double d, double b, double inv_b,
                                          bool pow2) {
  // (P * d) / b evaluated left to right in IEEE fp64 (balancer.py:57-59).
  // For b = 2^k, x / b and x * 2^-k are the same exactly-rounded real.
  double num = __dmul_rn(P, d);
  return pow2 ? __dmul_rn(num, inv_b) : __ddiv_rn(num, b);
}

__device__ __forceinline__ double neumaier_value(double s, double c) {
  // CPython 3.12 builtin sum(): `if (c && Py_IS_FINITE(c)) f_result += c`.
  return (c != 0.0 && isfinite(c)) ? __dadd_rn(s, c) : s;
}

__device__ __forceinline__ void neumaier_add(double& s, double& c, double x) {
  double t = __dadd_rn(s, x);
  if (fabs(s) >= fabs(x))
    c = __dadd_rn(c, __dadd_rn(__dsub_rn(s, t), x));
  else
    c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), s));
  s = t;
}

// v[m] for a run-time m in [0, K) as a log-depth select tree over registers
// (dynamic indexing would spill the array to local memory).
template <int K, typename T>
__device__ __forceinline__ T tree_select(const T (&v)[K], int m) {
  T a[K];
#pragma unroll
  for (int k = 0; k < K; ++k) a[k] = v[k];
#pragma unroll
  for (int step = 1; step < K; step *= 2)
#pragma unroll
    for (int k = 0; k + step < K; k += 2 * step) a[k] = (m & step) ? a[k + step] : a[k];
  return a[0];
}

// select_model (balancer.py:63-77) on load bit patterns (non-negative doubles
// order like their IEEE bits): m_fast = argmin (L, index) as a log-depth
// tournament whose left operand always carries the lower indices (strict <
// keeps the lowest index on ties); limit = (1 + tau) * L_fast; the candidates
// {m : L_m <= limit and q_m >= q_fast + margin}; the first one in
// descending-q order. Rank space: rank r is bit (7 - r), so the first
// candidate is the highest set bit (one FLO) and `perm` nibble (7 - r) holds
// the model of rank r. `qual` byte f holds the gate set of m_fast = f in rank
// space, `rbits` byte k the rank bit of model k (both precomputed per row).
template <int K>
__device__ __forceinline__ int select_bits(const unsigned long long (&Lb)[K], double one_plus_slack,
                                           uint64_t qual, uint64_t rbits, uint32_t perm) {
  // (1 + tau) * L_k for every k and the gate set of every candidate ride
  // along the tournament: no multiply or shift after the argmin
  unsigned long long tv[K], tl[K];
  uint32_t tq[K];
  int ti[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    tv[k] = Lb[k];
    tl[k] = (unsigned long long)__double_as_longlong(
        __dmul_rn(one_plus_slack, __longlong_as_double((long long)Lb[k])));
    tq[k] = (uint32_t)(qual >> (8 * k)) & 0xffu;
    ti[k] = k;
  }
#pragma unroll
  for (int step = 1; step < K; step *= 2)
#pragma unroll
    for (int k = 0; k + step < K; k += 2 * step) {
      const bool lt = tv[k + step] < tv[k];
      tv[k] = lt ? tv[k + step] : tv[k];
      tl[k] = lt ? tl[k + step] : tl[k];
      tq[k] = lt ? tq[k + step] : tq[k];
      ti[k] = lt ? ti[k + step] : ti[k];
    }
  const unsigned long long limb = tl[0];
  uint32_t okr = 0;
#pragma unroll
  for (int k = 0; k < K; ++k)
    okr |= (Lb[k] <= limb) ? ((uint32_t)(rbits >> (8 * k)) & 0xffu) : 0u;
  const uint32_t crk = tq[0] & okr;
  const int pos = (31 - __clz(crk)) & 7;
  const int mc = (int)((perm >> (4 * pos)) & 15u);
  return crk ? mc : ti[0];
}

// argmin (L, index) over load bit patterns with the winner's limit carried
// along (the tournament of select_bits on its own).
template <int K>
__device__ __forceinline__ void argmin_limit(const unsigned long long (&L)[K],
                                             const unsigned long long (&Lim)[K], int& mf,
                                             unsigned long long& lim) {
  unsigned long long tv[K], tl[K];
  int ti[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    tv[k] = L[k];
    tl[k] = Lim[k];
    ti[k] = k;
  }
#pragma unroll
  for (int step = 1; step < K; step *= 2)
#pragma unroll
    for (int k = 0; k + step < K; k += 2 * step) {
      const bool lt = tv[k + step] < tv[k];
      tv[k] = lt ? tv[k + step] : tv[k];
      tl[k] = lt ? tl[k + step] : tl[k];
      ti[k] = lt ? ti[k + step] : ti[k];
    }
  mf = ti[0];
  lim = tl[0];
}

// Tie band (north star: "ties inside the tolerance band are reported"): for a
// routed row with scores q and the loads L it saw, TIE_QUAL = some model
// inside the latency slack other than m_fast has |q_m - (q_fast + margin)| <=
// tol (the confidence gate could flip under a router error of tol);
// TIE_RANK = the chosen candidate and another candidate differ by <= tol in q
// (their descending-q order could flip). Same fp64 operations as the decision.
enum : uint8_t { DF_TIE_RANK = 8u, DF_TIE_QUAL = 16u };

template <int K>
__device__ __forceinline__ uint8_t tie_bits(const double (&q)[K], const double (&L)[K],
                                            const SelectParams& prm, int m) {
  int mf = 0;
  double lmin = L[0];
#pragma unroll
  for (int k = 1; k < K; ++k) {
    const bool lt = L[k] < lmin;
    mf = lt ? k : mf;
    lmin = lt ? L[k] : lmin;
  }
  const double limit = __dmul_rn(prm.one_plus_slack, lmin);
  double qf = q[0];
#pragma unroll
  for (int k = 1; k < K; ++k) qf = (k == mf) ? q[k] : qf;
  const double thr = __dadd_rn(qf, prm.margin);
  double qm = q[0];
#pragma unroll
  for (int k = 1; k < K; ++k) qm = (k == m) ? q[k] : qm;
  bool any_cand = false, tq = false, tr = false;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const bool ok = L[k] <= limit;
    if (ok && k != mf && fabs(__dsub_rn(q[k], thr)) <= prm.tie_tol) tq = true;
    const bool cand = ok && q[k] >= thr;
    any_cand |= cand;
    if (cand && k != m && __dsub_rn(qm, q[k]) <= prm.tie_tol) tr = true;
  }
  return (uint8_t)((tq ? DF_TIE_QUAL : 0) | ((any_cand && tr) ? DF_TIE_RANK : 0));
}

template <int K, bool SPEC>
__global__ void __launch_bounds__(kThreads, 1) schedule_rows_kernel(
    SelectParams prm, chm_monitor_state mon, chm_rows rows, chm_row_scratch sc,
    const double* __restrict__ scores, const double* __restrict__ yhat, chm_decisions out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ChunkBuf<K>* bufs = reinterpret_cast<ChunkBuf<K>*>(smem_raw);
  __shared__ int s_committed;
  const int B = rows.n_rows;
  const int tid = threadIdx.x;
  // A predictor / trace-gather error already recorded for row r stops the
  // batch there: rows < r are scheduled, row r gets the effects the reference
  // applied before predictor.predict raised (monitor.assign for a routed
  // row, balancer.py:113-115), later rows nothing.
  const int pred_stop = (out.error && out.error[0] != 0) ? min(out.error[1], B) : B;

  // ---- phase P: per-row precompute (independent of the in-flight state) ----
  // It also decides the chain mode: the fast chain has no error exits and
  // defers the engine bookkeeping (seq, admission, clock) to a parallel
  // post-pass, which is exact unless a row could raise (bad score, negative /
  // NaN prediction, clock going backwards, negative out_tokens, predictor
  // error) or needs the in-batch duplicate scan.
  double max_clk0 = 0.0;
#pragma unroll
  for (int m = 0; m < K; ++m) max_clk0 = fmax(max_clk0, mon.engine_clock[m]);
  int slow = pred_stop < B;
  // Dyadic mode: every prediction a multiple of 2^-8 below 2^29 (and the
  // tick-start sums likewise, compensation 0). Every partial sum is then a
  // multiple of 2^-8 below 2^44, exact in fp64, so Neumaier's compensation
  // stays exactly 0 and the running sum is a plain add (bit-identical).
  int dyadic_rows = 1;
  for (int i = tid; i < B; i += blockDim.x) {
    const int p = rows.program[i];
    const int st = rows.stage[i];
    {
      const double a = rows.arrival[i];
      const double prev = i ? rows.arrival[i - 1] : max_clk0;
      if (i ? (a < prev) : (a < __dsub_rn(prev, 1e-9))) slow = 1;
#pragma unroll
      for (int m = 0; m < K; ++m) {
        if (rows.out_tokens) slow |= rows.out_tokens[(size_t)i * K + m] < 0;
        const double y = yhat[(size_t)i * K + m];
        slow |= !(y >= 0.0);
        const double y8 = y * 256.0;
        dyadic_rows &= (y < 536870912.0 && y8 == trunc(y8)) ? 1 : 0;
      }
    }
    uint32_t fl = 0;
    uint64_t qual = 0;
    uint32_t rank = 0;
    if (p < 0 || p >= mon.n_programs) {
      fl |= RF_BAD_PROGRAM;
    } else {
      const int pre = sc.pre_model[i];
      const int first = sc.first_row[i];
      if (pre >= 0) fl |= RF_CACHED_PRE;
      else if (first != i) fl |= RF_REPEAT;
      else fl |= RF_ROUTE;
      if (st < 1 || st > CHM_MAX_STAGES) {
        fl |= RF_BAD_STAGE;
      } else if (__ldcg(mon.stage_bits + p) & (1u << (st - 1))) {
        fl |= RF_DUP_PRE;
      }
    }
    if (fl & RF_ROUTE) {
      double q[K];
      bool bad = false;
#pragma unroll
      for (int m = 0; m < K; ++m) {
        const double qm = scores[(size_t)i * K + m];
        // ConfidenceVector.__post_init__: `not 0.0 <= q <= 1.0` (NaN fails too).
        if (!(qm >= 0.0 && qm <= 1.0)) bad = true;
        q[m] = qm;
      }
      if (bad) fl |= RF_BAD_SCORE;
      // rank[m] = position of m in sorted(models, key=(-q[m], m)).
#pragma unroll
      for (int m = 0; m < K; ++m) {
        uint32_t r = 0;
#pragma unroll
        for (int o = 0; o < K; ++o)
          r += (q[o] > q[m] || (q[o] == q[m] && o < m)) ? 1u : 0u;
        rank |= r << (4 * m);
      }
      // qual byte mf = { m : q[m] >= q[mf] + margin } (balancer.py:73-75),
      // model-space bits (load_chunk derives the rank-space form)
#pragma unroll
      for (int mf = 0; mf < K; ++mf) {
        const double thr = __dadd_rn(q[mf], prm.margin);
        uint64_t bits = 0;
#pragma unroll
        for (int m = 0; m < K; ++m) bits |= q[m] >= thr ? (1u << m) : 0u;
        qual |= bits << (8 * mf);
      }
    }
    if (fl & ~(RF_ROUTE | RF_CACHED_PRE)) slow = 1;
    sc.flags[i] = fl;
    sc.qual[i] = qual;
    sc.rank[i] = rank;
  }
  const bool exact = __syncthreads_or(slow) != 0;
  bool dyadic = __syncthreads_and(dyadic_rows) != 0;
#pragma unroll
  for (int m = 0; m < K; ++m) {
    const double f = mon.inflight_sum[m];
    dyadic = dyadic && mon.inflight_comp[m] == 0.0 && f >= 0.0 &&
             f * 256.0 == trunc(f * 256.0) && f + (double)B * 536870912.0 < 17592186044416.0;
  }

  auto load_chunk = [&](int chunk, ChunkBuf<K>* buf, int t0, int nt) {
    const int r0 = chunk * kChunk;
    const int n = min(kChunk, B - r0);
    if (n <= 0) return;
    for (int j = t0; j < n; j += nt) {
      const uint64_t qm = __ldcg(sc.qual + r0 + j);
      const uint32_t rk = __ldcg(sc.rank + r0 + j);
      uint32_t pm = 0;  // perm: rank r -> model, at nibble 7 - r
      uint64_t rb = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const uint32_t r = (rk >> (4 * k)) & 15u;
        pm |= (uint32_t)k << (4 * (7 - r));
        rb |= (uint64_t)(0x80u >> r) << (8 * k);
      }
      uint64_t qr = 0;  // gate sets in rank space
#pragma unroll
      for (int f = 0; f < K; ++f)
#pragma unroll
        for (int k = 0; k < K; ++k)
          if ((qm >> (8 * f + k)) & 1ull) qr |= ((rb >> (8 * k)) & 0xffull) << (8 * f);
      buf->qual[j] = qr;
      buf->qualm[j] = qm;
      buf->rank[j] = rk;
      buf->perm[j] = pm;
      buf->rbits[j] = rb;
      buf->flags[j] = __ldcg(sc.flags + r0 + j);
      buf->arrival[j] = rows.arrival[r0 + j];
      buf->first_row[j] = sc.first_row[r0 + j];
      buf->pre_model[j] = sc.pre_model[r0 + j];
    }
    for (int j = t0; j < n * K; j += nt) {
      buf->yhat[j] = yhat[(size_t)r0 * K + j];
      buf->out_tokens[j] = rows.out_tokens ? rows.out_tokens[(size_t)r0 * K + j] : 0;
    }
  };

  const int n_chunks = (B + kChunk - 1) / kChunk;
  if (n_chunks > 0) load_chunk(0, &bufs[0], tid, blockDim.x);
  if (tid == 0) s_committed = B;
  __syncthreads();

  // Chain state (thread 0 only). Per-engine counters that do not feed back
  // into the selection live in shared memory.
  double L[K];
  __shared__ double s_f[K], s_c[K], s_clk[K], s_d[K], s_b[K], s_invb[K], s_L0[K], s_f0[K], s_dq[K];
  __shared__ long long s_seq[K], s_cnt[K], s_it[K];
  __shared__ int s_run[K], s_que[K], s_bmax[K], s_pow2[K];
  bool stop = false;
  if (tid == 0) {
#pragma unroll
    for (int m = 0; m < K; ++m) {
      const double f = mon.inflight_sum[m], c = mon.inflight_comp[m];
      const bool pw = (prm.b_pow2_mask >> m) & 1u;
      L[m] = load_of(neumaier_value(f, c), prm.d[m], prm.b[m], prm.inv_b[m], pw);
      s_L0[m] = L[m];
      s_f0[m] = f;
      s_dq[m] = __dmul_rn(prm.d[m], prm.inv_b[m]);
      s_f[m] = f;
      s_c[m] = c;
      s_d[m] = prm.d[m];
      s_b[m] = prm.b[m];
      s_invb[m] = prm.inv_b[m];
      s_pow2[m] = pw;
      s_bmax[m] = prm.b_int[m];
      s_clk[m] = mon.engine_clock[m];
      s_seq[m] = mon.engine_seq[m];
      s_cnt[m] = mon.inflight_count[m];
      s_it[m] = mon.engine_iterations[m];
      s_run[m] = mon.engine_running[m];
      s_que[m] = mon.engine_queued[m];
      // Work conservation: free slots imply an empty queue (engine.py:328-338).
      if (s_run[m] < prm.b_int[m] && s_que[m] > 0 && !stop) {
        report_error(out.error, CHM_ERR_INVALID_STATE, 0, m, s_que[m]);
        s_committed = 0;
        stop = true;
      }
    }
  }
  // Fast-chain state: everything the serial step touches lives in registers.
  // Loads are compared as IEEE bit patterns (all non-negative), which orders
  // them exactly like the fp64 values, with integer compares.
  unsigned long long Lb[K];
  double fr[K], cv[K], dd[K], bdiv[K], dq[K];
#pragma unroll
  for (int m = 0; m < K; ++m) {
    Lb[m] = (unsigned long long)__double_as_longlong(L[m]);
    // only thread 0 runs these chains (and wrote s_f / s_c just above)
    fr[m] = tid == 0 ? s_f[m] : 0.0;
    cv[m] = tid == 0 ? s_c[m] : 0.0;
    dd[m] = prm.d[m];
    bdiv[m] = ((prm.b_pow2_mask >> m) & 1u) ? prm.inv_b[m] : prm.b[m];
    dq[m] = __dmul_rn(prm.d[m], prm.inv_b[m]);  // d / b, exact for b = 2^k
  }
  const uint32_t pow2_mask = prm.b_pow2_mask;
  const double one_plus_slack = prm.one_plus_slack;
  // dyadic chain: the current m_fast and its limit, every engine's limit
  unsigned long long Lim[K];
#pragma unroll
  for (int m = 0; m < K; ++m)
    Lim[m] = (unsigned long long)__double_as_longlong(
        __dmul_rn(one_plus_slack, __longlong_as_double((long long)Lb[m])));
  int cmf;
  unsigned long long climb;
  argmin_limit<K>(Lb, Lim, cmf, climb);

  // ---- warp chain (dyadic, every b a power of two): lane k owns engine k ----
  // Per row every lane tests its own engine (gate of m_fast, slack limit)
  // and one integer min-reduction over the lanes picks the first candidate
  // in descending-q order (key = rank * 8 + engine); m_fast for the next row
  // is the argmin over the lanes of the loads with m_fast's speculative
  // update in place (three min-reductions: high word, low word, lowest
  // index), computed while the decision resolves. ~60 warp instructions per
  // row instead of ~160 for one thread (profiles/r2_k6_chain.md).
  const bool warp_chain = SPEC && dyadic && !exact;
  const int lane = tid & 31;
  double w_s = 0.0, w_L = __longlong_as_double(0x7ff0000000000000ll), w_dq = 0.0;
  double w_Lmin = 0.0, w_lim = 0.0;
  int w_cmf = 0;
  bool w_stop = false;
  if (warp_chain && tid < 32) {
    __syncwarp();
    w_stop = __shfl_sync(0xffffffffu, stop ? 1 : 0, 0) != 0;
    if (lane < K) {
      w_s = s_f[lane];  // dyadic: compensation 0
      w_dq = __dmul_rn(prm.d[lane], prm.inv_b[lane]);
      w_L = __dmul_rn(w_s, w_dq);
    }
    // argmin (L, index) over the lanes: high word, low word, index
    const unsigned long long lb = (unsigned long long)__double_as_longlong(w_L);
    const uint32_t hi = (uint32_t)(lb >> 32), lo = (uint32_t)lb;
    const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    const unsigned long long lm = ((unsigned long long)mh << 32) | ml;
    w_cmf = (int)__reduce_min_sync(0xffffffffu, lb == lm ? (uint32_t)lane : 31u);
    w_Lmin = __longlong_as_double((long long)lm);
    w_lim = __dmul_rn(prm.one_plus_slack, w_Lmin);
  }

  for (int ch = 0; ch < n_chunks; ++ch) {
    ChunkBuf<K>* cur = &bufs[ch & 1];
    if (tid >= 32) {
      if (ch + 1 < n_chunks) load_chunk(ch + 1, &bufs[(ch + 1) & 1], tid - 32, blockDim.x - 32);
    } else if (warp_chain) {
      if (!w_stop) {
        const int r0 = ch * kChunk;
        const int n = min(kChunk, B - r0);
        const double ops = prm.one_plus_slack;
        int32_t* __restrict__ model_out = out.model + r0;
        const int rsh = 4 * lane;  // this lane's rank nibble
        int mb = 0;  // lane l keeps the decision of row (j & ~31) + l until the group is full
        // software pipeline: row j + 1's inputs are read while row j resolves
        uint32_t nfl = cur->flags[0];
        uint64_t nqm = cur->qualm[0];
        uint32_t nrk = cur->rank[0];
        int npre = cur->pre_model[0];
        double ny = lane < K ? cur->yhat[lane] : 0.0;
        for (int j = 0; j < n; ++j) {
          const uint32_t fl = nfl;
          const uint64_t qm = nqm;
          const uint32_t rk = nrk;
          const int pre = npre;
          const double y = ny;
          {
            const int jn = j + 1 < n ? j + 1 : j;
            nfl = cur->flags[jn];
            nqm = cur->qualm[jn];
            nrk = cur->rank[jn];
            npre = cur->pre_model[jn];
            ny = lane < K ? cur->yhat[jn * K + lane] : 0.0;
          }
          // speculative: this engine's sum and load if the row lands here
          const double ls_d = __dadd_rn(w_s, y);
          const double ls = lane < K ? __dmul_rn(ls_d, w_dq) : w_L;
          // decision: candidates (gate of m_fast, within the slack) by rank
          const bool gate = (qm >> (8 * w_cmf + lane)) & 1ull;
          const bool cand = lane < K && gate && w_L <= w_lim;
          const uint32_t key = cand ? (((rk >> rsh) & 15u) << 3) | (uint32_t)lane : 0xffu;
          const uint32_t mn = __reduce_min_sync(0xffffffffu, key);
          int m = mn == 0xffu ? w_cmf : (int)(mn & 7u);
          m = (fl & RF_CACHED_PRE) ? pre : m;
          // m_fast after the row if it lands on m_fast (speculative argmin)
          const double lx = lane == w_cmf ? ls : w_L;
          const unsigned long long lb = (unsigned long long)__double_as_longlong(lx);
          const uint32_t hi = (uint32_t)(lb >> 32), lo = (uint32_t)lb;
          const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
          const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
          const unsigned long long lm = ((unsigned long long)mh << 32) | ml;
          const int mf2 = (int)__reduce_min_sync(0xffffffffu, lb == lm ? (uint32_t)lane : 31u);
          // update
          const bool hit = lane == m;
          w_s = hit ? ls_d : w_s;
          w_L = hit ? ls : w_L;
          const bool moved = m == w_cmf;
          const double lmd = __longlong_as_double((long long)lm);
          w_cmf = moved ? mf2 : w_cmf;
          w_lim = moved ? __dmul_rn(ops, lmd) : w_lim;
          // decisions leave in coalesced groups of 32 rows; the loads each
          // row saw are rebuilt in the post-pass from exact prefix sums
          mb = lane == (j & 31) ? m : mb;
          if ((j & 31) == 31 || j == n - 1) {
            if (lane <= (j & 31)) model_out[(j & ~31) + lane] = mb;
          }
        }
      }
    } else if (tid == 0 && !stop && !exact) {
      // ---------------- fast chain (no error exits) ----------------
      // Per row: decision from the loads (the only loop-carried input), then
      // the chosen model's in-flight update and new load. With SPEC (every b
      // a power of two) the K candidate updates are computed while the
      // decision resolves and the chosen one is selected afterwards, so the
      // loop-carried path is the decision alone. In dyadic mode every
      // partial sum is exact, the Neumaier compensation stays 0 and an
      // update is one add and one multiply (L = s * (d / b), exact scaling).
      const int r0 = ch * kChunk;
      const int n = min(kChunk, B - r0);
      if (SPEC && dyadic) {
        // Loads only grow and only the dispatched engine's changes, so
        // m_fast moves only when the row dispatches to m_fast itself. The
        // argmin for that case is computed speculatively while the row's
        // decision resolves; the loop-carried path is then: slack mask ->
        // first candidate in rank order -> m -> state select. Row j + 1's
        // inputs are read from shared memory while row j resolves.
        uint32_t nfl = cur->flags[0];
        uint64_t nqual = cur->qual[0], nrb = cur->rbits[0];
        uint32_t npm = cur->perm[0];
        int npre = cur->pre_model[0];
        double ny[K];
#pragma unroll
        for (int k = 0; k < K; ++k) ny[k] = cur->yhat[k];
        for (int j = 0; j < n; ++j) {
          const int i = r0 + j;
          const uint32_t fl = nfl;
          const uint64_t qual = nqual, rb = nrb;
          const uint32_t pm = npm;
          const int pre = npre;
          // speculative: every engine's sum, load and limit after this row
          double ls_d[K];
          unsigned long long ls[K], lsl[K], lt[K], ltl[K];
#pragma unroll
          for (int k = 0; k < K; ++k) {
            ls_d[k] = __dadd_rn(fr[k], ny[k]);
            const double lv = __dmul_rn(ls_d[k], dq[k]);
            ls[k] = (unsigned long long)__double_as_longlong(lv);
            lsl[k] = (unsigned long long)__double_as_longlong(__dmul_rn(one_plus_slack, lv));
            lt[k] = k == cmf ? ls[k] : Lb[k];
            ltl[k] = k == cmf ? lsl[k] : Lim[k];
          }
          int mf2;
          unsigned long long lim2;
          argmin_limit<K>(lt, ltl, mf2, lim2);  // m_fast if this row dispatches to m_fast
          const int jn = j + 1 < n ? j + 1 : j;
          nfl = cur->flags[jn];
          nqual = cur->qual[jn];
          nrb = cur->rbits[jn];
          npm = cur->perm[jn];
          npre = cur->pre_model[jn];
#pragma unroll
          for (int k = 0; k < K; ++k) ny[k] = cur->yhat[jn * K + k];
          // the decision (select_model with m_fast and its limit known)
          const uint32_t tq = (uint32_t)(qual >> (8 * cmf)) & 0xffu;
          uint32_t okr = 0;
#pragma unroll
          for (int k = 0; k < K; ++k)
            okr |= (Lb[k] <= climb) ? ((uint32_t)(rb >> (8 * k)) & 0xffu) : 0u;
          const uint32_t crk = tq & okr;
          const int pos = (31 - __clz(crk)) & 7;
          int m = crk ? (int)((pm >> (4 * pos)) & 15u) : cmf;
          m = (fl & RF_CACHED_PRE) ? pre : m;
#pragma unroll
          for (int k = 0; k < K; ++k) {
            const bool hit = k == m;
            fr[k] = hit ? ls_d[k] : fr[k];
            Lb[k] = hit ? ls[k] : Lb[k];
            Lim[k] = hit ? lsl[k] : Lim[k];
          }
          const bool moved = m == cmf;
          cmf = moved ? mf2 : cmf;
          climb = moved ? lim2 : climb;
          out.model[i] = m;
          sc.lnew[i] = __longlong_as_double((long long)tree_select<K>(ls, m));
        }
      } else {
#pragma unroll 2
        for (int j = 0; j < n; ++j) {
          const int i = r0 + j;
          const uint32_t fl = cur->flags[j];
          const uint64_t qual = cur->qual[j], rb = cur->rbits[j];
          const uint32_t pm = cur->perm[j];
          const int pre = cur->pre_model[j];
          double yr[K];
#pragma unroll
          for (int k = 0; k < K; ++k) yr[k] = cur->yhat[j * K + k];
          int m = select_bits<K>(Lb, one_plus_slack, qual, rb, pm);
          m = (fl & RF_CACHED_PRE) ? pre : m;
          unsigned long long lmb;
          if constexpr (SPEC) {
            double fs[K], cs[K];
            unsigned long long ls[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
              fs[k] = fr[k];
              cs[k] = cv[k];
              neumaier_add(fs[k], cs[k], yr[k]);
              ls[k] = (unsigned long long)__double_as_longlong(
                  __dmul_rn(__dmul_rn(neumaier_value(fs[k], cs[k]), dd[k]), bdiv[k]));
            }
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const bool hit = k == m;
              fr[k] = hit ? fs[k] : fr[k];
              cv[k] = hit ? cs[k] : cv[k];
              Lb[k] = hit ? ls[k] : Lb[k];
            }
            lmb = tree_select<K>(ls, m);
          } else {
            const double y = tree_select<K>(yr, m);
            double fm = tree_select<K>(fr, m), cm = tree_select<K>(cv, m);
            neumaier_add(fm, cm, y);
            const double num = __dmul_rn(neumaier_value(fm, cm), tree_select<K>(dd, m));
            const double bdm = tree_select<K>(bdiv, m);
            const double lm =
                ((pow2_mask >> m) & 1u) ? __dmul_rn(num, bdm) : __ddiv_rn(num, bdm);
            lmb = (unsigned long long)__double_as_longlong(lm);
#pragma unroll
            for (int k = 0; k < K; ++k) {
              const bool hit = k == m;
              fr[k] = hit ? fm : fr[k];
              cv[k] = hit ? cm : cv[k];
              Lb[k] = hit ? lmb : Lb[k];
            }
          }
          out.model[i] = m;
          sc.lnew[i] = __longlong_as_double((long long)lmb);
        }
      }
    } else if (tid == 0 && !stop && exact) {
      const int r0 = ch * kChunk;
      const int n = min(kChunk, B - r0);
      for (int j = 0; j < n; ++j) {
        const int i = r0 + j;
        const uint32_t fl = cur->flags[j];
        int err = 0, err_aux = 0;
        // stage how far the reference got before raising:
        // 0 nothing, 1 assigned, 2 + dispatched, 3 + clock advanced
        int partial = 0;
        if (fl & (RF_BAD_PROGRAM | RF_BAD_STAGE)) {
          err = (fl & RF_BAD_PROGRAM) ? CHM_ERR_INVALID_ARG : CHM_ERR_UNSUPPORTED;
          report_error(out.error, err, i, -1, 0);
          s_committed = i;
          stop = true;
          break;
        }
        int m;
        bool cached = true;
        if (fl & RF_CACHED_PRE) {
          m = cur->pre_model[j];
        } else if (fl & RF_REPEAT) {
          // The first occurrence (already decided by this thread) assigned it.
          m = out.model[cur->first_row[j]];
        } else {
          if (fl & RF_BAD_SCORE) {
            report_error(out.error, CHM_ERR_VALIDATION, i, -1, 1);
            s_committed = i;
            stop = true;
            break;
          }
          cached = false;
          unsigned long long lb[K];
#pragma unroll
          for (int k = 0; k < K; ++k) lb[k] = (unsigned long long)__double_as_longlong(L[k]);
          m = select_bits<K>(lb, prm.one_plus_slack, cur->qual[j], cur->rbits[j], cur->perm[j]);
          partial = 1;  // monitor.assign (balancer.py:113)
        }
        if (i == pred_stop) {
          // predictor.predict raised for this row (error already recorded)
          if (partial >= 1) mon.assignment[rows.program[i]] = (int8_t)m;
          s_committed = i;
          stop = true;
          break;
        }
        // predictor.predict + record_dispatch (balancer.py:115-116, monitor.py:86-96)
        const double y = cur->yhat[j * K + m];
        if (is_nan64(y)) err = CHM_ERR_NAN_PREDICTION;
        else if (y < 0.0) err = CHM_ERR_NEGATIVE_PREDICTION;
        else if (fl & RF_DUP_PRE) err = CHM_ERR_DUPLICATE_REQUEST;
        else if (fl & RF_REPEAT) {
          // Same (program, stage) earlier in this batch -> DuplicateRequest.
          const int p = rows.program[i], st = rows.stage[i];
          for (int o = cur->first_row[j]; o < i; ++o)
            if (rows.program[o] == p && rows.stage[o] == st) {
              err = CHM_ERR_DUPLICATE_REQUEST;
              break;
            }
        }
        if (!err) {
          partial = 2;
          double fs = s_f[m], cs = s_c[m];
          neumaier_add(fs, cs, y);
          s_f[m] = fs;
          s_c[m] = cs;
          const double lm = load_of(neumaier_value(fs, cs), s_d[m], s_b[m], s_invb[m],
                                    s_pow2[m] != 0);
#pragma unroll
          for (int k = 0; k < K; ++k) L[k] = (k == m) ? lm : L[k];
          sc.lnew[i] = lm;
          log_append(mon, m, s_cnt[m], rows.program[i], rows.stage[i], y, out.error, i);
          s_cnt[m] += 1;
          // EngineSim.enqueue: _advance_clock (engine.py:140-143), then
          // _make_entry validates out_tokens (engine.py:285-286).
          const double arr = cur->arrival[j];
          const double ck = s_clk[m];
          if (arr < __dsub_rn(ck, 1e-9)) {
            err = CHM_ERR_TIME_BACKWARDS;
          } else {
            partial = 3;
            s_clk[m] = arr > ck ? arr : ck;
            if (cur->out_tokens[j * K + m] < 0) {
              err = CHM_ERR_VALIDATION;
              err_aux = 2;
            }
          }
        }
        if (err) {
          report_error(out.error, err, i, m, err_aux);
          // Apply the side effects the reference performed before raising.
          const int p = rows.program[i];
          if (partial >= 1 && !cached) mon.assignment[p] = (int8_t)m;
          if (partial >= 2) atomicOr(mon.stage_bits + p, 1u << (rows.stage[i] - 1));
          s_committed = i;
          stop = true;
          break;
        }
        const long long sq = s_seq[m];
        s_seq[m] = sq + 1;
        uint8_t dfl = cached ? DF_CACHED : 0;
        const int rn = s_run[m];
        if (rn < s_bmax[m]) {
          // enqueue -> _iterate admits the only queued entry (engine.py:157-158)
          s_run[m] = rn + 1;
          s_it[m] += 1;
          dfl |= DF_ADMITTED;
        } else {
          s_que[m] += 1;
          dfl |= DF_QUEUED;
        }
        out.model[i] = m;
        out.priority[i] = y;
        out.flags[i] = dfl;
        out.seq[i] = sq;
      }
    }
    __syncthreads();
  }

  // Per-thread contiguous row ranges for the parallel post-passes.
  __shared__ int s_cntm[K][kThreads];
  __shared__ int s_lastm[K][kThreads];
  __shared__ int s_tot[K], s_last[K];
  const int n_ok = s_committed;
  const int per = (n_ok + kThreads - 1) / kThreads;
  const int lo = min(tid * per, n_ok), hi = min(lo + per, n_ok);
  const int warp = tid >> 5;
  if (warp_chain) {
    if (tid < K) s_f[tid] = w_s;  // compensation stays 0 (dyadic)
  } else if (tid == 0 && !exact) {
#pragma unroll
    for (int m = 0; m < K; ++m) {
      s_f[m] = fr[m];
      s_c[m] = cv[m];
    }
  }
#pragma unroll
  for (int m = 0; m < K; ++m) {
    s_cntm[m][tid] = 0;
    s_lastm[m][tid] = -1;
  }
  for (int i = lo; i < hi; ++i) {
    const int m = out.model[i];
    s_cntm[m][tid] += 1;
    s_lastm[m][tid] = i;
  }
  __syncthreads();
  // per model (warp m): exclusive prefix sums of the counts and exclusive
  // running max of the last row index over the thread ranges
  if (warp < K) {
    int v[kThreads / 32], lv[kThreads / 32], sum = 0, last = -1;
#pragma unroll
    for (int e = 0; e < kThreads / 32; ++e) {
      v[e] = s_cntm[warp][lane * (kThreads / 32) + e];
      lv[e] = s_lastm[warp][lane * (kThreads / 32) + e];
      sum += v[e];
      last = max(last, lv[e]);
    }
    int incl = sum, linc = last;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      const int tl = __shfl_up_sync(0xffffffffu, linc, o);
      if (lane >= o) {
        incl += t;
        linc = max(linc, tl);
      }
    }
    int run = incl - sum;
    int lrun = __shfl_up_sync(0xffffffffu, linc, 1);
    if (lane == 0) lrun = -1;
#pragma unroll
    for (int e = 0; e < kThreads / 32; ++e) {
      s_cntm[warp][lane * (kThreads / 32) + e] = run;
      s_lastm[warp][lane * (kThreads / 32) + e] = lrun;
      run += v[e];
      lrun = max(lrun, lv[e]);
    }
    if (lane == 31) {
      s_tot[warp] = incl;
      s_last[warp] = linc;
    }
  }
  __syncthreads();

  if (!exact) {
    // ---- fast-chain bookkeeping, in parallel (EngineSim.enqueue effects) ----
    // Rows choosing engine m take consecutive seq numbers; the first
    // max(0, b - running) of them are admitted by the enqueue-triggered
    // iteration, the rest queue; the engine clock ends at the arrival of the
    // last row it received (arrivals are non-decreasing in fast mode).
    for (int i = lo; i < hi; ++i) {
      const int m = out.model[i];
      const int r = s_cntm[m][tid]++;
      const double y = yhat[(size_t)i * K + m];
      log_append(mon, m, s_cnt[m] + r, rows.program[i], rows.stage[i], y, out.error, i);
      out.priority[i] = y;
      out.seq[i] = s_seq[m] + r;
      out.flags[i] = ((sc.flags[i] & RF_CACHED_PRE) ? DF_CACHED : 0) |
                     ((s_run[m] + r < s_bmax[m]) ? DF_ADMITTED : DF_QUEUED);
    }
    __syncthreads();
    if (tid < K) {
      const int m = tid, tot = s_tot[m];
      const int adm = min(max(s_bmax[m] - s_run[m], 0), tot);
      s_seq[m] += tot;
      s_run[m] += adm;
      s_que[m] += tot - adm;
      s_it[m] += adm;
      s_cnt[m] += tot;
      if (tot) s_clk[m] = fmax(s_clk[m], rows.arrival[s_last[m]]);
    }
  }
  // ---- Decision.estimated_loads + tie band, in parallel ----
  // The loads row i saw: L0, then for each model the new load recorded by the
  // last earlier row that dispatched to it (lnew). The warp chain records no
  // loads: in dyadic mode every partial sum is exact in any order, so each
  // thread rebuilds them as (s0 + prefix sum of the dispatched predictions) *
  // (d / b), the chain's own arithmetic.
  __shared__ double s_ysum[warp_chain_smem ? K : 1][warp_chain_smem ? kThreads : 1];
  double w_run[K];
  if (warp_chain_smem && warp_chain) {
#pragma unroll
    for (int k = 0; k < K; ++k) w_run[k] = 0.0;
    for (int i = lo; i < hi; ++i) {
      const int m = out.model[i];
      const double y = yhat[(size_t)i * K + m];
#pragma unroll
      for (int k = 0; k < K; ++k) w_run[k] = __dadd_rn(w_run[k], k == m ? y : 0.0);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) s_ysum[k][tid] = w_run[k];
    __syncthreads();
    if (warp < K) {  // exclusive prefix over the thread ranges (exact: dyadic)
      double v[kThreads / 32], tot = 0.0;
#pragma unroll
      for (int e = 0; e < kThreads / 32; ++e) {
        v[e] = s_ysum[warp][lane * (kThreads / 32) + e];
        tot = __dadd_rn(tot, v[e]);
      }
      double incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl = __dadd_rn(incl, t);
      }
      double run = __dsub_rn(incl, tot);
#pragma unroll
      for (int e = 0; e < kThreads / 32; ++e) {
        s_ysum[warp][lane * (kThreads / 32) + e] = run;
        run = __dadd_rn(run, v[e]);
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k)
      w_run[k] = __dadd_rn(s_f0[k], s_ysum[k][tid]);
  }
  {
    double Lc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = s_lastm[k][tid];
      Lc[k] = c >= 0 ? sc.lnew[c] : s_L0[k];
      if (warp_chain_smem && warp_chain) Lc[k] = __dmul_rn(w_run[k], s_dq[k]);
    }
    int n_rank = 0, n_qual = 0, n_any = 0;
    for (int i = lo; i < hi; ++i) {
      const int m = out.model[i];
      if (sc.flags[i] & RF_ROUTE) {
        double q[K];
#pragma unroll
        for (int k = 0; k < K; ++k) q[k] = scores[(size_t)i * K + k];
        if (out.loads) {
#pragma unroll
          for (int k = 0; k < K; ++k) out.loads[(size_t)i * K + k] = Lc[k];
        }
        const uint8_t tb = tie_bits<K>(q, Lc, prm, m);
        if (tb) {
          out.flags[i] |= tb;  // this thread wrote the row's other flag bits
          n_rank += (tb & DF_TIE_RANK) ? 1 : 0;
          n_qual += (tb & DF_TIE_QUAL) ? 1 : 0;
          n_any += 1;
        }
      }
      double ln;
      if (warp_chain_smem && warp_chain) {
        const double y = yhat[(size_t)i * K + m];
#pragma unroll
        for (int k = 0; k < K; ++k) w_run[k] = k == m ? __dadd_rn(w_run[k], y) : w_run[k];
        double wm = w_run[0], dm = s_dq[0];
#pragma unroll
        for (int k = 1; k < K; ++k) {
          wm = k == m ? w_run[k] : wm;
          dm = k == m ? s_dq[k] : dm;
        }
        ln = __dmul_rn(wm, dm);
      } else {
        ln = sc.lnew[i];
      }
#pragma unroll
      for (int k = 0; k < K; ++k) Lc[k] = (k == m) ? ln : Lc[k];
    }
    __shared__ int s_ties[3];
    if (tid < 3) s_ties[tid] = 0;
    __syncthreads();
    if (n_any) {
      atomicAdd(&s_ties[0], n_rank);
      atomicAdd(&s_ties[1], n_qual);
      atomicAdd(&s_ties[2], n_any);
    }
    __syncthreads();
    if (tid < 3 && out.tie_counts) out.tie_counts[tid] = s_ties[tid];
  }

  if (tid == 0) {
#pragma unroll
    for (int m = 0; m < K; ++m) {
      mon.inflight_sum[m] = s_f[m];
      mon.inflight_comp[m] = s_c[m];
      mon.engine_clock[m] = s_clk[m];
      mon.engine_seq[m] = s_seq[m];
      mon.inflight_count[m] = s_cnt[m];
      mon.engine_iterations[m] = s_it[m];
      mon.engine_running[m] = s_run[m];
      mon.engine_queued[m] = s_que[m];
    }
    *out.n_committed = s_committed;
  }
  // ---- post-pass: commit assignments and in-flight stage bits ----
  for (int i = tid; i < n_ok; i += blockDim.x) {
    const int p = rows.program[i];
    if (sc.flags[i] & RF_ROUTE) mon.assignment[p] = (int8_t)out.model[i];
    atomicOr(mon.stage_bits + p, 1u << (rows.stage[i] - 1));
  }
}

template <int K>
static chm_status launch_schedule(const SelectParams& prm, const chm_monitor_state& mon,
                                  const chm_rows& rows, const chm_row_scratch& sc,
                                  const double* scores, const double* yhat,
                                  const chm_decisions& out, cudaStream_t s) {
  const size_t smem = 2 * sizeof(ChunkBuf<K>);
  const bool spec = prm.b_pow2_mask == (1u << K) - 1u;
  auto kern = spec ? schedule_rows_kernel<K, true> : schedule_rows_kernel<K, false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  prof::begin(prof::K_SELECT, s);
  kern<<<1, kThreads, smem, s>>>(prm, mon, rows, sc, scores, yhat, out);
  // bytes per row: q 4K + yhat 8K + out_tokens 4K + program/stage/arrival 16 +
  // scratch 16 + outputs 21 (+ loads 8K)
  prof::end(prof::K_SELECT, s, (double)rows.n_rows * (24.0 * K + 53.0));
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace chm

extern "C" chm_status chm_prepare_rows(const chm_monitor_state* mon, const chm_rows* rows,
                                       const chm_row_scratch* scratch,
                                       uint32_t* epoch_counter, void* stream) {
  if (!mon || !rows || !scratch || !epoch_counter || rows->n_rows < 0)
    return CHM_ERR_INVALID_ARG;
  chm::prof::begin(chm::prof::K_PREPARE, (cudaStream_t)stream);
  chm::prepare_rows_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(*mon, *rows, *scratch,
                                                                  epoch_counter);
  chm::prof::end(chm::prof::K_PREPARE, (cudaStream_t)stream, (double)rows->n_rows * 26.0);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_schedule_rows(const chm_pool* pool, const chm_balancer_cfg* cfg,
                                        const chm_monitor_state* mon, const chm_rows* rows,
                                        const chm_row_scratch* scratch, const double* scores,
                                        const double* yhat, const chm_decisions* out,
                                        void* stream) {
  if (!pool || !cfg || !mon || !rows || !scratch || !out || !yhat || !scores)
    return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS || rows->n_rows < 0) return CHM_ERR_INVALID_ARG;
  if (!(cfg->latency_slack >= 0.0) || !(cfg->confidence_margin >= 0.0) ||
      !(cfg->confidence_margin <= 1.0))
    return CHM_ERR_INVALID_ARG;
  chm::SelectParams prm{};
  for (int m = 0; m < K; ++m) {
    const int bi = pool->max_batch_size[m];
    if (bi < 1 || !(pool->decode_ms_per_token[m] > 0.0)) return CHM_ERR_INVALID_ARG;
    prm.d[m] = pool->decode_ms_per_token[m];
    prm.b[m] = (double)bi;
    prm.b_int[m] = bi;
    if ((bi & (bi - 1)) == 0) {
      prm.b_pow2_mask |= 1u << m;
      prm.inv_b[m] = 1.0 / (double)bi;
    }
  }
  prm.one_plus_slack = 1.0 + cfg->latency_slack;
  prm.margin = cfg->confidence_margin;
  prm.tie_tol = cfg->tie_tolerance;
  if (!scratch->lnew) return CHM_ERR_INVALID_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  switch (K) {
    case 1: return chm::launch_schedule<1>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
    case 2: return chm::launch_schedule<2>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
    case 3: return chm::launch_schedule<3>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
    case 4: return chm::launch_schedule<4>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
    case 5: return chm::launch_schedule<5>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
    case 6: return chm::launch_schedule<6>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
    case 7: return chm::launch_schedule<7>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
    default: return chm::launch_schedule<8>(prm, *mon, *rows, *scratch, scores, yhat, *out, s);
  }
}
