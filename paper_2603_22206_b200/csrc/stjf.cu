// K7 -- STJF + aging engine queues.
//
// Reference: EngineSim (engine.py:265-374). Queue order is ascending
// QueueEntry.sort_key = (starvation_level, priority, arrival, seq)
// (engine.py:55-69). A scheduling iteration (`_iterate`, engine.py:328-338)
// admits the queue minimum while the running batch has free slots, then ages
// every still-queued entry (`_age_queued`, engine.py:340-374): count += 1 and,
// at count >= S, level -= 1, count = 0, quantum = 0.
//
// Device layout: engine m owns segment [m*cap, (m+1)*cap) of SoA arrays kept in
// seq order, so "seq" comparisons are storage-index comparisons and a stable
// sort over storage order needs no seq digits. One CTA per engine runs an LSD
// radix sort (8-bit digits, digits equal across the segment skipped) by
// (count, level, priority[, arrival]). Entries with equal count age in lock
// step, so each count group keeps its internal order for the whole call: R
// iterations become R rounds of "admit the minimum of the group heads, then
// shift each group's (count, level offset)". A final radix sort by
// (level, priority[, arrival]) writes the STJF order of what remains.
//
// Key storage: segments up to kQMax entries keep the sort keys in shared
// memory (16-bit indices); larger segments (the 64k-entry cfg4 stress) keep
// them in a global scratch area (32-bit indices, L2 resident) with the same
// algorithm -- chosen on the host from the segment capacity.
//
// HBM bytes per queued entry per call (algorithmic): read 40 (priority 8,
// arrival 8, handle 8, out_tokens 4, level 4, count 4, quantum 4; seq is
// implicit) + write 40 + order 4.
#include "common.cuh"
#include "prof.cuh"
#include "stjf_common.cuh"

namespace chm {

constexpr int kQMax = 10240;       // entries per engine segment held in smem
constexpr int kQThreads = 1024;
constexpr int kQWarps = kQThreads / 32;
constexpr size_t kScratchBytesPerEntry = 8 + 2 + 2 + 4 + 4;  // prio, lvl, cnt, idx a/b
constexpr int kQHuge = 1 << 18;    // larger segments: grid-wide passes (stjf_huge.cu)

size_t queue_huge_scratch_bytes(int capacity);
unsigned long long queue_huge_fast_calls();
chm_status launch_queue_huge(const QueueParams& prm, const chm_monitor_state& mon,
                             const chm_queue_state& q, const chm_rows& rows,
                             const chm_decisions& dec, const int32_t* n_complete,
                             int n_iterations, int mode, int32_t* err, cudaStream_t s);

// Shared control state (both storage modes).
struct QueueCtl {
  int wcnt[kQWarps][256];
  int g_start[kMaxGroups], g_end[kMaxGroups], g_cur[kMaxGroups];
  int g_count[kMaxGroups], g_lvloff[kMaxGroups];
  unsigned long long red_or[4], red_and[4];
  int scan[kQWarps];
  int misc[8];
};

template <typename Idx>
struct Keys {
  unsigned long long* prio;  // order-preserving bits of priority
  uint16_t* lvl;             // starvation_level + 32768
  uint16_t* cnt;             // starvation_count
  Idx* a;
  Idx* b;
};

// Small segments: keys right after the control block in shared memory.
struct SmallKeysSmem {
  unsigned long long prio[kQMax];
  uint16_t lvl[kQMax];
  uint16_t cnt[kQMax];
  uint16_t a[kQMax];
  uint16_t b[kQMax];
};

// One stable LSD counting-sort pass over `n` indices.
// src: 0 = arrival (global), 1 = priority, 2 = level, 3 = count; byte = digit index.
// Warp w owns the contiguous slice [w C, (w + 1) C) of `in`: a per-warp digit
// histogram, one block-wide exclusive scan in (digit, warp) order, then each
// warp scatters its slice in order (match_any ranks within 32-entry steps), so
// the pass is stable with three block barriers in total. (The round-1 pass
// walked 1024-entry blocks with a 32-step serial per-digit warp scan and three
// barriers per block: ~5x slower at 8k entries.)
template <typename Idx>
__device__ void radix_pass(QueueCtl& s, const Keys<Idx>& k, const Idx* in, Idx* out, int n,
                           int src, int byte, const double* __restrict__ arrival) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto digit = [&](int e) -> int {
    unsigned long long v;
    if (src == 0) v = f64_key(arrival[e]);
    else if (src == 1) v = k.prio[e];
    else if (src == 2) v = k.lvl[e];
    else v = k.cnt[e];
    return (int)((v >> (8 * byte)) & 255ull);
  };
  const int chunk = (n + kQWarps - 1) / kQWarps;
  const int lo = min(n, warp * chunk), hi = min(n, lo + chunk);
  const unsigned lt = (1u << lane) - 1u;
  // 1. per-warp histogram
#pragma unroll
  for (int j = 0; j < 8; ++j) s.wcnt[warp][lane * 8 + j] = 0;
  __syncwarp();
  for (int blk = lo; blk < hi; blk += 32) {
    const int i = blk + lane;
    const bool valid = i < hi;
    const int d = valid ? digit((int)in[i]) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (valid && (peers & lt) == 0) s.wcnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // 2. exclusive scan over L = 32 d + w; thread t covers L in [8 t, 8 t + 8)
  {
    const int d = tid >> 2, w0 = (tid & 3) * 8;
    int v[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { v[j] = s.wcnt[w0 + j][d]; tot += v[j]; }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s.scan[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const int x = s.scan[lane];
      int xi = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, xi, o);
        if (lane >= o) xi += t;
      }
      s.scan[lane] = xi - x;
    }
    __syncthreads();
    int run = s.scan[warp] + incl - tot;
#pragma unroll
    for (int j = 0; j < 8; ++j) { s.wcnt[w0 + j][d] = run; run += v[j]; }
  }
  __syncthreads();
  // 3. in-order scatter of each warp's slice
  for (int blk = lo; blk < hi; blk += 32) {
    const int i = blk + lane;
    const bool valid = i < hi;
    const Idx e = valid ? in[i] : (Idx)0;
    const int d = valid ? digit((int)e) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & lt);
    if (valid) out[s.wcnt[warp][d] + rank] = e;
    __syncwarp();
    if (valid && rank == 0) s.wcnt[warp][d] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
}

// Stable sort of [0, n) by the given key sources (most significant last in
// `srcs`), skipping digits that are equal across all entries.
template <typename Idx>
__device__ void radix_sort(QueueCtl& s, const Keys<Idx>& k, int n, const int* srcs, int n_srcs,
                           const double* __restrict__ arrival, bool use_arrival, Idx*& sorted,
                           Idx*& spare) {
  const int tid = threadIdx.x;
  if (tid < 4) { s.red_or[tid] = 0ull; s.red_and[tid] = ~0ull; }
  for (int i = tid; i < n; i += blockDim.x) k.a[i] = (Idx)i;
  __syncthreads();
  unsigned long long o[4] = {0, 0, 0, 0}, a[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  for (int i = tid; i < n; i += blockDim.x) {
    const unsigned long long v0 = use_arrival ? f64_key(arrival[i]) : 0ull;
    o[0] |= v0; a[0] &= v0;
    o[1] |= k.prio[i]; a[1] &= k.prio[i];
    o[2] |= k.lvl[i]; a[2] &= k.lvl[i];
    o[3] |= k.cnt[i]; a[3] &= k.cnt[i];
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    for (int off = 16; off; off >>= 1) {
      o[j] |= __shfl_xor_sync(0xffffffffu, o[j], off);
      a[j] &= __shfl_xor_sync(0xffffffffu, a[j], off);
    }
  }
  if ((tid & 31) == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) { atomicOr(&s.red_or[j], o[j]); atomicAnd(&s.red_and[j], a[j]); }
  }
  __syncthreads();
  Idx* in = k.a;
  Idx* out = k.b;
  for (int qi = 0; qi < n_srcs; ++qi) {
    const int src = srcs[qi];
    if (src == 0 && !use_arrival) continue;
    const int n_bytes = (src <= 1) ? 8 : 2;
    const unsigned long long diff = s.red_or[src] ^ s.red_and[src];
    for (int byte = 0; byte < n_bytes; ++byte) {
      if (((diff >> (8 * byte)) & 255ull) == 0) continue;
      radix_pass(s, k, in, out, n, src, byte, arrival);
      Idx* t = in; in = out; out = t;
    }
  }
  sorted = in;
  spare = out;
}

// Cross-GPU admission merge inputs (mode 2, chm_queue_admit_merged).
struct MergeArgs {
  const chm_queue_key* gathered;  // [G][K][F]
  int G, F, rank;
  const int32_t* release;         // [K] slots freed before the iteration (nullable)
  const double* target;           // [K] mode 3: advance_to target per engine
};

// Engine clock: start a stint for an admitted entry at `now`
// (_BatchEngine._admit, engine.py:202-227). Plain (unfused) double rounding,
// as Python evaluates now + prefill and decode_start + tokens * d.
__device__ __forceinline__ bool run_admit(const chm_engine_run& er, int m, int n_run,
                                          int64_t handle, int64_t seq, int32_t tokens,
                                          int32_t input, double now, double d) {
  if (n_run >= er.capacity) return false;
  const size_t b = (size_t)m * er.capacity + n_run;
  const double ds = __dadd_rn(now, __dmul_rn(er.prefill_ms_per_token[m], (double)input));
  er.handle[b] = handle;
  er.seq[b] = seq;
  er.decode_start[b] = ds;
  er.stint_end[b] = __dadd_rn(ds, __dmul_rn((double)tokens, d));
  er.stint_tokens[b] = tokens;
  return true;
}

__device__ __forceinline__ bool cand_less(const chm_queue_key& a, const chm_queue_key& b) {
  if (a.level != b.level) return a.level < b.level;
  if (a.priority != b.priority) return a.priority < b.priority;
  if (a.arrival != b.arrival) return a.arrival < b.arrival;
  return a.seq < b.seq;
}

// Engine m's admissions this iteration: a_global = min(free slots, gathered
// candidates) of the global minimum keys; a_local = how many of them are this
// rank's (its candidates are its STJF head, so it admits its first a_local).
__device__ void merge_counts(const MergeArgs& ma, int m, int K, int free_slots, int* misc) {
  const int n_c = ma.G * ma.F;
  __shared__ int n_real, n_own;
  if (threadIdx.x == 0) { n_real = 0; n_own = 0; }
  __syncthreads();
  int real = 0;
  for (int i = threadIdx.x; i < n_c; i += blockDim.x) {
    const chm_queue_key& c = ma.gathered[((size_t)(i / ma.F) * K + m) * ma.F + i % ma.F];
    real += c.level != INT64_MAX;
  }
  atomicAdd(&n_real, real);
  __syncthreads();
  const int a_global = min(free_slots, n_real);
  int own = 0;
  for (int j = threadIdx.x; j < ma.F; j += blockDim.x) {
    const chm_queue_key mine = ma.gathered[((size_t)ma.rank * K + m) * ma.F + j];
    if (mine.level == INT64_MAX) continue;
    int rank_j = 0;
    for (int i = 0; i < n_c && rank_j < a_global; ++i) {
      const chm_queue_key c = ma.gathered[((size_t)(i / ma.F) * K + m) * ma.F + i % ma.F];
      if (c.level != INT64_MAX && cand_less(c, mine)) ++rank_j;
    }
    own += rank_j < a_global;
  }
  atomicAdd(&n_own, own);
  __syncthreads();
  if (threadIdx.x == 0) { misc[0] = n_own; misc[1] = a_global; }
  __syncthreads();
}

__global__ void candidates_kernel(QueueParams prm, chm_monitor_state mon, chm_queue_state q,
                                  int F, chm_queue_key* __restrict__ out) {
  const int m = blockIdx.x;
  const size_t seg = (size_t)m * q.capacity;
  const int n = mon.engine_queued[m];
  const int take = min(n, prm.b[m]);
  for (int j = threadIdx.x; j < F; j += blockDim.x) {
    chm_queue_key k;
    if (j < take) {
      const int e = q.order[seg + j];
      k.level = q.level[seg + e];
      k.priority = q.priority[seg + e];
      k.arrival = q.arrival[seg + e];
      k.seq = q.seq[seg + e];
      k.handle = q.handle[seg + e];
    } else {
      k.level = INT64_MAX;
      k.priority = 0; k.arrival = 0; k.seq = 0; k.handle = -1;
    }
    out[(size_t)m * F + j] = k;
  }
}

// Engine clock, one warp: the running request with the smallest
// (stint_end, seq) ends if stint_end <= target (advance_to, engine.py:174-183):
// lane 0 records the completion (_finish_stint + _on_stint_end, 229-239,
// 396-407) and moves the last entry into its slot. Returns 1 when a stint
// ended (bt = its end), 0 when none is due, 2 on a clock violation.
__device__ int finish_next_stint(const chm_engine_run& er, int m, size_t rb, int n_run, int lane,
                                 double tgt, double clock, int32_t* err, double& bt_out) {
  double bt = 0;
  long long bs = LLONG_MAX;
  int bj = -1;
  for (int j = lane; j < n_run; j += 32) {
    const double te = er.stint_end[rb + j];
    const long long sq = er.seq[rb + j];
    if (bj < 0 || te < bt || (te == bt && sq < bs)) { bt = te; bs = sq; bj = j; }
  }
  for (int off = 16; off; off >>= 1) {
    const double ot = __shfl_xor_sync(0xffffffffu, bt, off);
    const long long os = __shfl_xor_sync(0xffffffffu, bs, off);
    const int oj = __shfl_xor_sync(0xffffffffu, bj, off);
    if (oj >= 0 && (bj < 0 || ot < bt || (ot == bt && os < bs))) { bt = ot; bs = os; bj = oj; }
  }
  bt_out = bt;
  if (bj < 0 || !(bt <= tgt)) return 0;
  if (bt < clock - 1e-9) {  // _finish_stint -> _advance_clock (engine.py:140-143, 233)
    if (lane == 0) report_error(err, CHM_ERR_TIME_BACKWARDS, 0, m, 1);
    return 2;
  }
  if (lane == 0) {
    const int nd = er.n_done[m];
    if (nd < er.done_capacity) {
      er.done_handle[(size_t)m * er.done_capacity + nd] = er.handle[rb + bj];
      er.done_time[(size_t)m * er.done_capacity + nd] = bt;
      er.n_done[m] = nd + 1;
    } else {
      report_error(err, CHM_ERR_CAPACITY, 0, m, nd);
    }
    er.tokens_emitted[m] += er.stint_tokens[rb + bj];
    er.served[m] += 1;
    const size_t last = rb + n_run - 1, at = rb + bj;
    er.handle[at] = er.handle[last];
    er.seq[at] = er.seq[last];
    er.stint_end[at] = er.stint_end[last];
    er.decode_start[at] = er.decode_start[last];
    er.stint_tokens[at] = er.stint_tokens[last];
  }
  return 1;
}

// mode 0: completions (R = n_complete[m], each frees one running slot first)
// mode 1: tick (append queued rows, then R = n_iterations explicit iterations)
// mode 2: one iteration with a cross-GPU admission merge (MergeArgs)
template <typename Idx, bool kBig>
__global__ void __launch_bounds__(kQThreads, 1) queue_kernel(
    QueueParams prm, chm_monitor_state mon, chm_queue_state q, chm_rows rows,
    chm_decisions dec, const int32_t* __restrict__ n_complete, int n_iterations, int mode,
    int32_t* err, MergeArgs ma, chm_engine_run er) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  QueueCtl& s = *reinterpret_cast<QueueCtl*>(smem_raw);
  const int m = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t seg = (size_t)m * q.capacity;
  const int cap = min(q.capacity, prm.cap_limit);
  Keys<Idx> k;
  if constexpr (kBig) {
    uint8_t* base = reinterpret_cast<uint8_t*>(q.scratch) +
                    (size_t)m * q.capacity * kScratchBytesPerEntry;
    const size_t C = (size_t)q.capacity;
    k.prio = reinterpret_cast<unsigned long long*>(base);
    k.lvl = reinterpret_cast<uint16_t*>(base + 8 * C);
    k.cnt = reinterpret_cast<uint16_t*>(base + 10 * C);
    k.a = reinterpret_cast<Idx*>(base + 12 * C);
    k.b = reinterpret_cast<Idx*>(base + 16 * C);
  } else {
    SmallKeysSmem& ks = *reinterpret_cast<SmallKeysSmem*>(smem_raw + sizeof(QueueCtl));
    k.prio = ks.prio;
    k.lvl = ks.lvl;
    k.cnt = ks.cnt;
    k.a = reinterpret_cast<Idx*>(ks.a);
    k.b = reinterpret_cast<Idx*>(ks.b);
  }
  double* prio_g = q.priority + seg;
  double* arr_g = q.arrival + seg;
  int64_t* seq_g = q.seq + seg;
  int64_t* handle_g = q.handle + seg;
  int32_t* out_g = q.out_tokens + seg;
  int32_t* lvl_g = q.level + seg;
  int32_t* cnt_g = q.count + seg;
  int32_t* qnt_g = q.quantum + seg;

  int n = mon.engine_queued[m];
  int run = mon.engine_running[m];
  const int bmax = prm.b[m];
  // engine clock (running set) tracking
  const bool track = er.handle != nullptr;
  int n_run = track ? er.n[m] : 0;
  double clock = mon.engine_clock[m];
  int32_t* qin_g = track ? er.queue_input_tokens + seg : nullptr;
  const double tgt = mode == 3 ? ma.target[m] : 0.0;
  if (mode == 3 && tgt < clock - 1e-9) {  // EngineSim._advance_clock (engine.py:140-143)
    if (tid == 0) report_error(err, CHM_ERR_TIME_BACKWARDS, 0, m, 0);
    return;
  }

  // ---- mode 1: append rows queued on this engine by chm_schedule_rows ----
  if (mode == 1) {
    // rows queued this batch were already counted in engine_queued by K6
    const int n_new_total = count_queued_rows(m, dec, s.scan, s.misc);
    const int n_old = n - n_new_total;
    if (n_old < 0 || n > cap) {
      if (tid == 0) report_error(err, n > cap ? CHM_ERR_CAPACITY : CHM_ERR_INVALID_STATE,
                                 0, m, n);
      return;
    }
    append_queued_rows(m, prm.K, rows, dec, seg, q, n_old, s.scan, s.misc,
                       track ? er.queue_input_tokens : nullptr);
    if (track) {
      // rows admitted at enqueue (EngineSim.enqueue -> _iterate, engine.py:145-158)
      // start their stints at their arrival, in row (= seq) order
      const int n_rows = *dec.n_committed;
      for (int blk = 0; blk < n_rows; blk += blockDim.x) {
        const int i = blk + tid;
        const bool take = i < n_rows && dec.model[i] == m && (dec.flags[i] & 2u);
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (lane == 0) s.scan[warp] = __popc(bal);
        __syncthreads();
        if (warp == 0) {
          int v = lane < kQWarps ? s.scan[lane] : 0, incl = v;
          for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
          }
          if (lane < kQWarps) s.scan[lane] = incl - v;
          if (lane == 31) s.misc[1] = incl;
        }
        __syncthreads();
        if (take) {
          const int pos = n_run + s.scan[warp] + __popc(bal & ((1u << lane) - 1u));
          if (!run_admit(er, m, pos, rows.handle ? rows.handle[i] : (int64_t)i, dec.seq[i],
                         rows.out_tokens ? rows.out_tokens[(size_t)i * prm.K + m] : 0,
                         rows.input_tokens ? rows.input_tokens[i] : 1, rows.arrival[i],
                         prm.d[m]))
            report_error(err, CHM_ERR_CAPACITY, i, m, pos);
        }
        n_run += s.misc[1];
        __syncthreads();
      }
    }
    __threadfence_block();
  } else {
    if (n > cap) {
      if (tid == 0) report_error(err, CHM_ERR_CAPACITY, 0, m, n);
      return;
    }
  }
  __syncthreads();

  // ---- stage keys ----
  int unsorted = 0;
  for (int i = tid; i < n; i += blockDim.x) {
    k.prio[i] = f64_key(prio_g[i]);
    k.lvl[i] = (uint16_t)(lvl_g[i] + 32768);
    k.cnt[i] = (uint16_t)min(max(cnt_g[i], 0), 65535);
    if (i > 0 && arr_g[i] < arr_g[i - 1]) unsorted = 1;
  }
  unsorted = __syncthreads_or(unsorted);
  const bool use_arr = unsorted != 0;

  const int R = (mode == 0) ? n_complete[m]
                : (mode == 2 ? 1 : (mode == 3 ? 0x7fffffff : n_iterations));
  int iters = 0;  // scheduling iterations run by this call
  // mode 2: this rank's and the global admission counts from the gathered keys
  // release[m] < 0: engine m runs no iteration this call
  const int rel = (mode == 2 && ma.release) ? ma.release[m] : 0;
  int a_local = 0, a_global = 0;
  if (mode == 2 && rel < 0) {
    // nothing to do; the order from the previous call stays valid
    return;
  }
  if (mode == 2) {
    merge_counts(ma, m, prm.K, max(0, bmax - max(run - rel, 0)), &s.misc[0]);
    a_local = s.misc[0];
    a_global = s.misc[1];
    __syncthreads();
  }
  // Admissions of this call are appended after those already reported since
  // the host last zeroed n_admitted (completions and tick share the list).
  const int n_adm0 = q.n_admitted[m];
  int n_adm = 0, n_prom = 0;

  if (R > 0 && prm.demote) {
    // ---- generic iterations (demote_while_queued, engine.py:340-374): a
    // promoted entry's quantum runs per entry, so equal-count entries no
    // longer age in lock step. Per admission a block-wide argmin of the live
    // entries' keys; aging per entry, in place. ----
    Idx* flag = k.b;  // 1 = admitted this call
    for (int i = tid; i < n; i += blockDim.x) flag[i] = 0;
    __shared__ int gen_e[kQWarps];
    __shared__ int gen_l[kQWarps];
    __shared__ unsigned long long gen_p[kQWarps], gen_a[kQWarps];
    __shared__ double gen_t;
    __shared__ int gen_prom;
    if (tid == 0) gen_prom = 0;
    __syncthreads();
    int remaining = n;
    const size_t rb = (size_t)m * (track ? er.capacity : 0);
    auto less = [](int l1, unsigned long long p1, unsigned long long a1, int e1, int l2,
                   unsigned long long p2, unsigned long long a2, int e2) {
      if (e2 < 0) return e1 >= 0;
      if (e1 < 0) return false;
      if (l1 != l2) return l1 < l2;
      if (p1 != p2) return p1 < p2;
      if (a1 != a2) return a1 < a2;
      return e1 < e2;
    };
    for (int r = 0; r < R; ++r) {
      double t_iter = clock;
      if (mode == 3) {
        if (warp == 0) {
          double bt;
          const int st3 = finish_next_stint(er, m, rb, n_run, lane, tgt, clock, err, bt);
          if (lane == 0) { s.misc[6] = st3; gen_t = bt; }
        }
        __syncthreads();
        const int st3 = s.misc[6];
        const double bt = gen_t;
        __syncthreads();
        if (st3 != 1) break;
        --n_run;
        run = max(run - 1, 0);
        clock = bt;
        t_iter = bt;
      }
      ++iters;
      if (mode == 0) run = max(run - 1, 0);
      if (mode == 2) run = max(run - rel, 0);
      const int a = mode == 2 ? min(a_local, remaining) : max(0, min(bmax - run, remaining));
      for (int t = 0; t < a; ++t) {
        int bl = 0, be = -1;
        unsigned long long bp = 0, ba = 0;
        for (int i = tid; i < n; i += blockDim.x) {
          if (flag[i]) continue;
          const int l = lvl_g[i];
          const unsigned long long pk = k.prio[i];
          const unsigned long long av = use_arr ? f64_key(arr_g[i]) : 0ull;
          if (less(l, pk, av, i, bl, bp, ba, be)) { bl = l; bp = pk; ba = av; be = i; }
        }
        for (int off = 16; off; off >>= 1) {
          const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
          const unsigned long long op = __shfl_xor_sync(0xffffffffu, bp, off);
          const unsigned long long oa = __shfl_xor_sync(0xffffffffu, ba, off);
          const int oe = __shfl_xor_sync(0xffffffffu, be, off);
          if (less(ol, op, oa, oe, bl, bp, ba, be)) { bl = ol; bp = op; ba = oa; be = oe; }
        }
        if (lane == 0) { gen_l[warp] = bl; gen_p[warp] = bp; gen_a[warp] = ba; gen_e[warp] = be; }
        __syncthreads();
        if (warp == 0) {
          bl = gen_l[lane]; bp = gen_p[lane]; ba = gen_a[lane]; be = gen_e[lane];
          for (int off = 16; off; off >>= 1) {
            const int ol = __shfl_xor_sync(0xffffffffu, bl, off);
            const unsigned long long op = __shfl_xor_sync(0xffffffffu, bp, off);
            const unsigned long long oa = __shfl_xor_sync(0xffffffffu, ba, off);
            const int oe = __shfl_xor_sync(0xffffffffu, be, off);
            if (less(ol, op, oa, oe, bl, bp, ba, be)) { bl = ol; bp = op; ba = oa; be = oe; }
          }
          if (lane == 0) {
            flag[be] = 1;
            q.admitted[seg + n_adm0 + n_adm + t] = handle_g[be];
            if (track && !run_admit(er, m, n_run + t, handle_g[be], seq_g[be], out_g[be],
                                    qin_g[be], t_iter, prm.d[m]))
              report_error(err, CHM_ERR_CAPACITY, 0, m, n_run + t);
          }
        }
        __syncthreads();
      }
      n_adm += a;
      remaining -= a;
      run += mode == 2 ? a_global : a;
      if (track) n_run += a;
      if (prm.aging_enabled && remaining > 0) {
        int np = 0;
        for (int i = tid; i < n; i += blockDim.x) {
          if (flag[i]) continue;
          const int c2 = cnt_g[i] + 1;
          if (c2 >= prm.S) {  // promote
            cnt_g[i] = 0;
            lvl_g[i] -= 1;
            qnt_g[i] = 0;
            ++np;
          } else {
            cnt_g[i] = c2;
            if (lvl_g[i] < 0) {  // demote_while_queued
              const int q2 = qnt_g[i] + 1;
              if (q2 >= prm.Q) {
                qnt_g[i] = 0;
                lvl_g[i] += 1;
              } else {
                qnt_g[i] = q2;
              }
            }
          }
        }
        for (int off = 16; off; off >>= 1) np += __shfl_xor_sync(0xffffffffu, np, off);
        if (lane == 0 && np) atomicAdd(&gen_prom, np);
      }
      __syncthreads();
    }
    n_prom = gen_prom;
    // ---- compact survivors in seq (storage) order ----
    int out_base = 0;
    for (int blk = 0; blk < n; blk += blockDim.x) {
      const int i = blk + tid;
      const bool keep = i < n && !flag[i];
      double pr = 0, ar = 0;
      int64_t sq = 0, hd = 0;
      int ot = 0, lv = 0, ct = 0, qn = 0, in = 0;
      if (keep) {
        pr = prio_g[i]; ar = arr_g[i]; sq = seq_g[i]; hd = handle_g[i]; ot = out_g[i];
        lv = lvl_g[i]; ct = cnt_g[i]; qn = qnt_g[i];
        if (track) in = qin_g[i];
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) s.scan[warp] = __popc(bal);
      __syncthreads();
      if (warp == 0) {
        int v = s.scan[lane], incl = v;
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        s.scan[lane] = incl - v;
        if (lane == 31) s.misc[6] = incl;
      }
      __syncthreads();
      if (keep) {
        const int pos = out_base + s.scan[warp] + __popc(bal & ((1u << lane) - 1u));
        prio_g[pos] = pr; arr_g[pos] = ar; seq_g[pos] = sq; handle_g[pos] = hd;
        out_g[pos] = ot; lvl_g[pos] = lv; cnt_g[pos] = ct; qnt_g[pos] = qn;
        if (track) qin_g[pos] = in;
        k.prio[pos] = f64_key(pr);
        k.lvl[pos] = (uint16_t)(lv + 32768);
        k.cnt[pos] = (uint16_t)min(max(ct, 0), 65535);
      }
      out_base += s.misc[6];
      __syncthreads();
    }
    n = out_base;
  } else if (R > 0) {
    // ---- sort by (count, level, priority[, arrival]) and form count groups ----
    const int srcs[4] = {0, 1, 2, 3};
    Idx *sorted, *spare;
    radix_sort(s, k, n, srcs, 4, arr_g, use_arr, sorted, spare);
    if (tid == 0) s.misc[2] = 0;
    __syncthreads();
    for (int p = tid; p < n; p += blockDim.x) {
      const bool head = (p == 0) || k.cnt[sorted[p]] != k.cnt[sorted[p - 1]];
      if (head) {
        const int g = atomicAdd(&s.misc[2], 1);
        if (g < kMaxGroups) {
          s.g_start[g] = p;
          s.g_count[g] = k.cnt[sorted[p]];
        }
      }
    }
    __syncthreads();
    const int G = s.misc[2];
    if (G > kMaxGroups) {
      if (tid == 0) report_error(err, CHM_ERR_UNSUPPORTED, 0, m, G);
      return;
    }
    if (tid == 0) {
      // groups were discovered out of order; insertion sort by start (G small)
      for (int a = 1; a < G; ++a) {
        int st = s.g_start[a], ct = s.g_count[a], b2 = a - 1;
        while (b2 >= 0 && s.g_start[b2] > st) {
          s.g_start[b2 + 1] = s.g_start[b2];
          s.g_count[b2 + 1] = s.g_count[b2];
          --b2;
        }
        s.g_start[b2 + 1] = st;
        s.g_count[b2 + 1] = ct;
      }
      for (int g = 0; g < G; ++g) {
        s.g_end[g] = (g + 1 < G) ? s.g_start[g + 1] : n;
        s.g_cur[g] = s.g_start[g];
        s.g_lvloff[g] = 0;
      }
    }
    __syncthreads();

    // ---- R scheduling iterations (warp 0) ----
    if (warp == 0) {
      int remaining = n;
      const size_t rb = (size_t)m * (track ? er.capacity : 0);
      for (int r = 0; r < R; ++r) {
        double t_iter = clock;
        if (mode == 3) {
          // next stint end: min (stint_end, seq) of the running set (engine.py:178-183)
          double bt;
          const int st3 = finish_next_stint(er, m, rb, n_run, lane, tgt, clock, err, bt);
          if (st3 != 1) break;
          __syncwarp();
          --n_run;
          run = max(run - 1, 0);
          clock = bt;
          t_iter = bt;
        }
        ++iters;
        if (mode == 0) run = max(run - 1, 0);
        if (mode == 2) run = max(run - rel, 0);
        const int a = mode == 2 ? min(a_local, remaining) : max(0, min(bmax - run, remaining));
        for (int t = 0; t < a; ++t) {
          HeadKey best;
          best.g = -1;
          for (int g0 = 0; g0 < G; g0 += 32) {
            const int g = g0 + lane;
            HeadKey hk;
            hk.g = -1;
            if (g < G && s.g_cur[g] < s.g_end[g]) {
              const int e = (int)sorted[s.g_cur[g]];
              hk.e = e;
              hk.g = g;
              hk.lvl = (int)k.lvl[e] - 32768 + s.g_lvloff[g];
              hk.prio = k.prio[e];
              hk.arr = use_arr ? f64_key(arr_g[e]) : 0ull;
            }
            for (int off = 16; off; off >>= 1) {
              HeadKey o;
              o.lvl = __shfl_xor_sync(0xffffffffu, hk.lvl, off);
              o.prio = __shfl_xor_sync(0xffffffffu, hk.prio, off);
              o.arr = __shfl_xor_sync(0xffffffffu, hk.arr, off);
              o.e = __shfl_xor_sync(0xffffffffu, hk.e, off);
              o.g = __shfl_xor_sync(0xffffffffu, hk.g, off);
              if (o.g >= 0 && (hk.g < 0 || key_less(o, hk))) hk = o;
            }
            if (hk.g >= 0 && (best.g < 0 || key_less(hk, best))) best = hk;
          }
          if (lane == 0) {
            q.admitted[seg + n_adm0 + n_adm] = handle_g[best.e];
            s.g_cur[best.g] += 1;
            if (track && !run_admit(er, m, n_run, handle_g[best.e], seq_g[best.e],
                                    out_g[best.e], qin_g[best.e], t_iter, prm.d[m]))
              report_error(err, CHM_ERR_CAPACITY, 0, m, n_run);
          }
          if (track) ++n_run;
          __syncwarp();
          ++n_adm;
          --remaining;
        }
        run += mode == 2 ? a_global : a;
        if (prm.aging_enabled && remaining > 0) {
          for (int g = lane; g < G; g += 32) {
            if (s.g_cur[g] < s.g_end[g]) {
              int c2 = s.g_count[g] + 1;
              if (c2 >= prm.S) {
                c2 = 0;
                s.g_lvloff[g] -= 1;
                n_prom += s.g_end[g] - s.g_cur[g];
              }
              s.g_count[g] = c2;
            }
          }
          __syncwarp();
        }
      }
      for (int off = 16; off; off >>= 1) n_prom += __shfl_xor_sync(0xffffffffu, n_prom, off);
      if (lane == 0) {
        s.misc[3] = n_adm; s.misc[4] = n_prom; s.misc[5] = run;
        s.misc[0] = iters; s.misc[7] = n_run;
        reinterpret_cast<double*>(s.red_or)[0] = clock;
      }
    }
    __syncthreads();
    n_adm = s.misc[3];
    n_prom = s.misc[4];
    run = s.misc[5];
    iters = s.misc[0];
    n_run = s.misc[7];
    clock = reinterpret_cast<double*>(s.red_or)[0];
    // ---- per-entry outcome: spare[e] = group or kAdmitted ----
    for (int p = tid; p < n; p += blockDim.x) {
      int lo = 0, hi = G - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s.g_start[mid] <= p) lo = mid; else hi = mid - 1;
      }
      const int e = (int)sorted[p];
      spare[e] = (p < s.g_cur[lo]) ? (Idx)kAdmitted : (Idx)lo;
    }
    __syncthreads();
    // ---- compact survivors in seq (storage) order, applying the aging ----
    int out_base = 0;
    for (int blk = 0; blk < n; blk += blockDim.x) {
      const int i = blk + tid;
      const bool valid = i < n;
      const Idx g = valid ? spare[i] : (Idx)kAdmitted;
      const bool keep = valid && g != (Idx)kAdmitted;
      double pr = 0, ar = 0;
      int64_t sq = 0, hd = 0;
      int ot = 0, lv = 0, ct = 0, qn = 0, in = 0;
      unsigned long long pk = 0;
      if (keep) {
        pr = prio_g[i]; ar = arr_g[i]; sq = seq_g[i]; hd = handle_g[i]; ot = out_g[i];
        if (track) in = qin_g[i];
        lv = (int)k.lvl[i] - 32768 + s.g_lvloff[g];
        ct = prm.aging_enabled ? s.g_count[g] : cnt_g[i];
        qn = (s.g_lvloff[g] != 0) ? 0 : qnt_g[i];
        pk = k.prio[i];
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) s.scan[warp] = __popc(bal);
      __syncthreads();
      if (warp == 0) {
        int v = s.scan[lane], incl = v;
        for (int o = 1; o < 32; o <<= 1) {
          int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        s.scan[lane] = incl - v;
        if (lane == 31) s.misc[6] = incl;
      }
      __syncthreads();
      if (keep) {
        const int pos = out_base + s.scan[warp] + __popc(bal & ((1u << lane) - 1u));
        prio_g[pos] = pr; arr_g[pos] = ar; seq_g[pos] = sq; handle_g[pos] = hd;
        out_g[pos] = ot; lvl_g[pos] = lv; cnt_g[pos] = ct; qnt_g[pos] = qn;
        if (track) qin_g[pos] = in;
        k.prio[pos] = pk;
        k.lvl[pos] = (uint16_t)(lv + 32768);
        k.cnt[pos] = (uint16_t)ct;
      }
      out_base += s.misc[6];
      __syncthreads();
    }
    n = out_base;
  }

  // ---- final STJF order of the remaining queue: (level, priority[, arrival], seq) ----
  {
    int unsorted2 = 0;
    for (int i = tid + 1; i < n; i += blockDim.x)
      if (arr_g[i] < arr_g[i - 1]) unsorted2 = 1;
    const bool ua = __syncthreads_or(unsorted2) != 0;
    const int srcs[3] = {0, 1, 2};
    Idx *sorted, *spare;
    radix_sort(s, k, n, srcs, 3, arr_g, ua, sorted, spare);
    for (int r = tid; r < n; r += blockDim.x) q.order[seg + r] = (int32_t)sorted[r];
    if (tid == 0) q.arrival_unsorted[m] = ua ? 1 : 0;
  }
  if (tid == 0) {
    q.n_admitted[m] = n_adm0 + n_adm;
    q.n_promoted[m] += n_prom;
    mon.engine_queued[m] = n;
    mon.engine_running[m] = run;
    mon.engine_iterations[m] += iters;
    if (track) er.n[m] = n_run;
    if (mode == 3) mon.engine_clock[m] = fmax(clock, tgt);
  }
}

static chm_status launch_queue(const chm_pool* pool, const chm_aging_cfg* aging,
                               const chm_monitor_state* mon, const chm_queue_state* q,
                               const chm_rows* rows, const chm_decisions* dec,
                               const int32_t* n_complete, int n_iterations, int mode,
                               int32_t* err, cudaStream_t s, MergeArgs ma = MergeArgs{}) {
  if (!pool || !aging || !mon || !q) return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS || q->capacity < 1) return CHM_ERR_INVALID_ARG;
  if (aging->enabled && (aging->starvation_threshold < 1 || aging->starvation_threshold > 65535))
    return CHM_ERR_UNSUPPORTED;
  // demote_while_queued: the generic per-entry path (not on the grid-wide one)
  if (aging->enabled && aging->demote_while_queued && q->capacity > kQHuge)
    return CHM_ERR_UNSUPPORTED;
  if (aging->enabled && aging->demote_while_queued && aging->running_quantum < 1)
    return CHM_ERR_INVALID_ARG;
  const bool big = q->capacity > kQMax;
  if (big && !q->scratch) return CHM_ERR_INVALID_ARG;
  const bool huge = q->capacity > kQHuge;
  QueueParams prm{};
  prm.K = K;
  for (int m = 0; m < K; ++m) {
    prm.b[m] = pool->max_batch_size[m];
    prm.d[m] = pool->decode_ms_per_token[m];
  }
  prm.aging_enabled = aging->enabled;
  chm_engine_run er{};
  if (q->run) {
    er = *q->run;
    if (mode == 0 || mode == 2 || huge) return CHM_ERR_UNSUPPORTED;
    if (!er.handle || !er.seq || !er.stint_end || !er.decode_start || !er.stint_tokens ||
        !er.n || !er.tokens_emitted || !er.served || !er.done_handle || !er.done_time ||
        !er.n_done || !er.queue_input_tokens || er.capacity < 1 || er.done_capacity < 0)
      return CHM_ERR_INVALID_ARG;
    for (int m = 0; m < K; ++m)
      if (er.capacity < pool->max_batch_size[m]) return CHM_ERR_INVALID_ARG;
  } else if (mode == 3) {
    return CHM_ERR_INVALID_ARG;
  }
  prm.S = aging->starvation_threshold;
  prm.Q = aging->running_quantum;
  prm.demote = aging->enabled && aging->demote_while_queued;
  prm.cap_limit = big ? 0x7fffffff : kQMax;
  chm_rows r{};
  chm_decisions d{};
  if (rows) r = *rows;
  if (dec) d = *dec;
  prof::begin(prof::K_QUEUE, s);
  if (huge && mode == 2) {
    prof::end(prof::K_QUEUE, s, 0.0);
    return CHM_ERR_UNSUPPORTED;
  }
  if (huge) {
    const chm_status rc = launch_queue_huge(prm, *mon, *q, r, d, n_complete, n_iterations, mode,
                                            err, s);
    prof::end(prof::K_QUEUE, s, 0.0);
    return rc;
  }
  if (big) {
    const size_t smem = sizeof(QueueCtl);
    cudaFuncSetAttribute(queue_kernel<uint32_t, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    queue_kernel<uint32_t, true><<<K, kQThreads, smem, s>>>(prm, *mon, *q, r, d, n_complete,
                                                             n_iterations, mode, err, ma, er);
  } else {
    const size_t smem = sizeof(QueueCtl) + sizeof(SmallKeysSmem);
    cudaFuncSetAttribute(queue_kernel<uint16_t, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    queue_kernel<uint16_t, false><<<K, kQThreads, smem, s>>>(prm, *mon, *q, r, d, n_complete,
                                                              n_iterations, mode, err, ma, er);
  }
  prof::end(prof::K_QUEUE, s, 0.0);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace chm

extern "C" uint64_t chm_queue_fast_calls(void) {
  return (uint64_t)chm::queue_huge_fast_calls();
}

extern "C" uint64_t chm_queue_scratch_bytes(int32_t capacity) {
  if (capacity <= chm::kQMax) return 0;
  if (capacity <= chm::kQHuge) return (uint64_t)capacity * chm::kScratchBytesPerEntry;
  return (uint64_t)chm::queue_huge_scratch_bytes(capacity);
}

extern "C" chm_status chm_queue_complete(const chm_pool* pool, const chm_aging_cfg* aging,
                                         const chm_monitor_state* mon,
                                         const chm_queue_state* q, const int32_t* n_complete,
                                         int32_t* error, void* stream) {
  if (!n_complete) return CHM_ERR_INVALID_ARG;
  return chm::launch_queue(pool, aging, mon, q, nullptr, nullptr, n_complete, 0, 0, error,
                           (cudaStream_t)stream);
}

extern "C" chm_status chm_queue_tick(const chm_pool* pool, const chm_aging_cfg* aging,
                                     const chm_monitor_state* mon, const chm_queue_state* q,
                                     const chm_rows* rows, const chm_decisions* dec,
                                     int32_t n_iterations, int32_t* error, void* stream) {
  if (!rows || !dec || n_iterations < 0) return CHM_ERR_INVALID_ARG;
  return chm::launch_queue(pool, aging, mon, q, rows, dec, nullptr, n_iterations, 1, error,
                           (cudaStream_t)stream);
}

extern "C" chm_status chm_queue_candidates(const chm_pool* pool, const chm_monitor_state* mon,
                                           const chm_queue_state* q, int32_t F,
                                           chm_queue_key* out, void* stream) {
  if (!pool || !mon || !q || !out || F < 1) return CHM_ERR_INVALID_ARG;
  const int K = pool->n_models;
  if (K < 1 || K > CHM_MAX_MODELS) return CHM_ERR_INVALID_ARG;
  chm::QueueParams prm{};
  prm.K = K;
  for (int m = 0; m < K; ++m) {
    prm.b[m] = pool->max_batch_size[m];
    if (prm.b[m] > F) return CHM_ERR_INVALID_ARG;  // F must cover every engine's slots
  }
  chm::candidates_kernel<<<K, 256, 0, (cudaStream_t)stream>>>(prm, *mon, *q, F, out);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

extern "C" chm_status chm_queue_admit_merged(const chm_pool* pool, const chm_aging_cfg* aging,
                                             const chm_monitor_state* mon,
                                             const chm_queue_state* q,
                                             const chm_queue_key* gathered, int32_t G,
                                             int32_t F, int32_t rank, const int32_t* release,
                                             int32_t* error, void* stream) {
  if (!gathered || G < 1 || F < 1 || rank < 0 || rank >= G) return CHM_ERR_INVALID_ARG;
  chm::MergeArgs ma{gathered, G, F, rank, release};
  return chm::launch_queue(pool, aging, mon, q, nullptr, nullptr, nullptr, 1, 2, error,
                           (cudaStream_t)stream, ma);
}

extern "C" chm_status chm_engine_advance(const chm_pool* pool, const chm_aging_cfg* aging,
                                         const chm_monitor_state* mon,
                                         const chm_queue_state* q, const double* target,
                                         int32_t* error, void* stream) {
  if (!target || !q || !q->run) return CHM_ERR_INVALID_ARG;
  chm::MergeArgs ma{};
  ma.target = target;
  return chm::launch_queue(pool, aging, mon, q, nullptr, nullptr, nullptr, 0, 3, error,
                           (cudaStream_t)stream, ma);
}
