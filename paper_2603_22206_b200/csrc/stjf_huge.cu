// K7 for very large engine queues (segments above 2^18 entries; the N_q = 16M
// bandwidth case of SURVEY §8d). Same semantics as stjf.cu (EngineSim
// engine.py:265-374: STJF order (level, priority, arrival, seq), admission of
// the minimum into free slots, aging of the rest), restated as grid-wide
// passes so the whole GPU works on one engine's queue:
//
//   prep        (1 CTA / engine)  append the batch's queued rows, reset control
//   stage       keys (priority bits, level, count) + their OR/AND (which radix
//               digits vary) + "arrival not monotone" flag
//   sort 1      LSD radix by (count, level, priority[, arrival]): per varying
//               byte a histogram / scan / stable-scatter triple of kernels
//               (4096-entry tiles, one CTA each); constant bytes are skipped on
//               the device (the ping-pong buffer index is carried in `cur[]`)
//   groups      count-group heads of the sorted order
//   rounds      (1 warp / engine) the R scheduling iterations on group heads
//   outcome     per entry: admitted, or its group (aging applied at compaction)
//   compact     survivors in seq order: tile counts / scan / scatter into a
//               staging copy, then copied back with the final sort keys
//   sort 2      LSD radix by (level, priority[, arrival]) -> q.order
//   finish      STJF order + engine counters
//
// HBM bytes per queued entry per call (algorithmic, as stjf.cu): 40 read + 40
// written + 4 (order); the radix passes add 2 x 4 (index) + the gathered key
// bytes per varying byte.
#include "common.cuh"
#include "prof.cuh"
#include "stjf_common.cuh"

namespace chm {
namespace qh {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kTile = 4096;      // entries per CTA in grid-wide passes
constexpr int kPass1 = 20;       // byte passes of sort 1: arrival 8, priority 8, level 2, count 2
constexpr int kPass2 = 18;       // sort 2: arrival 8, priority 8, level 2
constexpr int kMaxPasses = kPass1 + kPass2;

struct Ctl {
  unsigned long long kor[2][4], kand[2][4];  // [sort][src] OR / AND of the keys
  int unsorted[2];                           // arrival not monotone in seq (per sort)
  int n, R, G, n_new, n_adm0, n_adm, n_prom, run, err;
  int cur[kMaxPasses + 1];                   // index buffer holding the order before pass p
  uint32_t rowtot[256];                      // current pass: entries per digit
  int g_start[kMaxGroups], g_end[kMaxGroups], g_cur[kMaxGroups];
  int g_count[kMaxGroups], g_lvloff[kMaxGroups];
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }
__host__ __device__ inline size_t n_tiles(size_t C) { return (C + kTile - 1) / kTile; }

__host__ __device__ inline size_t seg_bytes(size_t C) {
  return align_up(8 * C) + 2 * align_up(2 * C) + 2 * align_up(4 * C) + 6 * align_up(8 * C) +
         4 * align_up(4 * C) + align_up(4 * 256 * n_tiles(C)) + align_up(4 * n_tiles(C)) +
         align_up(sizeof(Ctl));
}

struct Layout {
  unsigned long long* prio;
  uint16_t* lvl;
  uint16_t* cnt;
  uint32_t* idx[2];
  unsigned long long* kv[2];  // the current radix source's key, moved with idx
  double* s_prio;
  double* s_arr;
  int64_t* s_seq;
  int64_t* s_handle;
  int32_t* s_out;
  int32_t* s_lvl;
  int32_t* s_cnt;
  int32_t* s_qnt;
  uint32_t* hist;  // [256][T], digit-major
  uint32_t* tcnt;  // [T]
  Ctl* ctl;
};

__device__ inline Layout layout(void* scratch, size_t C, int m) {
  uint8_t* p = reinterpret_cast<uint8_t*>(scratch) + (size_t)m * seg_bytes(C);
  auto take = [&](size_t bytes) {
    uint8_t* r = p;
    p += align_up(bytes);
    return r;
  };
  Layout L;
  L.prio = reinterpret_cast<unsigned long long*>(take(8 * C));
  L.lvl = reinterpret_cast<uint16_t*>(take(2 * C));
  L.cnt = reinterpret_cast<uint16_t*>(take(2 * C));
  L.idx[0] = reinterpret_cast<uint32_t*>(take(4 * C));
  L.idx[1] = reinterpret_cast<uint32_t*>(take(4 * C));
  L.kv[0] = reinterpret_cast<unsigned long long*>(take(8 * C));
  L.kv[1] = reinterpret_cast<unsigned long long*>(take(8 * C));
  L.s_prio = reinterpret_cast<double*>(take(8 * C));
  L.s_arr = reinterpret_cast<double*>(take(8 * C));
  L.s_seq = reinterpret_cast<int64_t*>(take(8 * C));
  L.s_handle = reinterpret_cast<int64_t*>(take(8 * C));
  L.s_out = reinterpret_cast<int32_t*>(take(4 * C));
  L.s_lvl = reinterpret_cast<int32_t*>(take(4 * C));
  L.s_cnt = reinterpret_cast<int32_t*>(take(4 * C));
  L.s_qnt = reinterpret_cast<int32_t*>(take(4 * C));
  L.hist = reinterpret_cast<uint32_t*>(take(4 * 256 * n_tiles(C)));
  L.tcnt = reinterpret_cast<uint32_t*>(take(4 * n_tiles(C)));
  L.ctl = reinterpret_cast<Ctl*>(take(sizeof(Ctl)));
  return L;
}

struct Args {
  QueueParams prm;
  chm_monitor_state mon;
  chm_queue_state q;
  chm_rows rows;
  chm_decisions dec;
  const int32_t* n_complete;
  int n_iterations;
  int mode;
  int32_t* err;
};

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) prep_kernel(Args a) {
  __shared__ int scan[kWarps], misc[8];
  const int m = blockIdx.x, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  const size_t seg = (size_t)m * q.capacity;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  const int n = a.mon.engine_queued[m];
  bool bad = false;
  if (a.mode == 1) {
    const int n_new = count_queued_rows(m, a.dec, scan, misc);
    const int n_old = n - n_new;
    bad = n_old < 0 || n > q.capacity;
    if (!bad) append_queued_rows(m, a.prm.K, a.rows, a.dec, seg, q, n_old, scan, misc);
  } else {
    bad = n > q.capacity;
  }
  if (tid == 0) {
    if (bad) report_error(a.err, n > q.capacity ? CHM_ERR_CAPACITY : CHM_ERR_INVALID_STATE, 0,
                          m, n);
    c.err = bad ? 1 : 0;
    c.n = bad ? 0 : n;
    c.R = bad ? 0 : (a.mode == 0 ? a.n_complete[m] : a.n_iterations);
    c.G = 0;
    c.n_new = 0;
    c.n_adm0 = q.n_admitted[m];
    c.n_adm = 0;
    c.n_prom = 0;
    c.run = a.mon.engine_running[m];
    for (int s2 = 0; s2 < 2; ++s2) {
      c.unsorted[s2] = 0;
      for (int j = 0; j < 4; ++j) {
        c.kor[s2][j] = 0ull;
        c.kand[s2][j] = ~0ull;
      }
    }
    c.cur[0] = 0;
  }
}

// OR/AND of up to 4 key sources over the block, merged into ctl.
__device__ __forceinline__ void merge_masks(unsigned long long (&o)[4],
                                            unsigned long long (&an)[4], int unsorted,
                                            Ctl& c, int sort) {
  __shared__ unsigned long long s_or[4], s_and[4];
  __shared__ int s_uns;
  const int tid = threadIdx.x;
  if (tid < 4) {
    s_or[tid] = 0ull;
    s_and[tid] = ~0ull;
  }
  if (tid == 0) s_uns = 0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    for (int off = 16; off; off >>= 1) {
      o[j] |= __shfl_xor_sync(0xffffffffu, o[j], off);
      an[j] &= __shfl_xor_sync(0xffffffffu, an[j], off);
    }
  }
  unsorted = __any_sync(0xffffffffu, unsorted);
  if ((tid & 31) == 0) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      atomicOr(&s_or[j], o[j]);
      atomicAnd(&s_and[j], an[j]);
    }
    if (unsorted) s_uns = 1;
  }
  __syncthreads();
  if (tid < 4) {
    atomicOr(&c.kor[sort][tid], s_or[tid]);
    atomicAnd(&c.kand[sort][tid], s_and[tid]);
  }
  if (tid == 0 && s_uns) atomicOr(&c.unsorted[sort], 1);
}

// Sort-1 keys of the queue as it stands (after the append).
__device__ __forceinline__ void stage_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  const int n = c.n;
  const int base = tile * kTile;
  if (base >= n) return;
  const size_t seg = (size_t)m * q.capacity;
  const int end = min(base + kTile, n);
  unsigned long long o[4] = {0, 0, 0, 0}, an[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  int unsorted = 0;
  for (int i = base + tid; i < end; i += kThreads) {
    const unsigned long long ak = f64_key(q.arrival[seg + i]);
    const unsigned long long pk = f64_key(q.priority[seg + i]);
    const unsigned long long lk = (unsigned long long)(q.level[seg + i] + 32768);
    const unsigned long long ck = (unsigned long long)min(max(q.count[seg + i], 0), 65535);
    L.prio[i] = pk;
    L.lvl[i] = (uint16_t)lk;
    L.cnt[i] = (uint16_t)ck;
    L.idx[0][i] = (uint32_t)i;
    o[0] |= ak; an[0] &= ak;
    o[1] |= pk; an[1] &= pk;
    o[2] |= lk; an[2] &= lk;
    o[3] |= ck; an[3] &= ck;
    if (i > 0 && q.arrival[seg + i] < q.arrival[seg + i - 1]) unsorted = 1;
  }
  merge_masks(o, an, unsorted, c, 0);
}

struct PassSpec {
  int sort;  // 0: (count, level, priority, arrival) before the rounds; 1: final order
  int src;   // 0 arrival, 1 priority, 2 level, 3 count
  int byte;
  int p;     // pass index (cur[p] -> cur[p + 1])
};

__device__ __forceinline__ int pass_n(const Ctl& c, int sort) { return sort == 0 ? c.n : c.n_new; }

__device__ __forceinline__ bool pass_active(const Ctl& c, const PassSpec& ps) {
  if (ps.sort == 0 && c.R <= 0) return false;
  if (pass_n(c, ps.sort) < 2) return false;
  if (ps.src == 0 && !c.unsorted[ps.sort]) return false;
  const unsigned long long diff = c.kor[ps.sort][ps.src] ^ c.kand[ps.sort][ps.src];
  return ((diff >> (8 * ps.byte)) & 255ull) != 0;
}

__device__ __forceinline__ int src_bytes(int src) { return src <= 1 ? 8 : 2; }

// Any byte of this source active in this sort?
__device__ __forceinline__ bool src_active(const Ctl& c, int sort, int src) {
  PassSpec ps{sort, src, 0, 0};
  for (int b = 0; b < src_bytes(src); ++b) {
    ps.byte = b;
    if (pass_active(c, ps)) return true;
  }
  return false;
}

// Before the byte passes of a source: kv[cur][i] = that source's key of the
// entry at position i of the current order (one gather per source instead of
// one per byte; the passes then move (index, key) pairs sequentially).
__device__ __forceinline__ void gather_tile(int tile, Args a, PassSpec ps) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!src_active(c, ps.sort, ps.src)) return;
  const int n = pass_n(c, ps.sort);
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const int cur = c.cur[ps.p];
  const uint32_t* in = L.idx[cur];
  unsigned long long* kv = L.kv[cur];
  const double* arr = q.arrival + (size_t)m * q.capacity;
  for (int i = base + tid; i < end; i += kThreads) {
    const uint32_t e = in[i];
    unsigned long long v;
    if (ps.src == 0) v = f64_key(arr[e]);
    else if (ps.src == 1) v = L.prio[e];
    else if (ps.src == 2) v = L.lvl[e];
    else v = L.cnt[e];
    kv[i] = v;
  }
}

__device__ __forceinline__ void hist_tile(int tile, Args a, PassSpec ps) {
  __shared__ int h[256];
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!pass_active(c, ps)) return;
  const int n = pass_n(c, ps.sort);
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const unsigned long long* kv = L.kv[c.cur[ps.p]];
  if (tid < 256) h[tid] = 0;
  __syncthreads();
  // warp-aggregated: one shared atomic per distinct digit per warp (few
  // distinct digits -- exponent bytes, levels -- would serialise otherwise)
  for (int i0 = base; i0 < end; i0 += kThreads) {
    const int i = i0 + tid;
    const int d = i < end ? (int)((kv[i] >> (8 * ps.byte)) & 255ull) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (d < 256 && (peers & ((1u << (tid & 31)) - 1u)) == 0) atomicAdd(&h[d], __popc(peers));
  }
  __syncthreads();
  const size_t T = n_tiles(q.capacity);
  if (tid < 256) L.hist[(size_t)tid * T + tile] = (uint32_t)h[tid];
}

// Exclusive scan of n_vals values of a strided 2D array (value f at
// addr(f)), in place, one CTA. Returns the total (all threads).
template <typename Addr>
__device__ uint32_t block_scan_inplace(uint32_t* data, long long n_vals, Addr addr) {
  __shared__ uint32_t part[kThreads];
  __shared__ uint32_t total;
  const int tid = threadIdx.x;
  const long long per = (n_vals + kThreads - 1) / kThreads;
  const long long f0 = tid * per, f1 = min(f0 + per, n_vals);
  uint32_t s = 0;
  for (long long f = f0; f < f1; ++f) s += data[addr(f)];
  part[tid] = s;
  __syncthreads();
  if (tid < 32) {
    // 32 lanes x 32 partials each
    uint32_t v[32], t = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) { v[j] = part[tid * 32 + j]; t += v[j]; }
    uint32_t incl = t;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (tid >= o) incl += x;
    }
    uint32_t run = incl - t;
#pragma unroll
    for (int j = 0; j < 32; ++j) { part[tid * 32 + j] = run; run += v[j]; }
    if (tid == 31) total = incl;
  }
  __syncthreads();
  uint32_t run = part[tid];
  for (long long f = f0; f < f1; ++f) {
    const size_t ad = addr(f);
    const uint32_t v = data[ad];
    data[ad] = run;
    run += v;
  }
  __syncthreads();
  return total;
}

// Digit offsets of a pass, one CTA per digit row: hist[d][0..Tn) is scanned
// in place (exclusive) and its total goes to ctl.rowtot[d]; the scatter
// kernel adds the exclusive prefix of the row totals.
__global__ void __launch_bounds__(kThreads) scan_kernel(Args a, PassSpec ps) {
  __shared__ uint32_t wsum[kWarps];
  const int d = blockIdx.x, m = blockIdx.y, tid = threadIdx.x, lane = tid & 31,
            warp = tid >> 5;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  const bool act = pass_active(c, ps);
  const int cur = c.cur[ps.p];
  if (act) {
    const int Tn = (pass_n(c, ps.sort) + kTile - 1) / kTile;
    uint32_t* row = L.hist + (size_t)d * n_tiles(q.capacity);
    uint32_t carry = 0;
    for (int t0 = 0; t0 < Tn; t0 += kThreads) {
      const int t = t0 + tid;
      const uint32_t v = t < Tn ? row[t] : 0u;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      if (lane == 31) wsum[warp] = incl;
      __syncthreads();
      if (warp == 0) {
        const uint32_t wv = wsum[lane];
        uint32_t wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t x = __shfl_up_sync(0xffffffffu, wi, o);
          if (lane >= o) wi += x;
        }
        wsum[lane] = wi - wv;
      }
      __syncthreads();
      if (t < Tn) row[t] = carry + wsum[warp] + incl - v;
      // chunk total = exclusive prefix of the last warp + its inclusive total
      __syncthreads();
      if (tid == kThreads - 1) wsum[0] = wsum[kWarps - 1] + incl;
      __syncthreads();
      carry += wsum[0];
      __syncthreads();
    }
    if (tid == 0) c.rowtot[d] = carry;
  }
  if (d == 0 && tid == 0) c.cur[ps.p + 1] = act ? (cur ^ 1) : cur;
}

// Stable scatter of one tile: the tile is first counting-sorted by digit in
// shared memory (local stable ranks), then written out in local order, so
// each digit's run of the tile lands as one contiguous (coalesced) span at
// rowoff[d] + hist[d][tile].
struct ScatterSmem {
  unsigned long long s_k[kTile];
  uint32_t s_e[kTile];
  uint16_t wcnt[kWarps][256];
  int glob_d[256];  // global start of this tile's digit-d run, minus its local start
  int loc_d[256];   // local start of the digit-d run (then running)
  uint32_t rowoff[256];
};

__device__ __forceinline__ void scatter_tile(int tile, Args a, PassSpec ps) {
  extern __shared__ __align__(16) unsigned char sc_raw[];
  ScatterSmem& sm = *reinterpret_cast<ScatterSmem*>(sc_raw);
  auto& wcnt = sm.wcnt;
  auto& loc_d = sm.loc_d;
  auto& glob_d = sm.glob_d;
  const int m = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!pass_active(c, ps)) return;
  const int n = pass_n(c, ps.sort);
  const int base = tile * kTile;
  if (base >= n) return;
  const int len = min(kTile, n - base);
  const int cur = c.cur[ps.p];
  const uint32_t* in = L.idx[cur] + base;
  const unsigned long long* kin = L.kv[cur] + base;
  uint32_t* out = L.idx[cur ^ 1];
  unsigned long long* kout = L.kv[cur ^ 1];
  const size_t T = n_tiles(q.capacity);
  const int sh = 8 * ps.byte;
  // local digit histogram -> local run starts; global row offsets from totals
  if (tid < 256) loc_d[tid] = 0;
  if (warp == 1) {
    uint32_t v[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { v[j] = c.rowtot[lane * 8 + j]; tot += v[j]; }
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    uint32_t run = incl - tot;
#pragma unroll
    for (int j = 0; j < 8; ++j) { sm.rowoff[lane * 8 + j] = run; run += v[j]; }
  }
  __syncthreads();
  constexpr int kPer = kTile / kThreads;
  uint32_t ev[kPer];
  unsigned long long kvv[kPer];
  int dv[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = j * kThreads + tid;
    ev[j] = i < len ? in[i] : 0u;
    kvv[j] = i < len ? kin[i] : 0ull;
    dv[j] = i < len ? (int)((kvv[j] >> sh) & 255ull) : 256;
    const unsigned peers = __match_any_sync(0xffffffffu, dv[j]);
    if (dv[j] < 256 && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&loc_d[dv[j]], __popc(peers));
  }
  __syncthreads();
  if (warp == 0) {
    int v[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { v[j] = loc_d[lane * 8 + j]; tot += v[j]; }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int x = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += x;
    }
    int run = incl - tot;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int dd = lane * 8 + j;
      glob_d[dd] = (int)(sm.rowoff[dd] + L.hist[(size_t)dd * T + tile]) - run;
      loc_d[dd] = run;
      run += v[j];
    }
  }
  __syncthreads();
  // stable local ranks, 1024 entries at a time
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int d = dv[j];
#pragma unroll
    for (int k = 0; k < 8; ++k) wcnt[warp][lane * 8 + k] = 0;
    __syncwarp();
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (d < 256 && rank == 0) wcnt[warp][d] = (uint16_t)__popc(peers);
    __syncthreads();
    if (tid < 256) {
      int run = loc_d[tid];
#pragma unroll 8
      for (int w = 0; w < kWarps; ++w) {
        const int cnum = wcnt[w][tid];
        wcnt[w][tid] = (uint16_t)run;
        run += cnum;
      }
      loc_d[tid] = run;
    }
    __syncthreads();
    if (d < 256) {
      const int lp = wcnt[warp][d] + rank;
      sm.s_e[lp] = ev[j];
      sm.s_k[lp] = kvv[j];
    }
    __syncthreads();
  }
  // coalesced write-out in local (digit-run) order
  for (int lp = tid; lp < len; lp += kThreads) {
    const unsigned long long k = sm.s_k[lp];
    const int pos = glob_d[(int)((k >> sh) & 255ull)] + lp;
    out[pos] = sm.s_e[lp];
    kout[pos] = k;
  }
}

// ---------------------------------------------------------------------------
__device__ __forceinline__ void groups_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  const int n = c.n;
  if (c.R <= 0) return;
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const uint32_t* sorted = L.idx[c.cur[kPass1]];
  for (int p = base + tid; p < end; p += kThreads) {
    const uint16_t ct = L.cnt[sorted[p]];
    if (p == 0 || ct != L.cnt[sorted[p - 1]]) {
      const int g = atomicAdd(&c.G, 1);
      if (g < kMaxGroups) {
        c.g_start[g] = p;
        c.g_count[g] = ct;
      }
    }
  }
}

// The R scheduling iterations (engine.py:328-338) on the count-group heads:
// entries with equal starvation count age in lock step, so each group keeps
// its internal (level, priority, arrival, seq) order for the whole call.
__global__ void __launch_bounds__(32) rounds_kernel(Args a) {
  __shared__ int g_start[kMaxGroups], g_end[kMaxGroups], g_cur[kMaxGroups];
  __shared__ int g_count[kMaxGroups], g_lvloff[kMaxGroups];
  const int m = blockIdx.x, lane = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  const int R = c.R;
  if (R <= 0) return;
  const int n = c.n, G = c.G;
  if (G > kMaxGroups) {
    if (lane == 0) {
      report_error(a.err, CHM_ERR_UNSUPPORTED, 0, m, G);
      c.err = 1;
    }
    return;
  }
  const size_t seg = (size_t)m * q.capacity;
  const double* arr_g = q.arrival + seg;
  const bool use_arr = c.unsorted[0] != 0;
  const uint32_t* sorted = L.idx[c.cur[kPass1]];
  for (int g = lane; g < G; g += 32) {
    g_start[g] = c.g_start[g];
    g_count[g] = c.g_count[g];
  }
  __syncwarp();
  if (lane == 0) {
    for (int x = 1; x < G; ++x) {
      const int st = g_start[x], ct = g_count[x];
      int y = x - 1;
      while (y >= 0 && g_start[y] > st) {
        g_start[y + 1] = g_start[y];
        g_count[y + 1] = g_count[y];
        --y;
      }
      g_start[y + 1] = st;
      g_count[y + 1] = ct;
    }
    for (int g = 0; g < G; ++g) {
      g_end[g] = (g + 1 < G) ? g_start[g + 1] : n;
      g_cur[g] = g_start[g];
      g_lvloff[g] = 0;
    }
  }
  __syncwarp();
  const int bmax = a.prm.b[m];
  int run = c.run, n_adm = 0, n_prom = 0, remaining = n;
  for (int r = 0; r < R; ++r) {
    if (a.mode == 0) run = max(run - 1, 0);
    const int adm = max(0, min(bmax - run, remaining));
    for (int t = 0; t < adm; ++t) {
      HeadKey best;
      best.g = -1;
      for (int g0 = 0; g0 < G; g0 += 32) {
        const int g = g0 + lane;
        HeadKey hk;
        hk.g = -1;
        if (g < G && g_cur[g] < g_end[g]) {
          const int e = (int)sorted[g_cur[g]];
          hk.e = e;
          hk.g = g;
          hk.lvl = (int)L.lvl[e] - 32768 + g_lvloff[g];
          hk.prio = L.prio[e];
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
        q.admitted[seg + c.n_adm0 + n_adm] = q.handle[seg + best.e];
        g_cur[best.g] += 1;
      }
      __syncwarp();
      ++n_adm;
      --remaining;
    }
    run += adm;
    if (a.prm.aging_enabled && remaining > 0) {
      for (int g = lane; g < G; g += 32) {
        if (g_cur[g] < g_end[g]) {
          int c2 = g_count[g] + 1;
          if (c2 >= a.prm.S) {
            c2 = 0;
            g_lvloff[g] -= 1;
            n_prom += g_end[g] - g_cur[g];
          }
          g_count[g] = c2;
        }
      }
      __syncwarp();
    }
  }
  for (int off = 16; off; off >>= 1) n_prom += __shfl_xor_sync(0xffffffffu, n_prom, off);
  for (int g = lane; g < G; g += 32) {
    c.g_start[g] = g_start[g];
    c.g_end[g] = g_end[g];
    c.g_cur[g] = g_cur[g];
    c.g_count[g] = g_count[g];
    c.g_lvloff[g] = g_lvloff[g];
  }
  if (lane == 0) {
    c.n_adm = n_adm;
    c.n_prom = n_prom;
    c.run = run;
  }
}

// spare[e] = kAdmitted, or the count group of a surviving entry.
__device__ __forceinline__ void outcome_tile(int tile, Args a) {
  __shared__ int g_start[kMaxGroups], g_cur[kMaxGroups];
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (c.R <= 0 || c.err) return;
  const int n = c.n, G = c.G;
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  for (int g = tid; g < G; g += kThreads) {
    g_start[g] = c.g_start[g];
    g_cur[g] = c.g_cur[g];
  }
  __syncthreads();
  const int cur = c.cur[kPass1];
  const uint32_t* sorted = L.idx[cur];
  uint32_t* spare = L.idx[cur ^ 1];
  for (int p = base + tid; p < end; p += kThreads) {
    int lo = 0, hi = G - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (g_start[mid] <= p) lo = mid; else hi = mid - 1;
    }
    spare[sorted[p]] = (p < g_cur[lo]) ? kAdmitted : (uint32_t)lo;
  }
}

__device__ __forceinline__ bool survives(const Ctl& c, const Layout& L, int i) {
  if (c.R <= 0) return true;
  return L.idx[c.cur[kPass1] ^ 1][i] != kAdmitted;
}

__device__ __forceinline__ void compact_count_tile(int tile, Args a) {
  __shared__ int wsum[kWarps];
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  const int n = c.n;
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  int k = 0;
  for (int i = base + tid; i < end; i += kThreads) k += survives(c, L, i) ? 1 : 0;
  for (int off = 16; off; off >>= 1) k += __shfl_xor_sync(0xffffffffu, k, off);
  if ((tid & 31) == 0) wsum[tid >> 5] = k;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < kWarps; ++w) t += wsum[w];
    L.tcnt[tile] = (uint32_t)t;
  }
}

__global__ void __launch_bounds__(kThreads) compact_scan_kernel(Args a) {
  const int m = blockIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  const long long Tn = (c.n + kTile - 1) / kTile;
  const uint32_t tot = block_scan_inplace(L.tcnt, Tn, [](long long f) { return (size_t)f; });
  if (threadIdx.x == 0) c.n_new = c.err ? 0 : (int)tot;
}

// Survivors in seq order into the staging copy, aging applied.
__device__ __forceinline__ void compact_scatter_tile(int tile, Args a) {
  __shared__ int wpre[kWarps];
  __shared__ int blk_tot;
  __shared__ int g_count[kMaxGroups], g_lvloff[kMaxGroups];
  const int m = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (c.err) return;
  const int n = c.n;
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const bool aged = c.R > 0;
  if (aged)
    for (int g = tid; g < c.G; g += kThreads) {
      g_count[g] = c.g_count[g];
      g_lvloff[g] = c.g_lvloff[g];
    }
  const size_t seg = (size_t)m * q.capacity;
  const uint32_t* grp = L.idx[c.cur[kPass1] ^ 1];
  int out = (int)L.tcnt[tile];
  __syncthreads();
  for (int blk = base; blk < end; blk += kThreads) {
    const int i = blk + tid;
    const bool keep = i < end && survives(c, L, i);
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wpre[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      const int v = wpre[lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      wpre[lane] = incl - v;
      if (lane == 31) blk_tot = incl;
    }
    __syncthreads();
    if (keep) {
      const int pos = out + wpre[warp] + __popc(bal & ((1u << lane) - 1u));
      int lv = q.level[seg + i], ct = q.count[seg + i], qn = q.quantum[seg + i];
      if (aged) {
        const uint32_t g = grp[i];
        lv += g_lvloff[g];
        if (a.prm.aging_enabled) ct = g_count[g];
        if (g_lvloff[g] != 0) qn = 0;
      }
      L.s_prio[pos] = q.priority[seg + i];
      L.s_arr[pos] = q.arrival[seg + i];
      L.s_seq[pos] = q.seq[seg + i];
      L.s_handle[pos] = q.handle[seg + i];
      L.s_out[pos] = q.out_tokens[seg + i];
      L.s_lvl[pos] = lv;
      L.s_cnt[pos] = ct;
      L.s_qnt[pos] = qn;
    }
    out += blk_tot;
    __syncthreads();
  }
}

// Staging -> queue SoA, with the sort-2 keys and their OR/AND.
__device__ __forceinline__ void copy_back_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  if (tile == 0 && tid == 0) c.cur[kPass1] = 0;
  const int n = c.n_new;
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const size_t seg = (size_t)m * q.capacity;
  unsigned long long o[4] = {0, 0, 0, 0}, an[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  int unsorted = 0;
  for (int i = base + tid; i < end; i += kThreads) {
    const double pr = L.s_prio[i], ar = L.s_arr[i];
    const int lv = L.s_lvl[i];
    q.priority[seg + i] = pr;
    q.arrival[seg + i] = ar;
    q.seq[seg + i] = L.s_seq[i];
    q.handle[seg + i] = L.s_handle[i];
    q.out_tokens[seg + i] = L.s_out[i];
    q.level[seg + i] = lv;
    q.count[seg + i] = L.s_cnt[i];
    q.quantum[seg + i] = L.s_qnt[i];
    const unsigned long long ak = f64_key(ar), pk = f64_key(pr);
    const unsigned long long lk = (unsigned long long)(lv + 32768);
    L.prio[i] = pk;
    L.lvl[i] = (uint16_t)lk;
    L.idx[0][i] = (uint32_t)i;
    o[0] |= ak; an[0] &= ak;
    o[1] |= pk; an[1] &= pk;
    o[2] |= lk; an[2] &= lk;
    if (i > 0 && ar < L.s_arr[i - 1]) unsorted = 1;
  }
  merge_masks(o, an, unsorted, c, 1);
}

__device__ __forceinline__ void finish_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  const size_t seg = (size_t)m * q.capacity;
  if (c.err) return;
  const int n = c.n_new;
  if (tile == 0 && tid == 0) {
    q.n_admitted[m] = c.n_adm0 + c.n_adm;
    q.n_promoted[m] += c.n_prom;
    a.mon.engine_queued[m] = n;
    a.mon.engine_running[m] = c.run;
    a.mon.engine_iterations[m] += c.R;
    q.arrival_unsorted[m] = c.unsorted[1] ? 1 : 0;
  }
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const uint32_t* sorted = L.idx[c.cur[kMaxPasses]];
  for (int r = base + tid; r < end; r += kThreads) q.order[seg + r] = (int32_t)sorted[r];
}

// Grid-stride wrappers: a fixed grid of a few CTAs per SM walks the tiles, so
// passes whose digit turns out constant (checked on the device) cost one
// short wave instead of a launch of every tile.
// The loop bound is the live entry count (c.n before the compaction, c.n_new
// after), read once per CTA, and inactive passes exit before the loop.
template <void (*F)(int, Args), int kAfterCompaction>
__global__ void __launch_bounds__(kThreads) tiles(Args a) {
  const int m = blockIdx.y;
  const Ctl& c = *layout(a.q.scratch, a.q.capacity, m).ctl;
  const int n = kAfterCompaction ? c.n_new : c.n;
  // tile 0 always runs (it may carry per-engine bookkeeping)
  const int T = n > 0 ? (n + kTile - 1) / kTile : 1;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    F(t, a);
    __syncthreads();
  }
}
template <void (*F)(int, Args, PassSpec), bool kWholeSource>
__global__ void __launch_bounds__(kThreads) tiles_pass(Args a, PassSpec ps) {
  const int m = blockIdx.y;
  const Ctl& c = *layout(a.q.scratch, a.q.capacity, m).ctl;
  if (kWholeSource ? !src_active(c, ps.sort, ps.src) : !pass_active(c, ps)) return;
  const int T = (pass_n(c, ps.sort) + kTile - 1) / kTile;
  for (int t = blockIdx.x; t < T; t += gridDim.x) {
    F(t, a, ps);
    __syncthreads();
  }
}

}  // namespace qh

size_t queue_huge_scratch_bytes(int capacity) { return qh::seg_bytes((size_t)capacity); }

chm_status launch_queue_huge(const QueueParams& prm, const chm_monitor_state& mon,
                             const chm_queue_state& q, const chm_rows& rows,
                             const chm_decisions& dec, const int32_t* n_complete,
                             int n_iterations, int mode, int32_t* err, cudaStream_t s) {
  using namespace qh;
  Args a{prm, mon, q, rows, dec, n_complete, n_iterations, mode, err};
  const int K = prm.K;
  const int T = (int)n_tiles((size_t)q.capacity);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(tiles_pass<scatter_tile, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(ScatterSmem));
  }
  // two 1024-thread CTAs per SM walk the tiles
  const dim3 grid((unsigned)(T < 2 * sms ? T : 2 * sms), (unsigned)K);
  prep_kernel<<<K, kThreads, 0, s>>>(a);
  tiles<stage_tile, 0><<<grid, kThreads, 0, s>>>(a);
  auto pass = [&](int sort, int src, int byte, int p) {
    PassSpec ps{sort, src, byte, p};
    if (byte == 0) tiles_pass<gather_tile, true><<<grid, kThreads, 0, s>>>(a, ps);
    tiles_pass<hist_tile, false><<<grid, kThreads, 0, s>>>(a, ps);
    scan_kernel<<<dim3(256, K), kThreads, 0, s>>>(a, ps);
    tiles_pass<scatter_tile, false><<<grid, kThreads, sizeof(ScatterSmem), s>>>(a, ps);
  };
  int p = 0;
  // sort 1, least significant first: arrival, priority, level, count
  const int srcs1[4] = {0, 1, 2, 3}, bytes1[4] = {8, 8, 2, 2};
  for (int j = 0; j < 4; ++j)
    for (int b = 0; b < bytes1[j]; ++b) pass(0, srcs1[j], b, p++);
  tiles<groups_tile, 0><<<grid, kThreads, 0, s>>>(a);
  rounds_kernel<<<K, 32, 0, s>>>(a);
  tiles<outcome_tile, 0><<<grid, kThreads, 0, s>>>(a);
  tiles<compact_count_tile, 0><<<grid, kThreads, 0, s>>>(a);
  compact_scan_kernel<<<K, kThreads, 0, s>>>(a);
  tiles<compact_scatter_tile, 0><<<grid, kThreads, 0, s>>>(a);
  // copy_back (tile 0 resets the sort-2 buffer index) runs after n_new is known
  tiles<copy_back_tile, 1><<<grid, kThreads, 0, s>>>(a);
  // sort 2: arrival, priority, level
  const int srcs2[3] = {0, 1, 2}, bytes2[3] = {8, 8, 2};
  for (int j = 0; j < 3; ++j)
    for (int b = 0; b < bytes2[j]; ++b) pass(1, srcs2[j], b, p++);
  tiles<finish_tile, 1><<<grid, kThreads, 0, s>>>(a);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace chm
