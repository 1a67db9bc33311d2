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
//
// Incremental fast path (taken when the queue is exactly what the previous
// call left -- a 64-bit hash of (index, priority, arrival, level, count) over
// the old entries matches the one stored then -- and the call appends <=
// kNewMax rows and admits <= kAcapMax): the STJF order of the previous call is
// kept in scratch as a key array in that order (level, count, index, priority
// and arrival keys), so no full sort runs:
//   check       hash of the old entries, histogram of starvation counts
//   insert      the appended rows ranked among themselves, binary-searched
//               into the kept order; the kept keys stream into the merged
//               order (skipped when nothing is appended)
//   heads       per count group the first positions in that order (a tile
//               histogram + scan; only tiles holding a group's first
//               admissions are walked)
//   rounds      as below, on those per-group head lists
//   compact     in place: survivors shift left by the admissions before them
//               (<= kAcapMax), each tile's last kAcapMax entries saved to a
//               halo first; aging applied, the new hash accumulated
//   final       the merged order minus the admitted, aging applied: with one
//               level offset among the survivors it is already the STJF
//               order (one streaming pass); with two (a promoted class) the
//               classes are split and merged (merge path); more fall back to
//               the radix sort 2
// ~150 B per entry per call instead of ~900 B for the radix path.
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
constexpr int kNewMax = 8192;    // fast path: rows appended per call
constexpr int kAcapMax = 512;    // fast path: admissions per call (halo depth)
constexpr int kMergeTile = 2048; // output entries per merge-path CTA
constexpr size_t kMergeSmem = (size_t)kMergeTile * (8 + 8 + 4 + 4 + 2);
constexpr unsigned kValidMagic = 0x5A17C0DEu;

struct Ctl {
  unsigned long long kor[2][4], kand[2][4];  // [sort][src] OR / AND of the keys
  int unsorted[2];                           // arrival not monotone in seq (per sort)
  int n, R, G, n_new, n_adm0, n_adm, n_prom, run, err;
  int cur[kMaxPasses + 1];                   // index buffer holding the order before pass p
  uint32_t rowtot[256];                      // current pass: entries per digit
  int g_start[kMaxGroups], g_end[kMaxGroups], g_cur[kMaxGroups];
  int g_count[kMaxGroups], g_lvloff[kMaxGroups];
  // ---- incremental fast path ----
  int n_old, n_app, fast, need_sort2, big_count, A_cap, A, D, first_adm, nU, n_surv;
  int cnt_hist[kMaxGroups];  // entries per starvation count (counts < kMaxGroups)
  int cls[kMaxGroups];       // class (distinct level offset) of a count group
  unsigned long long hash_acc;  // this call: hash of the old entries as found
  unsigned long long hash_new;  // this call: hash of the state it leaves
  // persistent across calls (scratch is not cleared between them)
  unsigned valid;               // kValidMagic once a call left keys + hash
  int n_prev, kcur;
  unsigned long long hash_prev;
};

__host__ __device__ inline size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }
__host__ __device__ inline size_t n_tiles(size_t C) { return (C + kTile - 1) / kTile; }

// Fast-path key arrays, one entry per queue position in STJF order.
struct KeyBuf {
  int32_t* lvl;
  uint16_t* cnt;
  uint32_t* idx;
  unsigned long long* prio;
  unsigned long long* arr;
};

__host__ __device__ inline size_t keybuf_bytes(size_t C) {
  return align_up(4 * C) + align_up(2 * C) + align_up(4 * C) + 2 * align_up(8 * C);
}
__host__ __device__ inline size_t halo_bytes(size_t C) {
  return 4 * align_up(8 * (size_t)kAcapMax * n_tiles(C)) +
         4 * align_up(4 * (size_t)kAcapMax * n_tiles(C));
}

__host__ __device__ inline size_t seg_bytes(size_t C) {
  return align_up(8 * C) + 2 * align_up(2 * C) + 2 * align_up(4 * C) + 6 * align_up(8 * C) +
         4 * align_up(4 * C) + align_up(4 * 256 * n_tiles(C)) + align_up(4 * n_tiles(C)) +
         align_up(sizeof(Ctl)) + 2 * keybuf_bytes(C) + halo_bytes(C) +
         2 * align_up(4 * kNewMax) + align_up(4 * (size_t)kMaxGroups * kAcapMax) +
         2 * align_up(4 * kAcapMax);
}

struct Layout {
  unsigned long long* prio;
  uint16_t* lvl;
  uint16_t* cnt;
  uint32_t* idx0;
  uint32_t* idx1;
  unsigned long long* kv0;  // the current radix source's key, moved with idx
  unsigned long long* kv1;
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
  KeyBuf ks0, ks1;
  unsigned long long *h64_0, *h64_1, *h64_2, *h64_3;  // halo [T][kAcapMax]: priority, arrival, seq, handle
  int32_t *h32_0, *h32_1, *h32_2, *h32_3;             // out_tokens, level, count, quantum
  uint32_t* new_sorted;        // [kNewMax] appended entries in key order
  uint32_t* ins;               // [kNewMax] their insertion points in the kept order
  uint32_t* hl;                // [kMaxGroups][kAcapMax] head positions per count group
  uint32_t* adm_idx;           // [kAcapMax] admitted storage indices (sorted)
  uint32_t* adm_pos;           // [kAcapMax] admitted positions in the merged order (sorted)
  // selects, not arrays: a dynamically indexed member array would put the
  // whole layout in local memory
  __device__ __forceinline__ uint32_t* idxb(int b) const { return b ? idx1 : idx0; }
  __device__ __forceinline__ unsigned long long* kvb(int b) const { return b ? kv1 : kv0; }
  __device__ __forceinline__ KeyBuf ksb(int b) const { return b ? ks1 : ks0; }
  __device__ __forceinline__ unsigned long long* h64b(int f) const {
    return f == 0 ? h64_0 : f == 1 ? h64_1 : f == 2 ? h64_2 : h64_3;
  }
  __device__ __forceinline__ int32_t* h32b(int f) const {
    return f == 0 ? h32_0 : f == 1 ? h32_1 : f == 2 ? h32_2 : h32_3;
  }
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
  L.idx0 = reinterpret_cast<uint32_t*>(take(4 * C));
  L.idx1 = reinterpret_cast<uint32_t*>(take(4 * C));
  L.kv0 = reinterpret_cast<unsigned long long*>(take(8 * C));
  L.kv1 = reinterpret_cast<unsigned long long*>(take(8 * C));
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
  for (KeyBuf* kb : {&L.ks0, &L.ks1}) {
    kb->lvl = reinterpret_cast<int32_t*>(take(4 * C));
    kb->cnt = reinterpret_cast<uint16_t*>(take(2 * C));
    kb->idx = reinterpret_cast<uint32_t*>(take(4 * C));
    kb->prio = reinterpret_cast<unsigned long long*>(take(8 * C));
    kb->arr = reinterpret_cast<unsigned long long*>(take(8 * C));
  }
  const size_t H = (size_t)kAcapMax * n_tiles(C);
  L.h64_0 = reinterpret_cast<unsigned long long*>(take(8 * H));
  L.h64_1 = reinterpret_cast<unsigned long long*>(take(8 * H));
  L.h64_2 = reinterpret_cast<unsigned long long*>(take(8 * H));
  L.h64_3 = reinterpret_cast<unsigned long long*>(take(8 * H));
  L.h32_0 = reinterpret_cast<int32_t*>(take(4 * H));
  L.h32_1 = reinterpret_cast<int32_t*>(take(4 * H));
  L.h32_2 = reinterpret_cast<int32_t*>(take(4 * H));
  L.h32_3 = reinterpret_cast<int32_t*>(take(4 * H));
  L.new_sorted = reinterpret_cast<uint32_t*>(take(4 * kNewMax));
  L.ins = reinterpret_cast<uint32_t*>(take(4 * kNewMax));
  L.hl = reinterpret_cast<uint32_t*>(take(4 * (size_t)kMaxGroups * kAcapMax));
  L.adm_idx = reinterpret_cast<uint32_t*>(take(4 * kAcapMax));
  L.adm_pos = reinterpret_cast<uint32_t*>(take(4 * kAcapMax));
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
  int n_app = 0;
  if (a.mode == 1) {
    n_app = count_queued_rows(m, a.dec, scan, misc);
    const int n_old = n - n_app;
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
    c.n_old = bad ? 0 : n - n_app;
    c.n_app = bad ? 0 : n_app;
    c.fast = 0;
    c.need_sort2 = 0;
    c.big_count = 0;
    c.A = 0;
    c.D = 0;
    c.hash_acc = 0ull;
    c.hash_new = 0ull;
    if (bad) c.valid = 0u;
  }
  for (int g = tid; g < kMaxGroups; g += blockDim.x) c.cnt_hist[g] = 0;
}

// ---------------------------------------------------------------------------
// Incremental fast path (see the header).
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}
// Order-independent state hash: the sum over entries of this.
__device__ __forceinline__ unsigned long long entry_hash(uint32_t i, double pr, double ar, int lv,
                                                         int ct) {
  unsigned long long h = mix64((unsigned long long)i * 0x9E3779B97F4A7C15ull ^
                               (unsigned long long)__double_as_longlong(pr));
  h = mix64(h ^ (unsigned long long)__double_as_longlong(ar));
  return mix64(h ^ ((unsigned long long)(uint32_t)lv << 32 | (uint32_t)ct));
}

struct FKey {
  int lvl;
  unsigned long long prio, arr;
  uint32_t idx;
};
__device__ __forceinline__ bool fk_less(const FKey& x, const FKey& y) {
  if (x.lvl != y.lvl) return x.lvl < y.lvl;
  if (x.prio != y.prio) return x.prio < y.prio;
  if (x.arr != y.arr) return x.arr < y.arr;
  return x.idx < y.idx;
}
__device__ __forceinline__ FKey fk_at(const KeyBuf& k, size_t r) {
  return FKey{k.lvl[r], k.prio[r], k.arr[r], k.idx[r]};
}
__device__ __forceinline__ void fk_put(const KeyBuf& k, size_t r, const FKey& v, uint16_t cnt) {
  k.lvl[r] = v.lvl;
  k.prio[r] = v.prio;
  k.arr[r] = v.arr;
  k.idx[r] = v.idx;
  k.cnt[r] = cnt;
}
__device__ __forceinline__ FKey fk_entry(const chm_queue_state& q, size_t seg, uint32_t e) {
  return FKey{q.level[seg + e], f64_key(q.priority[seg + e]), f64_key(q.arrival[seg + e]), e};
}
// #{v in a[0, n) : v < x} for ascending a
__device__ __forceinline__ int count_less(const uint32_t* a, int n, uint32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
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
  if (c.fast) return;
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
    L.idxb(0)[i] = (uint32_t)i;
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
  if (ps.sort == 0 && (c.R <= 0 || c.fast)) return false;
  if (ps.sort == 1 && c.fast && !c.need_sort2) return false;
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
  const uint32_t* in = L.idxb(cur);
  unsigned long long* kv = L.kvb(cur);
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
  const unsigned long long* kv = L.kvb(c.cur[ps.p]);
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
  const uint32_t* in = L.idxb(cur) + base;
  const unsigned long long* kin = L.kvb(cur) + base;
  uint32_t* out = L.idxb(cur ^ 1);
  unsigned long long* kout = L.kvb(cur ^ 1);
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
  if (c.fast) return;
  const int n = c.n;
  if (c.R <= 0) return;
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const uint32_t* sorted = L.idxb(c.cur[kPass1]);
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
  if (c.fast) return;
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
  const uint32_t* sorted = L.idxb(c.cur[kPass1]);
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
  if (c.fast) return;
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
  const uint32_t* sorted = L.idxb(cur);
  uint32_t* spare = L.idxb(cur ^ 1);
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
  return L.idxb(c.cur[kPass1] ^ 1)[i] != kAdmitted;
}

__device__ __forceinline__ void compact_count_tile(int tile, Args a) {
  __shared__ int wsum[kWarps];
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (c.fast) return;
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
  if (c.fast) return;
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
  if (c.fast) return;
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
  const uint32_t* grp = L.idxb(c.cur[kPass1] ^ 1);
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
  if (c.fast) return;
  if (tile == 0 && tid == 0) c.cur[kPass1] = 0;
  const int n = c.n_new;
  const int base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const size_t seg = (size_t)m * q.capacity;
  unsigned long long o[4] = {0, 0, 0, 0}, an[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  int unsorted = 0;
  unsigned long long hs = 0ull;
  for (int i = base + tid; i < end; i += kThreads) {
    const double pr = L.s_prio[i], ar = L.s_arr[i];
    const int lv = L.s_lvl[i];
    hs += entry_hash((uint32_t)i, pr, ar, lv, L.s_cnt[i]);
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
    L.idxb(0)[i] = (uint32_t)i;
    o[0] |= ak; an[0] &= ak;
    o[1] |= pk; an[1] &= pk;
    o[2] |= lk; an[2] &= lk;
    if (i > 0 && ar < L.s_arr[i - 1]) unsorted = 1;
  }
  for (int off = 16; off; off >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, off);
  if ((tid & 31) == 0) atomicAdd(&c.hash_new, hs);
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
  if (c.fast && !c.need_sort2) return;  // the fast path wrote q.order
  const uint32_t* sorted = L.idxb(c.cur[kMaxPasses]);
  for (int r = base + tid; r < end; r += kThreads) q.order[seg + r] = (int32_t)sorted[r];
}

// Hash of the old entries, starvation-count histogram (all entries).
__device__ __forceinline__ void check_tile(int tile, Args a) {
  __shared__ int h[kMaxGroups];
  __shared__ unsigned long long s_hash;
  __shared__ int s_big;
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  const int n = c.n;
  const int base = tile * kTile;
  if (c.err || base >= n) return;
  for (int g = tid; g < kMaxGroups; g += kThreads) h[g] = 0;
  if (tid == 0) { s_hash = 0ull; s_big = 0; }
  __syncthreads();
  const size_t seg = (size_t)m * q.capacity;
  const int end = min(base + kTile, n), n_old = c.n_old;
  unsigned long long hs = 0ull;
  int big = 0;
  for (int i = base + tid; i < end; i += kThreads) {
    const int ct = q.count[seg + i];
    if (i < n_old)
      hs += entry_hash((uint32_t)i, q.priority[seg + i], q.arrival[seg + i], q.level[seg + i], ct);
    if (ct < 0 || ct >= kMaxGroups) big = 1; else atomicAdd(&h[ct], 1);
  }
  for (int off = 16; off; off >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, off);
  if ((tid & 31) == 0) atomicAdd(&s_hash, hs);
  if (big) s_big = 1;
  __syncthreads();
  for (int g = tid; g < kMaxGroups; g += kThreads)
    if (h[g]) atomicAdd(&c.cnt_hist[g], h[g]);
  if (tid == 0) {
    atomicAdd(&c.hash_acc, s_hash);
    if (s_big) atomicOr(&c.big_count, 1);
  }
}

// calls that took the incremental path (diagnostic: chm_queue_fast_calls)
__device__ unsigned long long g_fast_calls;

__global__ void decide_kernel(Args a, int allow) {
  const int m = blockIdx.x;
  if (threadIdx.x != 0) return;
  Layout L = layout(a.q.scratch, a.q.capacity, m);
  Ctl& c = *L.ctl;
  const int run0 = c.run, bmax = a.prm.b[m];
  long long acap = max(0, bmax - run0) + (a.mode == 0 ? max(c.R, 0) : 0);
  if (c.R <= 0) acap = 0;
  acap = acap < c.n ? acap : c.n;
  c.A_cap = (int)acap;
  c.fast = allow && !c.err && c.valid == kValidMagic && c.n_prev == c.n_old &&
           c.hash_prev == c.hash_acc && c.n_app <= kNewMax && !c.big_count &&
           acap <= kAcapMax && !a.prm.demote;
  if (c.fast) atomicAdd(&g_fast_calls, 1ull);
}

// Appended rows ranked among themselves (n_app <= kNewMax; indices ascend
// with seq, so the full key is a total order).
__global__ void __launch_bounds__(256) newsort_kernel(Args a) {
  __shared__ FKey tk[256];
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast) return;
  const int na = c.n_app, n_old = c.n_old;
  if ((int)blockIdx.x * 256 >= na) return;
  const size_t seg = (size_t)m * q.capacity;
  const int j = blockIdx.x * 256 + tid;
  const FKey mine = j < na ? fk_entry(q, seg, (uint32_t)(n_old + j)) : FKey{};
  int rank = 0;
  for (int t0 = 0; t0 < na; t0 += 256) {
    __syncthreads();
    if (t0 + tid < na) tk[tid] = fk_entry(q, seg, (uint32_t)(n_old + t0 + tid));
    __syncthreads();
    const int lim = min(256, na - t0);
    for (int k = 0; k < lim; ++k) rank += fk_less(tk[k], mine) ? 1 : 0;
  }
  if (j < na) L.new_sorted[rank] = (uint32_t)(n_old + j);
}

// Insertion point of each sorted appended row in the kept order; the row's
// keys go straight to its merged position ins + k.
__global__ void __launch_bounds__(256) insert_kernel(Args a) {
  const int m = blockIdx.y;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast) return;
  const int k = blockIdx.x * 256 + threadIdx.x;
  if (k >= c.n_app) return;
  const size_t seg = (size_t)m * q.capacity;
  const KeyBuf& ko = L.ksb(c.kcur);
  const KeyBuf& k1 = L.ksb(c.kcur ^ 1);
  const uint32_t e = L.new_sorted[k];
  const FKey key = fk_entry(q, seg, e);
  int lo = 0, hi = c.n_old;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (fk_less(fk_at(ko, mid), key)) lo = mid + 1; else hi = mid;
  }
  L.ins[k] = (uint32_t)lo;
  fk_put(k1, (size_t)lo + k, key, (uint16_t)q.count[seg + e]);
}

// Kept keys -> merged order: position r moves by #{k : ins[k] <= r}.
__device__ __forceinline__ void merge_old_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.n_app == 0) return;
  const int n_old = c.n_old, na = c.n_app;
  const int base = tile * kTile;
  if (base >= n_old) return;
  const int end = min(base + kTile, n_old);
  const KeyBuf& ko = L.ksb(c.kcur);
  const KeyBuf& k1 = L.ksb(c.kcur ^ 1);
  // insertion points inside this tile: ins[lo0, hi0)
  const int lo0 = count_less(L.ins, na, (uint32_t)base + 1);   // ins <= base
  const int hi0 = count_less(L.ins, na, (uint32_t)end);        // ins <= end - 1
  for (int r = base + tid; r < end; r += kThreads) {
    const int sh = lo0 == hi0 ? lo0 : lo0 + count_less(L.ins + lo0, hi0 - lo0, (uint32_t)r + 1);
    const size_t d = (size_t)r + sh;
    k1.lvl[d] = ko.lvl[r];
    k1.cnt[d] = ko.cnt[r];
    k1.idx[d] = ko.idx[r];
    k1.prio[d] = ko.prio[r];
    k1.arr[d] = ko.arr[r];
  }
}

// The merged order (position -> keys) of this call.
__device__ __forceinline__ const KeyBuf& merged_keys(const Layout& L, const Ctl& c) {
  return L.ksb(c.n_app > 0 ? (c.kcur ^ 1) : c.kcur);
}

// heads: entries per count group per tile (merged order) ...
__device__ __forceinline__ void heads_hist_tile(int tile, Args a) {
  __shared__ int h[kMaxGroups];
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.A_cap == 0) return;
  const int n = c.n, base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const KeyBuf& k1 = merged_keys(L, c);
  for (int g = tid; g < kMaxGroups; g += kThreads) h[g] = 0;
  __syncthreads();
  for (int r0 = base; r0 < end; r0 += kThreads) {  // warp-uniform trip count
    const int r = r0 + tid;
    const int g = r < end ? (int)k1.cnt[r] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, g);
    if (g >= 0 && (peers & ((1u << (tid & 31)) - 1u)) == 0) atomicAdd(&h[g], __popc(peers));
  }
  __syncthreads();
  const size_t T = n_tiles(q.capacity);
  for (int g = tid; g < kMaxGroups; g += kThreads) L.hist[(size_t)g * T + tile] = (uint32_t)h[g];
}

// ... scanned over tiles per group (one CTA per group) ...
__global__ void __launch_bounds__(kThreads) heads_scan_kernel(Args a) {
  const int g = blockIdx.x, m = blockIdx.y;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.A_cap == 0 || c.cnt_hist[g] == 0) return;
  const long long Tn = (c.n + kTile - 1) / kTile;
  uint32_t* row = L.hist + (size_t)g * n_tiles(q.capacity);
  block_scan_inplace(row, Tn, [](long long f) { return (size_t)f; });
}

// ... and the tiles holding a group's first A_cap members list them in order.
__device__ __forceinline__ void heads_select_tile(int tile, Args a) {
  __shared__ int need[kMaxGroups], run[kMaxGroups];
  __shared__ int any;
  const int m = blockIdx.y, tid = threadIdx.x, lane = tid & 31;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.A_cap == 0) return;
  const int n = c.n, base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const size_t T = n_tiles(q.capacity);
  if (tid == 0) any = 0;
  __syncthreads();
  for (int g = tid; g < kMaxGroups; g += kThreads) {
    const int b0 = c.cnt_hist[g] ? (int)L.hist[(size_t)g * T + tile] : 0x7fffffff;
    run[g] = b0;
    need[g] = b0 < c.A_cap;
    if (need[g]) any = 1;
  }
  __syncthreads();
  if (!any) return;
  const KeyBuf& k1 = merged_keys(L, c);
  // the tile's group ids staged in shared memory by the whole CTA; one warp
  // then lists the needed members in order
  __shared__ uint16_t s_cnt[kTile];
  for (int r = base + tid; r < end; r += kThreads) s_cnt[r - base] = k1.cnt[r];
  __syncthreads();
  if (tid >= 32) return;
  for (int r0 = base; r0 < end; r0 += 32) {
    const int r = r0 + lane;
    const int g = r < end ? (int)s_cnt[r - base] : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, g);
    if (g >= 0 && need[g]) {
      const int k = run[g] + __popc(peers & ((1u << lane) - 1u));
      if (k < c.A_cap) L.hl[(size_t)g * kAcapMax + k] = (uint32_t)r;
    }
    __syncwarp();
    if (g >= 0 && (peers & ((1u << lane) - 1u)) == 0) run[g] += __popc(peers);
    __syncwarp();
  }
}

// The R scheduling iterations on the count-group head lists (as rounds_kernel;
// a group is a starvation count value, its members in merged order).
__global__ void __launch_bounds__(32) fast_rounds_kernel(Args a) {
  __shared__ int g_size[kMaxGroups], g_cur[kMaxGroups], g_count[kMaxGroups],
      g_lvloff[kMaxGroups];
  // cached head of every count group (raw level; the group's level offset
  // is added at compare time): one admission reloads only its own group's
  // head instead of every group's from L2
  __shared__ int h_lvl[kMaxGroups], h_e[kMaxGroups];
  __shared__ unsigned long long h_prio[kMaxGroups], h_arr[kMaxGroups];
  const int m = blockIdx.x, lane = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  if (!c.fast) return;
  const int R = c.R, n = c.n;
  for (int g = lane; g < kMaxGroups; g += 32) {
    g_size[g] = c.cnt_hist[g];
    g_cur[g] = 0;
    g_count[g] = g;
    g_lvloff[g] = 0;
  }
  __syncwarp();
  const size_t seg = (size_t)m * q.capacity;
  const KeyBuf& k1 = merged_keys(L, c);
  const int bmax = a.prm.b[m];
  int run = c.run, n_adm = 0, n_prom = 0, remaining = n;
  // (a call admits at most A_cap entries, so no group needs a head past its
  // first A_cap members -- the only ones heads_select_tile lists in hl)
  auto load_head = [&](int g) {
    if (g_cur[g] < g_size[g] && g_cur[g] < c.A_cap) {
      const uint32_t p = L.hl[(size_t)g * kAcapMax + g_cur[g]];
      h_e[g] = (int)k1.idx[p];
      h_lvl[g] = k1.lvl[p];
      h_prio[g] = k1.prio[p];
      h_arr[g] = k1.arr[p];
    }
  };
  for (int g = lane; g < kMaxGroups; g += 32) load_head(g);
  __syncwarp();
  for (int r = 0; r < R; ++r) {
    if (a.mode == 0) run = max(run - 1, 0);
    const int adm = max(0, min(bmax - run, remaining));
    for (int t = 0; t < adm; ++t) {
      // this lane's best cached head, then the warp's
      HeadKey hk;
      hk.g = -1;
      for (int g = lane; g < kMaxGroups; g += 32) {
        if (g_cur[g] < g_size[g]) {
          HeadKey o;
          o.g = g;
          o.e = h_e[g];
          o.lvl = h_lvl[g] + g_lvloff[g];
          o.prio = h_prio[g];
          o.arr = h_arr[g];
          if (hk.g < 0 || key_less(o, hk)) hk = o;
        }
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
      const HeadKey best = hk;
      if (lane == 0) {
        q.admitted[seg + c.n_adm0 + n_adm] = q.handle[seg + best.e];
        L.adm_idx[n_adm] = (uint32_t)best.e;
        L.adm_pos[n_adm] = L.hl[(size_t)best.g * kAcapMax + g_cur[best.g]];
        g_cur[best.g] += 1;
        load_head(best.g);
      }
      __syncwarp();
      ++n_adm;
      --remaining;
    }
    run += adm;
    if (a.prm.aging_enabled && remaining > 0) {
      for (int g = lane; g < kMaxGroups; g += 32) {
        if (g_cur[g] < g_size[g]) {
          int c2 = g_count[g] + 1;
          if (c2 >= a.prm.S) {
            c2 = 0;
            g_lvloff[g] -= 1;
            n_prom += g_size[g] - g_cur[g];
          }
          g_count[g] = c2;
        }
      }
      __syncwarp();
    }
  }
  for (int off = 16; off; off >>= 1) n_prom += __shfl_xor_sync(0xffffffffu, n_prom, off);
  for (int g = lane; g < kMaxGroups; g += 32) {
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

// Admitted indices / positions sorted; survivor classes by level offset.
__global__ void __launch_bounds__(kThreads) fast_prep_kernel(Args a) {
  __shared__ uint32_t si[kAcapMax], sp[kAcapMax];
  const int m = blockIdx.x, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  if (!c.fast) return;
  const int A = c.n_adm;
  for (int t = tid; t < A; t += kThreads) {
    si[t] = L.adm_idx[t];
    sp[t] = L.adm_pos[t];
  }
  __syncthreads();
  for (int t = tid; t < A; t += kThreads) {
    int ri = 0, rp = 0;
    for (int u = 0; u < A; ++u) {
      ri += si[u] < si[t];
      rp += sp[u] < sp[t];
    }
    L.adm_idx[ri] = si[t];
    L.adm_pos[rp] = sp[t];
  }
  if (tid == 0) {
    const bool aged = c.R > 0;
    int vals[4], D = 0;
    for (int g = 0; g < kMaxGroups; ++g) {
      if (c.cnt_hist[g] - (aged ? c.g_cur[g] : 0) <= 0) { c.cls[g] = 0; continue; }
      const int off = aged ? c.g_lvloff[g] : 0;
      int k = 0;
      while (k < D && vals[k] != off) ++k;
      if (k == D) {
        if (D < 4) vals[D] = off;
        ++D;
      }
      c.cls[g] = k < 4 ? k : 3;
    }
    c.A = A;
    c.D = D;
    c.need_sort2 = D > 2;
    c.n_surv = c.n - A;
    c.n_new = c.n - A;
    int fa = c.n;
    for (int t = 0; t < A; ++t) fa = min(fa, (int)si[t]);
    c.first_adm = fa;
  }
}

// Each tile's last A entries (which the next tile's shifted writes overwrite).
// Every tile's last A entries, copied before compact_fast_tile overwrites
// them (flattened over (tile, entry): a tile holds only A <= kAcapMax of them).
__global__ void __launch_bounds__(256) halo_kernel(Args a) {
  const int m = blockIdx.y;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.A == 0) return;
  const int n = c.n, A = c.A;
  const long long T = (n + kTile - 1) / kTile;
  const size_t seg = (size_t)m * q.capacity;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < T * A;
       w += (long long)gridDim.x * blockDim.x) {
    const int tile = (int)(w / A), j = (int)(w - (long long)tile * A);
    const int base = tile * kTile, end = min(base + kTile, n);
    const int i = end - A + j;
    if (i < base) continue;
    const size_t hp = (size_t)tile * kAcapMax + j;
    L.h64b(0)[hp] = (unsigned long long)__double_as_longlong(q.priority[seg + i]);
    L.h64b(1)[hp] = (unsigned long long)__double_as_longlong(q.arrival[seg + i]);
    L.h64b(2)[hp] = (unsigned long long)q.seq[seg + i];
    L.h64b(3)[hp] = (unsigned long long)q.handle[seg + i];
    L.h32b(0)[hp] = q.out_tokens[seg + i];
    L.h32b(1)[hp] = q.level[seg + i];
    L.h32b(2)[hp] = q.count[seg + i];
    L.h32b(3)[hp] = q.quantum[seg + i];
  }
}

// In-place compaction with aging: survivors shift left by the admissions
// before them; a tile reads everything (its tail from the halo) before it
// writes. Accumulates the hash of the state it leaves.
__device__ __forceinline__ void compact_fast_tile(int tile, Args a) {
  constexpr int kPer = kTile / kThreads;
  __shared__ uint32_t sa[kAcapMax];
  __shared__ int g_count[kMaxGroups], g_lvloff[kMaxGroups];
  __shared__ unsigned long long s_hash;
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  if (!c.fast) return;
  const int n = c.n, base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n), A = c.A;
  const bool aged = c.R > 0;
  for (int t = tid; t < A; t += kThreads) sa[t] = L.adm_idx[t];
  for (int g = tid; g < kMaxGroups; g += kThreads) {
    g_count[g] = aged && a.prm.aging_enabled ? c.g_count[g] : g;
    g_lvloff[g] = aged ? c.g_lvloff[g] : 0;
  }
  if (tid == 0) s_hash = 0ull;
  __syncthreads();
  const size_t seg = (size_t)m * q.capacity;
  const int hbase = end - A;  // [hbase, end) comes from the halo
  double pr[kPer], ar[kPer];
  long long sq[kPer], hd[kPer];
  int ot[kPer], lv[kPer], ct[kPer], qn[kPer], sh[kPer];
  unsigned long long hs = 0ull;
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int i = base + j * kThreads + tid;
    sh[j] = -1;
    if (i >= end) continue;
    if (A > 0 && i >= hbase) {
      const size_t hp = (size_t)tile * kAcapMax + (i - hbase);
      pr[j] = __longlong_as_double((long long)L.h64b(0)[hp]);
      ar[j] = __longlong_as_double((long long)L.h64b(1)[hp]);
      sq[j] = (long long)L.h64b(2)[hp];
      hd[j] = (long long)L.h64b(3)[hp];
      ot[j] = L.h32b(0)[hp];
      lv[j] = L.h32b(1)[hp];
      ct[j] = L.h32b(2)[hp];
      qn[j] = L.h32b(3)[hp];
    } else {
      pr[j] = q.priority[seg + i];
      ar[j] = q.arrival[seg + i];
      sq[j] = q.seq[seg + i];
      hd[j] = q.handle[seg + i];
      ot[j] = q.out_tokens[seg + i];
      lv[j] = q.level[seg + i];
      ct[j] = q.count[seg + i];
      qn[j] = q.quantum[seg + i];
    }
    const int k = count_less(sa, A, (uint32_t)i);
    if (k < A && sa[k] == (uint32_t)i) continue;  // admitted
    sh[j] = k;
    const int g = ct[j];
    if (g_lvloff[g] != 0) qn[j] = 0;
    lv[j] += g_lvloff[g];
    ct[j] = g_count[g];
    hs += entry_hash((uint32_t)(i - k), pr[j], ar[j], lv[j], ct[j]);
  }
  __syncthreads();  // every read of this tile's range is done
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    if (sh[j] < 0) continue;
    const int i = base + j * kThreads + tid;
    const size_t d = seg + (size_t)(i - sh[j]);
    if (sh[j] > 0) {
      q.priority[d] = pr[j];
      q.arrival[d] = ar[j];
      q.seq[d] = sq[j];
      q.handle[d] = hd[j];
      q.out_tokens[d] = ot[j];
    }
    q.level[d] = lv[j];
    q.count[d] = ct[j];
    q.quantum[d] = qn[j];
  }
  for (int off = 16; off; off >>= 1) hs += __shfl_xor_sync(0xffffffffu, hs, off);
  if ((tid & 31) == 0) atomicAdd(&s_hash, hs);
  __syncthreads();
  if (tid == 0) atomicAdd(&c.hash_new, s_hash);
}

// Arrival monotone in seq over the compacted queue (q.arrival_unsorted).
__device__ __forceinline__ void unsorted_tile(int tile, Args a) {
  __shared__ int s_uns;
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  if (!c.fast) return;
  const int n = c.n_surv, base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const size_t seg = (size_t)m * q.capacity;
  if (tid == 0) s_uns = 0;
  __syncthreads();
  int u = 0;
  for (int i = max(base, 1) + tid; i < end; i += kThreads)
    if (q.arrival[seg + i] < q.arrival[seg + i - 1]) u = 1;
  if (u) s_uns = 1;
  __syncthreads();
  if (tid == 0 && s_uns) atomicOr(&c.unsorted[1], 1);
}

// Survivor at merged position r: its keys after this call (or false if admitted).
struct FinalCtx {
  const uint32_t* ai;
  const uint32_t* ap;
  const int* g_count;
  const int* g_lvloff;
  int A;
};
__device__ __forceinline__ bool final_key(const KeyBuf& k1, int r, const FinalCtx& f, FKey& out,
                                          uint16_t& cnt, int& pos, int& g) {
  const int kp = count_less(f.ap, f.A, (uint32_t)r);
  if (kp < f.A && f.ap[kp] == (uint32_t)r) return false;
  pos = r - kp;
  g = k1.cnt[r];
  const uint32_t e = k1.idx[r];
  out.lvl = k1.lvl[r] + f.g_lvloff[g];
  out.prio = k1.prio[r];
  out.arr = k1.arr[r];
  out.idx = e - (uint32_t)count_less(f.ai, f.A, e);
  cnt = (uint16_t)f.g_count[g];
  return true;
}

#define CHM_FINAL_SMEM                                                            \
  __shared__ uint32_t s_ai[kAcapMax], s_ap[kAcapMax];                            \
  __shared__ int s_gc[kMaxGroups], s_go[kMaxGroups], s_cls[kMaxGroups];          \
  const bool aged_ = c.R > 0;                                                     \
  for (int t = threadIdx.x; t < c.A; t += blockDim.x) {                           \
    s_ai[t] = L.adm_idx[t];                                                       \
    s_ap[t] = L.adm_pos[t];                                                       \
  }                                                                               \
  for (int g = threadIdx.x; g < kMaxGroups; g += blockDim.x) {                    \
    s_gc[g] = aged_ && a.prm.aging_enabled ? c.g_count[g] : g;                    \
    s_go[g] = aged_ ? c.g_lvloff[g] : 0;                                          \
    s_cls[g] = c.cls[g];                                                          \
  }                                                                               \
  __syncthreads();                                                                \
  const FinalCtx fx{s_ai, s_ap, s_gc, s_go, c.A};

// One level offset among the survivors: the merged order minus the admitted
// is the new STJF order.
__device__ __forceinline__ void final1_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.D > 1) return;
  const int n = c.n, base = tile * kTile;
  if (base >= n) return;
  CHM_FINAL_SMEM
  const int end = min(base + kTile, n);
  const KeyBuf& k1 = merged_keys(L, c);
  const KeyBuf& ko = L.ksb((c.n_app > 0 ? (c.kcur ^ 1) : c.kcur) ^ 1);
  const size_t seg = (size_t)m * q.capacity;
  for (int r = base + tid; r < end; r += kThreads) {
    FKey k;
    uint16_t cn;
    int pos, g;
    if (!final_key(k1, r, fx, k, cn, pos, g)) continue;
    fk_put(ko, pos, k, cn);
    q.order[seg + pos] = (int32_t)k.idx;
  }
}

// Two classes: survivors of class 1 per tile ...
__device__ __forceinline__ void final2_count_tile(int tile, Args a) {
  __shared__ int wsum[kWarps];
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.D != 2) return;
  const int n = c.n, base = tile * kTile;
  if (base >= n) return;
  CHM_FINAL_SMEM
  const int end = min(base + kTile, n);
  const KeyBuf& k1 = merged_keys(L, c);
  int cnt1 = 0;
  for (int r = base + tid; r < end; r += kThreads) {
    FKey k;
    uint16_t cn;
    int pos, g;
    if (final_key(k1, r, fx, k, cn, pos, g) && s_cls[g] == 1) ++cnt1;
  }
  for (int off = 16; off; off >>= 1) cnt1 += __shfl_xor_sync(0xffffffffu, cnt1, off);
  if ((tid & 31) == 0) wsum[tid >> 5] = cnt1;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < kWarps; ++w) t += wsum[w];
    L.tcnt[tile] = (uint32_t)t;
  }
}

__global__ void __launch_bounds__(kThreads) final2_scan_kernel(Args a) {
  const int m = blockIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  if (!c.fast || c.D != 2) return;
  const long long Tn = (c.n + kTile - 1) / kTile;
  const uint32_t tot = block_scan_inplace(L.tcnt, Tn, [](long long f) { return (size_t)f; });
  if (threadIdx.x == 0) c.nU = c.n_surv - (int)tot;
}

// ... split into U = class 0 (first nU) and P = class 1, each in merged order ...
__device__ __forceinline__ void final2_split_tile(int tile, Args a) {
  __shared__ int wpre[kWarps];
  __shared__ int blk_tot;
  const int m = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.D != 2) return;
  const int n = c.n, base = tile * kTile;
  if (base >= n) return;
  CHM_FINAL_SMEM
  const int end = min(base + kTile, n);
  const KeyBuf& k1 = merged_keys(L, c);
  const KeyBuf& kx = L.ksb((c.n_app > 0 ? (c.kcur ^ 1) : c.kcur) ^ 1);
  int p1 = (int)L.tcnt[tile];  // class-1 survivors before this tile
  for (int blk = base; blk < end; blk += kThreads) {
    const int r = blk + tid;
    FKey k{};
    uint16_t cn = 0;
    int pos = 0, g = 0;
    const bool live = r < end && final_key(k1, r, fx, k, cn, pos, g);
    const bool one = live && s_cls[g] == 1;
    const unsigned bal = __ballot_sync(0xffffffffu, one);
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
    if (live) {
      const int k1b = p1 + wpre[warp] + __popc(bal & ((1u << lane) - 1u));  // class-1 before r
      const int d = one ? c.nU + k1b : pos - k1b;
      fk_put(kx, d, k, cn);
    }
    p1 += blk_tot;
    __syncthreads();
  }
}

// ... and merged (merge path; keys are unique): kx[0, nU) + kx[nU, n_surv) -> k1.
__global__ void __launch_bounds__(kThreads) final2_merge_kernel(Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (!c.fast || c.D != 2) return;
  const int n = c.n_surv, nU = c.nU, nP = n - nU;
  const KeyBuf& out = merged_keys(L, c);
  const KeyBuf& kx = L.ksb((c.n_app > 0 ? (c.kcur ^ 1) : c.kcur) ^ 1);
  const size_t seg = (size_t)m * q.capacity;
  extern __shared__ __align__(16) unsigned char msm[];  // kMergeSmem: one staged output tile
  unsigned long long* s_prio = reinterpret_cast<unsigned long long*>(msm);
  unsigned long long* s_arr = s_prio + kMergeTile;
  int32_t* s_lvl = reinterpret_cast<int32_t*>(s_arr + kMergeTile);
  uint32_t* s_idx = reinterpret_cast<uint32_t*>(s_lvl + kMergeTile);
  uint16_t* s_cnt = reinterpret_cast<uint16_t*>(s_idx + kMergeTile);
  // merge-path splits of this CTA's tiles, found in parallel (one binary
  // search per tile boundary) for up to kSplitBatch tiles at a time: a serial
  // search per tile costs ~2 x 11 dependent L2 round trips
  constexpr int kSplitBatch = kThreads / 2;
  __shared__ int split[2 * kSplitBatch];
  const int n_tiles_all = (n + kMergeTile - 1) / kMergeTile;
  for (int tb = blockIdx.x; tb < n_tiles_all; tb += gridDim.x * kSplitBatch) {
  if (tid < 2 * kSplitBatch) {
    const int tt = tb + (tid >> 1) * gridDim.x;
    if (tt < n_tiles_all) {
      // i = #U among the first d outputs
      const int d = min((tt + (tid & 1)) * kMergeTile, n);
      int lo = max(0, d - nP), hi = min(d, nU);
      while (lo < hi) {
        const int i = (lo + hi) >> 1;  // take U[i] before P[d - i - 1]?
        if (fk_less(fk_at(kx, i), fk_at(kx, nU + d - i - 1))) lo = i + 1; else hi = i;
      }
      split[tid] = lo;
    }
  }
  __syncthreads();
  for (int bi = 0; bi < kSplitBatch; ++bi) {
    const int tt = tb + bi * gridDim.x;
    if (tt >= n_tiles_all) break;
    const int o0 = tt * kMergeTile, o1 = min(o0 + kMergeTile, n);
    const int u0 = split[2 * bi], u1 = split[2 * bi + 1];
    const int p0 = o0 - u0, p1 = o1 - u1;
    const int nu = u1 - u0, tot = nu + (p1 - p0);
    // stage the tile's U run then its P run in shared memory (coalesced)
    for (int t = tid; t < tot; t += kThreads) {
      const int src = t < nu ? u0 + t : nU + p0 + (t - nu);
      s_lvl[t] = kx.lvl[src];
      s_prio[t] = kx.prio[src];
      s_arr[t] = kx.arr[src];
      s_idx[t] = kx.idx[src];
      s_cnt[t] = kx.cnt[src];
    }
    __syncthreads();
    // each element's output slot: own offset + #(other run < it), by binary
    // search over the other run in shared memory
    for (int t = tid; t < tot; t += kThreads) {
      const bool isU = t < nu;
      const FKey k{s_lvl[t], s_prio[t], s_arr[t], s_idx[t]};
      int lo = isU ? nu : 0, hi = isU ? tot : nu;
      const int base = lo;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const FKey o{s_lvl[mid], s_prio[mid], s_arr[mid], s_idx[mid]};
        if (fk_less(o, k)) lo = mid + 1; else hi = mid;
      }
      const int d = o0 + (isU ? t : t - nu) + (lo - base);
      fk_put(out, d, k, s_cnt[t]);
      q.order[seg + d] = (int32_t)k.idx;
    }
    __syncthreads();
  }
  }
}

// D > 2 (several promotion classes): sort-2 keys from the compacted queue.
__device__ __forceinline__ void keys_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  Ctl& c = *L.ctl;
  if (!c.fast || !c.need_sort2) return;
  if (tile == 0 && tid == 0) c.cur[kPass1] = 0;
  const int n = c.n_new, base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const size_t seg = (size_t)m * q.capacity;
  unsigned long long o[4] = {0, 0, 0, 0}, an[4] = {~0ull, ~0ull, ~0ull, ~0ull};
  for (int i = base + tid; i < end; i += kThreads) {
    const unsigned long long ak = f64_key(q.arrival[seg + i]), pk = f64_key(q.priority[seg + i]);
    const int lv = q.level[seg + i];
    const unsigned long long lk = (unsigned long long)(lv + 32768);
    L.prio[i] = pk;
    L.lvl[i] = (uint16_t)lk;
    L.idxb(0)[i] = (uint32_t)i;
    o[0] |= ak; an[0] &= ak;
    o[1] |= pk; an[1] &= pk;
    o[2] |= lk; an[2] &= lk;
  }
  // the arrival flag of this call comes from unsorted_tile
  merge_masks(o, an, 0, c, 1);
}

// After a radix sort 2 (either path): the kept keys in the new order.
__device__ __forceinline__ void ks_build_tile(int tile, Args a) {
  const int m = blockIdx.y, tid = threadIdx.x;
  const chm_queue_state& q = a.q;
  Layout L = layout(q.scratch, q.capacity, m);
  const Ctl& c = *L.ctl;
  if (c.err || (c.fast && !c.need_sort2)) return;
  const int n = c.n_new, base = tile * kTile;
  if (base >= n) return;
  const int end = min(base + kTile, n);
  const size_t seg = (size_t)m * q.capacity;
  const uint32_t* sorted = L.idxb(c.cur[kMaxPasses]);
  const KeyBuf& k0 = L.ksb(0);
  for (int r = base + tid; r < end; r += kThreads) {
    const uint32_t e = sorted[r];
    fk_put(k0, r, fk_entry(q, seg, e), (uint16_t)min(max(q.count[seg + e], 0), 65535));
  }
}

__global__ void commit_kernel(Args a) {
  const int m = blockIdx.x;
  if (threadIdx.x != 0) return;
  Layout L = layout(a.q.scratch, a.q.capacity, m);
  Ctl& c = *L.ctl;
  if (c.err) {
    c.valid = 0u;
    return;
  }
  if (!c.fast || c.need_sort2) c.kcur = 0;
  else if (c.D == 2) c.kcur = c.n_app > 0 ? (c.kcur ^ 1) : c.kcur;          // merged back into k1
  else c.kcur = (c.n_app > 0 ? (c.kcur ^ 1) : c.kcur) ^ 1;                  // final1 wrote the other
  c.n_prev = c.n_new;
  c.hash_prev = c.hash_new;
  c.valid = kValidMagic;
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

unsigned long long queue_huge_fast_calls() {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, qh::g_fast_calls, sizeof(v));
  return v;
}

namespace qh {
// IF-node condition of a radix section: 1 if any engine runs it.
__global__ void section_cond_kernel(Args a, cudaGraphConditionalHandle h, int section) {
  if (threadIdx.x != 0) return;
  unsigned need = 0;
  for (int m = 0; m < a.prm.K; ++m) {
    const Ctl& c = *layout(a.q.scratch, a.q.capacity, m).ctl;
    need |= section == 0 ? (c.fast ? 0u : 1u) : ((!c.fast || c.need_sort2) ? 1u : 0u);
  }
  cudaGraphSetConditional(h, need);
}

// While `s` is being captured into a CUDA graph: a kernel sets the section's
// condition, an IF node follows it, and `body` is captured into the node's
// body graph on a side stream. Returns false (nothing enqueued) when `s` is
// not capturing or the graph API refuses, so the caller launches the body.
template <class Body>
bool cond_section(cudaStream_t s, const Args& a, int section, Body body) {
  cudaStreamCaptureStatus cs;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusActive)
    return false;
  cudaGraph_t g;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(s, &cs, &id, &g, &deps, &nd) != cudaSuccess) return false;
  cudaGraphConditionalHandle h;
  if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) != cudaSuccess)
    return false;
  section_cond_kernel<<<1, 32, 0, s>>>(a, h, section);
  if (cudaStreamGetCaptureInfo(s, &cs, &id, &g, &deps, &nd) != cudaSuccess) return false;
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  if (cudaGraphAddNode(&node, g, deps, nd, &cp) != cudaSuccess) return false;
  static cudaStream_t side = nullptr;
  if (!side) cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
  if (cudaStreamBeginCaptureToGraph(side, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                    cudaStreamCaptureModeRelaxed) != cudaSuccess)
    return false;
  body(side);
  cudaGraph_t done;
  cudaStreamEndCapture(side, &done);
  return cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies) ==
         cudaSuccess;
}
}  // namespace qh

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
    cudaFuncSetAttribute(final2_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMergeSmem);
    cudaFuncSetAttribute(tiles_pass<scatter_tile, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(ScatterSmem));
  }
  // two 1024-thread CTAs per SM walk the tiles
  const dim3 grid((unsigned)(T < 2 * sms ? T : 2 * sms), (unsigned)K);
  // CHM_QUEUE_FAST=0: always the radix path (measurement / tests)
  const char* fe = getenv("CHM_QUEUE_FAST");
  const int allow_fast = fe ? atoi(fe) != 0 : 1;
  prep_kernel<<<K, kThreads, 0, s>>>(a);
  tiles<check_tile, 0><<<grid, kThreads, 0, s>>>(a);
  decide_kernel<<<K, 32, 0, s>>>(a, allow_fast);
  // ---- incremental path (every kernel returns at once unless ctl.fast) ----
  const dim3 grid_new((kNewMax + 255) / 256, (unsigned)K);
  newsort_kernel<<<grid_new, 256, 0, s>>>(a);
  insert_kernel<<<grid_new, 256, 0, s>>>(a);
  tiles<merge_old_tile, 0><<<grid, kThreads, 0, s>>>(a);
  tiles<heads_hist_tile, 0><<<grid, kThreads, 0, s>>>(a);
  heads_scan_kernel<<<dim3(kMaxGroups, K), kThreads, 0, s>>>(a);
  tiles<heads_select_tile, 0><<<grid, kThreads, 0, s>>>(a);
  fast_rounds_kernel<<<K, 32, 0, s>>>(a);
  fast_prep_kernel<<<K, kThreads, 0, s>>>(a);
  halo_kernel<<<dim3(4 * sms, K), 256, 0, s>>>(a);
  tiles<compact_fast_tile, 0><<<grid, kThreads, 0, s>>>(a);
  tiles<unsorted_tile, 0><<<grid, kThreads, 0, s>>>(a);
  tiles<final1_tile, 0><<<grid, kThreads, 0, s>>>(a);
  tiles<final2_count_tile, 0><<<grid, kThreads, 0, s>>>(a);
  final2_scan_kernel<<<K, kThreads, 0, s>>>(a);
  tiles<final2_split_tile, 0><<<grid, kThreads, 0, s>>>(a);
  final2_merge_kernel<<<dim3(2 * sms, K), kThreads, kMergeSmem, s>>>(a);
  tiles<keys_tile, 1><<<grid, kThreads, 0, s>>>(a);
  // ---- radix path (every kernel returns at once if ctl.fast) ----
  auto pass = [&](cudaStream_t st, int sort, int src, int byte, int p) {
    PassSpec ps{sort, src, byte, p};
    if (byte == 0) tiles_pass<gather_tile, true><<<grid, kThreads, 0, st>>>(a, ps);
    tiles_pass<hist_tile, false><<<grid, kThreads, 0, st>>>(a, ps);
    scan_kernel<<<dim3(256, K), kThreads, 0, st>>>(a, ps);
    tiles_pass<scatter_tile, false><<<grid, kThreads, sizeof(ScatterSmem), st>>>(a, ps);
  };
  // section 0: sort 1 + the rounds + compaction (radix path only)
  auto section0 = [&](cudaStream_t st) {
    tiles<stage_tile, 0><<<grid, kThreads, 0, st>>>(a);
    int p = 0;
    // sort 1, least significant first: arrival, priority, level, count
    const int srcs1[4] = {0, 1, 2, 3}, bytes1[4] = {8, 8, 2, 2};
    for (int j = 0; j < 4; ++j)
      for (int b = 0; b < bytes1[j]; ++b) pass(st, 0, srcs1[j], b, p++);
    tiles<groups_tile, 0><<<grid, kThreads, 0, st>>>(a);
    rounds_kernel<<<K, 32, 0, st>>>(a);
    tiles<outcome_tile, 0><<<grid, kThreads, 0, st>>>(a);
    tiles<compact_count_tile, 0><<<grid, kThreads, 0, st>>>(a);
    compact_scan_kernel<<<K, kThreads, 0, st>>>(a);
    tiles<compact_scatter_tile, 0><<<grid, kThreads, 0, st>>>(a);
    // copy_back (tile 0 resets the sort-2 buffer index) runs after n_new is known
    tiles<copy_back_tile, 1><<<grid, kThreads, 0, st>>>(a);
  };
  // section 1: sort 2 (radix path, or the fast path with several promotion classes)
  auto section1 = [&](cudaStream_t st) {
    int p = kPass1;
    const int srcs2[3] = {0, 1, 2}, bytes2[3] = {8, 8, 2};
    for (int j = 0; j < 3; ++j)
      for (int b = 0; b < bytes2[j]; ++b) pass(st, 1, srcs2[j], b, p++);
  };
  // Under CUDA-graph capture each section is the body of an IF node whose
  // condition a one-thread kernel sets on the device (any engine needs it):
  // in the incremental steady state the ~230 radix launches, which would
  // all return at once, are skipped. Eager: launched as before.
  static const int use_cond = getenv("CHM_QUEUE_COND") ? atoi(getenv("CHM_QUEUE_COND")) : 1;
  if (!use_cond || !cond_section(s, a, 0, section0)) section0(s);
  if (!use_cond || !cond_section(s, a, 1, section1)) section1(s);
  tiles<finish_tile, 1><<<grid, kThreads, 0, s>>>(a);
  tiles<ks_build_tile, 1><<<grid, kThreads, 0, s>>>(a);
  commit_kernel<<<K, 32, 0, s>>>(a);
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

}  // namespace chm
