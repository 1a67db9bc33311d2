// Pieces shared by the STJF+aging queue kernels (stjf.cu: one CTA per engine
// segment; stjf_huge.cu: grid-wide passes for segments beyond 2^18 entries).
#pragma once
#include "common.cuh"

namespace chm {

constexpr int kMaxGroups = 256;             // distinct starvation counts per segment
constexpr uint32_t kAdmitted = 0xffffffffu;

struct QueueParams {
  int K;
  int b[CHM_MAX_MODELS];
  double d[CHM_MAX_MODELS];  // decode_ms_per_token (engine clock)
  int aging_enabled;
  int S;
  int Q;       // running_quantum
  int demote;  // AgingConfig.demote_while_queued
  int cap_limit;  // largest segment this kernel variant can hold
};

__device__ __forceinline__ unsigned long long f64_key(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  // priorities/arrivals are >= 0 (validated upstream); -0.0 == 0.0 in Python.
  return b == 0x8000000000000000ull ? 0ull : b;
}

// Lexicographic key of a count-group head: (level, priority, arrival?, storage idx).
struct HeadKey {
  int lvl;
  unsigned long long prio;
  unsigned long long arr;
  int e;
  int g;
};

__device__ __forceinline__ bool key_less(const HeadKey& x, const HeadKey& y) {
  if (x.lvl != y.lvl) return x.lvl < y.lvl;
  if (x.prio != y.prio) return x.prio < y.prio;
  if (x.arr != y.arr) return x.arr < y.arr;
  return x.e < y.e;
}

// Append the rows chm_schedule_rows queued on engine m (flag bit 2) at the end
// of the segment, in row order (= seq order). One CTA; `scan` needs
// blockDim/32 ints of shared memory, `misc` two. Returns the number of rows
// appended (already counted in engine_queued by K6).
__device__ __forceinline__ int append_queued_rows(int m, int K, const chm_rows& rows,
                                                  const chm_decisions& dec, size_t seg,
                                                  const chm_queue_state& q, int n_old,
                                                  int* scan, int* misc,
                                                  int32_t* q_input = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_warps = blockDim.x >> 5;
  const int n_rows = *dec.n_committed;
  int pos_base = n_old;
  for (int blk = 0; blk < n_rows; blk += blockDim.x) {
    const int i = blk + tid;
    const bool take = i < n_rows && dec.model[i] == m && (dec.flags[i] & 4u);
    const unsigned bal = __ballot_sync(0xffffffffu, take);
    if (lane == 0) scan[warp] = __popc(bal);
    __syncthreads();
    if (warp == 0) {
      int v = lane < n_warps ? scan[lane] : 0, incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane < n_warps) scan[lane] = incl - v;
      if (lane == 31) misc[1] = incl;
    }
    __syncthreads();
    if (take) {
      const size_t pos = seg + pos_base + scan[warp] + __popc(bal & ((1u << lane) - 1u));
      q.priority[pos] = dec.priority[i];
      q.arrival[pos] = rows.arrival[i];
      q.seq[pos] = dec.seq[i];
      q.handle[pos] = rows.handle ? rows.handle[i] : (int64_t)i;
      q.out_tokens[pos] = rows.out_tokens ? rows.out_tokens[(size_t)i * K + m] : 0;
      q.level[pos] = 0;
      q.count[pos] = 0;
      q.quantum[pos] = 0;
      if (q_input) q_input[pos] = rows.input_tokens ? rows.input_tokens[i] : 1;
    }
    pos_base += misc[1];
    __syncthreads();
  }
  return pos_base - n_old;
}

// Number of rows of this batch queued on engine m (all threads get it).
__device__ __forceinline__ int count_queued_rows(int m, const chm_decisions& dec, int* scan,
                                                 int* misc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_warps = blockDim.x >> 5;
  const int n_rows = *dec.n_committed;
  int c = 0;
  for (int i = tid; i < n_rows; i += blockDim.x)
    c += (dec.model[i] == m && (dec.flags[i] & 4u)) ? 1 : 0;
  for (int off = 16; off; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if (lane == 0) scan[warp] = c;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < n_warps; ++w) t += scan[w];
    misc[0] = t;
  }
  __syncthreads();
  const int r = misc[0];
  __syncthreads();
  return r;
}

}  // namespace chm
