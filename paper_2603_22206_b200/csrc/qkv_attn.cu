// K2+K3 fused: QKV projection + self-attention for S = 128 (the headline
// router shape), one pass, Q/K/V never written to HBM.
//
// An item is one (sequence, head): its 128 tokens are one MMA M tile, so the
// projection of that head is a 128 x 192 x H GEMM (rows = tokens, columns =
// the head's 64 Q + 64 K + 64 V output features of W_qkv), and its attention
// consumes the result straight from tensor memory.
//
// Default build path (PAIR, see the kernel template): two sequences of one
// head per CTA pair, the projection as a cta_group::2 pair MMA (28 KB of
// operands per SM per k-block), attention per CTA with cta_group::1 MMAs.
// The cta_group::1 description below is the CHM_QA_PAIR=0 path.
//
// Operand traffic: a lone CTA would stream 40 KB (x 16 KB + W 24 KB) from L2
// per 384 tensor cycles, ~2x what L2 can deliver to every SM at once. CTAs
// are therefore grouped in clusters of CS sequences x CH heads: the CH CTAs
// of one sequence share its x tile and the CS CTAs of one head share its W
// tile, each CTA loading a 1/CH slice of x and a 1/CS slice of W and
// multicasting it to the sharers (TMA .multicast::cluster). Stage reuse is
// released cluster-wide: each CTA's MMA commit arrives on the "empty"
// barrier of every CTA that writes into its stages (tcgen05.commit multicast).
//
//   warp 0      TMA producer: 4-stage ring of x[128 x 64] + W[192 x 64]
//   warp 1      MMA issuer (whole warp, warp-uniform; one elected lane issues
//               inside the asm). GEMM(i+1), GEMM(i+2) are issued while item
//               i's attention runs: between projection k-blocks it polls
//               (mbarrier test_wait) for "Q/K/V of item i staged" and
//               "P of item i written" and slots S(i) = Q K^T and O(i) = P V
//               into the tensor pipe as soon as they are ready; it blocks only
//               on the accumulator (drain of item i - 2)
//   warps 2-9   epilogue, 2 threads per token row (column halves hf = 0/1):
//               (1) acc(i) + bias -> bf16 Q (x 1/8), K, V tiles in smem
//                   (128B swizzle, the UMMA operand layout), accumulator freed
//               (2) softmax of S(i) (row max / sum exchanged between the two
//                   halves through smem), P bf16 over the Q|K tiles
//               (3) O(i) / rowsum -> ctx (bf16, HBM)
//
// TMEM (512 columns): accumulators acc[0] = [0,192), acc[1] = [192,384)
// (double-buffered across items), S = [384,512), O = [384,448) (after S is
// consumed). Numerics equal the unfused path (chm_gemm QKV epilogue + K3):
// fp32 accumulation, bias in fp32, bf16 Q/K/V, exp2-based softmax with the
// normaliser summed over the bf16-rounded P.
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "common.cuh"
#include "deferred_ln.cuh"
#include "prof.cuh"
#include "sm100.cuh"

namespace chm {
namespace gemm {
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, uint64_t rows, uint64_t cols,
                    uint32_t box_rows, uint32_t box_cols, uint64_t ld);
bool make_tmap_qkv3(CUtensorMap* map, const void* ptr, uint64_t hidden, uint32_t box_rows);
}
namespace qa {

constexpr int kS = 128;                        // tokens per sequence = MMA M
constexpr int kStages = 4;
#ifndef CHM_QA_PAIR_STAGES
#define CHM_QA_PAIR_STAGES 5
#endif
constexpr int kThreads = 320;                  // 10 warps
constexpr uint32_t kATile = kS * 64 * 2;       // x   [128][64] bf16, 16 KB
constexpr uint32_t kBTile = 192 * 64 * 2;      // W   [192][64] (Q | K | V rows), 24 KB
constexpr uint32_t kStageBytes = kATile + kBTile;  // 40 KB
constexpr uint32_t kWBox = 32;                 // W rows per TMA box (6 per head)
constexpr uint32_t kHeadTile = kS * 64 * 2;    // Q/K/V [128][64] bf16, 16 KB
constexpr uint32_t kAccCols = 192;
constexpr uint32_t kSCol = 384;
constexpr int kPairStages = CHM_QA_PAIR_STAGES;  // PAIR ring depth (28 KB stages)
#ifndef CHM_QA_POLY
#define CHM_QA_POLY 0
#endif
constexpr int kPolyPairs = CHM_QA_POLY;  // softmax exp2 pairs (of 4) on the FMA pipes

struct __align__(1024) Smem {
  // the operand ring: 4 x 40 KB (cta_group::1) or kPairStages x 28 KB (PAIR)
  uint8_t stages[kStages][kStageBytes];
  uint8_t stages_pair_extra[kPairStages * (kATile + kBTile / 2) > kStages * kStageBytes
                                ? kPairStages * (kATile + kBTile / 2) - kStages * kStageBytes
                                : 1];
  alignas(1024) uint8_t qkv[3][kHeadTile];  // Q, K, V; P key halves [0,64) / [64,128) overwrite Q / K
  float red_max[2][kS];
  float red_sum[2][kS];
  uint64_t full[8], empty[8], kdone[8];
  uint64_t acc_full[2], acc_empty[2];
  uint64_t qkv_ready, s_full, p_ready, o_full;
  uint64_t ev_pair;  // PAIR: both CTAs ready for the next S / O event
  uint32_t tmem_base;
};
constexpr size_t kSmemBytes = sizeof(Smem) + 1024;

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// dbg 11: per-item timeline of CTA 0, items [8, 16): 16 clock64 stamps per
// item into ctx (as int64; all ctx output is skipped in this mode).
__device__ __forceinline__ void stamp(int dbg, void* ctx, int it, int k) {
  if (dbg >= 11 && blockIdx.x == 0 && it >= 8 && it < 16)
    reinterpret_cast<long long*>(ctx)[(it - 8) * 16 + k] = clock64();
}

__device__ __forceinline__ void epi_sync() {
  asm volatile("bar.sync 1, 256;" ::: "memory");
}

// Cluster items: (group of CS sequences) x (group of CH heads). CTA (i, j) of
// the cluster (rank = i*CH + j) owns sequence sg*CS + i, head hg*CH + j.
// lag > 0: the MMA issuer keeps at most `lag` projection k-blocks queued on
// the tensor pipe, so S(i) / O(i) slotted between them start soon.
// FOLD: the deferred-LayerNorm instantiation (row affine + column sums); the
// plain one compiles without it.
// TS: Q and P stay in tensor memory as bf16 (FlashAttention-4 style): the
// S = Q K^T and O = P V MMAs read their A operand from TMEM (tcgen05.mma
// [d], [a_tmem], b_desc), saving the Q and P shared-memory round trips
// (96 KB per item) of a kernel bound by shared-memory traffic.
// PAIR (CS = 2, CH = 1): the projection is one cta_group::2 pair MMA per
// k-block (M = 256 = the two sequences, N = 192 split 96 / 96: each CTA stages
// its own x tile and half of the head's W rows, 28 KB instead of 40 KB, in
// kPairStages stages), issued by the leader into both CTAs' TMEM; each CTA runs its own
// sequence's S and O as cta_group::1 MMAs (tools/cta_group_mix_probe.cu).
template <int CS, int CH, bool FOLD, bool TS, bool PAIR = false>
__global__ void __launch_bounds__(kThreads, 1)
    qkv_attention_kernel(const __grid_constant__ CUtensorMap tm_x,
                         const __grid_constant__ CUtensorMap tm_w,
                         const float* __restrict__ b_qkv, const float* __restrict__ c_qkv,
                         const float2* __restrict__ stats_in, int n_part, float eps, int n_seq,
                         int n_heads, int hidden, __nv_bfloat16* __restrict__ ctx, int lag,
                         int dbg, int contiguous, const int32_t* __restrict__ n_live,
                         int pair_sync) {
  extern __shared__ uint8_t smem_raw[];
  Smem& s = sm100::align_smem_1024<Smem>(smem_raw);
  const int warp = sm100::warp_id(), lane = threadIdx.x & 31;
  const int k_blocks = hidden / 64;
  const uint32_t rank = sm100::cluster_ctarank();
  static_assert(!PAIR || (CS == 2 && CH == 1 && !TS), "pair projection: 2 sequences, one head");
  constexpr int NST = PAIR ? kPairStages : kStages;                // ring stages
  constexpr uint32_t SB = PAIR ? kATile + kBTile / 2 : kStageBytes;  // bytes per stage (per CTA)
  const bool leader = !PAIR || rank == 0;
  auto stage_ptr = [&](int i) { return &s.stages[0][0] + (size_t)i * SB; };
  const int ci = (int)rank / CH, cj = (int)rank % CH;
  const uint16_t row_mask = (uint16_t)(((1u << CH) - 1) << (ci * CH));  // same sequence
  uint16_t col_mask = 0;                                                 // same head
#pragma unroll
  for (int i = 0; i < CS; ++i) col_mask |= (uint16_t)(1u << (i * CH + cj));
  const int head_groups = n_heads / CH;
  // only the routed (live) sequences are encoded (balancer.py:104-114)
  if (n_live) n_seq = min(n_seq, __ldg(n_live));
  const int n_citems = ((n_seq + CS - 1) / CS) * head_groups;
  const int cl = (int)sm100::cluster_id_x(), n_cl = (int)sm100::n_clusters_x();
  // Item order: interleaved (cluster cl takes items cl, cl + n_cl, ...: the
  // clusters sweep the items together) or contiguous (a range per cluster, so
  // consecutive items of a CTA share a sequence and its cached LayerNorm row
  // affine). `contiguous` is chosen on the host.
  const int per = contiguous ? (n_citems + n_cl - 1) / n_cl : 0;
  const int c_lo = contiguous ? cl * per : cl;
  const int n_my = contiguous ? (c_lo < n_citems ? min(per, n_citems - c_lo) : 0)
                              : (cl < n_citems ? (n_citems - 1 - cl) / n_cl + 1 : 0);
  const int c_step = contiguous ? 1 : n_cl;
  auto item_of = [&](int it, int& seq, int& h) {
    const int c = c_lo + it * c_step;
    const int sg = c / head_groups, hg = c - sg * head_groups;
    seq = sg * CS + ci;
    h = hg * CH + cj;
  };

  if (warp == 0 && lane == 0) {
    sm100::tma_prefetch(&tm_x);
    sm100::tma_prefetch(&tm_w);
    for (int i = 0; i < NST; ++i) {
      sm100::mbar_init(&s.full[i], 1);
      sm100::mbar_init(&s.empty[i], PAIR ? 1 : CS + CH - 1);  // consumers of this CTA's slices
      sm100::mbar_init(&s.kdone[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      sm100::mbar_init(&s.acc_full[i], 1);
      sm100::mbar_init(&s.acc_empty[i], PAIR ? 2 * 8 : 256);  // PAIR: epilogue warps of both CTAs
    }
    sm100::mbar_init(&s.qkv_ready, 256);
    sm100::mbar_init(&s.s_full, 1);
    sm100::mbar_init(&s.p_ready, 256);
    sm100::mbar_init(&s.o_full, 1);
    sm100::mbar_init(&s.ev_pair, 2);
    sm100::fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR)
      sm100::tmem_alloc_cg2<512>(&s.tmem_base);
    else
      sm100::tmem_alloc<512>(&s.tmem_base);
  }
  sm100::tc_fence_before();
  sm100::cluster_sync();
  sm100::tc_fence_after();
  const uint32_t tmem = sm100::uniform(s.tmem_base);

  if (warp == 0) {
    // ---------------- TMA producer: this CTA's slices, multicast ----------------
    // (warp-uniform loop like the MMA issuer; one elected lane issues the copies)
    {
      constexpr int kARows = kS / CH;        // x rows this CTA loads
      constexpr int kBoxes = 6 / CS;         // 32-row W boxes this CTA loads
      int stage = 0;
      uint32_t phase = 0;
      for (int it = 0; it < (dbg >= 7 && dbg <= 10 ? 0 : n_my); ++it) {
        int seq, h;
        item_of(it, seq, h);
        const int a_row = seq * kS + cj * kARows;
        for (int kb = 0; kb < k_blocks; ++kb) {
          // every sharer of this stage has consumed its previous contents
          sm100::mbar_wait(&s.empty[stage], phase ^ 1);
          if constexpr (PAIR) {
            // own x tile + own half of the head's W rows (Q|K|V rows
            // [32 ci, +32) of each part), both signalling the leader's barrier
            if (sm100::elect_one()) {
              if (leader) sm100::mbar_arrive_expect_tx(&s.full[stage], 2 * SB);
              const uint32_t full_leader = sm100::mapa(sm100::smem_u32(&s.full[stage]), 0);
              uint8_t* st = stage_ptr(stage);
              sm100::tma_load_2d_cg2(st, &tm_x, full_leader, kb * 64, a_row);
              sm100::tma_load_3d_cg2(st + kATile, &tm_w, full_leader, kb * 64, h * 64 + ci * 32, 0);
            }
            __syncwarp();
            if (lane == 0 && (kb == 0 || kb == k_blocks - 1)) stamp(dbg, ctx, it, kb == 0 ? 11 : 12);
            if (++stage == NST) { stage = 0; phase ^= 1; }
            continue;
          }
          if (dbg >= 4 && dbg <= 10) {  // measurement: no operand loads (MMAs on stale smem)
            if (lane == 0) sm100::mbar_arrive(&s.full[stage]);
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          if (sm100::elect_one()) {
          // (dbg 14 / 15: full kernel, but only x / only W is loaded -- an
          // operand-traffic probe; results are garbage)
          sm100::mbar_arrive_expect_tx(&s.full[stage], dbg == 14   ? kATile
                                                       : dbg == 15 ? kStageBytes - kATile
                                                                   : kStageBytes);
          uint8_t* st = s.stages[stage];
          if (dbg != 15)
            sm100::tma_load_2d_mc(st + cj * kARows * 128, &tm_x, &s.full[stage], kb * 64, a_row,
                                  row_mask);
          if (dbg == 14) {
          } else if constexpr (TS || CS != 2) {
#pragma unroll
            for (int bb = 0; bb < kBoxes; ++bb) {
              const int b = ci * kBoxes + bb;  // box of the head's 6: part b/2, half b%2
              sm100::tma_load_2d_mc(st + kATile + b * kWBox * 128, &tm_w, &s.full[stage], kb * 64,
                                    (b >> 1) * hidden + h * 64 + (b & 1) * kWBox, col_mask);
            }
          } else {
            // one op: rows [64/CS * ci, +64/CS) of the head's Q, K and V parts
            // (tm_w is the 3-part view); B rows -- and accumulator columns --
            // are ordered (half, part, row)
            constexpr int kRowsPer = 64 / CS;
            sm100::tma_load_3d_mc(st + kATile + ci * 3 * kRowsPer * 128, &tm_w, &s.full[stage],
                                  kb * 64, h * 64 + ci * kRowsPer, 0, col_mask);
          }
          }
          __syncwarp();
          if (lane == 0 && (kb == 0 || kb == k_blocks - 1)) stamp(dbg, ctx, it, kb == 0 ? 11 : 12);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    // The whole warp runs the loop (waits, descriptors and counters stay
    // warp-uniform); the *_w helpers elect the issuing lane inside their asm.
    {
      // (dbg 5 / 6: N = 256 / 128 projection MMAs on stale shared memory -- an MMA-shape probe)
      const uint32_t idesc_g = dbg == 5   ? sm100::umma_idesc_bf16(128, 256)
                               : dbg == 6 ? sm100::umma_idesc_bf16(128, 128)
                                          : sm100::umma_idesc_bf16(128, 192);
      constexpr uint32_t idesc_s = sm100::umma_idesc_bf16(128, 128);
      constexpr uint32_t idesc_o = sm100::umma_idesc_bf16(128, 64) | (1u << 16);  // V MN-major
      const uint16_t share_mask = row_mask | col_mask;
      const uint32_t q_addr = sm100::smem_u32(s.qkv[0]);
      const uint32_t k_addr = sm100::smem_u32(s.qkv[1]);
      const uint32_t v_addr = sm100::smem_u32(s.qkv[2]);
      int stage = 0;
      uint32_t phase = 0;
      int g = 0;  // projection k-blocks issued so far
      auto gemm_kb = [&](int it, int kb) {
        if constexpr (PAIR) {
          // leader: one pair MMA group into both CTAs' accumulators. With a
          // lag, at most `lag` projection k-blocks are queued on the tensor
          // pipe, so S(i) / O(i) slotted between them start soon.
          if (lag > 0 && g >= lag) {
            const int d = g - lag;
            sm100::mbar_wait(&s.kdone[d % NST], (d / NST) & 1);
          }
          sm100::mbar_wait(&s.full[stage], phase);
          sm100::tc_fence_after();
          const uint32_t a = sm100::smem_u32(stage_ptr(stage));
          const uint32_t b = a + kATile;
          const uint32_t d = tmem + (uint32_t)(it & 1) * kAccCols;
          constexpr uint32_t idesc_p = sm100::umma_idesc_bf16(256, 192);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            sm100::mma_bf16_cg2_w(d, sm100::umma_desc_sw128(a + k * 32),
                                  sm100::umma_desc_sw128(b + k * 32), idesc_p, (kb | k) != 0);
          sm100::mma_commit_cg2_mc_w(&s.empty[stage], 0x3);
          if (lag > 0) sm100::mma_commit_cg2_mc_w(&s.kdone[stage], 0x1);
          if (kb == k_blocks - 1) sm100::mma_commit_cg2_mc_w(&s.acc_full[it & 1], 0x3);
          ++g;
          if (++stage == NST) { stage = 0; phase ^= 1; }
          return;
        }
        if (lag > 0 && g >= lag) {
          const int d = g - lag;
          sm100::mbar_wait(&s.kdone[d % kStages], (d / kStages) & 1);
        }
        // (dbg >= 7: no producer at all -- the issue loop alone, as
        // tools/mma_probe.cu; 8: + accumulators 256 apart, 9: + local commit
        // instead of the multicast one, 10: + no accumulator handshake)
        if (dbg < 7 || dbg > 10) sm100::mbar_wait(&s.full[stage], phase);
        sm100::tc_fence_after();
        const uint32_t a = sm100::smem_u32(s.stages[stage]);
        const uint32_t b = a + kATile;
        // (dbg == 3: projection only, accumulators 256 columns apart -- an
        // alignment probe; S is unused then)
        const uint32_t d = tmem + (uint32_t)(it & 1) * (dbg == 3 || dbg == 8 ? 256u : kAccCols);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          sm100::mma_bf16_w(d, sm100::umma_desc_sw128(a + k * 32), sm100::umma_desc_sw128(b + k * 32),
                            idesc_g, (kb | k) != 0);
        if (dbg == 9 || dbg == 10)
          sm100::mma_commit_w(&s.empty[stage]);
        else
          sm100::mma_commit_mc_w(&s.empty[stage], share_mask);
        if (lag > 0) sm100::mma_commit_w(&s.kdone[stage]);
        if (kb == k_blocks - 1 && dbg != 10) sm100::mma_commit_w(&s.acc_full[it & 1]);
        ++g;
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      };
      auto issue_s = [&](int it) {
        if (lane == 0) stamp(dbg, ctx, it, 6);
        sm100::tc_fence_after();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if constexpr (TS)  // Q bf16 in the drained accumulator's first 32 columns
            sm100::mma_bf16_ts_w(tmem + kSCol, tmem + (uint32_t)(it & 1) * kAccCols + k * 8,
                                 sm100::umma_desc_sw128(k_addr + k * 32), idesc_s, k);
          else
            sm100::mma_bf16_w(tmem + kSCol, sm100::umma_desc_sw128(q_addr + k * 32),
                              sm100::umma_desc_sw128(k_addr + k * 32), idesc_s, k);
        }
        sm100::mma_commit_w(&s.s_full);
      };
      auto issue_o = [&]() {
        sm100::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if constexpr (TS) {  // P bf16 over S's first 64 columns, O in its last 64
            sm100::mma_bf16_ts_w(tmem + kSCol + 64, tmem + kSCol + kk * 8,
                                 sm100::umma_desc_sw128(v_addr + kk * 2048), idesc_o, kk);
          } else {
            const uint32_t pa = ((kk >> 2) ? k_addr : q_addr) + (kk & 3) * 32;
            sm100::mma_bf16_w(tmem + kSCol, sm100::umma_desc_sw128(pa),
                              sm100::umma_desc_sw128(v_addr + kk * 2048), idesc_o, kk);
          }
        }
        sm100::mma_commit_w(&s.o_full);
      };
      // S(j) / O(j) "events": S(j) once Q/K/V(j) are staged (qkv_ready), O(j)
      // once P(j) is (p_ready). The epilogue produces them strictly in order
      // S(0) O(0) S(1) O(1) ..., so one counter `ev` (= 2 j + is_o) tracks the
      // next; the issuer polls it between projection k-blocks and only blocks
      // on the accumulator (drain of item it - 2), never on attention.
      // (dbg 1-10, 12, 13: projection only)
      int ev = (dbg >= 1 && dbg <= 10) || dbg == 12 || dbg == 13 ? 2 * n_my : 0;
      // PAIR + pair_sync: the two CTAs issue each S / O event together (each
      // arrives on both CTAs' ev_pair once its own inputs are staged), so
      // their cta_group::1 attention MMAs overlap instead of stalling the
      // pair projection twice
      bool armed = false;
      auto try_event = [&]() {
        if (ev >= 2 * n_my) return;
        const int j = ev >> 1;
        uint64_t* bar = (ev & 1) ? &s.p_ready : &s.qkv_ready;
        if (PAIR && pair_sync) {
          if (!armed) {
            if (!__shfl_sync(0xffffffffu, sm100::mbar_test(bar, j & 1), 0)) return;
            if (lane == 0) {
              sm100::mbar_arrive(&s.ev_pair);
              sm100::mbar_arrive_remote(sm100::mapa(sm100::smem_u32(&s.ev_pair), rank ^ 1u));
            }
            __syncwarp();
            armed = true;
          }
          if (!__shfl_sync(0xffffffffu, sm100::mbar_test(&s.ev_pair, ev & 1), 0)) return;
          armed = false;
        } else if (!__shfl_sync(0xffffffffu, sm100::mbar_test(bar, j & 1), 0)) {
          return;
        }
        if (ev & 1) {
          if (lane == 0) stamp(dbg, ctx, j, 7);
          issue_o();
        } else {
          issue_s(j);
        }
        ++ev;
      };
      // accumulator it & 1 free: item it - 2 drained (and, TS, its S -- which
      // reads Q from that accumulator -- issued)
      auto acc_wait = [&](int it) {
        if (dbg != 10)
          while (!__shfl_sync(0xffffffffu,
                              sm100::mbar_test(&s.acc_empty[it & 1], ((it >> 1) & 1) ^ 1), 0) ||
                 (TS && it >= 2 && ev <= 2 * (it - 2)))
            try_event();
        sm100::tc_fence_after();
      };
      for (int it = 0; it < (leader ? n_my : 0); ++it) {  // PAIR: the leader projects for both
        acc_wait(it);
        if (lane == 0) stamp(dbg, ctx, it, 8);
        for (int kb = 0; kb < k_blocks; ++kb) {
          gemm_kb(it, kb);
          if (lane == 0 && (kb == 0 || kb == k_blocks - 1)) stamp(dbg, ctx, it, kb == 0 ? 9 : 10);
          try_event();
        }
      }
      while (ev < 2 * n_my) try_event();
    }
    __syncwarp();
  } else {
    // ---------------- epilogue / softmax (warps 2-9) ----------------
    const int quarter = warp & 3;       // TMEM lane quarter this warp may access
    const int hf = (warp - 2) >> 2;     // column half
    const int r = quarter * 32 + lane;  // token row of the item
    const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
    constexpr float kLog2e = 1.4426950408889634f;
    int aff_seq = -1;           // sequence the cached row affine belongs to
    float rs_a = 1.f, rs_b = 0.f;
    for (int it = 0; it < (dbg == 10 ? 0 : n_my); ++it) {
      int seq, h;
      item_of(it, seq, h);
      const uint32_t par = it & 1;
      const int a = it & 1;
      // deferred LayerNorm of the input row (folded: x' = rs_a x + rs_b per
      // row, gamma inside the weights, W.beta inside the bias)
      if (FOLD && seq != aff_seq && seq < n_seq) {
        row_affine(stats_in + ((size_t)seq * kS + r) * n_part, n_part, eps, rs_a, rs_b);
        aff_seq = seq;
      }
      // (1) acc + bias -> bf16 Q/K/V tiles. Chunk c (32 columns) of the 192:
      // part t = c/2 (Q, K, V), columns (c&1)*32.. of that part.
      sm100::mbar_wait(&s.acc_full[a], (it >> 1) & 1);
      sm100::tc_fence_after();
      const bool tl = warp == 2 && lane == 0;
      if (tl) stamp(dbg, ctx, it, 0);
      // accumulator a drained: PAIR -> one arrive per warp on the leader's barrier
      auto release_acc = [&]() {
        sm100::tc_fence_before();
        if constexpr (PAIR) {
          __syncwarp();
          if (lane == 0)
            sm100::mbar_arrive_remote(sm100::mapa(sm100::smem_u32(&s.acc_empty[a]), 0));
        } else {
          sm100::mbar_arrive(&s.acc_empty[a]);
        }
      };
      if (dbg == 1 || (dbg >= 3 && dbg <= 10) || dbg == 12) {
        release_acc();
        continue;
      }
      uint32_t qp[32];  // TS: this row's Q in bf16 pairs (hf == 0 threads)
#pragma unroll 1
      for (int cc = 0; cc < 3; ++cc) {
        const int c = hf * 3 + cc;
        // accumulator chunk c (32 columns) -> (part t, 32-column half c32):
        // TS loads 6 boxes (Q0 Q1 K0 K1 V0 V1), otherwise one 3-part box per
        // CTA (Q0 K0 V0 Q1 K1 V1 for 2 sequences per cluster)
        constexpr bool kOneBox = !TS && CS == 2;
        const int t = kOneBox ? c % 3 : (c >> 1);
        const int c32 = kOneBox ? c / 3 : (c & 1);
        uint32_t raw[32];
        sm100::tmem_ld_32x32b_x32(lane_base + (uint32_t)a * kAccCols + c * 32, raw);
        sm100::tmem_ld_wait();
        const float* bp = b_qkv + t * hidden + h * 64 + c32 * 32;
        const float* cp = c_qkv + t * hidden + h * 64 + c32 * 32;
        const float scale = t == 0 ? 0.125f : 1.0f;
        uint8_t* rowp = s.qkv[t] + r * 128;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 b0 = __ldg(reinterpret_cast<const float4*>(bp + q4 * 8));
          const float4 b1 = __ldg(reinterpret_cast<const float4*>(bp + q4 * 8 + 4));
          float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
          if (FOLD) {
            const float4 c0 = __ldg(reinterpret_cast<const float4*>(cp + q4 * 8));
            const float4 c1 = __ldg(reinterpret_cast<const float4*>(cp + q4 * 8 + 4));
            const float cc[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
            for (int e = 0; e < 8; ++e) bb[e] = fmaf(rs_b, cc[e], bb[e]);
          }
          float v[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = fmaf(rs_a, __uint_as_float(raw[q4 * 8 + e]), bb[e]) * scale;
          uint4 u;
          u.x = pack_bf16(v[0], v[1]);
          u.y = pack_bf16(v[2], v[3]);
          u.z = pack_bf16(v[4], v[5]);
          u.w = pack_bf16(v[6], v[7]);
          const int piece = c32 * 4 + q4;
          if (TS && t == 0) {
            // (unrolled: cc is 0 or 1 here, so the indices are compile-time per branch)
            if (c32 == 0) {
              qp[q4 * 4 + 0] = u.x; qp[q4 * 4 + 1] = u.y; qp[q4 * 4 + 2] = u.z; qp[q4 * 4 + 3] = u.w;
            } else {
              qp[16 + q4 * 4 + 0] = u.x; qp[16 + q4 * 4 + 1] = u.y;
              qp[16 + q4 * 4 + 2] = u.z; qp[16 + q4 * 4 + 3] = u.w;
            }
          } else {
            *reinterpret_cast<uint4*>(rowp + ((piece ^ (r & 7)) << 4)) = u;
          }
        }
      }
      if (TS && hf == 0) {
        // Q (bf16, 64 per row = 32 columns) over the consumed Q accumulator
        sm100::tmem_st_32x32b_x32(lane_base + (uint32_t)a * kAccCols, qp);
        sm100::tmem_st_wait();
      }
      release_acc();
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive(&s.qkv_ready);
      if (tl) stamp(dbg, ctx, it, 1);
      if (dbg == 2 || dbg == 13) continue;
      // (2) softmax over this thread's 64 keys [64 hf, 64 hf + 64)
      sm100::mbar_wait(&s.s_full, par);
      sm100::tc_fence_after();
      if (tl) stamp(dbg, ctx, it, 2);
      uint32_t sv[2][32];
      sm100::tmem_ld_32x32b_x32(lane_base + kSCol + hf * 64, sv[0]);
      sm100::tmem_ld_32x32b_x32(lane_base + kSCol + hf * 64 + 32, sv[1]);
      sm100::tmem_ld_wait();
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < 32; ++e)
        mx = fmaxf(mx, fmaxf(__uint_as_float(sv[0][e]), __uint_as_float(sv[1][e])));
      s.red_max[hf][r] = mx;
      epi_sync();
      mx = fmaxf(mx, s.red_max[hf ^ 1][r]);
      const float mxl = mx * kLog2e;
      float sum = 0.f;
      uint8_t* prow = s.qkv[hf] + r * 128;  // P keys [64 hf, +64) over the Q (hf 0) / K tile
      uint32_t pp[32];  // TS: P in bf16 pairs, to TMEM over S (all S reads are done: epi_sync)
      // x = s log2e - m as FFMA2 pairs; kPolyPairs of every 4 pairs take the
      // FMA-pipe exp2 (sm100::exp2_poly2_bf16) instead of MUFU
      const uint64_t l2e2 = sm100::f2_pack(kLog2e, kLog2e), negm2 = sm100::f2_pack(-mxl, -mxl);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        __align__(16) __nv_bfloat162 pv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t* src = &sv[q >> 2][(q & 3) * 8 + 2 * e];
          const uint64_t x = sm100::f2_fma(
              sm100::f2_pack(__uint_as_float(src[0]), __uint_as_float(src[1])), l2e2, negm2);
          if (e < kPolyPairs) {
            const uint32_t u = sm100::exp2_poly2_bf16(x);
            pv[e] = *reinterpret_cast<const __nv_bfloat162*>(&u);
          } else {
            float x0, x1;
            sm100::f2_unpack(x, x0, x1);
            pv[e] = __floats2bfloat162_rn(sm100::ex2_approx(x0), sm100::ex2_approx(x1));
          }
          const float2 back = __bfloat1622float2(pv[e]);
          sum += back.x + back.y;
        }
        if (TS) {
#pragma unroll
          for (int e = 0; e < 4; ++e) pp[q * 4 + e] = *reinterpret_cast<uint32_t*>(&pv[e]);
        } else {
          *reinterpret_cast<uint4*>(prow + ((q ^ (r & 7)) << 4)) = *reinterpret_cast<uint4*>(pv);
        }
      }
      if (TS) {
        sm100::tmem_st_32x32b_x32(lane_base + kSCol + hf * 32, pp);
        sm100::tmem_st_wait();
      }
      s.red_sum[hf][r] = sum;
      sm100::fence_proxy_async_smem();
      sm100::tc_fence_before();
      sm100::mbar_arrive(&s.p_ready);
      if (tl) stamp(dbg, ctx, it, 3);
      // (3) O / rowsum -> ctx, this thread's 32 of the head's 64 features
      sm100::mbar_wait(&s.o_full, par);
      sm100::tc_fence_after();
      if (tl) stamp(dbg, ctx, it, 4);
      uint32_t ov[32];
      sm100::tmem_ld_32x32b_x32(lane_base + kSCol + (TS ? 64 : 0) + hf * 32, ov);
      sm100::tmem_ld_wait();
      epi_sync();
      const float inv = 1.0f / (sum + s.red_sum[hf ^ 1][r]);
      if (seq < n_seq && dbg < 11) {  // the last sequence group may be padded
        __nv_bfloat16* dst = ctx + ((size_t)seq * kS + r) * hidden + h * 64 + hf * 32;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          uint4 u;
          u.x = pack_bf16(__uint_as_float(ov[q4 * 8 + 0]) * inv, __uint_as_float(ov[q4 * 8 + 1]) * inv);
          u.y = pack_bf16(__uint_as_float(ov[q4 * 8 + 2]) * inv, __uint_as_float(ov[q4 * 8 + 3]) * inv);
          u.z = pack_bf16(__uint_as_float(ov[q4 * 8 + 4]) * inv, __uint_as_float(ov[q4 * 8 + 5]) * inv);
          u.w = pack_bf16(__uint_as_float(ov[q4 * 8 + 6]) * inv, __uint_as_float(ov[q4 * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(dst + q4 * 8) = u;
        }
      }
      if (tl) stamp(dbg, ctx, it, 5);
    }
  }
  sm100::tc_fence_before();
  // no CTA may leave while a sharer can still multicast into it or arrive on
  // its barriers
  sm100::cluster_sync();
  if (warp == 1) {
    sm100::tc_fence_after();
    if constexpr (PAIR)
      sm100::tmem_dealloc_cg2<512>(tmem);
    else
      sm100::tmem_dealloc<512>(tmem);
  }
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

}  // namespace qa

// Diagnostic overrides (measurement only): CHM_QA_DEBUG=1 projection alone,
// 2 + Q/K/V staging, 11 per-item timeline (see stamp()), 12 / 13 timeline of 1 / 2; CHM_QA_CLUSTER = "<CS><CH>"; CHM_QA_LAG = issue lag.
static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

template <int CS, int CH, bool FOLD, bool TS = false, bool PAIR = false>
static chm_status launch(const void* x, const void* w_qkv, const float* b_qkv,
                         const float* c_qkv, const float2* stats_in, int n_part, float eps,
                         void* ctx, int n_seq, int hidden, int lag, int dbg, cudaStream_t st,
                         const int32_t* n_live = nullptr) {
  // CHM_QA_ORDER: 0 interleaved, 1 contiguous (measurement override)
  static const int order_env = env_int("CHM_QA_ORDER", -1);
  // CHM_QA_PAIR_SYNC: issue the two CTAs' attention MMAs together (PAIR)
  static const int pair_sync = env_int("CHM_QA_PAIR_SYNC", 0);  // measured: no gain
  const int order = order_env >= 0 ? order_env : 0;
  const int n_heads = hidden / 64;
  if (n_heads % CH != 0) return CHM_ERR_UNSUPPORTED;
  constexpr int kCluster = CS * CH;
  const long long T = (long long)n_seq * qa::kS;
  CUtensorMap tm_x, tm_w;
  if (!gemm::make_tmap_bf16(&tm_x, x, (uint64_t)T, (uint64_t)hidden, qa::kS / CH, 64, 0))
    return CHM_ERR_CUDA;
  if (TS || CS != 2) {
    if (!gemm::make_tmap_bf16(&tm_w, w_qkv, (uint64_t)3 * hidden, (uint64_t)hidden, qa::kWBox, 64,
                              0))
      return CHM_ERR_CUDA;
  } else if (!gemm::make_tmap_qkv3(&tm_w, w_qkv, (uint64_t)hidden, 64 / CS)) {
    return CHM_ERR_CUDA;
  }
  auto kern = qa::qkv_attention_kernel<CS, CH, FOLD, TS, PAIR>;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(qa::kThreads, 1, 1);
  cfg.dynamicSmemBytes = qa::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_clusters = 0;
  if (!max_clusters) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qa::kSmemBytes);
    cfg.gridDim = dim3(kCluster * (qa::n_sms() / kCluster), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1)
      n = qa::n_sms() / kCluster;
    max_clusters = n;
  }
  const int citems = ((n_seq + CS - 1) / CS) * (n_heads / CH);
  const int n_cl = citems < max_clusters ? citems : max_clusters;
  cfg.gridDim = dim3(kCluster * n_cl, 1, 1);
  prof::begin(prof::K_QKV_ATTENTION, st);
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tm_x, tm_w, b_qkv, c_qkv, stats_in, n_part, eps,
                                     n_seq, n_heads, hidden,
                                     reinterpret_cast<__nv_bfloat16*>(ctx), lag, dbg, order,
                                     n_live, pair_sync);
  // tensor work: the projection (2 T 3H H) + S and O (4 S^2 64 per item)
  prof::end(prof::K_QKV_ATTENTION, st,
            2.0 * T * 3.0 * hidden * hidden + 4.0 * qa::kS * qa::kS * 64.0 * n_seq * n_heads);
  if (e != cudaSuccess) return CHM_ERR_CUDA;
  CHM_LAUNCH_CHECK();
  return CHM_OK;
}

// ctx = attention(x' . w_qkv^T + b_qkv) for n_seq sequences of 128 tokens,
// x' = x, or with stats_in the deferred LayerNorm of x folded in (w_qkv
// pre-scaled by gamma, b_qkv including W.beta, c_qkv = row sums of w_qkv).
chm_status qkv_attention_pair(const void* x, const void* w_qkv, const float* b_qkv,
                              const float* c_qkv, const float2* stats_in, int n_part, float eps,
                              void* ctx, int n_seq, int hidden, cudaStream_t st);

chm_status qkv_attention_duo(const void* x, const void* w_qkv, const float* b_qkv,
                             const float* c_qkv, const float2* stats_in, int n_part, float eps,
                             void* ctx, int n_seq, int hidden, cudaStream_t st,
                             const int32_t* n_live);

chm_status qkv_attention(const void* x, const void* w_qkv, const float* b_qkv,
                         const float* c_qkv, const float2* stats_in, int n_part, float eps,
                         void* ctx, int n_seq, int hidden, cudaStream_t st,
                         const int32_t* n_live = nullptr) {
  if (stats_in && (!c_qkv || n_part < 1 || n_part > kLnMaxParts)) return CHM_ERR_INVALID_ARG;
  // CHM_QA_DUO (default 1): the two-epilogue-group kernel (qkv_attn_duo.cu);
  // 0 selects the kernels below (measurement / A-B)
  static const int duo = env_int("CHM_QA_DUO", 1);
  if (duo && !env_int("CHM_QA_DEBUG", 0))
    return qkv_attention_duo(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden,
                             st, n_live);
  // CHM_QA_PAIR=1: the cta_group::2 kernel (qkv_attn_pair.cu)
  // default: the pair-projection kernel (fused 1.69 vs 1.76 ms for the
  // cta_group::1 one, tools/experiments/qa_pair2.sh); CHM_QA_PAIR=0 selects
  // the cta_group::1 kernel, 1 the all-cta_group::2 experiment
  static const int pair = env_int("CHM_QA_PAIR", 2);
  // CHM_QA_PAIR_LAG: projection k-blocks the pair kernel keeps queued ahead of
  // S / O (0 = the operand ring's depth)
  static const int pair_lag = env_int("CHM_QA_PAIR_LAG", 0) < qa::kPairStages
                                  ? env_int("CHM_QA_PAIR_LAG", 0) : qa::kPairStages - 1;
  if (pair == 2)  // pair-projection variant of the fused kernel (cta_group::2 + ::1)
    return stats_in ? launch<2, 1, true, false, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part,
                                                      eps, ctx, n_seq, hidden, pair_lag, 0, st,
                                                      n_live)
                    : launch<2, 1, false, false, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part,
                                                       eps, ctx, n_seq, hidden, pair_lag,
                                                       env_int("CHM_QA_DEBUG", 0), st, n_live);
  if (pair)
    return qkv_attention_pair(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden,
                              st);
  static const int cluster = env_int("CHM_QA_CLUSTER", 21);
  // (the kdone ring has kStages slots: larger lags would alias its phases)
  static const int lag = env_int("CHM_QA_LAG", 0) < qa::kStages ? env_int("CHM_QA_LAG", 0)
                                                                  : qa::kStages - 1;
  static const int dbg = env_int("CHM_QA_DEBUG", 0);
  // CHM_QA_TS: Q / P operands from tensor memory (cluster config 21 only)
  static const int ts = env_int("CHM_QA_TS", 0);
  switch (cluster) {
    case 11: return stats_in ? launch<1, 1, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st) : launch<1, 1, false>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st);
    case 12: return stats_in ? launch<1, 2, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st) : launch<1, 2, false>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st);
    case 21:
      if (ts)
        return stats_in ? launch<2, 1, true, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st)
                        : launch<2, 1, false, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st);
      return stats_in ? launch<2, 1, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st) : launch<2, 1, false>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st);
    case 24: return stats_in ? launch<2, 4, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st) : launch<2, 4, false>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st);
    default: return stats_in ? launch<2, 2, true>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st) : launch<2, 2, false>(x, w_qkv, b_qkv, c_qkv, stats_in, n_part, eps, ctx, n_seq, hidden, lag, dbg, st);
  }
}

}  // namespace chm

extern "C" chm_status chm_qkv_attention_bf16(const void* x, const void* w_qkv,
                                             const float* b_qkv, void* ctx, int32_t n_seq,
                                             int32_t hidden, void* stream) {
  if (!x || !w_qkv || !b_qkv || !ctx || n_seq < 0) return CHM_ERR_INVALID_ARG;
  if (hidden <= 0 || hidden % 64 != 0) return CHM_ERR_INVALID_ARG;
  if (n_seq == 0) return CHM_OK;
  return chm::qkv_attention(x, w_qkv, b_qkv, nullptr, nullptr, 0, 0.f, ctx, n_seq, hidden,
                            (cudaStream_t)stream);
}
