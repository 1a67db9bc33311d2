/*
 * chimera_b200.h -- C-ABI of libchimera_sm100a.so, the B200 (sm_100a) per-tick
 * scheduling hot path of Chimera (arxiv 2603.22206).
 *
 * Every entry point is stream-ordered and asynchronous: it enqueues kernels on
 * `stream` and returns. Device buffers are plain pointers owned by the caller
 * (the Python host layer allocates them as torch tensors); the library owns no
 * device memory. Nothing in these signatures is a C++ or torch type.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/pkg/src/hetsched):
 *   chm_prepare_rows       balancer.py:100-103   (assignment lookup `monitor.assignment`)
 *   chm_encoder_forward    router.py:39-42       (Router.score -> ConfidenceVector)
 *   chm_trace_*            workload.py:125-253, 454-495 (TraceRecord columns,
 *                          remaining_tokens, first/next_stage_request)
 *   chm_kendall_tau_*      predictor.py:132-251 (kendall_tau_distance,
 *                          evaluate_predictor, arrival_order_distance)
 *   chm_predict_*          predictor.py:22-27    (Predictor.predict) and the concrete
 *                          predictors at predictor.py:30-45, 65-108
 *   chm_schedule_rows      balancer.py:89-129    (schedule_request = Alg. 1), with
 *                          estimate_load 49-60, select_model 63-77,
 *                          monitor.py:55-63 (assign), 86-96 (record_dispatch),
 *                          122-129 (in_flight_sum), engine.py:145-158 (enqueue)
 *   chm_queue_tick         engine.py:309-374     (EngineSim._push/_pop_min/_iterate/
 *                          _age_queued, QueueEntry.sort_key 55-69)
 *
 * Errors: functions return chm_status. Conditions the reference raises as
 * exceptions inside a batch are detected on the device and reported in a
 * caller-provided int32[4] error word {code, row, model, aux}; the host maps
 * the code to the same hetsched.errors class (see paper_2603_22206_b200/errors.py).
 */
#ifndef CHIMERA_B200_H
#define CHIMERA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CHM_MAX_MODELS 8
#define CHM_MAX_STAGES 32

typedef enum chm_status {
  CHM_OK = 0,
  CHM_ERR_INVALID_ARG = 1,          /* bad sizes / null pointers (host-side check) */
  CHM_ERR_VALIDATION = 2,           /* errors.ValidationError: score outside [0,1]
                                       (router.py:27-28) or out_tokens < 0
                                       (engine.py:285-286) */
  CHM_ERR_NEGATIVE_PREDICTION = 3,  /* ValueError (monitor.py:89-90) */
  CHM_ERR_DUPLICATE_REQUEST = 4,    /* errors.DuplicateRequest (monitor.py:91-94) */
  CHM_ERR_TIME_BACKWARDS = 5,       /* ValueError (engine.py:140-143) */
  CHM_ERR_NAN_PREDICTION = 6,       /* NaN predicted tokens: rejected (reference
                                       behaviour is heap-order dependent) */
  CHM_ERR_INVALID_STATE = 7,        /* device state violates an engine invariant */
  CHM_ERR_CAPACITY = 8,             /* a queue segment exceeds its capacity */
  CHM_ERR_UNSUPPORTED = 9,          /* option not implemented on device */
  CHM_ERR_CUDA = 10,                /* CUDA launch / runtime failure */
  CHM_ERR_UNKNOWN_REQUEST = 11,     /* errors.UnknownRequest (monitor.py:104-105) */
  CHM_ERR_UNKNOWN_STAGE = 12,       /* errors.UnknownStage (workload.py:143-147) */
  CHM_ERR_NCCL = 13                 /* NCCL missing (libnccl.so.2) or a NCCL call failed */
} chm_status;

/* ---- static configuration ------------------------------------------------ */

/* Pool (profiles.py:17-71). Index order MUST be sorted(model_id), the
 * tie-break order everywhere in the reference (profiles.py:56-59). */
typedef struct chm_pool {
  int32_t n_models;
  int32_t max_batch_size[CHM_MAX_MODELS];
  double decode_ms_per_token[CHM_MAX_MODELS];
} chm_pool;

/* BalancerConfig (balancer.py:26-37) + the tie band reported per decision:
 * a routed decision is flagged when its confidence gate or its descending-q
 * choice compares two scores within tie_tolerance (chm_decisions.flags bits
 * 3/4). With the north star's router tolerance eps = 1e-2 on each score, a
 * band of 2*eps holds every decision a router error could flip. */
typedef struct chm_balancer_cfg {
  double latency_slack;
  double confidence_margin;
  double tie_tolerance;
} chm_balancer_cfg;

/* AgingConfig (engine.py:36-52). enabled=0 <=> starvation_threshold = inf. */
typedef struct chm_aging_cfg {
  int32_t enabled;
  int32_t starvation_threshold;
  int32_t running_quantum;
  int32_t demote_while_queued;
} chm_aging_cfg;

/* ---- activity monitor + per-engine counters (device state) --------------- */

typedef struct chm_monitor_state {
  int32_t n_programs;
  double* inflight_sum;      /* [K] Neumaier running sum of live predictions   */
  double* inflight_comp;     /* [K] Neumaier compensation term                 */
  int64_t* inflight_count;   /* [K] live in-flight entries                     */
  int8_t* assignment;        /* [n_programs] model index, -1 = unassigned      */
  uint32_t* stage_bits;      /* [n_programs] bit (stage-1) set while in flight */
  uint64_t* batch_stamp;     /* [n_programs] scratch, init 0xff.. (repeat detection) */
  double* engine_clock;      /* [K] EngineSim.now                              */
  int64_t* engine_seq;       /* [K] next QueueEntry.seq                        */
  int32_t* engine_running;   /* [K] len(EngineSim.running)                     */
  int32_t* engine_queued;    /* [K] len(EngineSim._queued)                     */
  int64_t* engine_iterations;/* [K] EngineSim.iterations                       */
  /* Optional live in-flight log (ActivityMonitor._in_flight, monitor.py:43-48,
   * 86-106): per model, the live entries in insertion order, [K * cap] each;
   * inflight_count[m] entries are live. Needed by chm_monitor_complete; NULL
   * keys disable it. key = program * 32 + (stage - 1) for dispatched rows
   * (negative keys: entries seeded by the caller). */
  int32_t inflight_capacity;
  int64_t* inflight_key;
  double* inflight_yhat;
  /* ActivityMonitor(decay_in_flight=True) (monitor.py:40-42, 108-129): the
   * tokens each live request has already emitted, parallel to the log
   * (0 on dispatch, set by chm_monitor_note_progress); the in-flight sum is
   * then the Neumaier sum of max(yhat - progress, 0) in insertion order.
   * NULL = decay off (the reference default). */
  double* inflight_progress;
  /* Request-sharded runs (optional, NULL = off): a global insertion stamp per
   * live entry, parallel to the log. chm_schedule_rows stamps row i with
   * *stamp_base + i (the host sets stamp_base = tick << 40 | rank << 32 each
   * tick), so the ranks' logs merge into the reference's one insertion order
   * (chm_inflight_merge_sum). */
  int64_t* inflight_stamp;
  const int64_t* stamp_base;
} chm_monitor_state;

/* ---- one batch of requests, in arrival order ----------------------------- */

typedef struct chm_rows {
  int32_t n_rows;
  const int32_t* program;    /* [B] dense program index                        */
  const int32_t* stage;      /* [B] 1-based stage index                        */
  const double* arrival;     /* [B] Request.arrival_time (ms)                  */
  const int32_t* out_tokens; /* [B*K] rec.out_tokens(stage, m) per model       */
  const int64_t* handle;     /* [B] opaque request handle stored in the queue  */
  const int32_t* input_tokens; /* [B] Request.input_tokens (prefill time; only
                                  read by the engine clock, may be NULL)       */
} chm_rows;

/* Scratch produced by chm_prepare_rows and consumed by chm_schedule_rows. */
typedef struct chm_row_scratch {
  int32_t* first_row;        /* [B] first row of the same program in the batch */
  int8_t* pre_model;         /* [B] assignment before the batch (-1 none)      */
  int32_t* route_rows;       /* [B] compacted rows that need the router        */
  int32_t* n_route;          /* [1]                                            */
  uint64_t* qual;            /* [B] per-row gate sets, byte f = models clearing
                                q_f + margin, as descending-q rank bits        */
  uint32_t* rank;            /* [B] per-row packed descending-q rank (4b/model)*/
  uint32_t* flags;           /* [B] per-row precomputed flags                  */
  double* lnew;              /* [B] load of the chosen engine after the row's
                                dispatch (estimated_loads are rebuilt from it) */
} chm_row_scratch;

typedef struct chm_decisions {
  int32_t* model;            /* [B] Decision.model (index)                     */
  double* priority;          /* [B] Decision.priority                          */
  uint8_t* flags;            /* [B] bit0 used_cached_assignment, bit1 admitted
                                    on enqueue, bit2 queued                    */
  int64_t* seq;              /* [B] QueueEntry.seq on the chosen engine        */
  double* loads;             /* [B*K] Decision.estimated_loads (NULL = skip)   */
  int32_t* n_committed;      /* [1] rows fully applied                         */
  int32_t* error;            /* [4] {code,row,model,aux}                       */
  int32_t* tie_counts;       /* [3] out (may be NULL): routed rows of this batch
                                with bit3, with bit4, with either              */
} chm_decisions;

/* ---- STJF + aging engine queues (device state, SoA, seq order) ----------- */

typedef struct chm_queue_state {
  int32_t capacity;          /* entries per engine segment                     */
  double* priority;          /* [K*cap] QueueEntry.priority                    */
  double* arrival;           /* [K*cap] QueueEntry.arrival                     */
  int64_t* seq;              /* [K*cap] QueueEntry.seq                         */
  int64_t* handle;           /* [K*cap]                                        */
  int32_t* out_tokens;       /* [K*cap]                                        */
  int32_t* level;            /* [K*cap] starvation_level                       */
  int32_t* count;            /* [K*cap] starvation_count                       */
  int32_t* quantum;          /* [K*cap] quantum_counter                        */
  int32_t* order;            /* [K*cap] out: STJF order of the remaining queue */
  int64_t* admitted;         /* [K*cap] out: handles admitted this call, in order */
  int32_t* n_admitted;       /* [K] out                                        */
  int32_t* n_promoted;       /* [K] out: promotions this call                  */
  uint8_t* arrival_unsorted; /* [K] out: arrival not monotone in seq           */
  void* scratch;             /* K * chm_queue_scratch_bytes(cap) bytes; required
                                when capacity > 10240 (sort keys then live in
                                L2/HBM instead of shared memory)               */
  const struct chm_engine_run* run; /* engine execution clock (NULL = off)    */
} chm_queue_state;

/* Engine execution clock (EngineSim running set,
 * engine.py:165-241): every admission (at enqueue, in an iteration, or after a
 * stint ends) starts a stint of out_tokens decode steps after a prefill of
 * prefill_ms_per_token * input_tokens; chm_engine_advance finishes stints in
 * (stint_end, seq) order up to a target time, running a scheduling iteration
 * at each end. Requires capacity <= 2^18 (not the grid-wide path); with it,
 * chm_queue_complete (external completions) and the merged admission are
 * CHM_ERR_UNSUPPORTED. */
typedef struct chm_engine_run {
  int32_t capacity;                      /* running entries per engine (>= b) */
  int32_t done_capacity;                 /* completion records per engine     */
  double prefill_ms_per_token[CHM_MAX_MODELS];
  int32_t* queue_input_tokens;           /* [K*queue cap] parallel to the queue */
  int64_t* handle;                       /* [K*cap] running set (unordered)   */
  int64_t* seq;                          /* [K*cap] QueueEntry.seq            */
  double* stint_end;                     /* [K*cap]                           */
  double* decode_start;                  /* [K*cap]                           */
  int32_t* stint_tokens;                 /* [K*cap]                           */
  int32_t* n;                            /* [K] live entries                  */
  int64_t* tokens_emitted;               /* [K] tokens_emitted_total          */
  int64_t* served;                       /* [K] requests_served               */
  int64_t* done_handle;                  /* [K*done cap] completions, in order */
  double* done_time;                     /* [K*done cap] Completion.time       */
  int32_t* n_done;                       /* [K] appended since the host zeroed */
} chm_engine_run;

/* One STJF candidate of an engine sub-queue, for the cross-GPU admission
 * merge: the reference sort key (QueueEntry.sort_key, engine.py:55-69) plus
 * the entry's handle. level == INT64_MAX marks "no candidate". */
typedef struct chm_queue_key {
  int64_t level;             /* starvation_level                               */
  double priority;
  double arrival;
  int64_t seq;               /* global per-engine enqueue counter              */
  int64_t handle;
} chm_queue_key;

/* Per-engine scratch bytes chm_queue_* need for a segment capacity: 0 up to
 * 10240 entries (keys in shared memory, one CTA per engine), 20/entry up to
 * 2^18 (keys in global memory, one CTA per engine), above that the
 * grid-wide path (radix passes over 4096-entry tiles, staging copy for the
 * compaction, plus the kept STJF key order of the incremental path and its
 * compaction halo): ~150/entry. The grid-wide path keeps state in this
 * scratch between calls: hand every call on a queue the same scratch. */
uint64_t chm_queue_scratch_bytes(int32_t capacity);

/* Diagnostic: grid-wide queue calls (capacity > 2^18) so far that ran
 * incrementally on the order the previous call kept (the queue unchanged
 * since, <= 8192 appended rows, <= 512 admissions); the others re-sort. */
uint64_t chm_queue_fast_calls(void);

/* ---- columnar trace store (TraceRecord, workload.py:111-253) ------------ */

/* Dense SoA columns of a trace: program p (dense index), 0-based stage s
 * (padded to max_stages), model m in pool order. The caller fills the input
 * columns (n_stages .. carried); chm_trace_derive fills the two derived ones. */
typedef struct chm_trace {
  int32_t n_programs, max_stages, n_models;
  const int32_t* n_stages;     /* [NP] number of stages                          */
  const int32_t* workflow;     /* [NP] predictor workflow index (-1: unknown)    */
  const double* user_arrival;  /* [NP] user_arrival_time_ms                      */
  const int32_t* base_input;   /* [NP*S] base_input_tokens                       */
  const int32_t* out_tokens;   /* [NP*S*K] out_tokens                            */
  const int32_t* carried;      /* [NP*S*K] carried_context_tokens                */
  int64_t* remaining;          /* [NP*S*K] derived: sum_{j>=s} out_tokens        */
  int64_t* carried_prefix;     /* [NP*S*K] derived: sum_{j<s} carried            */
} chm_trace;

/* ---- router encoder (BERT-style post-LN, CLS -> Linear(H,K) -> sigmoid) --- */

typedef struct chm_encoder_cfg {
  int32_t n_layers, hidden, n_heads, ffn, vocab, max_pos, n_models;
  float ln_eps;
  int32_t flags;  /* CHM_ENC_* */
} chm_encoder_cfg;

/* chm_encoder_cfg.flags: run the QKV projection and attention as two kernels
 * (QKV written to HBM) instead of the fused S = 128 kernel. Same numerics;
 * kept for A/B measurement and parity tests. */
#define CHM_ENC_UNFUSED_ATTENTION 1
/* chm_encoder_cfg.flags: normalise every post-LN sublayer inside its own GEMM
 * epilogue (rows owned by clusters of 2H/256 CTAs exchanging statistics over
 * DSMEM). This is the default; the flag is kept for explicitness. */
#define CHM_ENC_CLUSTER_LN 2
/* chm_encoder_cfg.flags: deferred LayerNorm (out-projection / FFN2 write the
 * pre-LN sum + row statistics on pair tiles; QKV and FFN1 fold the LayerNorm
 * into their epilogues). Same math; measured slower in the power-capped tick. */
#define CHM_ENC_DEFERRED_LN 4

/* bf16 weights, row-major [out_features, in_features] (nn.Linear layout). */
typedef struct chm_encoder_weights {
  const void* word_emb;      /* [vocab, H]  bf16 */
  const void* pos_emb;       /* [max_pos, H] bf16 */
  const void* type_emb;      /* [H] bf16 (token type 0) */
  const float* emb_ln_g; const float* emb_ln_b;           /* [H] */
  const void* const* w_qkv;  /* L x [3H, H] bf16 */
  const float* const* b_qkv; /* L x [3H] */
  const void* const* w_o;    /* L x [H, H] */
  const float* const* b_o;   /* L x [H] */
  const float* const* ln1_g; const float* const* ln1_b;   /* L x [H] */
  const void* const* w_1;    /* L x [F, H] */
  const float* const* b_1;   /* L x [F] */
  const void* const* w_2;    /* L x [H, F] */
  const float* const* b_2;   /* L x [H] */
  const float* const* ln2_g; const float* const* ln2_b;   /* L x [H] */
  const float* head_w;       /* [K, H] fp32 */
  const float* head_b;       /* [K] */
} chm_encoder_weights;

/* Activation workspace for up to `max_tokens` = B*S tokens (bf16 unless noted). */
typedef struct chm_encoder_workspace {
  int64_t max_tokens;
  void* x;                   /* [T, H]  residual stream                        */
  void* qkv;                 /* [T, 3H]                                        */
  void* ctx;                 /* [T, H]  attention output                       */
  void* tmp;                 /* [T, H]  pre-LN sum                             */
  void* ffn;                 /* [T, F]                                         */
  void* stats;               /* chm_encoder_stats_bytes(): deferred-LayerNorm row
                                statistics, (mean, M2) fp32 per 128 columns    */
  void* folded;              /* chm_encoder_folded_bytes(): LayerNorm-folded
                                QKV / FFN1 weights, written by
                                chm_encoder_fold_weights()                      */
} chm_encoder_workspace;

/* ---- entry points -------------------------------------------------------- */

const char* chm_version(void);
const char* chm_status_string(int32_t status);

/* Number of SMs and compute capability of `device` (for diagnostics). */
chm_status chm_device_info(int32_t device, int32_t* sm_count, int32_t* cc_major, int32_t* cc_minor);

/* Resolve, per row, the pre-batch assignment (balancer.py:100-103), the first
 * row of the same program inside the batch, and compact the rows that need
 * the router (first occurrence, no assignment). `epoch_counter` is a device
 * uint32 shared by every call on `mon->batch_stamp`; the kernel increments
 * it, so the call can be replayed from a CUDA graph. */
chm_status chm_prepare_rows(const chm_monitor_state* mon, const chm_rows* rows,
                            const chm_row_scratch* scratch, uint32_t* epoch_counter,
                            void* stream);

/* K5: EmpiricalQuantilePredictor (predictor.py:65-108) as a dense table with
 * the fallback chain resolved at build time: table[(wf*(S_cap+1) + st)*K + m],
 * wf in [0, n_wf] (n_wf = unseen workflow), st in [0, S_cap] (0 = unseen stage).
 * yhat[B*K] receives the prediction for every model. */
chm_status chm_predict_quantile(const double* table, int32_t n_wf, int32_t s_cap,
                                int32_t n_models, const int32_t* workflow,
                                const int32_t* stage, int32_t n_rows, double* yhat,
                                void* stream);
/* K5: OraclePredictor (predictor.py:30-36): suffix sum of stage outputs,
 * stage_out[(row*max_stages + j)*K + m], j 0-based. */
chm_status chm_predict_oracle(const int32_t* stage_out, const int32_t* n_stages,
                              const int32_t* stage, int32_t max_stages,
                              int32_t n_models, int32_t n_rows, double* yhat,
                              int32_t* error, void* stream);
/* K5: InputLengthPredictor (predictor.py:39-45). */
chm_status chm_predict_input_length(const int32_t* input_tokens, int32_t n_models,
                                    int32_t n_rows, double* yhat, void* stream);

/* K6: serial-exact fused monitor + load estimate + selection + dispatch for a
 * batch (B calls of schedule_request in row order). `scores` [B*K] must hold
 * router output for every routed row, in fp64 like the reference's
 * ConfidenceVector (router.py:21-31: Python floats); `yhat` [B*K] the
 * predictor output. */
chm_status chm_schedule_rows(const chm_pool* pool, const chm_balancer_cfg* cfg,
                             const chm_monitor_state* mon, const chm_rows* rows,
                             const chm_row_scratch* scratch, const double* scores,
                             const double* yhat, const chm_decisions* out,
                             void* stream);

/* Completion path (ActivityMonitor.record_completion, monitor.py:98-106): the
 * n requests (model[j], key[j]) finished; each is removed from model[j]'s
 * in-flight log (insertion order of the rest kept), its (program, stage)
 * in-flight bit cleared, and the model's Neumaier (sum, comp) recomputed over
 * the survivors exactly as builtin sum() would. n_complete[m] (optional, [K])
 * receives the per-model counts, ready for chm_queue_complete. Device errors:
 * UNKNOWN_REQUEST (not in flight on that model), VALIDATION (model index). */
chm_status chm_monitor_complete(const chm_pool* pool, const chm_monitor_state* mon,
                                const int32_t* model, const int64_t* key, int32_t n,
                                int32_t* n_complete, int32_t* error, void* stream);

/* K7 phase A: `n_complete[m]` running requests of engine m finish at `now`;
 * each frees a slot and runs one scheduling iteration (engine.py:232-241,
 * 328-338): admit the queue minimum, then age every queued entry. */
chm_status chm_queue_complete(const chm_pool* pool, const chm_aging_cfg* aging,
                              const chm_monitor_state* mon, const chm_queue_state* q,
                              const int32_t* n_complete, int32_t* error,
                              void* stream);

/* K7 phase B: append the rows chm_schedule_rows marked `queued`, then run
 * `n_iterations` explicit scheduling iterations per engine (admit into free
 * slots, age the rest), and write the final STJF order of every queue. */
chm_status chm_queue_tick(const chm_pool* pool, const chm_aging_cfg* aging,
                          const chm_monitor_state* mon, const chm_queue_state* q,
                          const chm_rows* rows, const chm_decisions* dec,
                          int32_t n_iterations, int32_t* error, void* stream);

/* Sharded engine queues (global admission). With requests
 * sharded over G GPUs, engine m's single reference queue (EngineSim._heap,
 * engine.py:309-326) is split into G sub-queues whose union, ordered by the
 * global sort key, is the reference queue (seq is the global enqueue counter,
 * relayed between ranks). One scheduling iteration (engine.py:328-338) then
 * is:
 *   chm_queue_candidates    each rank writes its first F = max_batch_size
 *                           entries per engine in STJF order ([K*F] keys);
 *   (all-gather of the [G*K*F] keys over NCCL);
 *   chm_queue_admit_merged  every rank frees release[m] slots (release NULL:
 *                           none; release[m] < 0: engine m skips this
 *                           iteration), takes the
 *                           global top min(free slots, candidates) of the
 *                           gathered keys, admits its own share of them from
 *                           its head (in order), adds the GLOBAL admitted
 *                           count to engine_running, ages the rest of its
 *                           sub-queue by one iteration and rewrites its order.
 * Requires capacity <= 2^18 (the huge path returns CHM_ERR_UNSUPPORTED). */
chm_status chm_queue_candidates(const chm_pool* pool, const chm_monitor_state* mon,
                                const chm_queue_state* q, int32_t F, chm_queue_key* out,
                                void* stream);
chm_status chm_queue_admit_merged(const chm_pool* pool, const chm_aging_cfg* aging,
                                  const chm_monitor_state* mon, const chm_queue_state* q,
                                  const chm_queue_key* gathered, int32_t G, int32_t F,
                                  int32_t rank, const int32_t* release, int32_t* error,
                                  void* stream);

/* EngineSim.advance_to(target[m]) for every engine (engine.py:174-183): finish
 * the running stints ending at or before the target in (stint_end, seq)
 * order; each frees its slot, is appended to the completion list and runs one
 * scheduling iteration at its end time (admissions start new stints, which
 * may end before the target too). The clock then moves to the target
 * (CHM_ERR_TIME_BACKWARDS if that is more than 1e-9 ms in the past). Needs
 * q->run. */
chm_status chm_engine_advance(const chm_pool* pool, const chm_aging_cfg* aging,
                              const chm_monitor_state* mon, const chm_queue_state* q,
                              const double* target, int32_t* error, void* stream);

/* ActivityMonitor.note_progress (monitor.py:108-111) for n (model index,
 * request key, emitted tokens) updates, in call order (a later update of the
 * same request wins); requests not in flight on that model are ignored, as in
 * the reference. Then the in-flight sums are recomputed with the decayed terms
 * (in_flight_sum, monitor.py:122-129): the snapshot the next
 * chm_schedule_rows starts from (simcore._sync_progress before a dispatch,
 * simcore.py:260-264, 278-279). Requires inflight_progress. */
chm_status chm_monitor_note_progress(const chm_pool* pool, const chm_monitor_state* mon,
                                     const int32_t* model, const int64_t* key,
                                     const double* emitted, int32_t n, int32_t* error,
                                     void* stream);

/* Trace store. chm_trace_derive: remaining (the suffix
 * sums TraceRecord.remaining_tokens returns, workload.py:160-165) and
 * carried_prefix (next_stage_request's carried context, workload.py:484-486),
 * validating n_stages in 1..max_stages, token counts >= 0 and base >= 1
 * (TraceRecord.validate, workload.py:170-200): CHM_ERR_VALIDATION, row =
 * program. HBM bound: 8 bytes read + 16 written per (program, stage, model). */
chm_status chm_trace_derive(const chm_trace* t, int32_t* error, void* stream);
/* Per batch row (program, 1-based stage): out_tokens[B*K]
 * (rec.out_tokens(stage, m), the EngineSim.enqueue argument), workflow[B],
 * n_stages[B], oracle_yhat[B*K] (OraclePredictor.predict, predictor.py:30-36).
 * Any output may be NULL. Stage outside 1..n_stages -> CHM_ERR_UNKNOWN_STAGE
 * (TraceRecord._stage, workload.py:143-147). */
chm_status chm_trace_gather_rows(const chm_trace* t, const int32_t* program,
                                 const int32_t* stage, int32_t n_rows, int32_t* out_tokens,
                                 int32_t* workflow, int32_t* n_stages, double* oracle_yhat,
                                 int32_t* error, void* stream);
/* next_stage_request (workload.py:467-495) for n completions (program,
 * completed stage, completion time, assigned model index): the requests of
 * programs with a next stage, compacted in input order into next_* (stage
 * s+1, arrival = completion time, input = base + carried prefix),
 * *n_next = their count, source_row = the completion each came from
 * (next_workflow / source_row may be NULL). Completed stage outside
 * 1..n_stages -> CHM_ERR_UNKNOWN_STAGE. */
chm_status chm_trace_next_stage(const chm_trace* t, const int32_t* program,
                                const int32_t* completed_stage, const double* completion_time,
                                const int8_t* model, int32_t n, int32_t* next_program,
                                int32_t* next_stage, double* next_arrival,
                                int32_t* next_input_tokens, int32_t* next_workflow,
                                int32_t* source_row, int32_t* n_next, int32_t* error,
                                void* stream);
/* first_stage_request (workload.py:454-464): input = base of stage 1,
 * arrival = arrival_in[i] or the program's user_arrival_time_ms (NULL). */
chm_status chm_trace_first_stage(const chm_trace* t, const int32_t* program,
                                 const double* arrival_in, int32_t n, int32_t* input_tokens,
                                 double* arrival, int32_t* workflow, int32_t* error,
                                 void* stream);

/* Predictor evaluation: kendall_tau_distance
 * (predictor.py:182-214) of n >= 2 (predicted, truth) pairs on the device --
 * merge-sort strict-inversion count after sorting by (predicted, truth), tied
 * pairs by binary search -- exact int64 counts, *result = (discordant + 0.5 *
 * half) / (n(n-1)/2) in fp64 like the reference. counts_out (may be NULL) =
 * {discordant, ties_predicted, ties_truth, ties_both}. Scratch:
 * chm_kendall_tau_scratch_bytes(n). NaN inputs are not supported (the
 * reference's sorted() order is undefined for them). */
uint64_t chm_kendall_tau_scratch_bytes(int64_t n);
chm_status chm_kendall_tau_distance(const double* predicted, const double* truth, int64_t n,
                                    void* scratch, uint64_t scratch_bytes, double* result,
                                    int64_t* counts_out, void* stream);

/* EmpiricalQuantilePredictor training (predictor.py:78-98) on the device:
 * the table chm_predict_quantile reads, [n_wf + 1, s_cap + 1, K] fp64, from
 * the derived `remaining` column of a training trace (chm_trace_derive) and a
 * per-program workflow index in 0..n_wf-1 (sorted workflow ids). Values per
 * group = remaining tokens of every training (program, stage, model); numpy's
 * 'linear' quantile with its exact arithmetic; the (workflow, stage, model)
 * -> (stage, model) -> (model) -> global fallback resolved into the table
 * (row n_wf: unseen workflow, column 0: stage outside 1..s_cap). n_entries =
 * sum of n_stages * K. Scratch: chm_quantile_train_scratch_bytes. */
uint64_t chm_quantile_train_scratch_bytes(int64_t n_entries, int32_t n_wf, int32_t s_cap,
                                          int32_t n_models);
chm_status chm_quantile_train(const chm_trace* t, const int32_t* workflow, int32_t n_wf,
                              int32_t s_cap, double quantile, int64_t n_entries, void* scratch,
                              uint64_t scratch_bytes, double* table, void* stream);

/* Deferred LayerNorm. The encoder does not normalise a sublayer output where
 * it is produced: out-projection and FFN2 write the pre-LN sum plus per-row
 * partial statistics, and the next projection folds the LayerNorm in
 * (LN(x).W^T + b = rstd (x.W'^T) - rstd mean c + b', W' = W diag(gamma),
 * c = W' row sums, b' = b + W beta). The folded QKV / FFN1 weights live in
 * the workspace; chm_encoder_fold_weights() (re)computes them and must run
 * after the weights are loaded or changed, before chm_encoder_forward. */
uint64_t chm_encoder_folded_bytes(const chm_encoder_cfg* cfg);
uint64_t chm_encoder_stats_bytes(const chm_encoder_cfg* cfg, int64_t max_tokens);
chm_status chm_encoder_fold_weights(const chm_encoder_cfg* cfg, const chm_encoder_weights* w,
                                    const chm_encoder_workspace* ws, void* stream);

/* Router encoder forward over `n_seq` sequences of `seq_len` token ids, only
 * for the rows listed in `rows` (NULL = all, n_seq rows). Writes
 * q[rows[i]*K + m] = sigmoid(head(h_CLS)) as fp64 (the scheduler's score
 * buffer is fp64). */
chm_status chm_encoder_forward(const chm_encoder_cfg* cfg, const chm_encoder_weights* w,
                               const chm_encoder_workspace* ws, const int32_t* token_ids,
                               const int32_t* rows, const int32_t* n_rows_dev,
                               int32_t n_seq, int32_t seq_len, double* q_out,
                               void* stream);

/* Standalone tcgen05 GEMM: C[M,N] = A[M,K] . B[N,K]^T (+bias[N]) (+GELU)
 * (+residual[M,N]); bf16 in/out, fp32 accumulate. epilogue: 0 none, 1 bias,
 * 2 bias+gelu, 3 bias+residual. */
chm_status chm_gemm_bf16(const void* A, const void* B, void* C, const float* bias,
                         const void* residual, int32_t M, int32_t N, int32_t K,
                         int32_t epilogue, void* stream);

/* Fused post-LN sublayer: C = LayerNorm(A . B^T + bias + residual) * gamma + beta
 * (fp32 statistics over the full row of N = 256*g columns, g <= 4; rows are
 * spread over a cluster of 2g CTAs that exchange partial statistics through
 * distributed shared memory). C may alias residual (in-place update). */
chm_status chm_gemm_bf16_ln(const void* A, const void* B, void* C, const float* bias,
                            const void* residual, const float* gamma, const float* beta,
                            float eps, int32_t M, int32_t N, int32_t K, void* stream);

/* Deferred-LayerNorm GEMMs (the encoder's sublayers):
 *  epilogue 1 / 2 (bias / bias+GELU) with stats_in: C = [GELU](rstd (A.B^T)
 *      - rstd mean colsum + bias), i.e. the LayerNorm of A's rows folded in
 *      (B, colsum, bias from chm_encoder_fold_weights' rule);
 *  epilogue 6: C = A.B^T + bias + R, R = residual, or LN(residual) with
 *      gamma/beta when stats_in is given; writes stats_out[M][N/128].
 * stats_in = [M][n_part] (mean, M2) partials over 128 columns each. */
chm_status chm_gemm_bf16_deferred_ln(const void* A, const void* B, void* C, const float* bias,
                                     int32_t epilogue, const void* residual, const float* gamma,
                                     const float* beta, const void* stats_in, int32_t n_part,
                                     const float* colsum, void* stats_out, float eps, int32_t M,
                                     int32_t N, int32_t K, void* stream);

/* Encoder self-attention sublayer core (no mask, head dim 64), the kernel the
 * encoder runs between its QKV projection and out-projection:
 *   ctx[t, h*64:(h+1)*64] = softmax(Q_h K_h^T) V_h  per sequence,
 * qkv = [n_seq*seq_len, 3*hidden] bf16 with Q pre-scaled by 1/8, ctx =
 * [n_seq*seq_len, hidden] bf16. seq_len % 128 == 0, <= 512. */
chm_status chm_attention_bf16(const void* qkv, void* ctx, int32_t n_seq, int32_t seq_len,
                              int32_t hidden, void* stream);

/* Fused QKV projection + attention (S = 128 only): ctx as chm_attention_bf16
 * of qkv = x . w_qkv^T + b_qkv (Q columns scaled by 1/8), without writing qkv
 * to HBM. x = [n_seq*128, hidden] bf16, w_qkv = [3*hidden, hidden] bf16. */
chm_status chm_qkv_attention_bf16(const void* x, const void* w_qkv, const float* b_qkv,
                                  void* ctx, int32_t n_seq, int32_t hidden, void* stream);

/* Fused feed-forward sublayer for hidden = 256 (the small router):
 *   x <- LayerNorm(x + GELU(x . w1^T + b1) . w2^T + b2) * gamma + beta
 * in place, the [M, F] intermediate kept on chip. w1 = [F, 256], w2 = [256, F]
 * bf16, F % 128 == 0, 128 <= F <= 4096; replaces chm_gemm_bf16 (epilogue 2)
 * + chm_gemm_bf16_ln for the encoder's FFN (router.py:34-45's paper encoder). */
chm_status chm_ffn_fused_bf16(void* x, const void* w1, const float* b1, const void* w2,
                              const float* b2, const float* gamma, const float* beta, float eps,
                              int32_t M, int32_t hidden, int32_t ffn, void* stream);

/* Profiling: launch counters per kernel class (always on) and opt-in CUDA
 * event timing around every launch on its own stream. Classes: 0 GEMM,
 * 1 attention, 2 row-wise (embedding+LN, LayerNorm, head), 3 predictor,
 * 4 prepare, 5 select, 6 queue, 7 fused QKV+attention. chm_profile_read
 * synchronises on the recorded events, fills 8-entry arrays (timed launches, summed ms, summed algorithmic
 * work -- FLOPs or bytes --, cumulative launch counts) and clears the timings. */
chm_status chm_profile_enable(int32_t enable);
chm_status chm_profile_read(int32_t* timed, double* total_ms, double* work, int64_t* launches);

/* ---- multi-GPU: request shards exchange the in-flight vector --
 *
 * One process per GPU. Requests shard by program, so router, predictor,
 * assignment map, in-flight logs and engine sub-queues are rank-local; the
 * only cross-GPU state is the per-engine Neumaier pair (s, c) of P_m
 * (ActivityMonitor.in_flight_sum, monitor.py:122-129). NCCL is resolved at
 * run time (dlopen libnccl.so.2; CHM_NCCL_LIB overrides the path). The
 * canonical tick-end state of both modes is P_prev folded with rank 0's
 * dispatches in row order, then rank 1's, ... = the monitor of one serial
 * schedule_request loop (balancer.py:116) over the concatenated batch. */
#define CHM_COMM_ID_BYTES 128
typedef struct chm_comm chm_comm;

/* CHM_OK when libnccl could be loaded. */
chm_status chm_comm_available(void);
/* ncclGetUniqueId on one rank; the caller distributes the bytes. */
chm_status chm_comm_unique_id(uint8_t* id_out /* CHM_COMM_ID_BYTES */);
/* ncclCommInitRank on `device` (cudaSetDevice first; -1 = current). */
chm_status chm_comm_init(const uint8_t* id, int32_t rank, int32_t world, int32_t device,
                         chm_comm** out);
chm_status chm_comm_destroy(chm_comm* comm);
/* Plain collectives on the caller's stream (candidate gather of the merged
 * admission; the sharded-completion sums). */
chm_status chm_comm_allgather(chm_comm* comm, const void* send, void* recv, uint64_t bytes,
                              void* stream);
chm_status chm_comm_allreduce_i64(chm_comm* comm, int64_t* buf, int32_t n, void* stream);

/* Mode A tick end: every rank's chain started from the tick-start (s0, c0);
 * pack this rank's committed (model, yhat) rows, all-gather the records and
 * fold them in rank order into mon->inflight_sum / inflight_comp (an int64
 * sum when every value is a multiple of 2^-8 -- exact in any order -- else
 * the Neumaier recurrence on the device). workspace: (world + 1) *
 * chm_inflight_record_bytes(K, max_rows) bytes. The pack / fold halves are
 * exported for transports other than NCCL (the gloo tests). */
uint64_t chm_inflight_record_bytes(int32_t n_models, int32_t max_rows);
chm_status chm_inflight_pack(const chm_pool* pool, const chm_decisions* dec, int32_t max_rows,
                             void* record, void* stream);
chm_status chm_inflight_fold(const chm_pool* pool, const chm_monitor_state* mon,
                             const double* s0, const double* c0, const void* gathered,
                             int32_t world, int32_t max_rows, int32_t* error, void* stream);
chm_status chm_allreduce_inflight(chm_comm* comm, const chm_pool* pool,
                                  const chm_monitor_state* mon, const double* s0,
                                  const double* c0, const chm_decisions* dec, int32_t max_rows,
                                  void* workspace, int32_t* error, void* stream);

/* Mode B relay around the selection kernel only: rank g > 0 receives the
 * packed state (n doubles: (s, c) [+ relayed engine counters]) from g - 1
 * before chm_schedule_rows; after it, sends to g + 1 and the last rank
 * broadcasts the tick-end state. Routers / predictors are enqueued before
 * the receive, so they overlap the predecessors' chains. */
chm_status chm_inflight_relay_recv(chm_comm* comm, double* state, int32_t n, void* stream);
chm_status chm_inflight_relay_send(chm_comm* comm, double* state, int32_t n, void* stream);

/* Sharded completions (record_completion, monitor.py:98-106, on a log that
 * holds only this rank's dispatches): out[0..K) = exact sum of this rank's
 * live terms per engine in units of 2^-8, out[K] = number of non-dyadic
 * terms; all-reduce the K + 1 words (chm_comm_allreduce_i64), then
 * chm_inflight_set_sum installs (sum, 0) -- builtin sum() of the survivors
 * in any order -- or leaves the sums and reports UNSUPPORTED into `error`
 * (if non-NULL) when a survivor is not dyadic: then the merge path below. */
chm_status chm_inflight_local_sum(const chm_pool* pool, const chm_monitor_state* mon,
                                  int64_t* out, void* stream);
chm_status chm_inflight_set_sum(const chm_pool* pool, const chm_monitor_state* mon,
                                const int64_t* summed, int32_t* error, void* stream);
/* Sharded completions with non-dyadic survivors: every rank packs its live
 * (stamp, term) pairs per engine into [K][cap] records (16 B each; cap >=
 * every rank's live count), the records are all-gathered ([G][K][cap]), and
 * chm_inflight_merge_sum merges the G stamp-ordered lists per engine and
 * replays CPython's Neumaier recurrence over them: builtin sum() of the
 * survivors in the reference's insertion order, bit for bit. counts: the
 * gathered live counts [G][K]. Requires inflight_stamp. */
chm_status chm_inflight_pack_live(const chm_pool* pool, const chm_monitor_state* mon,
                                  int32_t cap, void* records, void* stream);
chm_status chm_inflight_merge_sum(const chm_pool* pool, const chm_monitor_state* mon,
                                  const void* gathered, const int64_t* counts, int32_t world,
                                  int32_t cap, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CHIMERA_B200_H */
