/*
 * cdx_c.h — C-ABI of the B200-native Certaindex hot path (libcdx.so).
 *
 * Plain pointers and sizes only; no C++ or torch types cross this boundary.  Every entry
 * point is the batched replacement of a scalar routine of the reference library
 * (proj/include/cdx/ headers, CPU, one program at a time); the comment above each one
 * cites the reference interface it replaces.  The reference has no scheduler code: the
 * scheduler rows restate SPEC.md:385-486.
 *
 * Conventions
 *   - All array arguments of the compute entry points are DEVICE pointers owned by the
 *     caller (cudaMalloc / torch tensors).  The cdx_*_host entry points take HOST
 *     pointers and stream them through the device themselves.
 *   - Calls are asynchronous on the context stream; cdx_sync() waits and reports
 *     device-side validation errors (e.g. a reward outside [0,1]).
 *   - Status codes map 1:1 onto the reference's exception types:
 *       CDX_EINVAL   <-> std::invalid_argument     CDX_ERUNTIME <-> std::runtime_error
 *       CDX_ERANGE   <-> std::out_of_range         CDX_ELOGIC   <-> std::logic_error
 *     cdx_last_error() returns the reference's message text for the failure.
 *   - There is no CPU fallback: without a usable sm_100 device every call returns
 *     CDX_ECUDA.
 */
#ifndef CDX_C_H
#define CDX_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CDX_ABI_VERSION 4

typedef enum {
    CDX_OK = 0,
    CDX_EINVAL = 1,
    CDX_ERUNTIME = 2,
    CDX_ERANGE = 3,
    CDX_ELOGIC = 4,
    CDX_ECUDA = 5,
    CDX_ENCCL = 6
} cdx_status;

/* metrics.hpp:85 SignalKind (same ordinals) */
enum { CDX_SIG_ENTROPY = 0, CDX_SIG_REWARD = 1, CDX_SIG_MEAN_LEN = 2, CDX_SIG_LOGPROB = 3 };
/* Batched-API extension (no SignalKind ordinal in the reference): the majority-fraction
 * certaindex of Self-Consistency = size of the plurality cluster / n, the share of the answer
 * weighted_plurality returns (runtime.cpp:317-334, unweighted).  Only cdx_sc_certaindex(_ex)
 * and the SC archetype of cdx_mixed_allocate accept thresholds on it.                       */
enum { CDX_SIG_MAJORITY = 4 };
/* metrics.hpp:105 ThresholdDir */
enum { CDX_DIR_GE = 0, CDX_DIR_LE = 1 };
/* metrics.hpp:72 RewardAggregation */
enum { CDX_AGG_MEAN = 0, CDX_AGG_MAX = 1 };
/* probe.hpp:52 ExitDecision; also the `reason` byte of the batched outputs */
enum { CDX_EXIT_CONTINUE = 0, CDX_EXIT_CERTAIN = 1, CDX_EXIT_BUDGET = 2 };
/* runtime.hpp:32 Archetype */
enum { CDX_ARCH_SC = 0, CDX_ARCH_REBASE = 1, CDX_ARCH_MCTS = 2, CDX_ARCH_COT = 3 };
/* SPEC.md:391 AllocationPolicy.kind */
enum {
    CDX_POL_EVEN = 0,
    CDX_POL_LENGTH_PROXY = 1,
    CDX_POL_STATIC_THRESHOLD = 2,
    CDX_POL_INITIAL_CURVE_FIT = 3,
    CDX_POL_K_STEP_THRESHOLD = 4,
    CDX_POL_DYNAMIC_CURVE_FIT = 5
};
/* SPEC.md:395 InterSchedPolicy.order */
enum { CDX_ORDER_FIFO = 0, CDX_ORDER_SJF = 1, CDX_ORDER_LPM = 2 };

/* metrics.hpp:107-112 SignalThreshold */
typedef struct {
    uint8_t signal; /* CDX_SIG_* */
    uint8_t dir;    /* CDX_DIR_* */
    uint8_t _pad[6];
    double cutoff;
} cdx_threshold;

/* SPEC.md:390-393 AllocationPolicy (batched subset: even / static / k-step threshold) */
typedef struct {
    uint8_t kind; /* CDX_POL_EVEN | CDX_POL_STATIC_THRESHOLD | CDX_POL_K_STEP_THRESHOLD */
    uint8_t _pad[3];
    int32_t detect_at;       /* detect_at_knob, 1-based knob unit (<= resource_cap) */
    int32_t recheck_every;   /* k_step_threshold: re-test every this many units (>= 1) */
    int32_t resource_cap;    /* knob units, <= probes per request */
    int64_t tokens_per_unit; /* token budget of one knob unit (interval_tokens * samples) */
} cdx_alloc_policy;

/* probe.hpp:25-33 ProbeConfig (markers travel separately, see cdx_canon_intern) */
typedef struct {
    int32_t interval_tokens;
    int32_t window;
    double threshold;
    int64_t max_tokens;
} cdx_probe_cfg;

/* SPEC.md:394-397 InterSchedPolicy */
typedef struct {
    uint8_t gang;  /* requests grouped by program (always 1 for the program-level order) */
    uint8_t order; /* CDX_ORDER_FIFO | CDX_ORDER_SJF */
    uint8_t _pad[6];
    double starvation_limit; /* > 0 */
    double prior_tokens;     /* estimate_iteration_tokens prior */
} cdx_inter_policy;

/* Per-program scheduler state, structure of arrays (device pointers).
 * runtime.hpp:123-133 ReasoningProgram + runtime.hpp:191-192 iteration_tokens(). */
typedef struct {
    const double* arrival;        /* program arrival time */
    const double* last_service;   /* last time the program was serviced */
    const int64_t* iter_tok_sum;  /* sum of completed iteration token counts */
    const uint32_t* iter_count;   /* number of completed iterations */
    const int32_t* knob;          /* units granted so far (ReasoningProgram::knob, int) */
    const int32_t* cap;           /* resource cap (ReasoningProgram::resource_cap, int) */
    const uint8_t* terminated;    /* nonzero: dropped from the order */
    const uint32_t* program_id;   /* nullable: program id = id_base + index (the last tie-break) */
    uint32_t id_base;
    uint32_t _pad;
} cdx_prog_soa;

/* Synthetic trace parameters (counter-based restatement of runtime.hpp:45-69 and
 * runtime.cpp:91-117).  Answer ids: 0 = the stationary
 * answer "S", 1..M-1 = distractors "D1".."D{M-1}", M+a = the hesitant form "wait, "+name(a). */
typedef struct {
    uint64_t seed;
    uint32_t groups;            /* M >= 2 */
    uint32_t conv_lo, conv_hi;  /* convergence knob ~ U{lo..hi} */
    uint32_t _pad;
    double noise_level;         /* before convergence */
    double residual_noise;      /* from convergence on */
    double solvable_fraction;
    double hesitation_prob;     /* CoT */
    uint32_t reward_start_k;    /* reward model means in units of 2^-24 */
    uint32_t reward_final_k;
    uint32_t reward_unsolvable_k;
    uint32_t reward_jitter_k;   /* uniform jitter half-width */
} cdx_gen_params;

typedef struct cdx_ctx cdx_ctx;

/* ---- context ----------------------------------------------------------------------- */
int cdx_ctx_create(int device, cdx_ctx** out);
int cdx_ctx_destroy(cdx_ctx* ctx);
/* Run subsequent calls on this cudaStream_t (NULL = the device's legacy default stream).
 * A new context runs on its own non-blocking stream; cdx_ctx_use_own_stream restores it. */
int cdx_ctx_set_stream(cdx_ctx* ctx, void* cuda_stream);
int cdx_ctx_use_own_stream(cdx_ctx* ctx);
void* cdx_ctx_stream(cdx_ctx* ctx);
int cdx_sync(cdx_ctx* ctx);
const char* cdx_last_error(const cdx_ctx* ctx);
int cdx_abi_version(void);
/* Number of kernel launches this context has issued (the bench's gpu_launches count). */
uint64_t cdx_launch_count(const cdx_ctx* ctx);

/* ---- CUDA graphs: capture a sequence of cdx_* calls on the context stream and replay it
 * with one launch (small, launch-bound batches).  The stream must not be a default stream;
 * calls that synchronise with the host (buffer growth, canon_intern, gang_priority, jsonl)
 * cannot be captured.  Captured calls replay on the same buffers with the same arguments. */
typedef struct cdx_graph cdx_graph;
int cdx_graph_begin(cdx_ctx* ctx);
int cdx_graph_end(cdx_ctx* ctx, cdx_graph** out);
int cdx_graph_launch(cdx_ctx* ctx, cdx_graph* g);
int cdx_graph_destroy(cdx_graph* g);

/* ---- synthetic trace generation on the device (runtime.cpp:91-117 restated) ------- */
int cdx_gen_sc(cdx_ctx* ctx, const cdx_gen_params* g, uint64_t r0, uint64_t R, uint32_t P,
               uint32_t S, uint32_t* ids);
int cdx_gen_cot(cdx_ctx* ctx, const cdx_gen_params* g, uint64_t r0, uint64_t R, uint32_t P,
                uint32_t* ids, uint64_t* hes);
int cdx_gen_reward(cdx_ctx* ctx, const cdx_gen_params* g, uint64_t g0, uint64_t G, uint32_t T,
                   uint32_t W, float* rewards, uint32_t* ids);

/* ---- K2: Self-Consistency certaindex ------------------------------------------------
 * Replaces, per (request r, probe p) row of S sampled answers,
 *   metrics::certaindex_entropy(metrics::cluster_exact(row))        metrics.hpp:44,66
 *   metrics::combined_meets_thresholds({H~}, thresholds)            metrics.hpp:116
 * ids: u32[R][P][S] interned answer ids (equal id <=> equal trimmed bytes), 1 <= S <= 4096
 * (S <= 32: 32-row groups through the TMA / bulk-copy engines; S > 32: a warp per row).
 * hcert: f32[R][P] (nullable).  meets_bits: u32[R][ceil(P/32)], bit p%32 of word p/32.
 * Decisions are taken on the FP64 certaindex; hcert is its fp32 rounding.               */
int cdx_sc_certaindex(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                      const cdx_threshold* th, uint32_t n_th, float* hcert, uint32_t* meets_bits);
/* The same plus the majority-fraction certaindex (north_star (2)): majority f32[R][P]
 * (nullable) = largest cluster size / S of each row, the fp32 rounding of the double
 * (double)max_size / S on which CDX_SIG_MAJORITY thresholds are decided.  Thresholds may mix
 * CDX_SIG_ENTROPY and CDX_SIG_MAJORITY (an AND, metrics.cpp:159-171).                      */
int cdx_sc_certaindex_ex(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                         const cdx_threshold* th, uint32_t n_th, float* hcert, float* majority,
                         uint32_t* meets_bits);

/* Per-row clusters in first-seen order (the full metrics::Clustering of every row), 1 <= S <= 4096:
 * n_clusters u32[rows], leader u32[rows][S] (sample index of the cluster's first answer,
 * first n_clusters entries valid), size u32[rows][S].  metrics.cpp:21-37               */
int cdx_cluster_rows(cdx_ctx* ctx, const uint32_t* ids, uint64_t rows, uint32_t S,
                     uint32_t* n_clusters, uint32_t* leader, uint32_t* size);

/* Entropy of explicit clusterings (façade path of semantic_entropy/certaindex_entropy):
 * sizes u32[rows][max_m] in cluster order, m u32[rows] clusters per row, totals u32[rows]
 * (Clustering::total; nullable = the sum of the sizes).  Every row's total must be
 * <= max_n (host bound, sizes the term table); outputs f64 (nullable).  Fails at cdx_sync
 * with the reference's messages: "semantic_entropy: invalid clustering" (total < 1, m == 0,
 * or — a documented restriction — a cluster larger than the total), "semantic_entropy:
 * empty cluster".  The n == 1 -> 1.0 shortcut of certaindex_entropy applies to Hcert.
 * metrics.cpp:107-125                                                                    */
int cdx_entropy_from_sizes(cdx_ctx* ctx, const uint32_t* sizes, const uint32_t* m,
                           const uint32_t* totals, uint64_t rows, uint32_t max_m, uint32_t max_n,
                           double* H, double* Hcert);

/* One clustering whose total n is known on the host (the scalar façade's path, any n up to
 * 2^26): sizes u32[m] in cluster order (device).  Same semantics and messages as above. */
int cdx_entropy_one(cdx_ctx* ctx, const uint32_t* sizes, uint32_t m, uint32_t total, double* H,
                    double* Hcert);

/* One explicit Clustering of the scalar façade (metrics::semantic_entropy /
 * certaindex_entropy, metrics.cpp:107-125) with HOST cluster sizes in cluster order and any
 * total, a cluster larger than the total included (p > 1, as the reference computes it).
 * One term (c/total)*log(c/total) per cluster from the host libm, folded on the device in
 * cluster order.  H, Hcert: DEVICE f64 (nullable).  Errors as the reference, in its order. */
int cdx_entropy_sizes_host(cdx_ctx* ctx, const int32_t* sizes, uint32_t m, int32_t total, double* H,
                           double* Hcert);

/* ---- ragged rows behind the scalar C++ API (include/cdx/metrics.hpp, probe.hpp) -------
 * Rows are concatenated records, row r = [row_off[r], row_off[r+1]).  ids are interned
 * answers (K1: equal id <=> equal trimmed bytes), hes u8 hesitation flags, step_index i32
 * and token_offset i64 per record, in trace order.                                        */
/* probe::consistency(records, k[r], window)  probe.cpp:64-75.  C f64 = agree / window;
 * ready u8 = 0 where the reference returns nullopt (fewer than window usable records). */
int cdx_probe_consistency(cdx_ctx* ctx, const uint32_t* ids, const uint8_t* hes,
                          const int32_t* step_index, const uint64_t* row_off, const int32_t* k,
                          uint64_t rows, int32_t window, double* C, uint8_t* ready);
/* probe::should_exit(trace, cfg)  probe.cpp:77-85 -> decision u8 (CDX_EXIT_*).
 * cfg is validated first with ProbeConfig::validate's messages (probe.cpp:19-25).       */
int cdx_probe_should_exit(cdx_ctx* ctx, const uint32_t* ids, const uint8_t* hes,
                          const int32_t* step_index, const int64_t* token_offset,
                          const uint64_t* row_off, uint64_t rows, const cdx_probe_cfg* cfg,
                          uint8_t* decision);
/* probe::final_answer(trace)  probe.cpp:87-102 -> pos u64 (record index within the row of
 * the reported answer) and low_conf u8.  terminated_at i32[rows] (nullable; INT32_MIN =
 * nullopt), termination_reason u8[rows] (nullable; probe.hpp:42 ordinals: 0 Certain,
 * 1 Budget, 2 CriteriaExternal).  Rows must be non-empty (the caller raises
 * "final_answer: empty trace").                                                          */
int cdx_probe_final_answer(cdx_ctx* ctx, const uint8_t* hes, const int32_t* step_index,
                           const uint64_t* row_off, const int32_t* terminated_at,
                           const uint8_t* termination_reason, uint64_t rows, uint64_t* pos,
                           uint8_t* low_conf);
/* metrics::combined_meets_thresholds per row  metrics.cpp:159-171.  signals f64[rows][4]
 * in SignalKind order, present u8[rows] (bit k = signal k present); meets u8[rows].  An
 * absent signal reached in threshold order fails at cdx_sync with "combined_meets_
 * thresholds: signal '<name>' absent".                                                   */
int cdx_meets_thresholds_rows(cdx_ctx* ctx, const double* signals, const uint8_t* present,
                              uint64_t rows, const cdx_threshold* th, uint32_t n_th,
                              uint8_t* meets);
/* Cluster sizes of dense first-seen ids (output of cdx_canon_intern): counts u32[n_unique]
 * = the cluster sizes of metrics::cluster_exact in first-seen order (metrics.cpp:21-37). */
int cdx_id_histogram(cdx_ctx* ctx, const uint32_t* ids, uint64_t n, uint32_t n_unique,
                     uint32_t* counts);

/* SPEC.md:431-439 estimate_iteration_tokens per program: tokens i64 (completed iteration
 * token counts, concatenated), row_off u64[rows+1]; est f64 = mean, or prior if empty.  */
int cdx_iteration_tokens_rows(cdx_ctx* ctx, const int64_t* tokens, const uint64_t* row_off,
                              uint64_t rows, double prior, double* est);

/* ---- device buffers, stream-ordered on the context stream (hosts without cudart) ------ */
int cdx_alloc(cdx_ctx* ctx, uint64_t bytes, void** out);
int cdx_free(cdx_ctx* ctx, void* p);
int cdx_memcpy(cdx_ctx* ctx, void* dst, const void* src, uint64_t bytes); /* any direction */
int cdx_memset(cdx_ctx* ctx, void* dst, int value, uint64_t bytes);

/* ---- K5: SPEC allocate + exclusive scan of token budgets + stable compaction --------
 * Replaces scheduler.allocate for a batch of requests whose certaindex
 * threshold outcome per knob unit is meets_bits (from K2/K4).  Outputs per request:
 *   exit_knob  i32  knob unit at which the request terminates (always set: cap at latest)
 *   reason     u8   CDX_EXIT_CERTAIN (threshold met) | CDX_EXIT_BUDGET (resource cap)
 *   granted    i32  knob units granted (== exit_knob)
 *   offsets    i64  base_offset + exclusive prefix sum of granted*tokens_per_unit
 *   kept       u32  stable list of request indices continuing past detect_at
 * Device scalars: n_kept (u64), tokens_saved (i64) = sum (cap-granted)*tokens_per_unit,
 * total_budget (i64, nullable) = sum of budgets.                                         */
int cdx_allocate_scan(cdx_ctx* ctx, const uint32_t* meets_bits, uint64_t R, uint32_t P,
                      const cdx_alloc_policy* pol, int64_t base_offset, uint32_t kept_base,
                      int32_t* exit_knob, uint8_t* reason, int32_t* granted, int64_t* offsets,
                      uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved,
                      int64_t* total_budget);

/* K2 + K5 in one call: cdx_sc_certaindex (meets_bits required, hcert nullable) followed by
 * cdx_allocate_scan over its meets bits, with the same arguments and results as those two
 * calls (the SC update_certaindex + scheduler.allocate of runtime.cpp:264-313 /
 * SPEC.md:404-412 for a whole batch).  The policy is validated before anything launches.
 * Two launches back to back: running K5's tiles inside K2's tail was measured slower on the
 * B200 (the per-tile release of K2's finished meets words costs more than K5's launch). */
int cdx_sc_decide(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S, const cdx_threshold* th,
                  uint32_t n_th, float* hcert, uint32_t* meets_bits, const cdx_alloc_policy* pol, int64_t base_offset,
                  uint32_t kept_base, int32_t* exit_knob, uint8_t* reason, int32_t* granted, int64_t* offsets,
                  uint32_t* kept, uint64_t* n_kept, int64_t* tokens_saved, int64_t* total_budget);

/* ---- mixed-archetype batch: per-archetype certaindex + allocation at the current knob ------
 * The batched form of ProgramDriver::update_certaindex's dispatch (runtime.cpp:264-313)
 * followed by scheduler.allocate, for N programs of any archetypes, each at
 * its own current knob.  Programs of one archetype group share one trace tensor; program i has
 * archetype archetype[i] (CDX_ARCH_*) and is row slot[i] of its group's tensor (MCTS and Rebase
 * share the reward group).  Signals per knob unit u (1-based):
 *   SC      H~ = certaindex_entropy(cluster_exact(the S answers of probe row u-1))  (K2)
 *   CoT     C_k = consistency(records up to probe u-1, window), 0.0 while not ready (runtime.cpp:298)
 *   MCTS    H~ and mean reward over every path of steps 0..u-1 (cumulative, K4)
 *   Rebase  H~ and max reward over steps 0..u-1
 * Each archetype's thresholds (combined_meets_thresholds, metrics.cpp:159-171) and allocation
 * policy (even | static_threshold | k_step_threshold) come from policy[CDX_ARCH_*].          */
typedef struct {
    const uint32_t* sc_ids;      /* u32[sc_n][sc_P][sc_S] */
    uint64_t sc_n;
    uint32_t sc_P, sc_S;
    const uint32_t* cot_ids;     /* u32[cot_n][cot_P] */
    const uint64_t* cot_hes;     /* u64[cot_n][ceil(cot_P/64)] hesitation bits */
    uint64_t cot_n;
    uint32_t cot_P, cot_window;
    const float* rw_rewards;     /* f32[rw_n][rw_T][rw_W] */
    const uint32_t* rw_ids;      /* u32[rw_n][rw_T][rw_W] (nullable: no entropy signal) */
    uint64_t rw_n;
    uint32_t rw_T, rw_W;
} cdx_mixed_trace;

typedef struct {
    cdx_threshold th[4];         /* this archetype's thresholds, in order */
    uint32_t n_th;
    uint32_t _pad;
    cdx_alloc_policy alloc;      /* kind, detect_at, recheck_every, resource_cap, tokens_per_unit */
} cdx_arch_policy;

/* knob i32[N]: units the program holds now (0 <= knob <= its resource_cap).  Outputs:
 *   decision u8[N]  CDX_EXIT_CONTINUE (granted) | CDX_EXIT_CERTAIN (a test point <= knob met its
 *                   thresholds) | CDX_EXIT_BUDGET (knob == resource_cap); nonzero = terminated,
 *                   so it serves directly as cdx_prog_soa.terminated of the gang order
 *   grant   i32[N]  (nullable) units granted now: up to the next decision point
 *   cap     i32[N]  (nullable) the archetype's resource_cap (cdx_prog_soa.cap)
 *   offsets i64[N]  (nullable) exclusive scan of grant * tokens_per_unit, program order
 *   total_budget    (device i64, nullable) the scan's total
 * policy: cdx_arch_policy[4] (host).  A bad archetype, slot or knob fails at cdx_sync.      */
int cdx_mixed_allocate(cdx_ctx* ctx, const cdx_mixed_trace* trace, const uint8_t* archetype,
                       const uint32_t* slot, const int32_t* knob, uint64_t N,
                       const cdx_arch_policy* policy, uint8_t* decision, int32_t* grant,
                       int32_t* cap, int64_t* offsets, int64_t* total_budget);

/* The CoT signal as threshold bits: bit p of meets_bits u32[R][ceil(P/32)] =
 * combined_meets_thresholds({C_k(p)}, th) where C_k(p) = consistency over the records up to
 * probe p (probe.cpp:64-75), 0.0 while fewer than `window` are usable (runtime.cpp:298).
 * ids u32[R][P], hes u64[R][ceil(P/64)]; window <= 62; thresholds on the entropy slot only. */
int cdx_cot_meets(cdx_ctx* ctx, const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P,
                  int32_t window, const cdx_threshold* th, uint32_t n_th, uint32_t* meets_bits);

/* ---- K3: CoT probe-window exit ------------------------------------------------------
 * Replaces, for every prefix of each request's probe trace,
 *   probe::should_exit(trace, cfg)        probe.cpp:77-85  (consistency probe.cpp:64-75)
 *   probe::final_answer(trace)            probe.cpp:87-102
 * ids u32[R][P]; hes u64[R][ceil(P/64)] hesitation bits; offsets i64[R][P] token offsets
 * (nullable: offset of probe p = (p+1)*interval_tokens).  Outputs: exit_step i32 (0-based
 * probe index, -1 = no exit), reason u8, final_id u32, low_conf u8, ck f32[R][P] (nullable:
 * consistency at every probe, 0.0 while the window is not ready, runtime.cpp:298).        */
int cdx_cot_exit(cdx_ctx* ctx, const uint32_t* ids, const uint64_t* hes, const int64_t* offsets,
                 uint64_t R, uint32_t P, const cdx_probe_cfg* cfg, int32_t* exit_step,
                 uint8_t* reason, uint32_t* final_id, uint8_t* low_conf, float* ck);

/* ---- K4: reward certaindex (MCTS mean / Rebase max), cumulative over steps ----------
 * Replaces the MCTS/Rebase branch of ProgramDriver::update_certaindex (runtime.cpp:
 * 279-292): at step t, R = certaindex_reward(all rewards of steps 0..t) (metrics.cpp:
 * 127-137) and H~ = certaindex_entropy(cluster_exact(all answers of steps 0..t)).
 * rewards f32[G][T][W]; ids u32[G][T][W] (nullable: no entropy signal); agg u8[G]
 * (CDX_AGG_MEAN for MCTS, CDX_AGG_MAX for Rebase).  Thresholds are per aggregation kind.
 * Outputs R f32[G][T], H f32[G][T] (nullable), meets_bits u32[G][ceil(T/32)] (nullable). */
int cdx_reward_certaindex(cdx_ctx* ctx, const float* rewards, const uint32_t* ids,
                          const uint8_t* agg, uint64_t G, uint32_t T, uint32_t W,
                          const cdx_threshold* th_mean, uint32_t n_th_mean,
                          const cdx_threshold* th_max, uint32_t n_th_max, float* R, float* H,
                          uint32_t* meets_bits);

/* The same over f64 rewards (RewardSet / PathSample::reward hold doubles, metrics.hpp:74-77):
 * rewards f64[G][T][W]; every program is folded in the reference's left-fold order (one warp
 * per program); outputs as above (R, H fp32 stores of the FP64 values the decisions use).   */
int cdx_reward_certaindex_f64(cdx_ctx* ctx, const double* rewards, const uint32_t* ids,
                              const uint8_t* agg, uint64_t G, uint32_t T, uint32_t W,
                              const cdx_threshold* th_mean, uint32_t n_th_mean,
                              const cdx_threshold* th_max, uint32_t n_th_max, float* R, float* H,
                              uint32_t* meets_bits);

/* Scalar-façade reward path: RewardSet of f64 values, rows of variable length.
 * values f64 concatenated, row_off u64[rows+1], agg u8[rows]; out f64[rows]. */
int cdx_reward_sets(cdx_ctx* ctx, const double* values, const uint64_t* row_off,
                    const uint8_t* agg, uint64_t rows, double* out);

/* ---- K1: answer canonicalisation + interning + hesitation ---------------------------
 * Replaces metrics::trim + the unordered_map key of cluster_exact (metrics.cpp:12-37) and
 * probe::flag_hesitation (probe.cpp:36-44).  bytes: string arena (device), offsets
 * u64[n+1].  markers: host array of n_markers NUL-terminated strings.  Outputs: ids u32[n]
 * dense, in first-seen order of the trimmed bytes; hes u8[n] (nullable); first_index
 * u64[n_unique] (nullable, arena index of each id's first occurrence); *n_unique (host).  */
int cdx_canon_intern(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint64_t n,
                     const char* const* markers, uint32_t n_markers, uint32_t* ids,
                     uint8_t* hes, uint64_t* first_index, uint64_t* n_unique);

/* ---- K6: gang-scheduling program order ----------------------------------------------
 * Replaces scheduler.escalate / estimate_iteration_tokens / next_batch program order
 * (tie-break SPEC.md:470).  Order: escalated programs first (FIFO by
 * arrival), then the policy key (fifo: arrival; sjf: est_tokens_per_iter * (cap-knob)),
 * then arrival, then program id.  Terminated programs are dropped.  order u32[N] receives
 * program ids; *n_out (host) the count; escalated u8[N] (nullable) per input program.
 * keys (nullable, device u64[N][3]) receives the sortable composite key of each ordered
 * program, for the multi-GPU merge (cdx_gang_merge).                                     */
int cdx_gang_priority(cdx_ctx* ctx, const cdx_prog_soa* progs, uint64_t N,
                      const cdx_inter_policy* pol, double now, uint32_t* order, uint64_t* n_out,
                      uint8_t* escalated, uint64_t* keys);
/* Merge `runs` sorted runs of composite keys (from cdx_gang_priority's `keys`, u64[.][3] =
 * {priority word, arrival bits, program id}) into the global order.  Run q is
 * keys[q*stride .. q*stride + run_len[q]) — the receive layout of an allgather padded to
 * `stride` keys per rank.  run_len u64[runs] is a DEVICE array (the gathered per-rank
 * counts, so no host round trip).  order_out u32[sum run_len] receives program ids;
 * total (device u64, nullable) their count.  Used after the NCCL allgather (K6).        */
int cdx_gang_merge(cdx_ctx* ctx, const uint64_t* keys, const uint64_t* run_len, uint32_t runs,
                   uint64_t stride, uint32_t* order_out, uint64_t* total);

/* ---- multi-GPU: a context that owns its communicator -------------
 * One process (or host thread) per rank, one context per rank.  Requests / programs shard
 * into contiguous per-rank slices with no data-path exchange; the sharded entry points below
 * run the only two exchange steps (global token offsets, the global gang order) through the
 * context's communicator.  The transport is either
 *   - NCCL: nccl_id (128 bytes = ncclUniqueId, made once by cdx_nccl_unique_id on one rank and
 *     broadcast by the caller).  The context creates and owns an NCCL communicator over
 *     libnccl.so.2, loaded at run time (NVLink / NVSwitch on one box); or
 *   - caller callbacks (any transport: an NCCL communicator the caller owns, MPI, host
 *     staging between threads).  Buffers are DEVICE pointers; a callback must order its
 *     transfers after the work already queued on `stream` (a cudaStream_t) and complete them
 *     (or queue them on `stream`) before returning; nonzero return = failure (CDX_ENCCL).
 * The reference is single-process (proj/src/CMakeLists.txt:11-12), so these have no
 * reference counterpart: concatenating the ranks' outputs reproduces the 1-GPU result.    */
typedef struct {
    uint32_t rank, world;
    const uint8_t* nccl_id; /* non-null: NCCL transport (callbacks ignored) */
    void* user;             /* callbacks' first argument */
    /* recv[q*bytes .. (q+1)*bytes) <- rank q's send[0 .. bytes) */
    int (*allgather)(void* user, const void* send, void* recv, uint64_t bytes, void* stream);
    /* send[send_off[q] .. + send_bytes[q]) -> rank q; recv[recv_off[q] .. + recv_bytes[q]) <- rank q.
     * counts and offsets are HOST arrays of `world` entries (bytes) */
    int (*alltoallv)(void* user, const void* send, const uint64_t* send_bytes, const uint64_t* send_off,
                     void* recv, const uint64_t* recv_bytes, const uint64_t* recv_off, void* stream);
} cdx_comm;

/* A 128-byte NCCL unique id for cdx_comm.nccl_id (CDX_ENCCL when libnccl.so.2 is absent). */
int cdx_nccl_unique_id(uint8_t id[128]);
/* cdx_ctx_create plus a communicator (comm nullable = world 1, no exchange).  Collective:
 * with NCCL every rank must call it. */
int cdx_ctx_create_comm(int device, const cdx_comm* comm, cdx_ctx** out);
int cdx_ctx_comm_info(const cdx_ctx* ctx, uint32_t* rank, uint32_t* world);
/* recv[q*bytes ..] <- rank q's send (DEVICE), on the context stream. */
int cdx_allgather(cdx_ctx* ctx, const void* send, void* recv, uint64_t bytes);

/* K5 over this rank's request shard with GLOBAL results (SPEC.md:404-412 over the whole
 * batch): as cdx_allocate_scan, but offsets are the exclusive scan over all ranks' requests in
 * rank order, kept holds GLOBAL request indices (rank q's first request is the sum of the
 * requests of ranks < q), *n_kept (device) this rank's kept count, *tokens_saved and
 * *total_budget (device, nullable) the sums over all ranks.  shard_info (device u64[world][4],
 * nullable) receives every rank's {requests, budget total, kept, tokens saved}.  Collective.  */
int cdx_allocate_scan_sharded(cdx_ctx* ctx, const uint32_t* meets_bits, uint64_t R, uint32_t P,
                              const cdx_alloc_policy* pol, int32_t* exit_knob, uint8_t* reason,
                              int32_t* granted, int64_t* offsets, uint32_t* kept, uint64_t* n_kept,
                              int64_t* tokens_saved, int64_t* total_budget, uint64_t* shard_info);

/* K6 over this rank's programs (GLOBAL program ids via progs->program_id / id_base) with the
 * GLOBAL order on every rank: a distributed sample sort.  Each rank sorts its keys (as
 * cdx_gang_priority), allgathers cdx_shard_samples of its run, derives the same splitters
 * (cdx_shard_splitters), sends each key to the rank owning its bucket (alltoallv, about
 * 24 B x N_local x (world-1)/world per rank), merges the runs it received and the buckets'
 * program ids are allgathered in bucket order (4 B per program).  order: DEVICE u32 with room
 * for every rank's live programs; *n_out (host) = their count.  Identical to the 1-GPU order
 * (the composite key is a total order).  Collective.                                        */
int cdx_gang_priority_sharded(cdx_ctx* ctx, const cdx_prog_soa* progs, uint64_t N_local,
                              const cdx_inter_policy* pol, double now, uint32_t* order, uint64_t* n_out);

/* Building blocks of the sample sort (also used by torch.distributed hosts, sharding.py).
 * cdx_shard_samples: s keys of a sorted run keys u64[n][3] (DEVICE) at the midpoints of s
 * equal ranges -> samples u64[s][3] (DEVICE); all-ones sentinels when n == 0.
 * cdx_shard_splitters (HOST only, no device): samples u64[world][s][3] and counts u64[world]
 * (every rank's run length) -> world-1 splitters u64[world-1][3]: bucket b holds the keys k
 * with splitter[b-1] <= k < splitter[b]; each sample stands for counts[q]/s keys and
 * splitter b is the first sample at which the weight before it reaches b * total / world.
 * cdx_shard_bounds: bucket boundaries of a sorted run -> bounds u64[world+1] (DEVICE).
 * cdx_gang_merge_runs: merge sorted runs keys[run_off[q] .. run_off[q+1]) (run_off DEVICE
 * u64[runs+1]) -> program ids order_out u32[run_off[runs]].                                */
int cdx_shard_samples(cdx_ctx* ctx, const uint64_t* keys, uint64_t n, uint32_t s, uint64_t* samples);
int cdx_shard_splitters(const uint64_t* samples, const uint64_t* counts, uint32_t world, uint32_t s,
                        uint64_t* splitters);
int cdx_shard_bounds(cdx_ctx* ctx, const uint64_t* keys, uint64_t n, const uint64_t* splitters,
                     uint32_t world, uint64_t* bounds);
int cdx_gang_merge_runs(cdx_ctx* ctx, const uint64_t* keys, const uint64_t* run_off, uint32_t runs,
                        uint32_t* order_out);

/* Global token offsets across request shards (K5 multi-GPU): offsets[i] += sum of
 * shard_totals[q] for q < rank.  shard_totals i64[world] is the allgathered vector of
 * per-rank budget totals (DEVICE).  Concatenating the ranks' offsets then equals the
 * single-GPU exclusive scan.                                                             */
int cdx_offsets_rebase(cdx_ctx* ctx, int64_t* offsets, uint64_t R, const int64_t* shard_totals,
                       uint32_t rank);

/* ---- JSONL trace ingestion (probe::read_trace_jsonl, probe.cpp:126-165) ---------------
 * text: the whole JSON-lines file in DEVICE memory (nbytes < 4 GiB).  Per record, in line
 * order (blank lines skipped): program u32 (program ids interned exactly, dense, first-seen
 * order), step_index i32, token_offset i64, hesitant u8, the decoded answer in
 * answer_arena[answer_off[r] .. answer_off[r+1]) (capacity nbytes), the decoded program id in
 * program_arena[program_off[r] ..) (nullable pair), program_first u64[programs] (nullable:
 * first record of each program).  Arrays hold cap_records (>= the number of lines) entries,
 * offsets cap_records + 1.  The first bad line fails with CDX_ERUNTIME and the reference's
 * "trace line <n>: invalid JSON | missing or mistyped field | token_offset does not
 * increase | step_index does not increase" (detail text after the category may differ). */
int cdx_jsonl_parse(cdx_ctx* ctx, const char* text, uint64_t nbytes, uint64_t cap_records,
                    uint32_t* program, int32_t* step_index, int64_t* token_offset, uint8_t* hesitant,
                    uint64_t* answer_off, char* answer_arena, uint64_t* program_off,
                    char* program_arena, uint64_t* program_first, uint64_t* n_records,
                    uint64_t* n_programs);

/* ---- epsilon-accuracy stop test (alternative CoT stop rule) ----------------------------
 * probe::stationary_by_epsilon_test (probe.cpp:104-120) over theory::epsilon_stop_test
 * (theory.cpp:100-146).  Batched over CoT traces (ids u32[R][P], hes u64[R][ceil(P/64)],
 * P <= 64), evaluated at every prefix: eps_step i32[R] = first probe where it returns true
 * (-1 if none), state u8[R][P] (nullable) = 0 nullopt / 1 false / 2 true per prefix.
 * Errors as the reference: "epsilon_stop_test: k must be >= 1", "... epsilon must be > 0". */
int cdx_cot_eps_stop(cdx_ctx* ctx, const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P,
                     int32_t k, double epsilon, int32_t* eps_step, uint8_t* state);
/* The same test on ragged record rows (the scalar API): whole row r = one record span,
 * hes u8 per record; state u8[rows]; at most 1024 non-hesitant records per row.          */
int cdx_probe_eps_stop_rows(cdx_ctx* ctx, const uint32_t* ids, const uint8_t* hes,
                            const uint64_t* row_off, uint64_t rows, int32_t k, double epsilon,
                            uint8_t* state);

/* ---- aggregation: the final answer per archetype (ProgramDriver::aggregate_prefix,
 * runtime.cpp:318-403) --------------------------------------------------
 * SC: plurality over the exit row's answers, earliest-seen cluster wins ties.  ids
 * u32[R][P][S], exit_knob i32[R] (1-based knob unit, e.g. K5's exit_knob) -> answer u32[R].
 * A knob outside [1, P] fails at cdx_sync.                                                */
int cdx_sc_aggregate(cdx_ctx* ctx, const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                     const int32_t* exit_knob, uint32_t* answer);
/* MCTS (agg CDX_AGG_MEAN): answer of the first maximum-reward path over steps 0..t.
 * Rebase (agg CDX_AGG_MAX): softmax-weighted plurality (sum of exp(reward) per cluster in
 * path order) over the last full layer, step t.  rewards f32[G][T][W], ids u32[G][T][W],
 * exit_step i32[G] (0-based step t) -> answer u32[G]; W <= 256.  exp() is the host libm's
 * algorithm restated bit for bit on the device (cdx_libm_exp), so weights equal the
 * reference's for every reward.  A Rebase layer whose weights are all NaN has no winner (the
 * reference returns an empty string): answer = CDX_NO_ANSWER.  *inexact (device u64,
 * nullable; ABI v2) is zeroed: no weight is approximated.                                 */
#define CDX_NO_ANSWER 0xffffffffu
int cdx_reward_aggregate(cdx_ctx* ctx, const float* rewards, const uint32_t* ids, const uint8_t* agg,
                         uint64_t G, uint32_t T, uint32_t W, const int32_t* exit_step,
                         uint32_t* answer, uint64_t* inexact);
/* The same over f64 rewards (PathSample::reward and RewardSet hold doubles,
 * runtime.hpp / metrics.hpp:74-77).                                                        */
int cdx_reward_aggregate_f64(cdx_ctx* ctx, const double* rewards, const uint32_t* ids, const uint8_t* agg,
                             uint64_t G, uint32_t T, uint32_t W, const int32_t* exit_step,
                             uint32_t* answer);
/* y[i] = std::exp(x[i]) with the host libm's bits (glibc's table-driven exp, FMA build),
 * evaluated on the device; x, y DEVICE f64[n].  The weight function of the Rebase vote.   */
int cdx_libm_exp(cdx_ctx* ctx, const double* x, uint64_t n, double* y);

/* ---- end-to-end host entry: SC certaindex + allocate from HOST buffers ---------------
 * Streams ids (host, ideally pinned) through the device in chunks of whole requests,
 * overlapping H2D copies with K2+K5, and copies exit_knob/reason/granted/offsets and the
 * fp32 certaindex (nullable) back to host buffers.  Returns when the results are on host. */
int cdx_sc_decide_host(cdx_ctx* ctx, const uint32_t* ids_host, uint64_t R, uint32_t P,
                       uint32_t S, const cdx_threshold* th, uint32_t n_th,
                       const cdx_alloc_policy* pol, int32_t* exit_knob_host,
                       uint8_t* reason_host, int64_t* offsets_host, float* hcert_host,
                       int64_t* tokens_saved_host);

/* probe::should_exit at every prefix + final_answer (as cdx_cot_exit) from HOST buffers:
 * ids u32[R][P], hes u64[R][ceil(P/64)], offsets i64[R][P] (nullable: (p+1)*interval).
 * Outputs to host: exit_step i32[R], reason u8[R], final_id u32[R] (nullable), low_conf u8[R]
 * (nullable).  Chunked and double buffered like cdx_sc_decide_host.                        */
int cdx_cot_decide_host(cdx_ctx* ctx, const uint32_t* ids_host, const uint64_t* hes_host,
                        const int64_t* offsets_host, uint64_t R, uint32_t P, const cdx_probe_cfg* cfg,
                        int32_t* exit_step_host, uint8_t* reason_host, uint32_t* final_id_host,
                        uint8_t* low_conf_host);

/* MCTS/Rebase certaindex (as cdx_reward_certaindex) + allocate (as cdx_allocate_scan, knob
 * unit = step) from HOST buffers: rewards f32[G][T][W], ids u32[G][T][W] (nullable), agg
 * u8[G].  Outputs to host: exit_knob i32[G], reason u8[G], offsets i64[G] (global across
 * chunks), R f32[G][T] (nullable), *tokens_saved_host (nullable).                          */
int cdx_reward_decide_host(cdx_ctx* ctx, const float* rewards_host, const uint32_t* ids_host,
                           const uint8_t* agg_host, uint64_t G, uint32_t T, uint32_t W,
                           const cdx_threshold* th_mean, uint32_t n_th_mean,
                           const cdx_threshold* th_max, uint32_t n_th_max, const cdx_alloc_policy* pol,
                           int32_t* exit_knob_host, uint8_t* reason_host, int64_t* offsets_host,
                           float* R_host, int64_t* tokens_saved_host);

/* ---- one-round-trip scalar entries (k_scalar.cu) -------------------------------------
 * Host buffers in and out: ONE pinned host->device copy of every input, one launch, one
 * device->host copy of the outputs, one synchronisation.  They back the reference's scalar
 * C++ API (include/cdx/metrics.hpp, probe.hpp) for the per-program call sizes of
 * runtime.cpp:264-313; the batched entries above are the throughput path.  Answers are a
 * byte arena + offsets[n+1] (1..2048 answers, at most 1 MiB of text). */
/* metrics::cluster_exact (metrics.cpp:21-37) + probe::flag_hesitation (probe.cpp:36-44):
 * dense first-seen ids of the trimmed bytes, per cluster its first index and size; hes
 * (nullable) = the marker test on the raw answers.  Any output but n_unique may be NULL. */
int cdx_cluster_host(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint32_t n, const char* const* markers,
                     uint32_t n_markers, uint32_t* ids, uint8_t* hes, uint32_t* first_index, uint32_t* sizes,
                     uint32_t* n_unique);
/* probe::consistency(records, k, w) (probe.cpp:64-75): *ready = 0 for nullopt */
int cdx_consistency_host(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint32_t n, const uint8_t* hes,
                         const int32_t* step_index, int32_t k, int32_t w, double* C, uint8_t* ready);
/* probe::should_exit(trace, cfg) (probe.cpp:77-85): decision = cdx_exit_decision */
int cdx_should_exit_host(cdx_ctx* ctx, const char* bytes, const uint64_t* offsets, uint32_t n, const uint8_t* hes,
                         const int32_t* step_index, const int64_t* token_offset, const cdx_probe_cfg* cfg,
                         uint8_t* decision);
/* probe::final_answer(trace) (probe.cpp:87-102): record index + low-confidence flag;
 * terminated_at = INT32_MIN for nullopt, termination_reason = TerminationReason ordinal */
int cdx_final_answer_host(cdx_ctx* ctx, const uint8_t* hes, const int32_t* step_index, uint32_t n,
                          int32_t terminated_at, uint8_t termination_reason, uint64_t* pos, uint8_t* low_conf);
/* semantic_entropy / certaindex_entropy of one clustering (metrics.cpp:107-125), host outputs */
int cdx_entropy_host(cdx_ctx* ctx, const int32_t* sizes, uint32_t m, int32_t total, double* H, double* Hcert);
/* certaindex_reward (metrics.cpp:127-137): aggregation CDX_AGG_MEAN / CDX_AGG_MAX */
int cdx_reward_host(cdx_ctx* ctx, const double* rewards, uint64_t n, uint8_t aggregation, double* out);
/* combined_meets_thresholds (metrics.cpp:159-171): signals4 in SignalKind order, present
 * bit k = signal k present, at most 8 thresholds */
int cdx_meets_host(cdx_ctx* ctx, const double* signals4, uint8_t present, const cdx_threshold* th, uint32_t n_th,
                   uint8_t* meets);

#ifdef __cplusplus
}
#endif
#endif /* CDX_C_H */
