/*
 * cdx_oracle.h — CPU restatement of the Certaindex hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the checker, never the product: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  Every function cites
 * the reference file:line it restates (paths relative to the reference's proj/ tree, or
 * SPEC.md for the scheduler, which has no reference code).
 *
 * Parity pinning: the restatement is checked against (1) golden vectors produced by the
 * reference's own C++ sources compiled here (oracle/_ref, see oracle/Makefile and
 * tests/golden/make_golden.py) and (2) the SPEC.md examples.  The scheduler rows
 * (allocate / escalate / estimate_iteration_tokens / next_batch order) exist only in
 * for those the oracle is pinned by the SPEC examples only.
 */
#ifndef CDX_ORACLE_H
#define CDX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/cdx_c.h" /* shared plain-C parameter structs */

#ifdef __cplusplus
extern "C" {
#endif

/* ---- rng.hpp:25-34 ---------------------------------------------------------------- */
uint64_t cdxo_mix64(uint64_t x);
uint64_t cdxo_derive_seed(uint64_t master, uint64_t a, uint64_t b);

/* ---- synthetic trace generator (counter-based restatement of runtime.cpp:91-117) ---- */
int cdxo_solvable(const cdx_gen_params* g, uint64_t r);
uint32_t cdxo_convergence(const cdx_gen_params* g, uint64_t r);
uint32_t cdxo_answer(const cdx_gen_params* g, uint64_t r, uint64_t j, uint32_t knob);
int cdxo_hesitant(const cdx_gen_params* g, uint64_t r, uint32_t p);
uint32_t cdxo_reward_k(const cdx_gen_params* g, uint64_t r, uint64_t j, uint32_t knob);
/* ids[r][p][s] for r in [r0, r0+nreq) */
void cdxo_gen_sc(const cdx_gen_params* g, uint64_t r0, uint64_t nreq, uint32_t P, uint32_t S,
                 uint32_t* ids);
void cdxo_gen_sc_mt(const cdx_gen_params* g, uint64_t r0, uint64_t nreq, uint32_t P, uint32_t S,
                    uint32_t* ids, int nthreads);
/* ids[r][p] (hesitant probes carry id M + answer) and hes[r] bit p */
void cdxo_gen_cot(const cdx_gen_params* g, uint64_t r0, uint64_t nreq, uint32_t P, uint32_t* ids,
                  uint64_t* hes);
/* rewards[g][t][w] (on the 2^-24 grid) and ids[g][t][w] */
void cdxo_gen_reward(const cdx_gen_params* g, uint64_t g0, uint64_t ng, uint32_t T, uint32_t W,
                     float* rewards, uint32_t* ids);

/* ---- metrics.cpp ------------------------------------------------------------------ */
/* metrics.cpp:12-19: returns trimmed length, *begin = offset of first kept byte */
size_t cdxo_trim(const char* s, size_t len, size_t* begin);
/* metrics.cpp:21-37 on interned ids: first-seen cluster sizes (+ leader index), returns m */
int cdxo_cluster_exact_ids(const uint32_t* ids, int n, int* sizes, int* leaders);
/* metrics.cpp:107-118 */
double cdxo_semantic_entropy(const int* sizes, int m, int n);
/* metrics.cpp:120-125 */
double cdxo_certaindex_entropy(const int* sizes, int m, int n);
/* metrics.cpp:127-137; returns 0 ok, 1 = "reward outside [0,1]", 2 = empty */
int cdxo_certaindex_reward(const double* r, size_t n, int agg_max, double* out);
/* metrics.cpp:159-171; signals[kind] with present[kind]; returns -1 on absent signal */
int cdxo_meets_thresholds(const double* signals, const int* present, const cdx_threshold* th,
                          uint32_t n_th);

/* ---- batched SC certaindex (K2): per (r,p) row over S samples ----------------------- */
int cdxo_sc_certaindex(const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                       const cdx_threshold* th, uint32_t n_th, double* hcert64, float* hcert,
                       uint32_t* meets_bits);
/* ... plus the majority fraction (largest cluster / S, runtime.cpp:317-334's plurality) */
double cdxo_majority_fraction(const int* sizes, int m, int n);
int cdxo_sc_certaindex_ex(const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                          const cdx_threshold* th, uint32_t n_th, double* hcert64, float* hcert,
                          double* maj64, float* maj, uint32_t* meets_bits);

/* ---- SPEC allocate + exclusive scan + stable compaction (K5), SPEC.md:404-412 ------- */
int cdxo_allocate_scan(const uint32_t* meets_bits, uint64_t R, uint32_t P,
                       const cdx_alloc_policy* pol, int64_t base_offset, int32_t* exit_knob,
                       uint8_t* reason, int32_t* granted, int64_t* offsets, uint32_t* kept,
                       uint64_t* n_kept, int64_t* tokens_saved);

/* ---- CoT probe window (K3), probe.cpp:48-102 ----------------------------------------- */
/* Literal prefix replay of should_exit / consistency / final_answer (O(P^2) per request). */
int cdxo_cot_exit_replay(const uint32_t* ids, const uint64_t* hes, const int64_t* offsets,
                         uint64_t R, uint32_t P, const cdx_probe_cfg* cfg, int32_t* exit_step,
                         uint8_t* reason, uint32_t* final_id, uint8_t* low_conf, float* ck);
/* Batched single-pass form (integer compares after host a_min). */
int cdxo_cot_exit_batched(const uint32_t* ids, const uint64_t* hes, const int64_t* offsets,
                          uint64_t R, uint32_t P, const cdx_probe_cfg* cfg, int32_t* exit_step,
                          uint8_t* reason, uint32_t* final_id, uint8_t* low_conf, float* ck);
/* a_min = min{a : (double)a/(double)w >= tau} */
int cdxo_cot_amin(int w, double tau);

/* ---- reward certaindex (K4), metrics.cpp:127-137 + runtime.cpp:279-292 ------------ */
/* agg[g] (0 mean, 1 max) per program; ids nullable.  Cumulative over steps.            */
int cdxo_reward_certaindex(const float* rewards, const uint32_t* ids, const uint8_t* agg,
                           uint64_t G, uint32_t T, uint32_t W, double* R64, float* Rout,
                           float* Hout);
int cdxo_reward_certaindex2(const float* rewards, const uint32_t* ids, const uint8_t* agg,
                            uint64_t G, uint32_t T, uint32_t W, double* R64, float* Rout,
                            float* Hout, double* H64);
int cdxo_reward_certaindex_f64(const double* rewards, const uint32_t* ids, const uint8_t* agg,
                               uint64_t G, uint32_t T, uint32_t W, double* R64, float* Rout,
                               float* Hout, double* H64);

/* ---- gang priority order (K6), SPEC.md:422-448,467-472 ----------------------------- */
int cdxo_gang_order(const cdx_prog_soa* progs, uint64_t N, const cdx_inter_policy* pol,
                    double now, uint32_t* order, uint64_t* n_out, uint8_t* escalated);
double cdxo_estimate_iteration_tokens(int64_t sum, uint32_t count, double prior);

/* ---- canonicalisation + hesitation (K1), metrics.cpp:12-37, probe.cpp:36-44 ------ */
/* ids = dense first-seen ids of trimmed strings; hes = flag_hesitation(raw string) */
int cdxo_canon_intern(const char* bytes, const uint64_t* offsets, uint64_t n,
                      const char* markers, const uint32_t* marker_offsets, uint32_t n_markers,
                      uint32_t* ids, uint8_t* hes, uint64_t* n_unique);
int cdxo_flag_hesitation(const char* s, size_t len, const char* markers,
                         const uint32_t* marker_offsets, uint32_t n_markers);

/* ---- epsilon-accuracy stop test at every CoT prefix (probe.cpp:104-120) -------------- */
int cdxo_cot_eps_stop(const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P, int k, double epsilon,
                      int32_t* step, uint8_t* state);

/* ---- aggregation (runtime.cpp:316-403) ------------------------------------------------ */
int cdxo_sc_aggregate(const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S, const int32_t* exit_knob,
                      uint32_t* answer);
int cdxo_reward_aggregate(const float* rw, const uint32_t* ids, const uint8_t* agg, uint64_t G, uint32_t T,
                          uint32_t W, const int32_t* exit_step, uint32_t* answer);
int cdxo_reward_aggregate_f64(const double* rw, const uint32_t* ids, const uint8_t* agg, uint64_t G, uint32_t T,
                              uint32_t W, const int32_t* exit_step, uint32_t* answer);

int cdxo_cot_meets(const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P, int w,
                   const cdx_threshold* th, uint32_t n_th, uint32_t* meets);
int cdxo_mixed_decide(const uint8_t* arch, const uint32_t* slot, const int32_t* knob, uint64_t N,
                      const uint32_t* const* meets, const uint32_t* words, const uint64_t* n,
                      const cdx_arch_policy* pol, uint8_t* decision, int32_t* grant, int32_t* cap,
                      int64_t* offsets, int64_t* total);

int cdxo_gang_order_mt(const cdx_prog_soa* s, uint64_t N, const cdx_inter_policy* pol, double now,
                       uint32_t* order, uint64_t* n_out, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
