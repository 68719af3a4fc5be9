/*
 * cdx_oracle.c — CPU restatement of the Certaindex hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared against; the
 * product (libcdx.so) never links or calls it.  Compiled with -O2 -ffp-contract=off so
 * that every floating-point expression rounds exactly as the reference's (x86-64 SSE2,
 * no FMA contraction) — see tests/test_oracle.py for the pinning against the reference's
 * own sources (oracle/_ref) and the SPEC.md examples.
 *
 * Reference citations are relative to /root/reference/proj/ unless they name SPEC.md.
 */
#include "cdx_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ===================================================================================== */
/* rng.hpp:25-34                                                                          */
/* ===================================================================================== */
uint64_t cdxo_mix64(uint64_t x) {
    /* splitmix64 finalizer, rng.hpp:25-30 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t cdxo_derive_seed(uint64_t master, uint64_t a, uint64_t b) {
    /* rng.hpp:32-34 */
    return cdxo_mix64(cdxo_mix64(master ^ cdxo_mix64(a)) ^ cdxo_mix64(b ^ 0xa5a5a5a5a5a5a5a5ULL));
}

/* ===================================================================================== */
/* Synthetic traces: counter-based restatement of the reference's answer/reward oracle.  */
/* The reference draws from per-program mt19937_64 streams (rng.hpp:36-121, runtime.cpp: */
/* 56-58); a sequential stream cannot be evaluated in parallel, so every draw here is a   */
/* pure function of (seed, program, sample, knob) built from the reference's own mixing  */
/* functions.  Semantics follow runtime.cpp:91-117 and generate_workload :430-460.       */
/* ===================================================================================== */
#define TAG_SOLVABLE 0x50175ULL
#define TAG_CONV 0xC0117ULL
#define TAG_DISTRACT 0xD15ULL
#define TAG_JITTER 0x8E3AULL
#define HES_DOMAIN (1ULL << 63)

static double unit53(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; } /* rng.hpp:41 */

int cdxo_solvable(const cdx_gen_params* g, uint64_t r) {
    /* generate_workload: spec.solvable = rng.uniform() < solvable_fraction (runtime.cpp:439) */
    return unit53(cdxo_derive_seed(g->seed, r, TAG_SOLVABLE)) < g->solvable_fraction;
}

uint32_t cdxo_convergence(const cdx_gen_params* g, uint64_t r) {
    /* generate_workload: true_convergence_knob = uniform_int(lo, hi) (runtime.cpp:443) */
    const uint64_t span = (uint64_t)(g->conv_hi - g->conv_lo) + 1;
    return g->conv_lo + (uint32_t)(cdxo_mix64(cdxo_derive_seed(g->seed, r, TAG_CONV)) % span);
}

uint32_t cdxo_answer(const cdx_gen_params* g, uint64_t r, uint64_t j, uint32_t knob) {
    /* sample_answer, runtime.cpp:91-102: unsolvable -> distractor; before convergence a
     * distractor w.p. noise_level, from convergence on w.p. residual_noise; else "S". */
    const uint64_t h = cdxo_derive_seed(g->seed, r, (j << 32) | knob);
    const uint32_t distractor = 1 + (uint32_t)(cdxo_mix64(h ^ TAG_DISTRACT) % (g->groups - 1));
    if (!cdxo_solvable(g, r)) return distractor;
    const double noise = knob < cdxo_convergence(g, r) ? g->noise_level : g->residual_noise;
    if (noise > 0.0 && unit53(h) < noise) return distractor;
    return 0;
}

int cdxo_hesitant(const cdx_gen_params* g, uint64_t r, uint32_t p) {
    /* next_cot_record, runtime.cpp:128-131: hesitant w.p. hesitation_prob */
    return g->hesitation_prob > 0.0 &&
           unit53(cdxo_derive_seed(g->seed, r, HES_DOMAIN | p)) < g->hesitation_prob;
}

uint32_t cdxo_reward_k(const cdx_gen_params* g, uint64_t r, uint64_t j, uint32_t knob) {
    /* sample_reward, runtime.cpp:104-117: mean rises linearly to the convergence knob
     * (start -> final), unsolvable programs sit at unsolvable_mean; the Beta draw is
     * replaced by a uniform jitter so that values stay on the 2^-24 grid (integer math). */
    int64_t mean;
    if (!cdxo_solvable(g, r)) {
        mean = g->reward_unsolvable_k;
    } else {
        const uint32_t conv = cdxo_convergence(g, r);
        const uint32_t k = knob < conv ? knob : conv;
        mean = (int64_t)g->reward_start_k +
               ((int64_t)g->reward_final_k - (int64_t)g->reward_start_k) * k / conv;
    }
    const uint64_t h = cdxo_derive_seed(g->seed, r, (j << 32) | knob);
    const int64_t span = 2 * (int64_t)g->reward_jitter_k + 1;
    const int64_t jit = (int64_t)(cdxo_mix64(h ^ TAG_JITTER) % (uint64_t)span) - g->reward_jitter_k;
    int64_t v = mean + jit;
    if (v < 0) v = 0;
    if (v > (1 << 24)) v = 1 << 24;
    return (uint32_t)v;
}

static uint32_t answer_ps(const cdx_gen_params* g, int solvable, uint32_t conv, uint64_t r, uint64_t j,
                          uint32_t knob) {
    /* cdxo_answer with the per-program draws hoisted */
    const uint64_t h = cdxo_derive_seed(g->seed, r, (j << 32) | knob);
    const uint32_t distractor = 1 + (uint32_t)(cdxo_mix64(h ^ TAG_DISTRACT) % (g->groups - 1));
    if (!solvable) return distractor;
    const double noise = knob < conv ? g->noise_level : g->residual_noise;
    if (noise > 0.0 && unit53(h) < noise) return distractor;
    return 0;
}

void cdxo_gen_sc(const cdx_gen_params* g, uint64_t r0, uint64_t nreq, uint32_t P, uint32_t S,
                 uint32_t* ids) {
    for (uint64_t i = 0; i < nreq; ++i) {
        const int sv = cdxo_solvable(g, r0 + i);
        const uint32_t conv = cdxo_convergence(g, r0 + i);
        for (uint32_t p = 0; p < P; ++p)
            for (uint32_t s = 0; s < S; ++s)
                ids[(i * P + p) * S + s] = answer_ps(g, sv, conv, r0 + i, s, p + 1);
    }
}

typedef struct {
    const cdx_gen_params* g;
    uint64_t r0, n;
    uint32_t P, S;
    uint32_t* ids;
} gen_job;

static void* gen_sc_worker(void* a) {
    gen_job* j = (gen_job*)a;
    cdxo_gen_sc(j->g, j->r0, j->n, j->P, j->S, j->ids);
    return NULL;
}

void cdxo_gen_sc_mt(const cdx_gen_params* g, uint64_t r0, uint64_t nreq, uint32_t P, uint32_t S,
                    uint32_t* ids, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    pthread_t th[256];
    gen_job jobs[256];
    const uint64_t chunk = (nreq + (uint64_t)nthreads - 1) / (uint64_t)nthreads;
    int started = 0;
    for (int t = 0; t < nthreads; ++t) {
        const uint64_t b = (uint64_t)t * chunk;
        if (b >= nreq) break;
        jobs[t].g = g;
        jobs[t].r0 = r0 + b;
        jobs[t].n = (b + chunk > nreq) ? nreq - b : chunk;
        jobs[t].P = P;
        jobs[t].S = S;
        jobs[t].ids = ids + b * P * S;
        pthread_create(&th[t], NULL, gen_sc_worker, &jobs[t]);
        ++started;
    }
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
}

void cdxo_gen_cot(const cdx_gen_params* g, uint64_t r0, uint64_t nreq, uint32_t P, uint32_t* ids,
                  uint64_t* hes) {
    const uint32_t words = (P + 63) / 64;
    for (uint64_t i = 0; i < nreq; ++i) {
        for (uint32_t w = 0; w < words; ++w) hes[i * words + w] = 0;
        for (uint32_t p = 0; p < P; ++p) {
            const uint32_t a = cdxo_answer(g, r0 + i, 0, p + 1);
            const int h = cdxo_hesitant(g, r0 + i, p);
            /* runtime.cpp:131: the hesitant record's answer is "wait, " + ans -> id M + a */
            ids[i * P + p] = h ? g->groups + a : a;
            if (h) hes[i * words + p / 64] |= 1ULL << (p % 64);
        }
    }
}

void cdxo_gen_reward(const cdx_gen_params* g, uint64_t g0, uint64_t ng, uint32_t T, uint32_t W,
                     float* rewards, uint32_t* ids) {
    for (uint64_t i = 0; i < ng; ++i)
        for (uint32_t t = 0; t < T; ++t)
            for (uint32_t w = 0; w < W; ++w) {
                const uint64_t o = (i * T + t) * W + w;
                if (rewards) rewards[o] = (float)cdxo_reward_k(g, g0 + i, w, t + 1) * 0x1.0p-24f;
                if (ids) ids[o] = cdxo_answer(g, g0 + i, w, t + 1);
            }
}

/* ===================================================================================== */
/* metrics.cpp                                                                            */
/* ===================================================================================== */
static int is_space(char c) {
    /* metrics.cpp:13-15 */
    return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v';
}

size_t cdxo_trim(const char* s, size_t len, size_t* begin) {
    /* metrics.cpp:12-19 */
    size_t b = 0, e = len;
    while (b < e && is_space(s[b])) ++b;
    while (e > b && is_space(s[e - 1])) --e;
    if (begin) *begin = b;
    return e - b;
}

int cdxo_cluster_exact_ids(const uint32_t* ids, int n, int* sizes, int* leaders) {
    /* metrics.cpp:21-37: clusters in first-seen order; equality of interned ids is
     * equality of the trimmed bytes (the unordered_map<string_view> key, :28-29). */
    int m = 0;
    for (int i = 0; i < n; ++i) {
        int k = 0;
        while (k < m && ids[leaders[k]] != ids[i]) ++k;
        if (k == m) {
            leaders[m] = i;
            sizes[m] = 1;
            ++m;
        } else {
            ++sizes[k];
        }
    }
    return m;
}

double cdxo_semantic_entropy(const int* sizes, int m, int n) {
    /* metrics.cpp:107-118: h -= p * log(p) in cluster order, then max(0, h) */
    const double nn = (double)n;
    double h = 0.0;
    for (int k = 0; k < m; ++k) {
        const double p = (double)sizes[k] / nn;
        h -= p * log(p);
    }
    return (0.0 < h) ? h : 0.0; /* std::max(0.0, h) */
}

double cdxo_certaindex_entropy(const int* sizes, int m, int n) {
    /* metrics.cpp:120-125 */
    if (n == 1) return 1.0;
    const double log_n = log((double)n);
    const double h = cdxo_semantic_entropy(sizes, m, n);
    const double v = (log_n - h) / log_n;
    return v < 0.0 ? 0.0 : (1.0 < v ? 1.0 : v); /* std::clamp(v, 0.0, 1.0) */
}

int cdxo_certaindex_reward(const double* r, size_t n, int agg_max, double* out) {
    /* metrics.cpp:127-137 */
    if (n == 0) return 2;
    for (size_t i = 0; i < n; ++i)
        if (r[i] < 0.0 || r[i] > 1.0) return 1;
    if (agg_max) {
        size_t best = 0; /* std::max_element: first maximal element, comparing with < */
        for (size_t i = 1; i < n; ++i)
            if (r[best] < r[i]) best = i;
        *out = r[best];
        return 0;
    }
    double s = 0.0; /* std::accumulate left fold */
    for (size_t i = 0; i < n; ++i) s = s + r[i];
    *out = s / (double)n;
    return 0;
}

int cdxo_meets_thresholds(const double* signals, const int* present, const cdx_threshold* th,
                          uint32_t n_th) {
    /* metrics.cpp:159-171: inclusive comparisons, AND, absent signal -> error */
    for (uint32_t i = 0; i < n_th; ++i) {
        if (!present[th[i].signal]) return -1;
        const double v = signals[th[i].signal];
        const int ok = th[i].dir == CDX_DIR_GE ? v >= th[i].cutoff : v <= th[i].cutoff;
        if (!ok) return 0;
    }
    return 1;
}

/* ===================================================================================== */
/* K2 restated: SC certaindex per (r,p) row (runtime.cpp:266-271 applied per probe row)  */
/* ===================================================================================== */
/* Majority-fraction certaindex of one clustering: the weight of the answer the reference's
 * plurality vote returns, over n.  runtime.cpp:317-334 weighted_plurality (softmax off): every
 * path weighs 1.0, clusters are visited in first-seen order and a later cluster wins only with
 * a strictly larger weight, so the winner is the first largest cluster; its weight is its size
 * (an exact double sum of 1.0s).                                                              */
double cdxo_majority_fraction(const int* sizes, int m, int n) {
    double best_w = -1.0;
    for (int k = 0; k < m; ++k)
        if ((double)sizes[k] > best_w) best_w = (double)sizes[k];
    return best_w / (double)n;
}

int cdxo_sc_certaindex(const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                       const cdx_threshold* th, uint32_t n_th, double* hcert64, float* hcert,
                       uint32_t* meets_bits) {
    return cdxo_sc_certaindex_ex(ids, R, P, S, th, n_th, hcert64, hcert, NULL, NULL, meets_bits);
}

int cdxo_sc_certaindex_ex(const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                          const cdx_threshold* th, uint32_t n_th, double* hcert64, float* hcert,
                          double* maj64, float* maj, uint32_t* meets_bits) {
    if (S == 0) return CDX_EINVAL;
    int* sizes = (int*)malloc(sizeof(int) * S);
    int* leaders = (int*)malloc(sizeof(int) * S);
    const uint32_t words = (P + 31) / 32;
    double sig[5] = {0, 0, 0, 0, 0};
    int present[5] = {1, 0, 0, 0, 1};
    int st = CDX_OK;
    for (uint64_t r = 0; r < R && st == CDX_OK; ++r) {
        if (meets_bits)
            for (uint32_t w = 0; w < words; ++w) meets_bits[r * words + w] = 0;
        for (uint32_t p = 0; p < P; ++p) {
            const uint64_t row = r * P + p;
            const int m = cdxo_cluster_exact_ids(ids + row * S, (int)S, sizes, leaders);
            const double hc = cdxo_certaindex_entropy(sizes, m, (int)S);
            const double mf = cdxo_majority_fraction(sizes, m, (int)S);
            if (hcert64) hcert64[row] = hc;
            if (hcert) hcert[row] = (float)hc;
            if (maj64) maj64[row] = mf;
            if (maj) maj[row] = (float)mf;
            sig[CDX_SIG_ENTROPY] = hc;
            sig[CDX_SIG_MAJORITY] = mf;
            const int ok = cdxo_meets_thresholds(sig, present, th, n_th);
            if (ok < 0) {
                st = CDX_EINVAL;
                break;
            }
            if (ok && meets_bits) meets_bits[r * words + p / 32] |= 1u << (p % 32);
        }
    }
    free(sizes);
    free(leaders);
    return st;
}

/* ===================================================================================== */
/* K5 restated: SPEC.md:404-412 allocate, then exclusive scan + stable compaction         */
/* ===================================================================================== */
int cdxo_allocate_scan(const uint32_t* meets_bits, uint64_t R, uint32_t P,
                       const cdx_alloc_policy* pol, int64_t base_offset, int32_t* exit_knob,
                       uint8_t* reason, int32_t* granted, int64_t* offsets, uint32_t* kept,
                       uint64_t* n_kept, int64_t* tokens_saved) {
    const int cap = pol->resource_cap;
    if (cap < 1 || (uint32_t)cap > P) return CDX_EINVAL;
    if (pol->kind != CDX_POL_EVEN && (pol->detect_at < 1 || pol->detect_at > cap))
        return CDX_EINVAL; /* SPEC.md:392 detect_at_knob <= resource_cap */
    if (pol->kind == CDX_POL_K_STEP_THRESHOLD && pol->recheck_every < 1) return CDX_EINVAL;
    if (pol->kind != CDX_POL_EVEN && pol->kind != CDX_POL_STATIC_THRESHOLD &&
        pol->kind != CDX_POL_K_STEP_THRESHOLD)
        return CDX_EINVAL;
    const uint32_t words = (P + 31) / 32;
    int64_t acc = base_offset, saved = 0;
    uint64_t nk = 0;
    for (uint64_t r = 0; r < R; ++r) {
        int ek = cap;
        uint8_t why = CDX_EXIT_BUDGET; /* "always terminate at resource_cap" SPEC.md:407 */
        if (pol->kind != CDX_POL_EVEN) {
            /* static_threshold: test once at detect_at; k_step: re-test every e units */
            for (int k = pol->detect_at; k <= cap;
                 k += (pol->kind == CDX_POL_K_STEP_THRESHOLD ? pol->recheck_every : cap + 1)) {
                const uint32_t p = (uint32_t)(k - 1);
                if ((meets_bits[r * words + p / 32] >> (p % 32)) & 1u) {
                    ek = k;
                    why = CDX_EXIT_CERTAIN;
                    break;
                }
            }
        }
        const int detect = pol->kind == CDX_POL_EVEN ? 0 : pol->detect_at;
        if (exit_knob) exit_knob[r] = ek;
        if (reason) reason[r] = why;
        if (granted) granted[r] = ek;
        if (offsets) offsets[r] = acc;
        acc += (int64_t)ek * pol->tokens_per_unit;
        saved += (int64_t)(cap - ek) * pol->tokens_per_unit;
        if (ek > detect) {
            if (kept) kept[nk] = (uint32_t)r;
            ++nk;
        }
    }
    if (n_kept) *n_kept = nk;
    if (tokens_saved) *tokens_saved = saved;
    return CDX_OK;
}

/* ===================================================================================== */
/* K3 restated: CoT probe window (probe.cpp:48-102)                                       */
/* ===================================================================================== */
static int validate_probe_cfg(const cdx_probe_cfg* c) {
    /* probe.cpp:19-25 */
    if (c->interval_tokens < 1 || c->window < 1) return CDX_EINVAL;
    if (c->threshold <= 0.0 || c->threshold > 1.0) return CDX_EINVAL;
    if (c->max_tokens < 1) return CDX_EINVAL;
    return CDX_OK;
}

static int64_t probe_offset(const int64_t* offsets, uint64_t r, uint32_t P, uint32_t p,
                            const cdx_probe_cfg* c) {
    return offsets ? offsets[r * P + p] : (int64_t)(p + 1) * c->interval_tokens;
}

static int hes_bit(const uint64_t* hes, uint64_t r, uint32_t P, uint32_t p) {
    const uint32_t words = (P + 63) / 64;
    return (int)((hes[r * words + p / 64] >> (p % 64)) & 1ULL);
}

/* probe.cpp:64-75 consistency over records [0, n) of request r at k = latest step:
 * returns -1 ("nullopt") when fewer than w usable records exist, else agree count. */
static int consistency_prefix(const uint32_t* ids, const uint64_t* hes, uint64_t r, uint32_t P,
                              uint32_t n, int w) {
    /* usable_up_to (probe.cpp:53-60): non-hesitant records, step_index <= k (all, since
     * step_index = p+1 is increasing and k is the latest) */
    int usable = 0;
    for (uint32_t p = 0; p < n; ++p) usable += !hes_bit(hes, r, P, p);
    if (usable < w) return -1;
    /* window: last w usable records; compare against the last usable's answer */
    int last = -1;
    for (int p = (int)n - 1; p >= 0; --p)
        if (!hes_bit(hes, r, P, (uint32_t)p)) {
            last = p;
            break;
        }
    int agree = 0, seen = 0;
    for (int p = last; p >= 0 && seen < w; --p) {
        if (hes_bit(hes, r, P, (uint32_t)p)) continue;
        ++seen;
        if (ids[r * P + (uint32_t)p] == ids[r * P + (uint32_t)last]) ++agree;
    }
    return agree;
}

static void final_answer_prefix(const uint32_t* ids, const uint64_t* hes, uint64_t r, uint32_t P,
                                uint32_t n, int certain, uint32_t* fid, uint8_t* low) {
    /* probe.cpp:87-102: certain -> the terminating (= latest) record's answer; else the
     * latest non-hesitant answer; else the latest answer, low_confidence. */
    if (certain) {
        *fid = ids[r * P + n - 1];
        *low = 0;
        return;
    }
    for (int p = (int)n - 1; p >= 0; --p)
        if (!hes_bit(hes, r, P, (uint32_t)p)) {
            *fid = ids[r * P + (uint32_t)p];
            *low = 0;
            return;
        }
    *fid = ids[r * P + n - 1];
    *low = 1;
}

int cdxo_cot_exit_replay(const uint32_t* ids, const uint64_t* hes, const int64_t* offsets,
                         uint64_t R, uint32_t P, const cdx_probe_cfg* cfg, int32_t* exit_step,
                         uint8_t* reason, uint32_t* final_id, uint8_t* low_conf, float* ck) {
    if (validate_probe_cfg(cfg)) return CDX_EINVAL;
    if (P == 0) return CDX_EINVAL;
    const int w = cfg->window;
    for (uint64_t r = 0; r < R; ++r) {
        int32_t ex = -1;
        uint8_t why = CDX_EXIT_CONTINUE;
        for (uint32_t n = 1; n <= P; ++n) {
            /* should_exit on the prefix of n records (probe.cpp:77-85) */
            const int agree = consistency_prefix(ids, hes, r, P, n, w);
            const double c = agree < 0 ? 0.0 : (double)agree / (double)w;
            if (ck) ck[r * P + n - 1] = (float)c; /* update_certaindex: value_or(0.0) */
            if (ex >= 0) continue;
            if (agree >= 0 && c >= cfg->threshold) {
                ex = (int32_t)n - 1;
                why = CDX_EXIT_CERTAIN;
            } else if (probe_offset(offsets, r, P, n - 1, cfg) >= cfg->max_tokens) {
                ex = (int32_t)n - 1;
                why = CDX_EXIT_BUDGET;
            }
            if (ex >= 0 && !ck) break;
        }
        exit_step[r] = ex;
        reason[r] = why;
        /* terminate() (runtime.cpp:405-411) then final_answer on the trace so far; a
         * request that never exits reports the full trace (criteria_external). */
        const uint32_t n = ex >= 0 ? (uint32_t)ex + 1 : P;
        uint32_t fid;
        uint8_t low;
        final_answer_prefix(ids, hes, r, P, n, why == CDX_EXIT_CERTAIN, &fid, &low);
        if (final_id) final_id[r] = fid;
        if (low_conf) low_conf[r] = low;
    }
    return CDX_OK;
}

int cdxo_cot_amin(int w, double tau) {
    for (int a = 0; a <= w; ++a)
        if ((double)a / (double)w >= tau) return a;
    return w + 1; /* unreachable for tau <= 1 */
}

int cdxo_cot_exit_batched(const uint32_t* ids, const uint64_t* hes, const int64_t* offsets,
                          uint64_t R, uint32_t P, const cdx_probe_cfg* cfg, int32_t* exit_step,
                          uint8_t* reason, uint32_t* final_id, uint8_t* low_conf, float* ck) {
    /* One pass per request: the window of the last w usable answers slides over the
     * non-hesitant probes; certain_step = first non-hesitant probe whose window is full
     * with agree >= a_min; budget_step = first probe with offset >= max_tokens; certainty
     * wins ties.  Equivalent to the prefix replay above. */
    if (validate_probe_cfg(cfg)) return CDX_EINVAL;
    if (P == 0) return CDX_EINVAL;
    const int w = cfg->window;
    const int amin = cdxo_cot_amin(w, cfg->threshold);
    uint32_t* win = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)w);
    for (uint64_t r = 0; r < R; ++r) {
        int usable = 0, head = 0, last_agree = -1;
        int32_t cstep = -1, bstep = -1;
        int last_usable = -1;
        for (uint32_t p = 0; p < P; ++p) {
            if (!hes_bit(hes, r, P, p)) {
                const uint32_t v = ids[r * P + p];
                win[head] = v;
                head = (head + 1) % w;
                ++usable;
                last_usable = (int)p;
                if (usable >= w) {
                    int agree = 0;
                    for (int i = 0; i < w; ++i) agree += win[i] == v;
                    last_agree = agree;
                    if (cstep < 0 && agree >= amin) cstep = (int32_t)p;
                }
            }
            if (ck) ck[r * P + p] = last_agree < 0 ? 0.0f : (float)((double)last_agree / (double)w);
            if (bstep < 0 && probe_offset(offsets, r, P, p, cfg) >= cfg->max_tokens)
                bstep = (int32_t)p;
            if (!ck && cstep >= 0) break;
            if (!ck && bstep >= 0 && cstep < 0 && (uint32_t)bstep == p) break;
        }
        int32_t ex = -1;
        uint8_t why = CDX_EXIT_CONTINUE;
        if (cstep >= 0 && (bstep < 0 || cstep <= bstep)) {
            ex = cstep;
            why = CDX_EXIT_CERTAIN;
        } else if (bstep >= 0) {
            ex = bstep;
            why = CDX_EXIT_BUDGET;
        }
        exit_step[r] = ex;
        reason[r] = why;
        const uint32_t n = ex >= 0 ? (uint32_t)ex + 1 : P;
        uint32_t fid;
        uint8_t low;
        (void)last_usable;
        final_answer_prefix(ids, hes, r, P, n, why == CDX_EXIT_CERTAIN, &fid, &low);
        if (final_id) final_id[r] = fid;
        if (low_conf) low_conf[r] = low;
    }
    free(win);
    return CDX_OK;
}

/* ===================================================================================== */
/* K4 restated: MCTS/Rebase update_certaindex, cumulative (runtime.cpp:279-292)           */
/* ===================================================================================== */
int cdxo_reward_certaindex(const float* rewards, const uint32_t* ids, const uint8_t* agg,
                           uint64_t G, uint32_t T, uint32_t W, double* R64, float* Rout,
                           float* Hout) {
    return cdxo_reward_certaindex2(rewards, ids, agg, G, T, W, R64, Rout, Hout, NULL);
}

/* The same with the FP64 certaindex as well (H64, nullable): the value the thresholds are
 * applied to (runtime.cpp:279-292 -> combined_meets_thresholds, metrics.cpp:159-171). */
static int reward_certaindex_any(const float* rewards, const double* rewards64, const uint32_t* ids,
                                 const uint8_t* agg, uint64_t G, uint32_t T, uint32_t W, double* R64,
                                 float* Rout, float* Hout, double* H64);
int cdxo_reward_certaindex2(const float* rewards, const uint32_t* ids, const uint8_t* agg,
                            uint64_t G, uint32_t T, uint32_t W, double* R64, float* Rout,
                            float* Hout, double* H64) {
    return reward_certaindex_any(rewards, NULL, ids, agg, G, T, W, R64, Rout, Hout, H64);
}
/* f64 rewards (RewardSet holds doubles, metrics.hpp:74-77) */
int cdxo_reward_certaindex_f64(const double* rewards, const uint32_t* ids, const uint8_t* agg,
                               uint64_t G, uint32_t T, uint32_t W, double* R64, float* Rout,
                               float* Hout, double* H64) {
    return reward_certaindex_any(NULL, rewards, ids, agg, G, T, W, R64, Rout, Hout, H64);
}
static int reward_certaindex_any(const float* rewards, const double* rewards64, const uint32_t* ids,
                                 const uint8_t* agg, uint64_t G, uint32_t T, uint32_t W, double* R64,
                                 float* Rout, float* Hout, double* H64) {
    const size_t n_all = (size_t)T * W;
    int* sizes = (int*)malloc(sizeof(int) * (n_all ? n_all : 1));
    int* leaders = (int*)malloc(sizeof(int) * (n_all ? n_all : 1));
    int st = CDX_OK;
    for (uint64_t g = 0; g < G; ++g) {
        const float* rw = rewards ? rewards + g * n_all : NULL;
        const double* rw64 = rewards64 ? rewards64 + g * n_all : NULL;
        /* RewardSet over all paths so far; certaindex_reward validates every reward and
         * folds left (mean) or takes the first maximum (max).  Incremental evaluation of
         * the same left fold / running first-maximum. */
        double sum = 0.0;
        double best = 0.0;
        int bad = 0;
        for (uint32_t t = 0; t < T; ++t) {
            for (uint32_t w = 0; w < W; ++w) {
                const double v = rw64 ? rw64[(size_t)t * W + w] : (double)rw[(size_t)t * W + w];
                if (v < 0.0 || v > 1.0) bad = 1;
                sum = sum + v;
                if (t == 0 && w == 0)
                    best = v;
                else if (best < v)
                    best = v;
            }
            if (bad) {
                st = CDX_EINVAL;
                break;
            }
            const size_t n = (size_t)(t + 1) * W;
            const double rv = agg[g] == CDX_AGG_MAX ? best : sum / (double)n;
            if (R64) R64[g * T + t] = rv;
            if (Rout) Rout[g * T + t] = (float)rv;
            if (ids && (Hout || H64)) {
                const int m = cdxo_cluster_exact_ids(ids + g * n_all, (int)n, sizes, leaders);
                const double h = cdxo_certaindex_entropy(sizes, m, (int)n);
                if (Hout) Hout[g * T + t] = (float)h;
                if (H64) H64[g * T + t] = h;
            }
        }
        if (st) break;
    }
    free(sizes);
    free(leaders);
    return st;
}

/* ===================================================================================== */
/* K6 restated: SPEC.md:422-448 (gang order, escalation, SJF estimate), :467-472         */
/* ===================================================================================== */
double cdxo_estimate_iteration_tokens(int64_t sum, uint32_t count, double prior) {
    /* arithmetic mean of completed iteration token counts, else prior */
    return count ? (double)sum / (double)count : prior;
}

typedef struct {
    int esc;
    double key;
    double arrival;
    uint32_t id;
} gang_item;

static int gang_cmp(const void* a, const void* b) {
    const gang_item* x = (const gang_item*)a;
    const gang_item* y = (const gang_item*)b;
    if (x->esc != y->esc) return x->esc ? -1 : 1; /* escalated first */
    if (x->key < y->key) return -1;
    if (y->key < x->key) return 1;
    if (x->arrival < y->arrival) return -1; /* tie-break (priority, arrival, id) :470 */
    if (y->arrival < x->arrival) return 1;
    return x->id < y->id ? -1 : (x->id > y->id ? 1 : 0);
}

int cdxo_gang_order(const cdx_prog_soa* s, uint64_t N, const cdx_inter_policy* pol, double now,
                    uint32_t* order, uint64_t* n_out, uint8_t* escalated) {
    if (!(pol->starvation_limit > 0.0)) return CDX_EINVAL;
    if (pol->order != CDX_ORDER_FIFO && pol->order != CDX_ORDER_SJF) return CDX_EINVAL;
    gang_item* it = (gang_item*)malloc(sizeof(gang_item) * (N ? N : 1));
    uint64_t n = 0;
    for (uint64_t i = 0; i < N; ++i) {
        /* escalate: inclusive (now - last_service) >= limit */
        const int esc = (now - s->last_service[i]) >= pol->starvation_limit;
        if (escalated) escalated[i] = (uint8_t)esc;
        if (s->terminated[i]) continue;
        double key;
        if (esc || pol->order == CDX_ORDER_FIFO) {
            key = s->arrival[i]; /* FIFO among escalated */
        } else {
            /* SJF estimated remaining work = est tokens/iter x remaining knob, :425,469 */
            const double est = cdxo_estimate_iteration_tokens(s->iter_tok_sum[i], s->iter_count[i],
                                                              pol->prior_tokens);
            const int64_t rem = (int64_t)s->cap[i] - (int64_t)s->knob[i];
            key = est * (double)(rem > 0 ? rem : 0);
        }
        it[n].esc = esc;
        it[n].key = key;
        it[n].arrival = s->arrival[i];
        it[n].id = s->program_id ? s->program_id[i] : s->id_base + (uint32_t)i;
        ++n;
    }
    qsort(it, n, sizeof(gang_item), gang_cmp); /* total order => unique result */
    for (uint64_t i = 0; i < n; ++i) order[i] = it[i].id;
    *n_out = n;
    free(it);
    return CDX_OK;
}

/* ===================================================================================== */
/* K1 restated: trim + exact-match interning (metrics.cpp:12-37), flag_hesitation        */
/* (probe.cpp:36-44)                                                                      */
/* ===================================================================================== */
int cdxo_flag_hesitation(const char* s, size_t len, const char* markers,
                         const uint32_t* moff, uint32_t n_markers) {
    /* ASCII tolower of the answer (std::tolower in the "C" locale), then any NON-EMPTY
     * marker as a substring; markers are not lowered. */
    for (uint32_t k = 0; k < n_markers; ++k) {
        const char* m = markers + moff[k];
        const size_t ml = moff[k + 1] - moff[k];
        if (ml == 0 || ml > len) continue;
        for (size_t i = 0; i + ml <= len; ++i) {
            size_t j = 0;
            for (; j < ml; ++j) {
                unsigned char c = (unsigned char)s[i + j];
                if (c >= 'A' && c <= 'Z') c = (unsigned char)(c + 32);
                if ((char)c != m[j]) break;
            }
            if (j == ml) return 1;
        }
    }
    return 0;
}

typedef struct {
    const char* p;
    size_t n;
    uint32_t id;
    int used;
} intern_slot;

static uint64_t fnv1a(const char* p, size_t n) {
    uint64_t h = 1469598103934665603ULL;
    for (size_t i = 0; i < n; ++i) h = (h ^ (unsigned char)p[i]) * 1099511628211ULL;
    return h;
}

int cdxo_canon_intern(const char* bytes, const uint64_t* offsets, uint64_t n, const char* markers,
                      const uint32_t* marker_offsets, uint32_t n_markers, uint32_t* ids,
                      uint8_t* hes, uint64_t* n_unique) {
    uint64_t cap = 16;
    while (cap < 2 * n + 16) cap <<= 1;
    intern_slot* tab = (intern_slot*)calloc(cap, sizeof(intern_slot));
    uint32_t next = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const char* s = bytes + offsets[i];
        const size_t len = offsets[i + 1] - offsets[i];
        size_t b;
        const size_t tl = cdxo_trim(s, len, &b);
        const char* t = s + b;
        uint64_t h = fnv1a(t, tl) & (cap - 1);
        while (tab[h].used && !(tab[h].n == tl && memcmp(tab[h].p, t, tl) == 0)) h = (h + 1) & (cap - 1);
        if (!tab[h].used) {
            tab[h].used = 1;
            tab[h].p = t;
            tab[h].n = tl;
            tab[h].id = next++;
        }
        ids[i] = tab[h].id;
        if (hes) hes[i] = (uint8_t)cdxo_flag_hesitation(s, len, markers, marker_offsets, n_markers);
    }
    *n_unique = next;
    free(tab);
    return CDX_OK;
}

/* ===================================================================================== */
/* Aggregation, runtime.cpp:316-403 (weighted_plurality :316-336, aggregate_prefix       */
/* :345-403): SC plurality, MCTS first argmax, Rebase exp-weighted plurality over the     */
/* last full layer.  exp() is this libm's, the same glibc the reference links.           */
/* ===================================================================================== */
/* weighted plurality over n answers (ids) with optional weights: first-seen clusters,
 * strict > over the summed weights (weights summed in path order, starting from 0.0) */
static uint32_t plurality_ids(const uint32_t* v, const double* w, int n) {
    uint32_t keys[1024];
    double tot[1024];
    int m = 0;
    for (int i = 0; i < n; ++i) {
        int c = 0;
        while (c < m && keys[c] != v[i]) ++c;
        if (c == m) {
            keys[m] = v[i];
            tot[m] = 0.0;
            ++m;
        }
        tot[c] += w ? w[i] : 1.0;
    }
    uint32_t best = 0xffffffffu; /* std::string best stays empty when nothing beats -1.0 */
    double bw = -1.0;
    for (int c = 0; c < m; ++c)
        if (tot[c] > bw) {
            bw = tot[c];
            best = keys[c];
        }
    return best;
}

int cdxo_sc_aggregate(const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S, const int32_t* exit_knob,
                      uint32_t* answer) {
    if (S == 0 || S > 1024 || P == 0) return CDX_EINVAL;
    for (uint64_t r = 0; r < R; ++r) {
        if (exit_knob[r] < 1 || (uint32_t)exit_knob[r] > P) return CDX_EINVAL;
        answer[r] = plurality_ids(ids + (r * P + (uint64_t)(exit_knob[r] - 1)) * S, NULL, (int)S);
    }
    return CDX_OK;
}

/* rewards as doubles (PathSample::reward), either from f32 or f64 storage */
static int reward_aggregate_any(const float* rwf, const double* rwd, const uint32_t* ids, const uint8_t* agg,
                                uint64_t G, uint32_t T, uint32_t W, const int32_t* exit_step, uint32_t* answer) {
    if (W == 0 || W > 1024 || T == 0) return CDX_EINVAL;
    double w[1024];
#define RW(i) (rwd ? rwd[i] : (double)rwf[i])
    for (uint64_t g = 0; g < G; ++g) {
        const int32_t t = exit_step[g];
        if (t < 0 || (uint32_t)t >= T) return CDX_EINVAL;
        const uint64_t base = g * T * W;
        if (agg[g] == CDX_AGG_MEAN) { /* MCTS: runtime.cpp:380-389 */
            const uint64_t n = (uint64_t)(t + 1) * W;
            uint64_t best = 0;
            for (uint64_t i = 1; i < n; ++i)
                if (RW(base + i) > RW(base + best)) best = i;
            answer[g] = ids[base + best];
        } else { /* Rebase: runtime.cpp:357-378, last full layer = step t; std::exp :324 */
            const uint64_t l0 = base + (uint64_t)t * W;
            for (uint32_t i = 0; i < W; ++i) w[i] = exp(RW(l0 + i));
            answer[g] = plurality_ids(ids + l0, w, (int)W);
        }
    }
#undef RW
    return CDX_OK;
}

int cdxo_reward_aggregate(const float* rw, const uint32_t* ids, const uint8_t* agg, uint64_t G, uint32_t T,
                          uint32_t W, const int32_t* exit_step, uint32_t* answer) {
    return reward_aggregate_any(rw, NULL, ids, agg, G, T, W, exit_step, answer);
}

int cdxo_reward_aggregate_f64(const double* rw, const uint32_t* ids, const uint8_t* agg, uint64_t G, uint32_t T,
                              uint32_t W, const int32_t* exit_step, uint32_t* answer) {
    return reward_aggregate_any(NULL, rw, ids, agg, G, T, W, exit_step, answer);
}

/* ===================================================================================== */
/* Epsilon-accuracy stop test, probe.cpp:104-120 over theory.cpp:100-146, at every prefix */
/* of every CoT trace: state 0 nullopt / 1 false / 2 true; step = first true (or -1).     */
/* Restated with the reference's dense per-group vectors (window_counts, tv_raw).         */
/* ===================================================================================== */
static void eps_window_counts(const int* g, int start, int len, int m, double* out) {
    for (int i = 0; i < m; ++i) out[i] = 0.0;
    for (int t = 0; t < len; ++t) out[g[start + t]] += 1.0;
    for (int i = 0; i < m; ++i) out[i] /= (double)len;
}
static double eps_tv(const double* a, const double* b, int m) {
    double l1 = 0.0;
    for (int i = 0; i < m; ++i) l1 += fabs(a[i] - b[i]);
    return 0.5 * l1;
}
static int eps_test(const int* g, int n, int k, double epsilon) {
    if (n < 2 * k) return 0;
    const int anchor = n - 2 * k;
    int m = 0;
    for (int i = 0; i < n; ++i)
        if (g[i] + 1 > m) m = g[i] + 1;
    const double limit = epsilon / 3.0;
    double ref[1024], probe[1024];
    eps_window_counts(g, anchor, k, m, ref);
    for (int j = 1; j <= k; ++j) {
        eps_window_counts(g, anchor + j, k, m, probe);
        if (eps_tv(ref, probe, m) > limit) return 1;
    }
    if (k >= 2) {
        eps_window_counts(g, anchor, k - 1, m, ref);
        for (int j = 1; j <= k - 1; ++j) {
            eps_window_counts(g, anchor + j, k - 1, m, probe);
            if (eps_tv(ref, probe, m) > limit) return 1;
        }
    }
    return 2;
}

int cdxo_cot_eps_stop(const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P, int k, double epsilon,
                      int32_t* step, uint8_t* state) {
    if (k < 1 || !(epsilon > 0.0) || P == 0 || P > 1024) return CDX_EINVAL;
    const uint32_t hw = (P + 63) / 64;
    int g[1024];
    uint32_t seen[1024];
    for (uint64_t r = 0; r < R; ++r) {
        int n = 0, m = 0;
        int32_t first = -1;
        for (uint32_t p = 0; p < P; ++p) {
            if (!((hes[r * hw + p / 64] >> (p % 64)) & 1ull)) {
                const uint32_t v = ids[r * P + p];
                int c = 0;
                while (c < m && seen[c] != v) ++c;
                if (c == m) seen[m++] = v;
                g[n++] = c;
            }
            const int st = eps_test(g, n, k, epsilon);
            if (state) state[r * P + p] = (uint8_t)st;
            if (st == 2 && first < 0) first = (int32_t)p;
        }
        step[r] = first;
    }
    return CDX_OK;
}

/* ===================================================================================== */
/* Mixed-archetype step (cdx_mixed_allocate): the CoT signal of update_certaindex as     */
/* threshold bits, then scheduler.allocate at each program's current knob.              */
/* ===================================================================================== */
/* runtime.cpp:293-299: C = consistency(records, latest step, w).value_or(0.0) after probe p
 * (probe.cpp:64-75), then combined_meets_thresholds({C}, th) (metrics.cpp:159-171). */
int cdxo_cot_meets(const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P, int w,
                   const cdx_threshold* th, uint32_t n_th, uint32_t* meets) {
    if (w < 1) return CDX_EINVAL;
    const uint32_t words = (P + 31) / 32;
    const int present[4] = {1, 0, 0, 0};
    for (uint64_t r = 0; r < R; ++r) {
        for (uint32_t q = 0; q < words; ++q) meets[r * words + q] = 0;
        for (uint32_t p = 0; p < P; ++p) {
            const int agree = consistency_prefix(ids, hes, r, P, p + 1, w);
            double sig[4] = {agree < 0 ? 0.0 : (double)agree / (double)w, 0.0, 0.0, 0.0};
            const int ok = cdxo_meets_thresholds(sig, present, th, n_th);
            if (ok < 0) return CDX_EINVAL;
            if (ok) meets[r * words + p / 32] |= 1u << (p % 32);
        }
    }
    return CDX_OK;
}

/* SPEC.md:404-412 allocate at knob k for every program, as include/cdx/scheduler.hpp's
 * allocate: k >= cap -> terminate (resource cap); a test point t <= k (detect_at, then every
 * recheck_every for k_step) whose bit t-1 is set -> terminate (certain); else grant up to
 * the next decision point.  meets[g]/words[g]/n[g]: groups 0 SC, 1 CoT, 2 MCTS/Rebase. */
int cdxo_mixed_decide(const uint8_t* arch, const uint32_t* slot, const int32_t* knob, uint64_t N,
                      const uint32_t* const* meets, const uint32_t* words, const uint64_t* n,
                      const cdx_arch_policy* pol, uint8_t* decision, int32_t* grant, int32_t* cap,
                      int64_t* offsets, int64_t* total) {
    int64_t run = 0;
    for (uint64_t i = 0; i < N; ++i) {
        const uint8_t a = arch[i];
        if (a > 3) return CDX_EINVAL;
        const int g = a == CDX_ARCH_SC ? 0 : (a == CDX_ARCH_COT ? 1 : 2);
        const cdx_alloc_policy* q = &pol[a].alloc;
        const int32_t k = knob[i];
        if (slot[i] >= n[g] || k < 0 || k > q->resource_cap) return CDX_EINVAL;
        uint8_t dec = CDX_EXIT_CONTINUE;
        int32_t units = 0;
        if (k >= q->resource_cap) {
            dec = CDX_EXIT_BUDGET;
        } else {
            int met = 0;
            if (q->kind != CDX_POL_EVEN) {
                const uint32_t* row = meets[g] + (uint64_t)slot[i] * words[g];
                const int32_t step = q->kind == CDX_POL_K_STEP_THRESHOLD ? q->recheck_every : q->resource_cap + 1;
                for (int32_t t = q->detect_at; t <= k && !met; t += step) met = (row[(t - 1) / 32] >> ((t - 1) % 32)) & 1u;
            }
            if (met) {
                dec = CDX_EXIT_CERTAIN;
            } else {
                int32_t next = q->resource_cap;
                if (q->kind == CDX_POL_STATIC_THRESHOLD && k < q->detect_at) next = q->detect_at;
                if (q->kind == CDX_POL_K_STEP_THRESHOLD) {
                    next = q->detect_at;
                    while (next <= k) next += q->recheck_every;
                    if (next > q->resource_cap) next = q->resource_cap;
                }
                units = next - k;
            }
        }
        decision[i] = dec;
        grant[i] = units;
        cap[i] = q->resource_cap;
        offsets[i] = run;
        run += (int64_t)units * q->tokens_per_unit;
    }
    *total = run;
    return CDX_OK;
}

/* The same order on `nthreads` host threads (the CPU baseline of the gang order): items
 * are built and qsort-ed in per-thread chunks with the SPEC comparator, then merged in
 * parallel pairwise rounds.  Same total order, so the same result as cdxo_gang_order. */
typedef struct {
    const cdx_prog_soa* s;
    const cdx_inter_policy* pol;
    double now;
    uint64_t b, e;
    gang_item* it;  /* chunk output (live items, compacted within the chunk) */
    uint64_t n;
} gang_chunk;

static void* gang_chunk_build(void* arg) {
    gang_chunk* c = (gang_chunk*)arg;
    const cdx_prog_soa* s = c->s;
    uint64_t n = 0;
    for (uint64_t i = c->b; i < c->e; ++i) {
        if (s->terminated[i]) continue;
        const int esc = (c->now - s->last_service[i]) >= c->pol->starvation_limit;
        double key;
        if (esc || c->pol->order == CDX_ORDER_FIFO) {
            key = s->arrival[i];
        } else {
            const double est = cdxo_estimate_iteration_tokens(s->iter_tok_sum[i], s->iter_count[i],
                                                              c->pol->prior_tokens);
            const int64_t rem = (int64_t)s->cap[i] - (int64_t)s->knob[i];
            key = est * (double)(rem > 0 ? rem : 0);
        }
        c->it[n].esc = esc;
        c->it[n].key = key;
        c->it[n].arrival = s->arrival[i];
        c->it[n].id = s->program_id ? s->program_id[i] : s->id_base + (uint32_t)i;
        ++n;
    }
    c->n = n;
    qsort(c->it, n, sizeof(gang_item), gang_cmp);
    return NULL;
}

typedef struct {
    const gang_item *a, *b;
    uint64_t na, nb;
    gang_item* out;
} gang_merge_job;

static void* gang_merge2(void* arg) {
    gang_merge_job* m = (gang_merge_job*)arg;
    uint64_t i = 0, j = 0, k = 0;
    while (i < m->na && j < m->nb) m->out[k++] = gang_cmp(&m->b[j], &m->a[i]) < 0 ? m->b[j++] : m->a[i++];
    while (i < m->na) m->out[k++] = m->a[i++];
    while (j < m->nb) m->out[k++] = m->b[j++];
    return NULL;
}

int cdxo_gang_order_mt(const cdx_prog_soa* s, uint64_t N, const cdx_inter_policy* pol, double now,
                       uint32_t* order, uint64_t* n_out, int nthreads) {
    if (!(pol->starvation_limit > 0.0)) return CDX_EINVAL;
    if (pol->order != CDX_ORDER_FIFO && pol->order != CDX_ORDER_SJF) return CDX_EINVAL;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    gang_item* buf = (gang_item*)malloc(sizeof(gang_item) * (N ? N : 1) * 2);
    gang_chunk ch[256];
    pthread_t th[256];
    for (int t = 0; t < nthreads; ++t) {
        ch[t].s = s;
        ch[t].pol = pol;
        ch[t].now = now;
        ch[t].b = N * (uint64_t)t / (uint64_t)nthreads;
        ch[t].e = N * (uint64_t)(t + 1) / (uint64_t)nthreads;
        ch[t].it = buf + ch[t].b;
        pthread_create(&th[t], NULL, gang_chunk_build, &ch[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    /* runs: (start, length) in buf; merge pairwise into the other half until one run */
    uint64_t rs[256], rl[256];
    int runs = nthreads;
    for (int t = 0; t < nthreads; ++t) {
        rs[t] = ch[t].b;
        rl[t] = ch[t].n;
    }
    gang_item* src = buf;
    gang_item* dst = buf + (N ? N : 1);
    while (runs > 1) {
        gang_merge_job mj[128];
        int nm = 0;
        uint64_t ns[256], nl[256];
        for (int r = 0; r + 1 < runs; r += 2) {
            mj[nm].a = src + rs[r];
            mj[nm].na = rl[r];
            mj[nm].b = src + rs[r + 1];
            mj[nm].nb = rl[r + 1];
            mj[nm].out = dst + rs[r];
            ns[nm] = rs[r];
            nl[nm] = rl[r] + rl[r + 1];
            pthread_create(&th[nm], NULL, gang_merge2, &mj[nm]);
            ++nm;
        }
        for (int m = 0; m < nm; ++m) pthread_join(th[m], NULL);
        int nr = nm;
        if (runs % 2) { /* odd run out: copy across */
            memcpy(dst + rs[runs - 1], src + rs[runs - 1], rl[runs - 1] * sizeof(gang_item));
            ns[nr] = rs[runs - 1];
            nl[nr] = rl[runs - 1];
            ++nr;
        }
        for (int r = 0; r < nr; ++r) {
            rs[r] = ns[r];
            rl[r] = nl[r];
        }
        runs = nr;
        gang_item* t = src;
        src = dst;
        dst = t;
    }
    /* the merged runs are not contiguous across chunk gaps: compact while writing ids */
    const uint64_t n = runs ? rl[0] : 0;
    for (uint64_t i = 0; i < n; ++i) order[i] = src[rs[0] + i].id;
    *n_out = n;
    free(buf);
    return CDX_OK;
}
