// ref_harness.cpp — drives the REFERENCE's own C++ functions (compiled unmodified from
// /root/reference/proj/src/*.cpp into oracle/_ref/libcdxref.so by oracle/Makefile).
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Two uses:
//   1. golden vectors and randomized parity: tests pin the C restatement (cdx_oracle.c)
//      and the CUDA path against what the reference itself computes;
//   2. bench.py --impl reference and the cpu_baseline leg: the reference's CPU path on
//      all host threads (std::thread pool over contiguous shards, as BASELINE.md plans).
//
// Each batch entry point calls, per unit, exactly the reference routine the GPU kernel
// replaces: metrics::cluster_exact + certaindex_entropy + combined_meets_thresholds
// (SC rows), probe::should_exit / consistency / final_answer on every trace prefix (CoT),
// and metrics::certaindex_reward + cluster_exact over all paths so far (MCTS/Rebase).
// Answers are materialised as std::string from an id->string vocabulary, as the
// reference consumes them; that row-buffer fill is part of the timed work.

#include <algorithm>
#include <atomic>
#include <sstream>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "cdx/metrics.hpp"
#include "cdx/probe.hpp"
#include "cdx/rng.hpp"
#include "cdx/runtime.hpp"
#include "cdx/theory.hpp"

namespace m = cdx::metrics;
namespace pr = cdx::probe;

namespace {

struct CThreshold {
    uint8_t signal, dir, pad[6];
    double cutoff;
};
struct CProbeCfg {
    int32_t interval_tokens, window;
    double threshold;
    int64_t max_tokens;
};

std::vector<std::string> make_vocab(const char* const* vocab, uint32_t n) {
    std::vector<std::string> v;
    v.reserve(n);
    for (uint32_t i = 0; i < n; ++i) v.emplace_back(vocab[i]);
    return v;
}

std::vector<m::SignalThreshold> make_th(const CThreshold* th, uint32_t n) {
    std::vector<m::SignalThreshold> out;
    for (uint32_t i = 0; i < n; ++i) {
        m::SignalThreshold t;
        t.signal = static_cast<m::SignalKind>(th[i].signal);
        t.cutoff = th[i].cutoff;
        t.dir = static_cast<m::ThresholdDir>(th[i].dir);
        out.push_back(t);
    }
    return out;
}

template <class F>
void parallel_for(uint64_t n, int nthreads, F&& f) {
    if (nthreads <= 1 || n < 2) {
        f(uint64_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    const uint64_t chunk = (n + nthreads - 1) / nthreads;
    for (int t = 0; t < nthreads; ++t) {
        const uint64_t b = std::min<uint64_t>(n, t * chunk), e = std::min<uint64_t>(n, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& th : pool) th.join();
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
int ref_hardware_threads() { return static_cast<int>(std::thread::hardware_concurrency()); }

// ---- scalar reference calls (golden vectors) --------------------------------------------
// answers: n NUL-terminated strings.  Returns m (clusters), sizes/labels in first-seen order.
int ref_cluster_exact(const char* const* answers, uint32_t n, int32_t* sizes, char* labels,
                      uint32_t label_stride) {
    try {
        std::vector<std::string> a;
        for (uint32_t i = 0; i < n; ++i) a.emplace_back(answers[i]);
        const auto c = m::cluster_exact(a);
        for (int k = 0; k < c.group_count(); ++k) {
            sizes[k] = c.clusters[k].size;
            std::strncpy(labels + k * label_stride, c.clusters[k].label.c_str(), label_stride - 1);
            labels[k * label_stride + label_stride - 1] = 0;
        }
        return c.group_count();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_entropy(const int32_t* sizes, uint32_t mcl, int32_t total, double* H, double* Hc) {
    try {
        m::Clustering c;
        c.total = total;
        for (uint32_t k = 0; k < mcl; ++k) c.clusters.push_back({"c" + std::to_string(k), sizes[k]});
        *Hc = m::certaindex_entropy(c);
        *H = total == 1 && mcl == 1 ? 0.0 : m::semantic_entropy(c);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_certaindex_reward(const double* r, uint32_t n, int agg_max, double* out) {
    try {
        m::RewardSet rs;
        rs.rewards.assign(r, r + n);
        rs.aggregation = agg_max ? m::RewardAggregation::Max : m::RewardAggregation::Mean;
        *out = m::certaindex_reward(rs);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// signals[4] with present[4]; returns 0/1, or -1 on exception (message in ref_last_error)
int ref_meets(const double* signals, const int32_t* present, const CThreshold* th, uint32_t n) {
    try {
        m::SignalVector s;
        if (present[0]) s.certaindex_entropy = signals[0];
        if (present[1]) s.certaindex_reward = signals[1];
        if (present[2]) s.mean_output_length = signals[2];
        if (present[3]) s.mean_norm_logprob = signals[3];
        const auto t = make_th(th, n);
        return m::combined_meets_thresholds(s, t) ? 1 : 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

int ref_flag_hesitation(const char* answer, const char* const* markers, uint32_t n) {
    std::vector<std::string> mk;
    for (uint32_t i = 0; i < n; ++i) mk.emplace_back(markers[i]);
    return pr::flag_hesitation(answer, mk) ? 1 : 0;
}

int ref_trim(const char* s, uint64_t len, uint64_t* begin, uint64_t* tlen) {
    const std::string_view v(s, len);
    const auto t = m::trim(v);
    *begin = static_cast<uint64_t>(t.data() - v.data());
    *tlen = t.size();
    return 0;
}

uint64_t ref_mix64(uint64_t x) { return cdx::mix64(x); }
uint64_t ref_derive_seed(uint64_t a, uint64_t b, uint64_t c) { return cdx::derive_seed(a, b, c); }

// probe trace of explicit records; returns decision (0/1/2) or -1 on exception.
int ref_should_exit(const int32_t* step, const int64_t* off, const char* const* ans,
                    const uint8_t* hes, uint32_t n, const CProbeCfg* cfg) {
    try {
        pr::ProbeTrace t;
        for (uint32_t i = 0; i < n; ++i) t.records.push_back({step[i], off[i], ans[i], hes[i] != 0});
        pr::ProbeConfig c;
        c.interval_tokens = cfg->interval_tokens;
        c.window = cfg->window;
        c.threshold = cfg->threshold;
        c.max_tokens = cfg->max_tokens;
        return static_cast<int>(pr::should_exit(t, c));
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// consistency at k; returns 1 with *out set, 0 for nullopt, -1 on exception
int ref_consistency(const int32_t* step, const char* const* ans, const uint8_t* hes, uint32_t n,
                    int32_t k, int32_t w, double* out) {
    try {
        std::vector<pr::AnswerRecord> recs;
        for (uint32_t i = 0; i < n; ++i) recs.push_back({step[i], (long)(i + 1) * 64, ans[i], hes[i] != 0});
        const auto c = pr::consistency(recs, k, w);
        if (!c) return 0;
        *out = *c;
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// final_answer; terminated_at < 0 = none; reason 0 certain 1 budget 2 external
int ref_final_answer(const int32_t* step, const char* const* ans, const uint8_t* hes, uint32_t n,
                     int32_t terminated_at, int32_t reason, char* out, uint32_t out_len,
                     uint8_t* low) {
    try {
        pr::ProbeTrace t;
        for (uint32_t i = 0; i < n; ++i) t.records.push_back({step[i], (long)(i + 1) * 64, ans[i], hes[i] != 0});
        if (terminated_at >= 0) t.terminated_at = terminated_at;
        t.termination_reason = static_cast<pr::TerminationReason>(reason);
        const auto fa = pr::final_answer(t);
        std::strncpy(out, fa.answer.c_str(), out_len - 1);
        out[out_len - 1] = 0;
        *low = fa.low_confidence ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// JSONL ingestion error text: returns #lines or -1 with message.
int ref_read_trace_jsonl(const char* text) {
    try {
        std::string s(text);
        std::istringstream in(s);
        return static_cast<int>(pr::read_trace_jsonl(in).size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// read_trace_jsonl on `nthreads` host threads: the text is cut at line boundaries into one
// contiguous chunk per thread, each chunk parsed by the reference's own read_trace_jsonl
// (nlohmann parse, field checks, per-program order checks inside the chunk), then one
// sequential pass applies the per-program order checks across chunk boundaries (a program's
// first record in a chunk against its last record in the chunks before).  Valid traces
// give the reference's result; returns the record count or -1 (message in g_err).
int ref_read_trace_jsonl_mt(const char* text, int nthreads) {
    try {
        const std::string s(text);
        const size_t nt = static_cast<size_t>(std::max(1, nthreads));
        std::vector<size_t> cut(nt + 1, s.size());
        cut[0] = 0;
        for (size_t t = 1; t < nt; ++t) {
            size_t c = std::max(cut[t - 1], s.size() * t / nt);
            while (c < s.size() && c > 0 && s[c - 1] != '\n') ++c;
            cut[t] = c;
        }
        std::vector<std::vector<pr::TraceLine>> part(nt);
        std::vector<std::string> err(nt);
        std::vector<std::thread> pool;
        for (size_t t = 0; t < nt; ++t)
            pool.emplace_back([&, t] {
                try {
                    std::istringstream in(s.substr(cut[t], cut[t + 1] - cut[t]));
                    part[t] = pr::read_trace_jsonl(in);
                } catch (const std::exception& e) {
                    err[t] = e.what();
                }
            });
        for (auto& th : pool) th.join();
        for (size_t t = 0; t < nt; ++t)
            if (!err[t].empty()) throw std::runtime_error(err[t] + " (chunk " + std::to_string(t) + ")");
        std::unordered_map<std::string, std::pair<long, int>> last;  // program -> (offset, step)
        size_t n = 0;
        for (size_t t = 0; t < nt; ++t) {
            std::unordered_map<std::string, bool> seen_here;
            for (const auto& l : part[t]) {
                if (!seen_here.count(l.program_id)) {
                    seen_here[l.program_id] = true;
                    auto it = last.find(l.program_id);
                    if (it != last.end()) {
                        if (l.record.token_offset <= it->second.first) throw std::runtime_error("token_offset does not increase");
                        if (l.record.step_index <= it->second.second) throw std::runtime_error("step_index does not increase");
                    }
                }
                last[l.program_id] = {l.record.token_offset, l.record.step_index};
            }
            n += part[t].size();
        }
        return static_cast<int>(n);
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// read_trace_jsonl with every field returned (probe.cpp:126-165): strings packed with
// offsets; returns the record count, -1 with the reference's message, or -2 if max is small.
int ref_parse_jsonl(const char* text, uint64_t nbytes, uint64_t max, int32_t* step, int64_t* tok, uint8_t* hes,
                    char* pid_buf, uint64_t* pid_off, char* ans_buf, uint64_t* ans_off) {
    try {
        std::istringstream in(std::string(text, nbytes));
        const auto lines = pr::read_trace_jsonl(in);
        if (lines.size() > max) return -2;
        uint64_t po = 0, ao = 0;
        pid_off[0] = 0;
        ans_off[0] = 0;
        for (size_t i = 0; i < lines.size(); ++i) {
            const auto& l = lines[i];
            step[i] = l.record.step_index;
            tok[i] = l.record.token_offset;
            hes[i] = l.record.hesitant ? 1 : 0;
            std::memcpy(pid_buf + po, l.program_id.data(), l.program_id.size());
            po += l.program_id.size();
            pid_off[i + 1] = po;
            std::memcpy(ans_buf + ao, l.record.answer.data(), l.record.answer.size());
            ao += l.record.answer.size();
            ans_off[i + 1] = ao;
        }
        return static_cast<int>(lines.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// update_certaindex through a real ProgramDriver (runtime.cpp:264-313) for an SC/MCTS/
// Rebase synthetic spec: expand `units` one unit at a time, completing each request, and
// record the signal vector after each unit.  Returns #points or -1.
int ref_driver_signals(int archetype, uint64_t seed, int cap, int conv, int solvable,
                       int units, double* ent, double* rew, double* len) {
    try {
        cdx::runtime::SyntheticProgramSpec spec;
        spec.archetype = static_cast<cdx::runtime::Archetype>(archetype);
        spec.resource_cap = cap;
        spec.true_convergence_knob = conv;
        spec.solvable = solvable != 0;
        spec.difficulty_factor = solvable ? 1 : 3;
        if (spec.archetype != cdx::runtime::Archetype::SC) spec.rewards = cdx::runtime::RewardModel{};
        cdx::runtime::ProgramDriver d(7, "p", spec, seed);
        for (int u = 0; u < units; ++u) {
            auto reqs = d.expand(1, 0.0);
            std::vector<cdx::runtime::Request> q(reqs.begin(), reqs.end());
            while (!q.empty()) {
                auto r = q.back();
                q.pop_back();
                if (auto nx = d.on_request_complete(r, 1.0)) q.push_back(*nx);
            }
            const auto sv = d.update_certaindex();
            ent[u] = sv.certaindex_entropy.value_or(-1.0);
            rew[u] = sv.certaindex_reward.value_or(-1.0);
            len[u] = sv.mean_output_length.value_or(-1.0);
        }
        return units;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// ---- batched reference runs (parity and the CPU baseline) -----------------------------
// SC rows: ids[R][P][S] -> H~ (f64) per row and meets bits [R][ceil(P/32)].
// mode 0 = full reference work; mode 1 = row-buffer fill only (reported separately).
int ref_sc_batch(const uint32_t* ids, uint64_t R, uint32_t P, uint32_t S,
                 const char* const* vocab, uint32_t nvocab, const CThreshold* th, uint32_t n_th,
                 double* hcert, uint32_t* meets_bits, int nthreads, int mode) {
    const auto voc = make_vocab(vocab, nvocab);
    const auto thr = make_th(th, n_th);
    const uint32_t words = (P + 31) / 32;
    std::atomic<int> fail{0};
    uint64_t sink = 0;
    parallel_for(R, nthreads, [&](uint64_t b, uint64_t e) {
        std::vector<std::string> row(S);
        uint64_t local = 0;
        try {
            for (uint64_t r = b; r < e; ++r) {
                if (meets_bits)
                    for (uint32_t w = 0; w < words; ++w) meets_bits[r * words + w] = 0;
                for (uint32_t p = 0; p < P; ++p) {
                    const uint32_t* x = ids + (r * P + p) * S;
                    for (uint32_t s = 0; s < S; ++s) row[s] = voc[x[s]];  // row-buffer fill
                    if (mode == 1) {
                        local += row[0].size();
                        continue;
                    }
                    const double hc = m::certaindex_entropy(m::cluster_exact(row));
                    if (hcert) hcert[r * P + p] = hc;
                    m::SignalVector sv;
                    sv.certaindex_entropy = hc;
                    if (m::combined_meets_thresholds(sv, thr) && meets_bits)
                        meets_bits[r * words + p / 32] |= 1u << (p % 32);
                }
            }
        } catch (const std::exception& ex) {
            g_err = ex.what();
            fail = 1;
        }
        __atomic_add_fetch(&sink, local, __ATOMIC_RELAXED);
    });
    return fail ? -1 : 0;
}

// K1's reference work over a string arena (answers arena[off[i] .. off[i+1])), rows of S
// consecutive answers: each row is materialised as the std::string answers the reference
// consumes, clustered by metrics::cluster_exact (trim + unordered_map<string_view> key,
// metrics.cpp:12-37) and each answer flagged by probe::flag_hesitation (probe.cpp:36-44).
// ncl[row] = cluster count, hes[i] = flag (both nullable).
int ref_intern_batch(const char* arena, const uint64_t* off, uint64_t n, uint32_t S, const char* const* markers,
                     uint32_t n_markers, uint32_t* ncl, uint8_t* hes, int nthreads) {
    std::vector<std::string> mk;
    for (uint32_t k = 0; k < n_markers; ++k) mk.emplace_back(markers[k]);
    const uint64_t rows = (n + S - 1) / S;
    std::atomic<int> fail{0};
    parallel_for(rows, nthreads, [&](uint64_t b, uint64_t e) {
        std::vector<std::string> row;
        try {
            for (uint64_t r = b; r < e; ++r) {
                const uint64_t i0 = r * S, i1 = std::min<uint64_t>(n, i0 + S);
                row.clear();
                for (uint64_t i = i0; i < i1; ++i) row.emplace_back(arena + off[i], off[i + 1] - off[i]);
                const auto c = m::cluster_exact(row);
                if (ncl) ncl[r] = static_cast<uint32_t>(c.group_count());
                for (uint64_t i = i0; i < i1; ++i) {
                    const bool h = pr::flag_hesitation(row[i - i0], mk);
                    if (hes) hes[i] = h ? 1 : 0;
                }
            }
        } catch (const std::exception& ex) {
            g_err = ex.what();
            fail = 1;
        }
    });
    return fail ? -1 : 0;
}

// CoT: ids[R][P] (vocab), hes bits [R][ceil(P/64)], implicit offsets (p+1)*interval.
// Every prefix: should_exit(trace, cfg) (probe.cpp:77-85); on the first exit the trace is
// terminated (runtime.cpp:405-411) and final_answer taken.  ck = consistency(...).value_or(0)
// at every prefix (runtime.cpp:293-300).  exit_step -1 = never exited (final answer then
// from the full trace, criteria_external).
// The CoT signal ProgramDriver::update_certaindex records after every probe
// (runtime.cpp:293-299): consistency(records, latest step_index, window).value_or(0.0), with
// the reference's own probe::consistency (probe.cpp:64-75), as f64 per prefix.
int ref_cot_signal(const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P, const char* const* vocab,
                   uint32_t nvocab, int window, double* ck64, int nthreads) {
    const auto voc = make_vocab(vocab, nvocab);
    const uint32_t hw = (P + 63) / 64;
    std::atomic<int> fail{0};
    parallel_for(R, nthreads, [&](uint64_t b, uint64_t e) {
        try {
            std::vector<pr::AnswerRecord> recs;
            recs.reserve(P);
            for (uint64_t r = b; r < e; ++r) {
                recs.clear();
                for (uint32_t p = 0; p < P; ++p) {
                    const bool h = (hes[r * hw + p / 64] >> (p % 64)) & 1ULL;
                    recs.push_back({static_cast<int>(p + 1), static_cast<long>(p + 1) * 64, voc[ids[r * P + p]], h});
                    ck64[r * P + p] = pr::consistency(recs, recs.back().step_index, window).value_or(0.0);
                }
            }
        } catch (const std::exception& ex) {
            g_err = ex.what();
            fail = 1;
        }
    });
    return fail ? -1 : 0;
}

int ref_cot_batch(const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P,
                  const char* const* vocab, uint32_t nvocab, const CProbeCfg* cfgc,
                  int32_t* exit_step, uint8_t* reason, uint32_t* final_id, uint8_t* low_conf,
                  float* ck, int nthreads) {
    const auto voc = make_vocab(vocab, nvocab);
    pr::ProbeConfig cfg;
    cfg.interval_tokens = cfgc->interval_tokens;
    cfg.window = cfgc->window;
    cfg.threshold = cfgc->threshold;
    cfg.max_tokens = cfgc->max_tokens;
    const uint32_t hw = (P + 63) / 64;
    std::atomic<int> fail{0};
    parallel_for(R, nthreads, [&](uint64_t b, uint64_t e) {
        try {
            pr::ProbeTrace t;
            t.records.reserve(P);
            for (uint64_t r = b; r < e; ++r) {
                t.records.clear();
                t.terminated_at.reset();
                t.termination_reason = pr::TerminationReason::Budget;
                int32_t ex = -1;
                uint8_t why = 0;
                for (uint32_t p = 0; p < P; ++p) {
                    const bool h = (hes[r * hw + p / 64] >> (p % 64)) & 1ULL;
                    t.records.push_back({static_cast<int>(p + 1),
                                         static_cast<long>(p + 1) * cfg.interval_tokens,
                                         voc[ids[r * P + p]], h});
                    if (ck) {
                        const auto c = pr::consistency(t.records, static_cast<int>(p + 1), cfg.window);
                        ck[r * P + p] = static_cast<float>(c.value_or(0.0));
                    }
                    if (ex < 0) {
                        const auto d = pr::should_exit(t, cfg);
                        if (d != pr::ExitDecision::Continue) {
                            ex = static_cast<int32_t>(p);
                            why = d == pr::ExitDecision::ExitCertain ? 1 : 2;
                        }
                    }
                }
                exit_step[r] = ex;
                reason[r] = why;
                // final answer on the trace as terminated
                pr::ProbeTrace ft;
                const uint32_t n = ex >= 0 ? static_cast<uint32_t>(ex) + 1 : P;
                ft.records.assign(t.records.begin(), t.records.begin() + n);
                ft.terminated_at = ft.records.back().step_index;
                ft.termination_reason = why == 1   ? pr::TerminationReason::Certain
                                        : why == 2 ? pr::TerminationReason::Budget
                                                   : pr::TerminationReason::CriteriaExternal;
                const auto fa = pr::final_answer(ft);
                // map the answer string back to its vocabulary id
                uint32_t id = 0xffffffffu;
                for (uint32_t v = 0; v < voc.size(); ++v)
                    if (m::trim(voc[v]) == std::string_view(fa.answer)) {
                        id = v;
                        break;
                    }
                final_id[r] = id;
                low_conf[r] = fa.low_confidence ? 1 : 0;
            }
        } catch (const std::exception& ex) {
            g_err = ex.what();
            fail = 1;
        }
    });
    return fail ? -1 : 0;
}

// MCTS/Rebase cumulative: at step t, certaindex_reward over all rewards of steps 0..t and
// certaindex_entropy(cluster_exact(all answers so far)) (runtime.cpp:279-292).
// with_entropy = 0: reward certaindex only.
int ref_reward_batch(const float* rewards, const uint32_t* ids, const uint8_t* agg, uint64_t G,
                     uint32_t T, uint32_t W, const char* const* vocab, uint32_t nvocab,
                     double* R, double* H, int nthreads) {
    const auto voc = make_vocab(vocab, nvocab);
    std::atomic<int> fail{0};
    parallel_for(G, nthreads, [&](uint64_t b, uint64_t e) {
        try {
            m::RewardSet rs;
            std::vector<std::string> answers;
            for (uint64_t g = b; g < e; ++g) {
                rs.rewards.clear();
                answers.clear();
                rs.aggregation = agg[g] ? m::RewardAggregation::Max : m::RewardAggregation::Mean;
                for (uint32_t t = 0; t < T; ++t) {
                    for (uint32_t w = 0; w < W; ++w) {
                        const uint64_t o = (g * T + t) * W + w;
                        rs.rewards.push_back(static_cast<double>(rewards[o]));
                        if (ids) answers.push_back(voc[ids[o]]);
                    }
                    R[g * T + t] = m::certaindex_reward(rs);
                    if (ids && H) H[g * T + t] = m::certaindex_entropy(m::cluster_exact(answers));
                }
            }
        } catch (const std::exception& ex) {
            g_err = ex.what();
            fail = 1;
        }
    });
    return fail ? -1 : 0;
}

// ProgramDriver::aggregate_prefix (runtime.cpp:345-403) of an SC / Rebase / MCTS program
// whose paths are injected: answers vocab[ids[i]], rewards (nullable), Rebase layers of
// widths layer_w.  Writes the index into vocab of the trimmed answer; returns 0 or -1.
int ref_aggregate(int archetype, const uint32_t* ids, const double* rewards, int n, const int* layer_w,
                  int n_layers, int units, const char* const* vocab, uint32_t nvocab, uint32_t* out) {
    try {
        const auto voc = make_vocab(vocab, nvocab);
        cdx::runtime::SyntheticProgramSpec spec;
        spec.archetype = static_cast<cdx::runtime::Archetype>(archetype);
        spec.resource_cap = std::max(units, n);
        if (spec.archetype != cdx::runtime::Archetype::SC) spec.rewards = cdx::runtime::RewardModel{};
        cdx::runtime::ProgramDriver d(7, "p", spec, 1);
        auto& st = d.program().state;
        st.paths.clear();
        for (int i = 0; i < n; ++i) {
            cdx::runtime::PathSample ps;
            ps.knob_point = i + 1;
            ps.answer = voc[ids[i]];
            if (rewards) ps.reward = rewards[i];
            st.paths.push_back(ps);
        }
        st.layer_widths.assign(layer_w, layer_w + n_layers);
        const auto res = d.aggregate_prefix(units);
        if (res.answer.empty()) {  // weighted_plurality found no winner (NaN weights)
            *out = 0xffffffffu;
            return 0;
        }
        for (uint32_t k = 0; k < nvocab; ++k)
            if (cdx::metrics::trim(voc[k]) == res.answer) {
                *out = k;
                return 0;
            }
        g_err = "ref_aggregate: answer not in vocabulary: " + res.answer;
        return -1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// probe::stationary_by_epsilon_test (probe.cpp:104-120) of every prefix of each trace:
// ids[R][P] (answers vocab[id]), hes bits u64[R][ceil(P/64)] -> state u8[R][P] (0 nullopt,
// 1 false, 2 true).  Returns 0, or -1 with the exception text (k / epsilon validation).
int ref_eps_prefixes(const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P, int k, double epsilon,
                     const char* const* vocab, uint32_t nvocab, uint8_t* state) {
    try {
        const auto voc = make_vocab(vocab, nvocab);
        const uint32_t hw = (P + 63) / 64;
        for (uint64_t r = 0; r < R; ++r) {
            std::vector<cdx::probe::AnswerRecord> recs;
            for (uint32_t p = 0; p < P; ++p) {
                cdx::probe::AnswerRecord a;
                a.step_index = static_cast<int>(p) + 1;
                a.token_offset = 64L * (p + 1);
                a.answer = voc[ids[r * P + p]];
                a.hesitant = (hes[r * hw + p / 64] >> (p % 64)) & 1ull;
                recs.push_back(a);
                const auto res = cdx::probe::stationary_by_epsilon_test(recs, k, epsilon);
                state[r * P + p] = res ? (*res ? 2 : 1) : 0;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
