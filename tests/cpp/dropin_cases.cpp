// dropin_cases.cpp — the drop-in proof for the C++ API.
//
// ONE caller source, written only against the reference's public headers (cdx/metrics.hpp,
// cdx/probe.hpp), compiled twice:
//   oracle/_ref/dropin_ref   against /root/reference/proj/include + the reference's own
//                            metrics.cpp / probe.cpp / theory.cpp (oracle/Makefile)
//   tests/cpp/bin/dropin_ours against this repo's include/cdx + libcdxhost.so (Makefile)
// Both print one line per case; tests/test_gpu_dropin.py requires the outputs to be
// identical line for line (floats printed as hex, exceptions as type + message).
// The cases are the SPEC.md examples followed by seeded random cases over
// every declared function, edge cases included (empty inputs, whitespace-only answers,
// ties on thresholds, non-monotone step indices, invalid configs, malformed JSONL).

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <typeinfo>
#include <vector>

#include "cdx/metrics.hpp"
#include "cdx/probe.hpp"

using namespace cdx;

namespace {

uint64_t g_state = 0x2412209930ULL;
uint64_t next_u64() {  // xorshift64*
    g_state ^= g_state >> 12;
    g_state ^= g_state << 25;
    g_state ^= g_state >> 27;
    return g_state * 0x2545F4914F6CDD1DULL;
}
uint32_t below(uint32_t n) { return static_cast<uint32_t>(next_u64() % n); }
double unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }

std::string esc(const std::string& s) {
    std::string o;
    for (unsigned char c : s) {
        if (c >= 0x20 && c < 0x7f && c != '\\' && c != '|') {
            o += static_cast<char>(c);
        } else {
            char b[8];
            std::snprintf(b, sizeof b, "\\x%02x", c);
            o += b;
        }
    }
    return o;
}

std::string hex(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%a", v);
    return b;
}

const char* exc_type(const std::exception& e) {
    if (dynamic_cast<const std::invalid_argument*>(&e)) return "invalid_argument";
    if (dynamic_cast<const std::out_of_range*>(&e)) return "out_of_range";
    if (dynamic_cast<const std::logic_error*>(&e)) return "logic_error";
    if (dynamic_cast<const std::runtime_error*>(&e)) return "runtime_error";
    return "exception";
}

// JSONL errors: the reference's detail text after the category is nlohmann's exception
// message; the contract is the prefix "trace line <n>: <category>" (facade_jsonl.cpp).
std::string jsonl_message(const std::string& m) {
    for (const char* cat : {"invalid JSON", "missing or mistyped field"}) {
        const auto p = m.find(cat);
        if (p != std::string::npos) return m.substr(0, p + std::string(cat).size());
    }
    return m;
}

template <class F>
void run(const std::string& tag, F&& f) {
    std::string out;
    try {
        out = f();
    } catch (const std::exception& e) {
        out = std::string("EXC ") + exc_type(e) + " " + esc(e.what());
    }
    std::printf("%s | %s\n", tag.c_str(), out.c_str());
}

std::string show(const metrics::Clustering& c) {
    std::string o = "n=" + std::to_string(c.total) + " m=" + std::to_string(c.group_count());
    for (const auto& cl : c.clusters) o += " [" + esc(cl.label) + "]x" + std::to_string(cl.size);
    return o;
}

const std::vector<std::string> kAnswers = {"12", " 12", "12 ", "\t12\n", "13", " 13 ", "x", "y", "",
                                           "   ", "\v\f", "wait, 12", "Wait 13", "hmm", "HMM no", "12.0",
                                           "a b", " a b", "a  b", "\r\n"};

std::string random_answer() { return kAnswers[below(static_cast<uint32_t>(kAnswers.size()))]; }

std::vector<probe::AnswerRecord> random_records(int n, bool monotone) {
    std::vector<probe::AnswerRecord> r(static_cast<size_t>(n));
    int step = 0;
    long off = 0;
    for (auto& x : r) {
        step = monotone ? step + 1 + static_cast<int>(below(2)) : static_cast<int>(below(12)) - 1;
        off = off + 1 + static_cast<long>(below(100));
        x.step_index = step;
        x.token_offset = off;
        x.answer = random_answer();
        x.hesitant = below(4) == 0;
    }
    return r;
}

void spec_examples() {
    // metrics
    run("spec cluster_exact", [] {
        std::vector<std::string> a = {"12", " 12", "13"};
        return show(metrics::cluster_exact(a));
    });
    run("spec cluster_exact empty", [] { return show(metrics::cluster_exact(std::vector<std::string>{})); });
    for (std::vector<int> sizes : {std::vector<int>{2, 2}, {1}, {1, 1, 1, 1}, {3, 1, 1}, {5}, {4, 0}}) {
        metrics::Clustering c;
        for (int s : sizes) {
            c.clusters.push_back({"k" + std::to_string(c.clusters.size()), s});
            c.total += s;
        }
        std::string tag = "spec entropy";
        for (int s : sizes) tag += " " + std::to_string(s);
        run(tag + " H", [&] { return hex(metrics::semantic_entropy(c)); });
        run(tag + " Hc", [&] { return hex(metrics::certaindex_entropy(c)); });
    }
    run("spec entropy invalid", [] { return hex(metrics::semantic_entropy(metrics::Clustering{})); });
    run("spec reward mean", [] { return hex(metrics::certaindex_reward({{0.2, 0.4, 0.6}, metrics::RewardAggregation::Mean})); });
    run("spec reward max", [] { return hex(metrics::certaindex_reward({{0.2, 0.9, 0.6}, metrics::RewardAggregation::Max})); });
    run("spec reward empty", [] { return hex(metrics::certaindex_reward({})); });
    run("spec reward range", [] { return hex(metrics::certaindex_reward({{0.5, 1.5}})); });
    run("spec thresholds table3", [] {
        metrics::SignalVector s;
        s.certaindex_entropy = 0.99;
        s.certaindex_reward = 0.4;
        std::vector<metrics::SignalThreshold> t = {{metrics::SignalKind::CertaindexEntropy, 0.99},
                                                   {metrics::SignalKind::CertaindexReward, 0.4}};
        return std::to_string(metrics::combined_meets_thresholds(s, t));
    });
    run("spec thresholds absent", [] {
        metrics::SignalVector s;
        s.certaindex_entropy = 0.5;
        std::vector<metrics::SignalThreshold> t = {{metrics::SignalKind::CertaindexReward, 0.4}};
        return std::to_string(metrics::combined_meets_thresholds(s, t));
    });
    // probe
    const std::vector<std::string> mk = {"wait", "hmm"};
    for (const char* a : {"Wait, maybe 12", "12", "HMM", "ahmm", ""})
        run(std::string("spec flag_hesitation ") + esc(a), [&] { return std::to_string(probe::flag_hesitation(a, mk)); });
    run("spec consistency xyx", [] {
        std::vector<probe::AnswerRecord> r = {{1, 64, "x", false}, {2, 128, "y", false}, {3, 192, "x", false}};
        auto c = probe::consistency(r, 3, 3);
        return c ? hex(*c) : std::string("nullopt");
    });
    run("spec consistency hes", [] {
        std::vector<probe::AnswerRecord> r = {{1, 64, "x", false}, {2, 128, "x", true}, {3, 192, "x", false}};
        auto c = probe::consistency(r, 3, 2);
        return c ? hex(*c) : std::string("nullopt");
    });
    run("spec should_exit aabaa", [] {
        probe::ProbeTrace t;
        const char* ans[] = {"a", "a", "b", "a", "a"};
        for (int i = 0; i < 5; ++i) t.records.push_back({i + 1, 64L * (i + 1), ans[i], false});
        probe::ProbeConfig cfg;
        cfg.window = 5;
        cfg.threshold = 0.6;
        return std::to_string(static_cast<int>(probe::should_exit(t, cfg)));
    });
    run("spec final_answer all hesitant", [] {
        probe::ProbeTrace t;
        t.records = {{1, 64, " wait 3 ", true}, {2, 128, "hmm 4 ", true}};
        auto f = probe::final_answer(t);
        return esc(f.answer) + " low=" + std::to_string(f.low_confidence);
    });
}

void random_cases(int count) {
    for (int i = 0; i < count; ++i) {
        const std::string id = std::to_string(i);
        // clustering + entropies
        {
            const int n = static_cast<int>(1 + below(i % 7 == 0 ? 300 : 70));
            std::vector<std::string> a(static_cast<size_t>(n));
            for (auto& s : a) s = random_answer();
            run("cluster " + id, [&] {
                auto c = metrics::cluster_exact(a);
                return show(c) + " H=" + hex(metrics::semantic_entropy(c)) + " Hc=" + hex(metrics::certaindex_entropy(c));
            });
        }
        // explicit (possibly malformed) clusterings
        {
            metrics::Clustering c;
            const int m = static_cast<int>(below(6));
            for (int k = 0; k < m; ++k) c.clusters.push_back({"c", static_cast<int>(below(9)) - (below(10) == 0 ? 1 : 0)});
            for (auto& cl : c.clusters) c.total += cl.size > 0 ? cl.size : 0;
            if (below(8) == 0) c.total = static_cast<int>(below(3));
            // includes clusters larger than the total (p > 1), which the reference computes
            run("entropy " + id, [&] { return hex(metrics::semantic_entropy(c)); });
            run("certaindex " + id, [&] { return hex(metrics::certaindex_entropy(c)); });
        }
        // reward sets
        {
            metrics::RewardSet r;
            const int n = static_cast<int>(below(i % 5 == 0 ? 400 : 20));
            for (int k = 0; k < n; ++k) r.rewards.push_back(below(50) == 0 ? 1.0 + unit() : unit());
            r.aggregation = below(2) ? metrics::RewardAggregation::Max : metrics::RewardAggregation::Mean;
            run("reward " + id, [&] { return hex(metrics::certaindex_reward(r)); });
        }
        // thresholds
        {
            metrics::SignalVector s;
            const double v[4] = {unit(), unit(), 100 * unit(), -unit()};
            if (below(4)) s.certaindex_entropy = v[0];
            if (below(4)) s.certaindex_reward = v[1];
            if (below(3)) s.mean_output_length = v[2];
            if (below(3)) s.mean_norm_logprob = v[3];
            std::vector<metrics::SignalThreshold> t;
            const int nt = static_cast<int>(below(i % 9 == 0 ? 12 : 4));
            for (int k = 0; k < nt; ++k) {
                metrics::SignalThreshold x;
                x.signal = static_cast<metrics::SignalKind>(below(4));
                const int si = static_cast<int>(x.signal);
                x.cutoff = below(3) == 0 ? v[si] : (below(2) ? v[si] * 0.9 : v[si] * 1.1);
                x.dir = below(3) == 0 ? metrics::ThresholdDir::LessEq : metrics::ThresholdDir::GreaterEq;
                t.push_back(x);
            }
            run("meets " + id, [&] { return std::to_string(metrics::combined_meets_thresholds(s, t)); });
        }
        // hesitation
        {
            std::vector<std::string> mk;
            const char* pool[] = {"wait", "hmm", "WAIT", "", "a b", "12", "\t"};
            const int nm = static_cast<int>(below(4));
            for (int k = 0; k < nm; ++k) mk.push_back(pool[below(7)]);
            const std::string a = random_answer() + (below(2) ? random_answer() : std::string());
            run("hesitation " + id, [&] { return std::to_string(probe::flag_hesitation(a, mk)); });
        }
        // consistency / should_exit / final_answer
        {
            const int n = static_cast<int>(below(i % 11 == 0 ? 90 : 14));
            auto recs = random_records(n, below(3) != 0);
            const int k = static_cast<int>(below(16)) - 1;
            const int w = static_cast<int>(below(6)) - (below(12) == 0 ? 1 : 0);
            run("consistency " + id, [&] {
                auto c = probe::consistency(recs, k, w);
                return c ? hex(*c) : std::string("nullopt");
            });
            probe::ProbeTrace t;
            t.records = recs;
            probe::ProbeConfig cfg;
            cfg.window = 1 + static_cast<int>(below(5));
            const double taus[] = {0.5, 0.6, 2.0 / 3.0, 0.75, 0.9, 1.0, 0.0, 1.5};
            cfg.threshold = taus[below(below(10) == 0 ? 8 : 6)];
            cfg.max_tokens = 1 + static_cast<long>(below(1200));
            if (below(15) == 0) cfg.interval_tokens = 0;
            run("should_exit " + id, [&] { return std::to_string(static_cast<int>(probe::should_exit(t, cfg))); });
            if (!recs.empty() && below(2)) t.terminated_at = recs[below(static_cast<uint32_t>(recs.size()))].step_index + (below(5) == 0 ? 1 : 0);
            t.termination_reason = static_cast<probe::TerminationReason>(below(3));
            const int ek = static_cast<int>(below(5)) - (below(15) == 0 ? 1 : 0);
            const double eps = below(12) == 0 ? 0.0 : 0.05 + unit();
            run("eps_test " + id, [&] {
                auto e = probe::stationary_by_epsilon_test(recs, ek, eps);
                return e ? std::to_string(*e) : std::string("nullopt");
            });
            run("final_answer " + id, [&] {
                auto f = probe::final_answer(t);
                return esc(f.answer) + " low=" + std::to_string(f.low_confidence);
            });
        }
    }
}

// NaN / +-inf / -0.0 / subnormal inputs: every validation and comparison must take the
// reference's branch (e.g. probe.cpp:22 accepts a NaN threshold, theory.cpp:119 a NaN epsilon,
// metrics.cpp:131 a NaN reward, metrics.cpp:167 fails every compare against a NaN)
void nonfinite_cases() {
    const double nan = std::numeric_limits<double>::quiet_NaN(), inf = std::numeric_limits<double>::infinity();
    const double den = std::numeric_limits<double>::denorm_min();
    const std::vector<double> specials = {nan, -nan, inf, -inf, -0.0, 0.0, den, -den, 1.0, 0.5, 1.0 + 0x1p-52};
    for (size_t a = 0; a < specials.size(); ++a) {
        const std::string ta = std::to_string(a);
        for (auto agg : {metrics::RewardAggregation::Mean, metrics::RewardAggregation::Max}) {
            const std::string tg = agg == metrics::RewardAggregation::Max ? " max" : " mean";
            run("nf reward " + ta + tg, [&] { return hex(metrics::certaindex_reward({{specials[a]}, agg})); });
            run("nf reward mid " + ta + tg,
                [&] { return hex(metrics::certaindex_reward({{0.25, specials[a], 0.75}, agg})); });
            run("nf reward first " + ta + tg,
                [&] { return hex(metrics::certaindex_reward({{specials[a], 0.25, 0.75}, agg})); });
        }
        for (size_t b = 0; b < specials.size(); ++b) {
            metrics::SignalVector s;
            s.certaindex_entropy = specials[a];
            s.certaindex_reward = 0.5;
            for (auto dir : {metrics::ThresholdDir::GreaterEq, metrics::ThresholdDir::LessEq}) {
                std::vector<metrics::SignalThreshold> t = {{metrics::SignalKind::CertaindexEntropy, specials[b], dir},
                                                           {metrics::SignalKind::CertaindexReward, 0.5}};
                run("nf meets " + ta + " " + std::to_string(b) + " " + std::to_string(static_cast<int>(dir)),
                    [&] { return std::to_string(metrics::combined_meets_thresholds(s, t)); });
            }
        }
        probe::ProbeTrace tr;
        const char* ans[] = {"a", "a", "b", "a", "a", "a"};
        for (int i = 0; i < 6; ++i) tr.records.push_back({i + 1, 64L * (i + 1), ans[i], false});
        probe::ProbeConfig cfg;
        cfg.window = 3;
        cfg.threshold = specials[a];
        cfg.max_tokens = 300;
        run("nf should_exit tau " + ta, [&] { return std::to_string(static_cast<int>(probe::should_exit(tr, cfg))); });
        cfg.max_tokens = 1 << 20;
        run("nf should_exit tau nobudget " + ta,
            [&] { return std::to_string(static_cast<int>(probe::should_exit(tr, cfg))); });
        run("nf validate " + ta, [&] {
            cfg.validate();
            return std::string("ok");
        });
        for (int k : {1, 2, 3}) {
            run("nf eps " + ta + " k" + std::to_string(k), [&] {
                auto e = probe::stationary_by_epsilon_test(tr.records, k, specials[a]);
                return e ? std::to_string(*e) : std::string("nullopt");
            });
        }
    }
    // explicit clusterings with oversized clusters and large totals (metrics.cpp:107-125)
    for (std::vector<int> sizes : {std::vector<int>{5, 1}, {3}, {7, 7, 7}, {100000000, 3}, {1, 1 << 30}, {2, -1}}) {
        for (int total : {1, 2, 4, 1 << 28}) {
            metrics::Clustering c;
            for (int x : sizes) c.clusters.push_back({"c", x});
            c.total = total;
            std::string tag = "nf entropy";
            for (int x : sizes) tag += " " + std::to_string(x);
            tag += " /" + std::to_string(total);
            run(tag + " H", [&] { return hex(metrics::semantic_entropy(c)); });
            run(tag + " Hc", [&] { return hex(metrics::certaindex_entropy(c)); });
        }
    }
}

void jsonl_cases() {
    const std::vector<std::string> docs = {
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\" 12 \",\"hesitant\":false}\n"
        "\n  \n"
        "{\"program_id\":\"p\",\"step_index\":2,\"token_offset\":128,\"answer\":\"wait\\n\\u00e9\\ud83d\\ude00\"}\n"
        "{\"program_id\":\"q\",\"step_index\":1,\"token_offset\":64,\"answer\":\"x\\\"y\\\\z\\u0001\",\"hesitant\":true}\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\"a\"}\n"
        "{\"program_id\":\"p\",\"step_index\":2,\"token_offset\":64,\"answer\":\"b\"}\n",
        "{\"program_id\":\"p\",\"step_index\":3,\"token_offset\":64,\"answer\":\"a\"}\n"
        "{\"program_id\":\"p\",\"step_index\":3,\"token_offset\":65,\"answer\":\"b\"}\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\"a\"\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64}\n",
        "{\"program_id\":7,\"step_index\":1,\"token_offset\":64,\"answer\":\"a\"}\n",
        "{\"program_id\":\"p\",\"step_index\":1.9,\"token_offset\":64.5,\"answer\":\"a\",\"hesitant\":true,\"extra\":[1,{}]}\n",
        "{\"program_id\":\"p\",\"step_index\":true,\"token_offset\":64,\"answer\":\"a\"}\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":true,\"answer\":\"a\"}\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\"a\",\"hesitant\":1}\n",
        "[1,2,3]\n",
        "{\"program_id\":\"p\",\"step_index\":01,\"token_offset\":64,\"answer\":\"a\"}\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\"a\"} x\n",
        "{\"program_id\":\"p\",\"program_id\":\"r\",\"step_index\":-2,\"token_offset\":-9,\"answer\":\"\"}\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":1e2,\"answer\":\"a\"}\n",
        "{\"pro\\u0067ram_id\":\"p\",\"step_index\":1,\"token_offset\":2,\"answer\":\"c\"}\r\n"
        "{\"program_id\":\" p\",\"step_index\":1,\"token_offset\":2,\"answer\":\"\\ud83d\\ude00\"}\n \f \n"
        "{\"program_id\":\"p\",\"step_index\":2,\"token_offset\":3,\"answer\":\"caf\xc3\xa9\",\"x\":{\"y\":[[],{}]}}",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\"a\\u0001\"}\n"
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\"a\x01\"}\n",
        "{\"program_id\":\"q\",\"step_index\":5,\"token_offset\":9,\"answer\":\"a\"}\n"
        "{\"program_id\":\"r\",\"step_index\":1,\"token_offset\":1,\"answer\":\"a\"}\n"
        "{\"program_id\":\"q\",\"step_index\":5,\"token_offset\":10,\"answer\":\"b\"}\n",
        "{\"program_id\":\"p\",\"step_index\":1,\"token_offset\":64,\"answer\":\"a\",}",
        "{\"program_id\":\"p\",\"step_index\":-0,\"token_offset\":-9223372036854775808,\"answer\":\"\"}",
    };
    for (size_t d = 0; d < docs.size(); ++d) {
        run("jsonl " + std::to_string(d), [&] {
            std::istringstream in(docs[d]);
            std::vector<probe::TraceLine> lines;
            try {
                lines = probe::read_trace_jsonl(in);
            } catch (const std::runtime_error& e) {
                throw std::runtime_error(jsonl_message(e.what()));
            }
            std::ostringstream out;
            probe::write_trace_jsonl(out, lines);
            return esc(out.str());
        });
    }
    run("jsonl missing file", [] { return std::to_string(probe::read_trace_file("/nonexistent/trace.jsonl").size()); });
}

}  // namespace

// Sizes on both sides of the one-round-trip limit of this repo's scalar entries (2048
// answers / records): the results must not depend on which path took the call.
void size_edge_cases() {
    for (int n : {1, 2047, 2048, 2049, 5000}) {
        std::vector<std::string> a;
        for (int i = 0; i < n; ++i) a.push_back(random_answer() + (i % 97 == 5 ? std::to_string(i % 13) : ""));
        run("size cluster_exact " + std::to_string(n), [&] {
            const auto c = metrics::cluster_exact(a);
            return show(c) + " " + hex(metrics::certaindex_entropy(c));
        });
        auto recs = random_records(n, true);
        run("size consistency " + std::to_string(n), [&] {
            const auto v = probe::consistency(recs, recs.back().step_index - 1, 3);
            return v ? hex(*v) : std::string("nullopt");
        });
        probe::ProbeTrace t;
        t.records = recs;
        probe::ProbeConfig cfg;
        cfg.max_tokens = 1000000;
        run("size should_exit " + std::to_string(n), [&] { return std::to_string(static_cast<int>(probe::should_exit(t, cfg))); });
        run("size final_answer " + std::to_string(n), [&] {
            const auto f = probe::final_answer(t);
            return esc(f.answer) + (f.low_confidence ? " low" : "");
        });
    }
    // hand-built clusterings the reference still evaluates: a cluster larger than the total,
    // a total past 2^26
    for (auto [sz, tot] : {std::pair<int, int>{5, 4}, {3, 2}, {1 << 27, (1 << 27) + 3}, {7, 100000000}}) {
        metrics::Clustering c;
        c.total = tot;
        c.clusters = {{"a", sz}, {"b", 1}};
        run("size entropy " + std::to_string(sz) + "/" + std::to_string(tot),
            [&] { return hex(metrics::semantic_entropy(c)) + " " + hex(metrics::certaindex_entropy(c)); });
    }
    std::string big(1 << 21, 'x');  // one answer above the byte limit
    run("size flag_hesitation big", [&] { return std::to_string(probe::flag_hesitation(big + " WAIT", std::vector<std::string>{"wait"})); });
    run("size cluster_exact big", [&] { return show(metrics::cluster_exact(std::vector<std::string>{big, " " + big})).substr(0, 40); });
}

int main(int argc, char** argv) {
    const int count = argc > 1 ? std::atoi(argv[1]) : 400;
    spec_examples();
    random_cases(count);
    nonfinite_cases();
    jsonl_cases();
    size_edge_cases();
    return 0;
}
