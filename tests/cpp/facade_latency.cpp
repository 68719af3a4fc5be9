// facade_latency.cpp — per-call latency of the reference's scalar C++ API.
//
// Written only against the reference's public headers (cdx/metrics.hpp, cdx/probe.hpp) and
// compiled twice, like dropin_cases.cpp:
//   oracle/_ref/facade_latency_ref    the reference's own metrics.cpp / probe.cpp (host CPU)
//   tests/cpp/bin/facade_latency_ours this repo's headers + libcdxhost.so (B200 kernels)
// Each line: "<call> <microseconds per call> <checksum>" (median of 7 batches after a
// warm-up).  The checksum keeps the calls from being optimised away and lets the two builds
// be compared for equal results.  The shapes are the per-program calls of the reference's
// runtime.cpp update_certaindex: 32 answers per SC program, 16 rewards per
// MCTS step, a 64-record CoT trace.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "cdx/metrics.hpp"
#include "cdx/probe.hpp"

using namespace cdx;

namespace {

template <class F>
double time_us(F&& f, int reps) {
    for (int i = 0; i < 20; ++i) f();  // warm-up (first-call context creation, table uploads)
    std::vector<double> batches;
    for (int b = 0; b < 7; ++b) {
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < reps; ++i) f();
        const auto t1 = std::chrono::steady_clock::now();
        batches.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count() / reps);
    }
    std::sort(batches.begin(), batches.end());
    return batches[3];
}

}  // namespace

int main(int argc, char** argv) {
    const int reps = argc > 1 ? std::atoi(argv[1]) : 200;
    std::vector<std::string> answers;
    const char* vocab[] = {"42", " 42", "41", "wait, 42", "7 ", "\t42\n"};
    for (int i = 0; i < 32; ++i) answers.push_back(vocab[(i * 7 + i / 3) % 6]);
    metrics::Clustering cl = metrics::cluster_exact(answers);
    metrics::RewardSet rs;
    for (int i = 0; i < 16; ++i) rs.rewards.push_back((i * 37 % 100) / 128.0);
    metrics::SignalVector sv;
    sv.certaindex_entropy = 0.75;
    const metrics::SignalThreshold th[1] = {{metrics::SignalKind::CertaindexEntropy, 0.7, metrics::ThresholdDir::GreaterEq}};
    const std::vector<std::string> markers = {"wait", "hmm"};
    probe::ProbeTrace tr;
    for (int i = 0; i < 64; ++i)
        tr.records.push_back({i, (i + 1) * 64, vocab[(i * 5 + i / 7) % 6], (i % 11) == 3});
    probe::ProbeConfig cfg;
    cfg.interval_tokens = 64;
    cfg.window = 3;
    cfg.threshold = 0.9;
    cfg.max_tokens = 4096;

    double sink = 0;
    auto row = [&](const char* name, double us) { std::printf("%-28s %10.2f %.17g\n", name, us, sink); };
    row("cluster_exact[32]", time_us([&] { sink += metrics::cluster_exact(answers).group_count(); }, reps));
    row("certaindex_entropy", time_us([&] { sink += metrics::certaindex_entropy(cl); }, reps));
    row("semantic_entropy", time_us([&] { sink += metrics::semantic_entropy(cl); }, reps));
    row("certaindex_reward[16]", time_us([&] { sink += metrics::certaindex_reward(rs); }, reps));
    row("combined_meets_thresholds", time_us([&] { sink += metrics::combined_meets_thresholds(sv, th) ? 1 : 0; }, reps));
    row("flag_hesitation", time_us([&] { sink += probe::flag_hesitation("I think, WAIT, 42", markers) ? 1 : 0; }, reps));
    row("consistency[64]", time_us([&] { sink += probe::consistency(tr.records, 40, 3).value_or(-1.0); }, reps));
    row("should_exit[64]", time_us([&] { sink += static_cast<int>(probe::should_exit(tr, cfg)); }, reps));
    row("final_answer[64]", time_us([&] { sink += probe::final_answer(tr).answer.size(); }, reps));
    // one SC program's update_certaindex (runtime.cpp:264-313): cluster, entropy, thresholds
    row("sc_update[32]", time_us([&] {
            const auto c = metrics::cluster_exact(answers);
            metrics::SignalVector s;
            s.certaindex_entropy = metrics::certaindex_entropy(c);
            sink += metrics::combined_meets_thresholds(s, th) ? 1 : 0;
        }, reps));
    return 0;
}
