// sim_cases.cpp — the SPEC examples of the sim module through cdx::sim,
// whose scheduling decisions run on the B200 (scheduler::next_batch -> K6).  One line per
// case; tests/test_sim.py checks the values.

#include <cstdio>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "cdx/batch.hpp"
#include "cdx/metrics.hpp"
#include "cdx/sim.hpp"

using namespace cdx;

namespace {
template <class F>
void run(const char* tag, F&& f) {
    try {
        std::printf("%s | %s\n", tag, f().c_str());
    } catch (const std::exception& e) {
        std::printf("%s | EXC %s\n", tag, e.what());
    }
}
std::string num(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.9g", v);
    return b;
}

// Knob-unit SC programs from the synthetic answer process (cdx_gen_sc on the device, the
// counter-based restatement of runtime.cpp:91-117): unit k of program i samples S branches
// (S requests of `tok` tokens); its signals are the reference API's certaindex_entropy(
// cluster_exact(the S answers)) (metrics.hpp, on the B200) and correct_at[k-1] says whether
// the SC plurality vote (runtime.cpp:317-334) at unit k is the stationary answer "S".
std::vector<sim::SimProgram> sc_workload(int n, int cap, int S, uint64_t seed, long tok) {
    batch::Context cx(0);
    cdx_gen_params g{};
    g.seed = seed;
    g.groups = 5;
    g.conv_lo = 1;
    g.conv_hi = static_cast<uint32_t>(cap);
    g.noise_level = 0.5;
    g.residual_noise = 0.0;
    g.solvable_fraction = 0.9;
    batch::DeviceArray<uint32_t> ids(cx, static_cast<size_t>(n) * cap * S);
    cx.check(cdx_gen_sc(cx.raw(), &g, 0, static_cast<uint64_t>(n), static_cast<uint32_t>(cap),
                        static_cast<uint32_t>(S), ids.data()));
    const auto h = ids.download();
    const char* names[5] = {"S", "D1", "D2", "D3", "D4"};
    std::vector<sim::SimProgram> p(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
        p[i].program_id = static_cast<uint32_t>(i);
        p[i].resource_cap = cap;
        p[i].request_tokens.assign(static_cast<size_t>(S), tok);
        for (int k = 0; k < cap; ++k) {
            std::vector<std::string> row;
            for (int b = 0; b < S; ++b) row.push_back(names[h[(static_cast<size_t>(i) * cap + k) * S + b]]);
            metrics::SignalVector sv;
            sv.certaindex_entropy = metrics::certaindex_entropy(metrics::cluster_exact(row));
            p[i].signals.push_back(sv);
            std::vector<std::string> order;
            std::map<std::string, int> cnt;
            for (const auto& a : row)
                if (cnt[a]++ == 0) order.push_back(a);
            std::string best;
            int bw = -1;
            for (const auto& a : order)
                if (cnt[a] > bw) {
                    best = a;
                    bw = cnt[a];
                }
            p[i].correct_at.push_back(best == "S" ? 1 : 0);
        }
    }
    return p;
}

std::string summary(const sim::SimReport& r) {
    long units = 0, dec = 0, cert = 0, maxknob = 0;
    for (const auto& x : r.programs) {
        units += x.knob;
        dec += x.decisions;
        cert += x.cause == scheduler::TerminationCause::Certain ? 1 : 0;
        maxknob = std::max<long>(maxknob, x.knob);
    }
    return num(r.total_tokens) + " " + num(r.accuracy) + " " + std::to_string(units) + " " + std::to_string(dec) +
           " " + std::to_string(cert) + " " + std::to_string(maxknob) + " " + num(r.mean_latency * 1e3) + " " +
           num(r.makespan * 1e3) + " " + num(r.throughput) + " " + std::to_string(r.truncated);
}
}  // namespace

int main() {
    // deadline_for
    run("deadline 1 1 240", [] { return num(sim::deadline_for(1, 1, 240)); });
    run("deadline 1.5 2 60", [] { return num(sim::deadline_for(1.5, 2, 60)); });
    run("deadline 1 3 300", [] { return num(sim::deadline_for(1, 3, 300)); });
    // Fig. 5: 2 programs x 2 requests at t=0, 4 ms / 5 ms requests,
    // capacity 2; durations = tokens / token_rate (1 token per ms)
    std::vector<sim::SimProgram> fig5(2);
    fig5[0].program_id = 0;
    fig5[0].request_tokens = {4, 4};
    fig5[1].program_id = 1;
    fig5[1].request_tokens = {5, 5};
    sim::SimConfig cfg;
    cfg.batch_capacity = 2;
    cfg.token_rate = 1000.0;  // tokens per second: 4 tokens = 4 ms
    cfg.policy.starvation_limit = 1e9;
    run("fig5 gang", [&] { return num(sim::run(fig5, cfg).mean_latency * 1e3); });
    cfg.policy.gang = false;
    run("fig5 interleaved", [&] { return num(sim::run(fig5, cfg).mean_latency * 1e3); });
    cfg.policy.gang = true;
    run("zero programs", [&] {
        const auto r = sim::run({}, cfg);
        return std::to_string(r.programs.size()) + " " + num(r.total_tokens);
    });
    // single program: gang on/off identical
    run("single program", [&] {
        std::vector<sim::SimProgram> one(1);
        one[0].request_tokens = {3, 7, 2};
        auto c = cfg;
        const double a = sim::run(one, c).mean_latency;
        c.policy.gang = false;
        return num(a * 1e3) + " " + num(sim::run(one, c).mean_latency * 1e3);
    });
    // SJF by estimated remaining work: a later-arriving short program overtakes a long one
    run("sjf", [&] {
        std::vector<sim::SimProgram> p(3);
        p[0].program_id = 10;
        p[0].request_tokens = {10, 10, 10, 10, 10, 10};  // 6 requests: large remaining knob
        p[1].program_id = 11;
        p[1].arrival = 0.001;
        p[1].request_tokens = {10};
        p[2].program_id = 12;
        p[2].arrival = 0.001;
        p[2].request_tokens = {10, 10};
        auto c = cfg;
        c.batch_capacity = 1;
        c.policy.prior_tokens = 10.0;  // per-iteration estimate before any history
        const auto r = sim::run(p, c);
        return num(r.programs[0].completion * 1e3) + " " + num(r.programs[1].completion * 1e3) + " " +
               num(r.programs[2].completion * 1e3);
    });
    // attainment: deadlines met / total, horizon truncation = missed
    run("attainment", [&] {
        std::vector<sim::SimProgram> p(10);
        for (int i = 0; i < 10; ++i) {
            p[i].program_id = static_cast<uint32_t>(i);
            p[i].request_tokens = {10};
            p[i].deadline = i < 9 ? 1.0 : 0.005;  // the last one cannot make 5 ms behind 9 others
        }
        auto c = cfg;
        c.batch_capacity = 1;
        const auto r = sim::run(p, c);
        c.horizon = 0.035;
        const auto t = sim::run(p, c);
        return num(sim::attainment(r)) + " " + num(sim::attainment(t)) + " " + std::to_string(t.truncated);
    });
    run("attainment empty", [&] { return num(sim::attainment(sim::SimReport{})); });
    // Poisson arrivals: cumulative exponential gaps from derive_seed(seed, i)
    run("poisson", [&] {
        const auto t = sim::poisson_arrivals(6, 250.0, 99);
        std::string o;
        for (double x : t) o += num(x) + " ";
        return o;
    });
    // knob-unit SC programs under Poisson arrivals: allocate at the detect / recheck points
    // (SPEC.md:519).  One line per policy: total tokens, accuracy, units, allocate calls,
    // certain exits, largest knob, mean latency (ms), makespan (ms), tokens/s, truncated.
    const int NP = 48, CAP = 16, SS = 8;
    std::vector<sim::SimProgram> W;
    try {
        W = sc_workload(NP, CAP, SS, 20993, 64);
    } catch (const std::exception& e) {
        std::printf("knob workload | EXC %s\n", e.what());
        return 0;
    }
    sim::SimConfig kc;
    kc.batch_capacity = 16;
    kc.token_rate = 64000.0;  // 1 ms per 64-token request
    kc.policy.starvation_limit = 0.05;
    kc.arrival_rate = 400.0;
    kc.seed = 5;
    auto knob_run = [&](scheduler::AllocationKind kind, double tau, int detect, int every) {
        auto c = kc;
        c.allocation.kind = kind;
        c.allocation.detect_at_knob = detect;
        c.allocation.recheck_every = every;
        c.allocation.thresholds = {{metrics::SignalKind::CertaindexEntropy, tau}};
        return sim::run(W, c);
    };
    run("knob even", [&] { return summary(knob_run(scheduler::AllocationKind::Even, 1.0, 1, 1)); });
    run("knob static", [&] { return summary(knob_run(scheduler::AllocationKind::StaticThreshold, 1.0, 4, 1)); });
    run("knob kstep", [&] { return summary(knob_run(scheduler::AllocationKind::KStepThreshold, 1.0, 2, 1)); });
    run("knob kstep tau0.7", [&] { return summary(knob_run(scheduler::AllocationKind::KStepThreshold, 0.7, 2, 1)); });
    run("knob kstep repeat", [&] { return summary(knob_run(scheduler::AllocationKind::KStepThreshold, 1.0, 2, 1)); });
    // per-program knobs at two thresholds (threshold monotonicity)
    run("knob monotone", [&] {
        const auto lo = knob_run(scheduler::AllocationKind::KStepThreshold, 0.6, 2, 1);
        const auto hi = knob_run(scheduler::AllocationKind::KStepThreshold, 0.9, 2, 1);
        int bad = 0;
        for (size_t i = 0; i < lo.programs.size(); ++i) bad += hi.programs[i].knob < lo.programs[i].knob;
        return std::to_string(bad);
    });
    // the token-to-accuracy curve over resource caps under even allocation
    run("curve", [&] {
        std::vector<sim::SimReport> reps;
        for (int cap : {16, 8}) {
            auto w = W;
            for (auto& p : w) p.resource_cap = cap;
            auto c = kc;
            c.allocation.kind = scheduler::AllocationKind::Even;
            reps.push_back(sim::run(w, c));
        }
        std::string o;
        for (const auto& [t, a] : sim::token_accuracy_curve(reps)) o += num(t) + ":" + num(a) + " ";
        return o;
    });
    return 0;
}
