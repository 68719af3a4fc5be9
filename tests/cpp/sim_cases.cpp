// sim_cases.cpp — the SPEC examples of the sim module through cdx::sim,
// whose scheduling decisions run on the B200 (scheduler::next_batch -> K6).  One line per
// case; tests/test_sim.py checks the values.

#include <cstdio>
#include <exception>
#include <string>
#include <vector>

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
    return 0;
}
