// scheduler_cases.cpp — caller of include/cdx/scheduler.hpp on the B200.
// Prints the SPEC examples' outcomes, then seeded random program sets as
//   "order <case> <n> | <inputs...> | <ids...>"
// which tests/test_gpu_scheduler_facade.py re-evaluates with the SPEC restatement
// (oracle/cdx_oracle.c: cdxo_gang_order / cdxo_allocate_scan).

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>
#include <vector>

#include "cdx/scheduler.hpp"

using namespace cdx;

namespace {

uint64_t g_state = 0x5C4ED0ULL;
uint64_t next_u64() {
    g_state ^= g_state >> 12;
    g_state ^= g_state << 25;
    g_state ^= g_state >> 27;
    return g_state * 0x2545F4914F6CDD1DULL;
}
uint32_t below(uint32_t n) { return static_cast<uint32_t>(next_u64() % n); }

const char* action(const scheduler::AllocationDecision& d) {
    return d.action == scheduler::AllocationAction::Terminate
               ? (d.cause == scheduler::TerminationCause::Certain ? "terminate_certain" : "terminate_cap")
               : "grant";
}

template <class F>
void run(const std::string& tag, F&& f) {
    try {
        std::printf("%s | %s\n", tag.c_str(), f().c_str());
    } catch (const std::exception& e) {
        std::printf("%s | EXC %s\n", tag.c_str(), e.what());
    }
}

}  // namespace

int main(int argc, char** argv) {
    const int count = argc > 1 ? std::atoi(argv[1]) : 40;
    using metrics::SignalKind;
    scheduler::AllocationPolicy sc;  // Table 3 SC/GSM8K: H~ >= 0.7 at detect@5, cap 20
    sc.kind = scheduler::AllocationKind::StaticThreshold;
    sc.detect_at_knob = 5;
    sc.resource_cap = 20;
    sc.thresholds = {{SignalKind::CertaindexEntropy, 0.7}};
    auto hist = [](double h, int n) {
        std::vector<metrics::SignalVector> v(static_cast<size_t>(n));
        for (auto& s : v) s.certaindex_entropy = h;
        return v;
    };
    // SPEC.md:410-412
    run("spec allocate 0.72", [&] {
        auto d = scheduler::allocate(hist(0.72, 5), 5, sc);
        return std::string(action(d));
    });
    run("spec allocate 0.3", [&] {
        auto d = scheduler::allocate(hist(0.3, 5), 5, sc);
        return std::string(action(d)) + " " + std::to_string(d.grant_units);
    });
    run("spec allocate cap", [&] { return std::string(action(scheduler::allocate(hist(0.0, 20), 20, sc))); });
    run("spec allocate before detect", [&] {
        auto d = scheduler::allocate(hist(0.99, 3), 3, sc);
        return std::string(action(d)) + " " + std::to_string(d.grant_units);
    });
    run("spec allocate absent signal", [&] {
        std::vector<metrics::SignalVector> v(5);
        for (auto& s : v) s.certaindex_reward = 0.9;
        return std::string(action(scheduler::allocate(v, 5, sc)));
    });
    run("spec allocate kstep", [&] {
        auto p = sc;
        p.kind = scheduler::AllocationKind::KStepThreshold;
        p.recheck_every = 3;
        auto v = hist(0.1, 12);
        v[10].certaindex_entropy = 0.8;  // knob 11 = 5 + 2*3 is a recheck point
        auto a = scheduler::allocate(v, 10, p);
        auto b = scheduler::allocate(v, 11, p);
        return std::string(action(a)) + " " + std::to_string(a.grant_units) + " / " + action(b);
    });
    // SPEC.md:437-439
    run("spec estimate", [] {
        const long h1[] = {100, 200}, h3[] = {64};
        return std::to_string(scheduler::estimate_iteration_tokens(h1, 128.0)) + " " +
               std::to_string(scheduler::estimate_iteration_tokens({}, 128.0)) + " " +
               std::to_string(scheduler::estimate_iteration_tokens(h3, 128.0));
    });
    // SPEC.md:446-448
    run("spec escalate", [] {
        std::vector<scheduler::ProgramState> p(3);
        p[0] = {0, 0.0, 10.0};  // wait 0 < limit
        p[1] = {1, 1.0, 5.0};   // wait = limit
        p[2] = {2, 0.5, 4.0};   // wait > limit
        auto e = scheduler::escalate(p, 10.0, 5.0);
        return std::to_string(e[0]) + std::to_string(e[1]) + std::to_string(e[2]);
    });
    run("spec escalated fifo", [] {
        std::vector<scheduler::ProgramState> p(3);
        p[0] = {7, 2.0, 0.0, 0, 0, 0, 10};
        p[1] = {8, 1.0, 0.0, 0, 0, 0, 10};
        p[2] = {9, 0.5, 9.9, 0, 0, 0, 1};  // not escalated, shortest job
        scheduler::InterSchedPolicy pol;
        pol.starvation_limit = 5.0;
        std::string o;
        for (auto id : scheduler::program_order(p, pol, 10.0)) o += std::to_string(id) + " ";
        return o;
    });
    // Fig. 5: 2 programs x 2 requests, capacity 2, gang on
    run("spec next_batch gang", [] {
        std::vector<scheduler::ProgramState> p(2);
        p[0] = {0, 0.0, 0.0, 4 * 2, 2, 0, 2};
        p[1] = {1, 0.0, 0.0, 5 * 2, 2, 0, 2};
        std::vector<scheduler::Request> ready = {{0, 0}, {1, 0}, {0, 1}, {1, 1}};
        scheduler::InterSchedPolicy pol;
        pol.batch_capacity = 2;
        pol.starvation_limit = 100.0;
        std::string o;
        for (auto r : scheduler::next_batch(ready, p, pol, 0.0))
            o += std::to_string(r.program_id) + ":" + std::to_string(r.branch) + " ";
        pol.gang = false;
        o += "/ ";
        for (auto r : scheduler::next_batch(ready, p, pol, 0.0))
            o += std::to_string(r.program_id) + ":" + std::to_string(r.branch) + " ";
        return o;
    });
    // random program sets: inputs then the device order
    for (int c = 0; c < count; ++c) {
        const int n = 1 + static_cast<int>(below(c % 4 == 0 ? 5000 : 60));
        std::vector<scheduler::ProgramState> p(static_cast<size_t>(n));
        double t = 0.0;
        for (int i = 0; i < n; ++i) {
            auto& s = p[static_cast<size_t>(i)];
            // odd cases: shuffled, sparse program ids (the tie-break is the id, not the position)
            s.program_id = c % 2 ? static_cast<uint32_t>(i) * 7919u % 100003u + 11u * static_cast<uint32_t>(c)
                                 : static_cast<uint32_t>(i);
            t += below(3) == 0 ? 0.0 : static_cast<double>(below(1000)) * 0x1p-10;  // ties on arrival
            s.arrival = below(5) == 0 ? static_cast<double>(below(8)) : t;
            s.last_service = static_cast<double>(below(64)) * 0x1p-3;
            s.iteration_count = below(4);
            s.iteration_token_sum = static_cast<int64_t>(below(300)) * s.iteration_count;
            s.resource_cap = 1 + static_cast<int>(below(20));
            s.knob = static_cast<int>(below(static_cast<uint32_t>(s.resource_cap) + 1));
            s.terminated = below(6) == 0;
        }
        scheduler::InterSchedPolicy pol;
        pol.order = below(2) ? scheduler::InterOrder::SjfEstimated : scheduler::InterOrder::Fifo;
        pol.starvation_limit = 1.0 + static_cast<double>(below(8));
        const double now = 8.0;
        std::string line = "order " + std::to_string(c) + " " + std::to_string(n) + " " +
                           std::to_string(static_cast<int>(pol.order)) + " " + std::to_string(pol.starvation_limit) + " |";
        for (const auto& s : p) {
            char b[160];
            std::snprintf(b, sizeof b, " %a,%a,%lld,%u,%d,%d,%d,%u", s.arrival, s.last_service,
                          static_cast<long long>(s.iteration_token_sum), s.iteration_count, s.knob, s.resource_cap,
                          s.terminated ? 1 : 0, s.program_id);
            line += b;
        }
        line += " |";
        try {
            for (auto id : scheduler::program_order(p, pol, now)) line += " " + std::to_string(id);
        } catch (const std::exception& e) {
            line += std::string(" EXC ") + e.what();
        }
        std::printf("%s\n", line.c_str());
    }
    return 0;
}
