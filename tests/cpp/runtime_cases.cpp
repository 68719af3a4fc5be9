// runtime_cases.cpp — the reference's own hot-path caller, ProgramDriver (runtime.cpp), run
// unchanged: written only against the reference's headers (cdx/runtime.hpp), it drives
// synthetic programs of every archetype and a replayed CoT trace through expand /
// on_request_complete / update_certaindex / aggregate, printing every signal and decision.
//
// Built twice by oracle/Makefile, from the reference sources where they lie:
//   _ref/runtime_ref   runtime.cpp + metrics.cpp + probe.cpp + theory.cpp (all reference)
//   _ref/runtime_ours  runtime.cpp + theory.cpp compiled against include/cdx (this repo's
//                      metrics.hpp / probe.hpp first), linked with libcdxhost.so: every
//                      certaindex, clustering and probe decision then runs on the B200.
// tests/test_dropin.py requires identical output.

#include <cstdio>
#include <deque>
#include <exception>
#include <string>
#include <vector>

#include "cdx/runtime.hpp"

using namespace cdx;
using namespace cdx::runtime;

namespace {

void print_opt(const char* name, const std::optional<double>& v) {
    if (v) std::printf(" %s=%.17g", name, *v);
    else std::printf(" %s=-", name);
}

void print_signals(const metrics::SignalVector& s) {
    print_opt("H", s.certaindex_entropy);
    print_opt("R", s.certaindex_reward);
    print_opt("L", s.mean_output_length);
}

// One program driven unit by unit: expand one knob unit, complete its requests in issue
// order (chains continue through on_request_complete), evaluate the certaindex.
void drive(ProgramDriver& d, const char* tag, int max_units) {
    double now = 0.0;
    for (int unit = 0; unit < max_units; ++unit) {
        const auto& prog = d.program();
        if (prog.status == ProgramStatus::Terminated || prog.knob >= prog.resource_cap) break;
        std::vector<Request> reqs;
        try {
            reqs = d.expand(1, now);
        } catch (const std::exception& e) {
            std::printf("%s expand EXC %s\n", tag, e.what());
            break;
        }
        if (reqs.empty()) break;
        std::deque<Request> q(reqs.begin(), reqs.end());
        while (!q.empty()) {
            Request r = q.front();
            q.pop_front();
            now += 0.001 * static_cast<double>(r.tokens);
            if (auto nx = d.on_request_complete(r, now)) q.push_back(*nx);
        }
        try {
            const auto sv = d.update_certaindex();
            std::printf("%s unit=%d knob=%d done=%d tokens=%ld", tag, unit, d.program().knob, d.completed_units(),
                        d.program().tokens_used);
            print_signals(sv);
            std::printf("\n");
        } catch (const std::exception& e) {
            std::printf("%s unit=%d EXC %s\n", tag, unit, e.what());
        }
    }
    if (d.program().status != ProgramStatus::Terminated) d.terminate(probe::TerminationReason::CriteriaExternal);
    try {
        const auto a = d.aggregate();
        std::printf("%s final=%s correct=%d low=%d\n", tag, a.answer.c_str(), a.correct ? 1 : 0, a.low_confidence ? 1 : 0);
    } catch (const std::exception& e) {
        std::printf("%s final EXC %s\n", tag, e.what());
    }
    const auto& h = d.program().certaindex_history;
    std::printf("%s history=%zu", tag, h.size());
    for (const auto& pt : h) {
        std::printf(" k%d", pt.knob_point);
        print_opt("H", pt.signals.certaindex_entropy);
        print_opt("R", pt.signals.certaindex_reward);
    }
    std::printf("\n");
    for (int u = 1; u <= d.completed_units(); ++u) {
        try {
            const auto a = d.aggregate_prefix(u);
            std::printf("%s prefix=%d %s %d %d\n", tag, u, a.answer.c_str(), a.correct ? 1 : 0, a.low_confidence ? 1 : 0);
        } catch (const std::exception& e) {
            std::printf("%s prefix=%d EXC %s\n", tag, u, e.what());
        }
    }
}

}  // namespace

int main() {
    const Archetype kinds[4] = {Archetype::SC, Archetype::Rebase, Archetype::MCTS, Archetype::CoT};
    for (int ai = 0; ai < 4; ++ai) {
        WorkloadParams wp;
        wp.count = 12;
        wp.archetype = kinds[ai];
        wp.answer_groups = 4 + ai;
        wp.noise_level = 0.6;
        wp.solvable_fraction = 0.8;
        wp.hesitation_prob = kinds[ai] == Archetype::CoT ? 0.2 : 0.0;
        wp.convergence_max = 8;
        wp.caps = {6, 10, 14};
        wp.with_rewards = kinds[ai] == Archetype::MCTS || kinds[ai] == Archetype::Rebase;
        wp.mcts_chain_len = 2;
        wp.rebase_max_depth = 5;
        std::vector<SyntheticProgramSpec> specs;
        try {
            specs = generate_workload(wp, 20993 + ai);
        } catch (const std::exception& e) {
            std::printf("workload %d EXC %s\n", ai, e.what());
            continue;
        }
        for (size_t i = 0; i < specs.size(); ++i) {
            ProgramDriver d(i, std::string(archetype_name(kinds[ai])) + "-" + std::to_string(i), specs[i], 7 + ai);
            const std::string tag = std::string(archetype_name(kinds[ai])) + "#" + std::to_string(i);
            drive(d, tag.c_str(), 20);
        }
    }
    // a recorded CoT trace replayed through the driver (runtime.hpp:268-270)
    std::vector<probe::TraceLine> lines;
    const char* ans[6] = {"12", " 12", "wait, 13", "13", "13 ", "hmm 14"};
    for (int p = 0; p < 3; ++p)
        for (int k = 0; k < 9; ++k) {
            probe::TraceLine tl;
            tl.program_id = "trace-" + std::to_string(p);
            tl.record.step_index = k + 1;
            tl.record.token_offset = 64L * (k + 1);
            tl.record.answer = ans[(k + p) % 6];
            tl.record.hesitant = ((k + p) % 6) == 2 || ((k + p) % 6) == 5;
            lines.push_back(tl);
        }
    probe::ProbeConfig cfg;
    cfg.window = 3;
    cfg.threshold = 0.6;
    try {
        auto drivers = replay_trace_lines(lines, cfg);
        for (size_t i = 0; i < drivers.size(); ++i) drive(drivers[i], ("trace#" + std::to_string(i)).c_str(), 12);
    } catch (const std::exception& e) {
        std::printf("replay EXC %s\n", e.what());
    }
    return 0;
}
