// facade_sim.cpp — cdx::sim (include/cdx/sim.hpp).  An event loop on the
// host (the simulator is sequential by nature) whose every scheduling
// decision is scheduler::next_batch, i.e. K6's program order on the B200.

#include "cdx/sim.hpp"

#include <algorithm>
#include <queue>
#include <stdexcept>
#include <tuple>
#include <vector>

namespace cdx::sim {

double deadline_for(double slo_scale, double difficulty_factor, double base_deadline) {
    return slo_scale * difficulty_factor * base_deadline;
}

namespace {

struct Event {
    double time;
    int kind;  // 0 completion (frees a slot first), 1 arrival
    uint64_t id;
    bool operator>(const Event& o) const {
        return std::tie(time, kind, id) > std::tie(o.time, o.kind, o.id);
    }
};

struct ProgState {
    size_t total = 0, issued = 0, done = 0;
    double last_service = 0.0;
    int64_t tok_sum = 0;
    uint32_t tok_count = 0;
    bool arrived = false;
};

}  // namespace

SimReport run(std::span<const SimProgram> programs, const SimConfig& cfg) {
    if (cfg.batch_capacity < 1) throw std::invalid_argument("sim: batch_capacity must be >= 1");
    if (!(cfg.token_rate > 0.0)) throw std::invalid_argument("sim: token_rate must be > 0");
    SimReport rep;
    const size_t np = programs.size();
    rep.programs.resize(np);
    if (np == 0) return rep;
    std::vector<ProgState> ps(np);
    std::priority_queue<Event, std::vector<Event>, std::greater<Event>> ev;
    for (size_t i = 0; i < np; ++i) {
        rep.programs[i].program_id = programs[i].program_id;
        rep.programs[i].arrival = programs[i].arrival;
        rep.programs[i].deadline = programs[i].deadline;
        ps[i].total = programs[i].request_tokens.size();
        ps[i].last_service = programs[i].arrival;
        ev.push({programs[i].arrival, 1, i});
    }
    // in-flight requests: (program index, branch) by event id = np + request serial
    std::vector<std::pair<size_t, size_t>> flight;
    std::vector<scheduler::Request> ready;  // gang off keeps this order (round-robin, below)
    int running = 0;
    while (!ev.empty()) {
        const double now = ev.top().time;
        if (now > cfg.horizon) {
            rep.truncated = true;
            break;
        }
        while (!ev.empty() && ev.top().time == now) {  // every event at this instant
            const Event e = ev.top();
            ev.pop();
            if (e.kind == 1) {
                ps[e.id].arrived = true;
                for (size_t b = 0; b < ps[e.id].total; ++b)
                    ready.push_back({programs[e.id].program_id, static_cast<int>(b)});
                if (ps[e.id].total == 0) {
                    rep.programs[e.id].finished = true;
                    rep.programs[e.id].completion = now;
                }
            } else {
                const auto [pi, br] = flight[e.id - np];
                --running;
                const long tk = programs[pi].request_tokens[br];
                ps[pi].tok_sum += tk;
                ++ps[pi].tok_count;
                rep.programs[pi].tokens += tk;
                rep.total_tokens += static_cast<double>(tk);
                if (++ps[pi].done == ps[pi].total) {
                    rep.programs[pi].finished = true;
                    rep.programs[pi].completion = now;
                }
            }
        }
        // scheduling opportunity: fill the free slots (event-driven)
        const int free = cfg.batch_capacity - running;
        if (free <= 0 || ready.empty()) continue;
        std::vector<size_t> idx_of(np);  // program id -> index (ids are caller labels)
        std::vector<scheduler::ProgramState> states;
        for (size_t i = 0; i < np; ++i) {
            if (!ps[i].arrived || ps[i].issued == ps[i].total) continue;
            scheduler::ProgramState s;
            s.program_id = programs[i].program_id;
            s.arrival = programs[i].arrival;
            s.last_service = ps[i].last_service;
            s.iteration_token_sum = ps[i].tok_sum;
            s.iteration_count = ps[i].tok_count;
            s.knob = static_cast<int>(ps[i].issued);
            s.resource_cap = static_cast<int>(ps[i].total);
            states.push_back(s);
        }
        if (!cfg.policy.gang)  // request-level order: round-robin over programs (branch-major)
            std::stable_sort(ready.begin(), ready.end(), [&](const scheduler::Request& x, const scheduler::Request& y) {
                return x.branch < y.branch;
            });
        scheduler::InterSchedPolicy pol = cfg.policy;
        pol.batch_capacity = free;
        const auto batch = scheduler::next_batch(ready, states, pol, now);
        for (const auto& r : batch) {
            size_t pi = np;
            for (size_t i = 0; i < np; ++i)
                if (programs[i].program_id == r.program_id) pi = i;
            if (pi == np) continue;
            ++ps[pi].issued;
            ps[pi].last_service = now;
            ++running;
            flight.push_back({pi, static_cast<size_t>(r.branch)});
            const double dur = static_cast<double>(programs[pi].request_tokens[static_cast<size_t>(r.branch)]) /
                               cfg.token_rate;
            ev.push({now + dur, 0, np + flight.size() - 1});
            ready.erase(std::find_if(ready.begin(), ready.end(), [&](const scheduler::Request& x) {
                return x.program_id == r.program_id && x.branch == r.branch;
            }));
        }
    }
    double sum = 0.0;
    size_t fin = 0;
    for (size_t i = 0; i < np; ++i) {
        auto& pr = rep.programs[i];
        if (!pr.finished) {
            rep.truncated = true;
            continue;
        }
        pr.latency = pr.completion - pr.arrival;  // queueing included
        pr.met = pr.deadline <= 0.0 || pr.latency <= pr.deadline;
        sum += pr.latency;
        ++fin;
    }
    rep.mean_latency = fin ? sum / static_cast<double>(fin) : 0.0;
    return rep;
}

double attainment(const SimReport& report) {
    if (report.programs.empty()) throw std::invalid_argument("attainment: empty report");
    size_t met = 0;
    for (const auto& p : report.programs) met += (p.finished && p.met) ? 1 : 0;
    return static_cast<double>(met) / static_cast<double>(report.programs.size());
}

}  // namespace cdx::sim
