// facade_sim.cpp — cdx::sim (include/cdx/sim.hpp).  An event loop on the
// host (the simulator is sequential by nature) whose every scheduling
// decision is scheduler::next_batch, i.e. K6's program order on the B200, and whose every
// budget decision is scheduler::allocate (thresholds + K5 on the B200).

#include "cdx/sim.hpp"

#include <algorithm>
#include <cmath>
#include <queue>
#include <stdexcept>
#include <tuple>
#include <vector>

namespace cdx::sim {

double deadline_for(double slo_scale, double difficulty_factor, double base_deadline) {
    return slo_scale * difficulty_factor * base_deadline;
}

namespace {

// splitmix64 and the derived-seed mixing of the reference (rng.hpp:25-34)
uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
uint64_t derive_seed(uint64_t master, uint64_t a, uint64_t b) {
    return mix64(mix64(master ^ mix64(a)) ^ mix64(b ^ 0xa5a5a5a5a5a5a5a5ULL));
}

struct Event {
    double time;
    int kind;  // 0 completion (frees a slot first), 1 arrival
    uint64_t id;
    bool operator>(const Event& o) const {
        return std::tie(time, kind, id) > std::tie(o.time, o.kind, o.id);
    }
};

struct ProgState {
    size_t total = 0, issued = 0, done = 0;  // requests (fixed) / of the current unit (knob)
    double last_service = 0.0;
    int64_t tok_sum = 0;      // completed iteration token counts
    uint32_t tok_count = 0;
    int64_t unit_tokens = 0;  // tokens of the unit in flight
    int knob = 0;             // knob-unit programs: units completed
    bool arrived = false;
};

// a detect / recheck point of the policy at knob k (1-based), or the cap
bool decision_point(const scheduler::AllocationPolicy& pol, int k, int cap) {
    if (k >= cap) return true;
    switch (pol.kind) {
        case scheduler::AllocationKind::StaticThreshold: return k == pol.detect_at_knob;
        case scheduler::AllocationKind::KStepThreshold:
            return k >= pol.detect_at_knob && (k - pol.detect_at_knob) % pol.recheck_every == 0;
        default: return false;
    }
}

}  // namespace

std::vector<double> poisson_arrivals(size_t n, double rate, uint64_t seed) {
    if (!(rate > 0.0)) throw std::invalid_argument("sim: arrival rate must be > 0");
    std::vector<double> t(n);
    double now = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double u = static_cast<double>(derive_seed(seed, i, 0) >> 11) * 0x1.0p-53;  // [0, 1)
        now += -std::log1p(-u) / rate;
        t[i] = now;
    }
    return t;
}

SimReport run(std::span<const SimProgram> programs, const SimConfig& cfg) {
    if (cfg.batch_capacity < 1) throw std::invalid_argument("sim: batch_capacity must be >= 1");
    if (!(cfg.token_rate > 0.0)) throw std::invalid_argument("sim: token_rate must be > 0");
    SimReport rep;
    const size_t np = programs.size();
    rep.programs.resize(np);
    if (np == 0) return rep;
    std::vector<double> arrival(np);
    if (cfg.arrival_rate > 0.0) arrival = poisson_arrivals(np, cfg.arrival_rate, cfg.seed);
    else
        for (size_t i = 0; i < np; ++i) arrival[i] = programs[i].arrival;
    std::vector<ProgState> ps(np);
    std::priority_queue<Event, std::vector<Event>, std::greater<Event>> ev;
    for (size_t i = 0; i < np; ++i) {
        const SimProgram& p = programs[i];
        if (p.resource_cap > 0 && p.signals.size() < static_cast<size_t>(p.resource_cap))
            throw std::invalid_argument("sim: a knob-unit program needs a signal vector per unit");
        if (p.resource_cap > 0 && p.request_tokens.empty())
            throw std::invalid_argument("sim: a knob-unit program needs at least one branch");
        rep.programs[i].program_id = p.program_id;
        rep.programs[i].arrival = arrival[i];
        rep.programs[i].deadline = p.deadline;
        ps[i].total = p.request_tokens.size();
        ps[i].last_service = arrival[i];
        ev.push({arrival[i], 1, i});
    }
    auto finish = [&](size_t i, double now, scheduler::TerminationCause cause) {
        auto& pr = rep.programs[i];
        pr.finished = true;
        pr.completion = now;
        pr.knob = ps[i].knob;
        pr.cause = cause;
        const auto& c = programs[i].correct_at;
        pr.correct = ps[i].knob > 0 && static_cast<size_t>(ps[i].knob) <= c.size() && c[ps[i].knob - 1] != 0;
    };
    // in-flight requests: (program index, branch) by event id = np + request serial
    std::vector<std::pair<size_t, size_t>> flight;
    std::vector<scheduler::Request> ready;  // gang off keeps this order (round-robin, below)
    auto release_unit = [&](size_t i) {     // the branch requests of the next iteration
        ps[i].issued = ps[i].done = 0;
        ps[i].unit_tokens = 0;
        for (size_t b = 0; b < ps[i].total; ++b) ready.push_back({programs[i].program_id, static_cast<int>(b)});
    };
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
                if (ps[e.id].total == 0) finish(e.id, now, scheduler::TerminationCause::None);
                else release_unit(e.id);
                continue;
            }
            const auto [pi, br] = flight[e.id - np];
            --running;
            const long tk = programs[pi].request_tokens[br];
            rep.programs[pi].tokens += tk;
            rep.total_tokens += static_cast<double>(tk);
            ProgState& s = ps[pi];
            if (programs[pi].resource_cap == 0) {  // fixed program: one request = one iteration
                s.tok_sum += tk;
                ++s.tok_count;
                if (++s.done == s.total) finish(pi, now, scheduler::TerminationCause::None);
                continue;
            }
            s.unit_tokens += tk;
            if (++s.done < s.total) continue;
            // knob unit complete: its signals join the history; allocate at decision points
            s.tok_sum += s.unit_tokens;
            ++s.tok_count;
            const int k = ++s.knob;
            const int cap = programs[pi].resource_cap;
            if (!decision_point(cfg.allocation, k, cap)) {
                release_unit(pi);
                continue;
            }
            scheduler::AllocationPolicy pol = cfg.allocation;
            pol.resource_cap = cap;
            const auto d = scheduler::allocate(std::span<const metrics::SignalVector>(programs[pi].signals).first(k),
                                               k, pol);
            ++rep.programs[pi].decisions;
            if (d.action == scheduler::AllocationAction::Terminate) finish(pi, now, d.cause);
            else release_unit(pi);
        }
        // scheduling opportunity: fill the free slots (event-driven)
        const int free = cfg.batch_capacity - running;
        if (free <= 0 || ready.empty()) continue;
        std::vector<scheduler::ProgramState> states;
        for (size_t i = 0; i < np; ++i) {
            if (!ps[i].arrived || rep.programs[i].finished || ps[i].issued == ps[i].total) continue;
            scheduler::ProgramState s;
            s.program_id = programs[i].program_id;
            s.arrival = arrival[i];
            s.last_service = ps[i].last_service;
            s.iteration_token_sum = ps[i].tok_sum;
            s.iteration_count = ps[i].tok_count;
            if (programs[i].resource_cap > 0) {  // remaining work = (cap - units held) iterations
                s.knob = ps[i].knob;
                s.resource_cap = programs[i].resource_cap;
            } else {
                s.knob = static_cast<int>(ps[i].issued);
                s.resource_cap = static_cast<int>(ps[i].total);
            }
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
    size_t fin = 0, correct = 0;
    for (size_t i = 0; i < np; ++i) {
        auto& pr = rep.programs[i];
        if (!pr.finished) {
            rep.truncated = true;
            pr.knob = ps[i].knob;
            continue;
        }
        pr.latency = pr.completion - pr.arrival;  // queueing included
        pr.met = pr.deadline <= 0.0 || pr.latency <= pr.deadline;
        sum += pr.latency;
        ++fin;
        correct += pr.correct ? 1 : 0;
        rep.makespan = std::max(rep.makespan, pr.completion);
    }
    rep.mean_latency = fin ? sum / static_cast<double>(fin) : 0.0;
    rep.accuracy = static_cast<double>(correct) / static_cast<double>(np);
    rep.throughput = rep.makespan > 0.0 ? rep.total_tokens / rep.makespan : 0.0;
    return rep;
}

double attainment(const SimReport& report) {
    if (report.programs.empty()) throw std::invalid_argument("attainment: empty report");
    size_t met = 0;
    for (const auto& p : report.programs) met += (p.finished && p.met) ? 1 : 0;
    return static_cast<double>(met) / static_cast<double>(report.programs.size());
}

std::vector<std::pair<double, double>> token_accuracy_curve(std::span<const SimReport> reports) {
    std::vector<std::pair<double, double>> pts;
    pts.reserve(reports.size());
    for (const auto& r : reports) pts.emplace_back(r.total_tokens, r.accuracy);
    std::stable_sort(pts.begin(), pts.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    return pts;
}

}  // namespace cdx::sim
