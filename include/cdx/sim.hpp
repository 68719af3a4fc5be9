#pragma once
// cdx/sim.hpp — a deterministic discrete-event loop over a batched serving backend
// (the reference's absent sim.cpp): the caller of
// the hot path.  Programs are sets of requests with known token counts; a request holds
// one of batch_capacity slots for tokens / token_rate seconds; at every arrival and every
// completion (the scheduling opportunities) free slots are filled in the order
// scheduler::next_batch returns — on the B200, through K6's program order.
//
// Two program kinds:
//   * fixed programs (resource_cap == 0): every request of request_tokens is ready at arrival
//     (the Fig. 5 family);
//   * knob-unit programs (resource_cap > 0): knob unit k is one iteration issuing one request
//     per branch (request_tokens[b]); when unit k completes, the program's certaindex signals
//     for it (signals[k-1], computed by the caller with the hot path) are appended to its
//     history and, at each detect / recheck point of the allocation policy (and at the cap),
//     scheduler::allocate decides on the device whether it terminates or continues
//     ("at each program's detect/recheck points invokes scheduler.allocate").
// Arrivals are the given list or a Poisson process (SimConfig::arrival_rate, seeded).
// Scope: the SPEC's service model (linear, one request per slot, no batching speedup), gang
// on/off, fifo / sjf_estimated with starvation escalation, the SLO deadline rule,
// attainment, accuracy and the token-to-accuracy curve.

#include <cstdint>
#include <span>
#include <vector>

#include "cdx/scheduler.hpp"

namespace cdx::sim {

struct SimProgram {
    uint32_t program_id = 0;
    double arrival = 0.0;               // seconds (ignored when SimConfig::arrival_rate > 0)
    std::vector<long> request_tokens;   // fixed: one request per branch, all ready at arrival;
                                        // knob-unit: the branch requests of every iteration
    double deadline = 0.0;              // relative to arrival; <= 0: no deadline
    int resource_cap = 0;               // > 0: a knob-unit program with this many units at most
    std::vector<metrics::SignalVector> signals;  // knob-unit: signals[k-1] after unit k (>= cap)
    std::vector<uint8_t> correct_at;    // optional: answer correct if stopped after unit k
};

struct SimConfig {
    int batch_capacity = 1;        // concurrent request slots (>= 1)
    double token_rate = 1.0;       // tokens / second per slot (> 0)
    scheduler::InterSchedPolicy policy;  // gang, order, starvation_limit, prior_tokens
    double horizon = 1e30;         // programs unfinished at the horizon count as misses
    // knob-unit programs: kind, detect_at_knob, thresholds, recheck_every (resource_cap is each
    // program's own)
    scheduler::AllocationPolicy allocation;
    // Poisson arrivals: rate > 0 (programs / s) replaces SimProgram::arrival by
    // cumulative exponential gaps, gap i = -log(1 - u_i) / rate with u_i the 53-bit uniform of
    // derive_seed(seed, i) (rng.hpp:25-34), in program order
    double arrival_rate = 0.0;
    uint64_t seed = 0;
};

struct ProgramResult {
    uint32_t program_id = 0;
    double arrival = 0.0, completion = 0.0, latency = 0.0, deadline = 0.0;
    bool met = false, finished = false;
    long tokens = 0;
    int knob = 0;                       // knob-unit programs: units completed
    int decisions = 0;                  // scheduler::allocate calls
    scheduler::TerminationCause cause = scheduler::TerminationCause::None;
    bool correct = false;               // correct_at[knob-1] (finished programs only)
};

struct SimReport {
    std::vector<ProgramResult> programs;  // input order
    double mean_latency = 0.0;            // over finished programs
    double total_tokens = 0.0;
    double makespan = 0.0;                // last completion (0 without any)
    double throughput = 0.0;              // total_tokens / makespan (tokens / s)
    double accuracy = 0.0;                // correct / all programs (unfinished = wrong)
    bool truncated = false;               // some program was still running at the horizon
};

// slo_scale x difficulty_factor x base_deadline
double deadline_for(double slo_scale, double difficulty_factor, double base_deadline);

// SPEC.md:516-524.  Identical inputs give identical reports (events are ordered by
// (time, kind, id); the program order comes from the deterministic K6 sort).
SimReport run(std::span<const SimProgram> programs, const SimConfig& config);

// fraction of programs whose latency <= deadline (unfinished = missed).
double attainment(const SimReport& report);

// one (total tokens, accuracy) point per report, sorted by tokens.
std::vector<std::pair<double, double>> token_accuracy_curve(std::span<const SimReport> reports);

// The Poisson arrival times run() uses for `n` programs (SimConfig::arrival_rate, seed).
std::vector<double> poisson_arrivals(size_t n, double rate, uint64_t seed);

}  // namespace cdx::sim
