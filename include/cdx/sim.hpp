#pragma once
// cdx/sim.hpp — a deterministic discrete-event loop over a batched serving backend
// (the reference's absent sim.cpp): the caller of
// the hot path.  Programs are sets of requests with known token counts; a request holds
// one of batch_capacity slots for tokens / token_rate seconds; at every arrival and every
// completion (the scheduling opportunities) free slots are filled in the order
// scheduler::next_batch returns — on the B200, through K6's program order.
//
// Scope: the SPEC's service model (linear, one request per slot, no batching speedup),
// fixed arrival lists, gang on/off, fifo / sjf_estimated with starvation escalation, the
// SLO deadline rule and attainment.  Not modelled: Poisson arrival generation, synthetic
// program expansion (ProgramDriver chains), token-to-accuracy curves.

#include <cstdint>
#include <span>
#include <vector>

#include "cdx/scheduler.hpp"

namespace cdx::sim {

struct SimProgram {
    uint32_t program_id = 0;
    double arrival = 0.0;               // seconds
    std::vector<long> request_tokens;   // one request per branch, all ready at arrival
    double deadline = 0.0;              // relative to arrival; <= 0: no deadline
};

struct SimConfig {
    int batch_capacity = 1;        // concurrent request slots (>= 1)
    double token_rate = 1.0;       // tokens / second per slot (> 0)
    scheduler::InterSchedPolicy policy;  // gang, order, starvation_limit, prior_tokens
    double horizon = 1e30;         // programs unfinished at the horizon count as misses
};

struct ProgramResult {
    uint32_t program_id = 0;
    double arrival = 0.0, completion = 0.0, latency = 0.0, deadline = 0.0;
    bool met = false, finished = false;
    long tokens = 0;
};

struct SimReport {
    std::vector<ProgramResult> programs;  // input order
    double mean_latency = 0.0;            // over finished programs
    double total_tokens = 0.0;
    bool truncated = false;               // some program was still running at the horizon
};

// slo_scale x difficulty_factor x base_deadline
double deadline_for(double slo_scale, double difficulty_factor, double base_deadline);

// SPEC.md:516-524.  Identical inputs give identical reports (events are ordered by
// (time, kind, id); the program order comes from the deterministic K6 sort).
SimReport run(std::span<const SimProgram> programs, const SimConfig& config);

// fraction of programs whose latency <= deadline (unfinished = missed).
double attainment(const SimReport& report);

}  // namespace cdx::sim
