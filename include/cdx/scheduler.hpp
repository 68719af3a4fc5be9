#pragma once
// cdx/scheduler.hpp — the scheduler API the reference declares only in its spec
// (proj/src/CMakeLists.txt:6 lists scheduler.cpp but no code or header
// exists).  Authored from the spec so the north star's "token-budget decisions and
// gang-scheduling priority" have a C++ entry point; every decision runs on the B200:
//   allocate                   -> cdx_meets_thresholds_rows + K5 cdx_allocate_scan
//   estimate_iteration_tokens  -> cdx_iteration_tokens_rows
//   escalate / program_order   -> K6 cdx_gang_priority (radix-sorted total order)
// Parity here is against the repo's SPEC restatement (oracle/cdx_oracle.c), pinned by the
// SPEC examples.
//
// Not provided (calibration / reporting, not per-batch decisions):
// calibrate_threshold, fairness_report, the curve-fit policy kinds.

#include <cstdint>
#include <span>
#include <vector>

#include "cdx/metrics.hpp"

namespace cdx::scheduler {

// SPEC.md:390-393
enum class AllocationKind {
    Even,
    LengthProxy,
    StaticThreshold,
    InitialCurveFit,
    KStepThreshold,
    DynamicCurveFit
};

struct AllocationPolicy {
    AllocationKind kind = AllocationKind::StaticThreshold;
    int detect_at_knob = 1;  // knob unit where certaindex is first read (<= resource_cap)
    std::vector<metrics::SignalThreshold> thresholds;
    int recheck_every = 1;  // KStepThreshold
    int resource_cap = 1;   // knob units
};

enum class AllocationAction { Grant, Terminate };

enum class TerminationCause { None, Certain, ResourceCap };

struct AllocationDecision {
    AllocationAction action = AllocationAction::Grant;
    int grant_units = 0;  // further knob units granted (Grant only)
    TerminationCause cause = TerminationCause::None;
};

// SPEC.md:404-412.  history[i] = signals observed at knob unit i+1; `knob` = units the
// program holds now (history.size() >= knob).  Even, StaticThreshold, KStepThreshold.
// Throws std::invalid_argument on an invalid policy or a threshold on an absent signal.
AllocationDecision allocate(std::span<const metrics::SignalVector> history, int knob,
                            const AllocationPolicy& policy);

// arithmetic mean of completed iteration token counts, else the prior.
double estimate_iteration_tokens(std::span<const long> completed_iteration_tokens, double prior);

// SPEC.md:394-397
enum class InterOrder { Fifo, SjfEstimated, LpmLikeBaseline };

struct InterSchedPolicy {
    bool gang = true;
    InterOrder order = InterOrder::SjfEstimated;
    double starvation_limit = 1.0;  // > 0
    int batch_capacity = 1;
    double prior_tokens = 128.0;  // estimate_iteration_tokens prior
};

// Scheduler-visible state of one program (runtime.hpp:123-133 ReasoningProgram fields the
// spec's ordering reads).
struct ProgramState {
    uint32_t program_id = 0;
    double arrival = 0.0;
    double last_service = 0.0;
    int64_t iteration_token_sum = 0;   // sum of completed iteration token counts
    uint32_t iteration_count = 0;      // completed iterations
    int knob = 0;                      // units granted so far
    int resource_cap = 0;
    bool terminated = false;
};

// escalated[i] iff now - last_service >= starvation_limit (inclusive).
std::vector<bool> escalate(std::span<const ProgramState> programs, double now,
                           double starvation_limit);

// live programs in priority order — escalated first (FIFO by
// arrival), then fifo: arrival | sjf: est_tokens_per_iter * (cap - knob), then arrival,
// then program id.  Terminated programs are dropped.  Returns program ids.
std::vector<uint32_t> program_order(std::span<const ProgramState> programs,
                                    const InterSchedPolicy& policy, double now);

struct Request {
    uint32_t program_id = 0;
    int branch = 0;  // branch order within the program
};

// SPEC.md:422-430 next_batch with gang = true: ready requests grouped by program in
// program_order, branch order within a program, truncated to batch_capacity.  gang = false
// keeps request-level (ready-list) order.
std::vector<Request> next_batch(std::span<const Request> ready, std::span<const ProgramState> programs,
                                const InterSchedPolicy& policy, double now);

}  // namespace cdx::scheduler
