#pragma once
// cdx/batch.hpp — the batched (structure-of-arrays) C++ API over the hot path: one call
// scores a whole request batch resident in HBM.  This is the API the north star's
// throughput is measured through; the scalar reference API (metrics.hpp / probe.hpp) is
// the compatibility surface.  Thin RAII over the C-ABI (include/cdx_c.h): errors become
// the reference's exception types, buffers are stream-ordered device allocations.
//
//   sc_certaindex      K2  cluster_exact + certaindex_entropy + thresholds per (r,p) row
//   allocate_scan      K5  SPEC allocate + exclusive budget scan + stable compaction
//   cot_exit           K3  should_exit / consistency / final_answer over every prefix
//   reward_certaindex  K4  cumulative certaindex_reward (+ entropy) per (program, step)
//   canon_intern       K1  trim + intern + flag_hesitation over a string arena
//   gang_priority      K6  escalate + estimate + next_batch program order (radix sort)
//   sc_aggregate / reward_aggregate   final answers per archetype (runtime.cpp:316-403)
//   cot_eps_stop       the epsilon-accuracy stop rule at every CoT prefix (probe.cpp:104-120)
//   jsonl_parse        probe-trace JSONL ingestion (probe.cpp:126-165)
//   Graph              capture / replay of a call sequence (launch-bound small batches)
//   allocate_scan_sharded / gang_priority_sharded   K5 / K6 with global results across the
//                      ranks of a multi-GPU job (Context(device, comm))

#include <cstddef>
#include <cstdint>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "cdx/metrics.hpp"
#include "cdx/probe.hpp"
#include "cdx/scheduler.hpp"
#include "cdx_c.h"

namespace cdx::batch {

// Throws the exception type the status maps to (cdx_c.h conventions).
[[noreturn]] void raise(int status, const char* message);

class Context {
public:
    explicit Context(int device = 0);
    // A rank of a multi-GPU job: the context owns the communicator (NCCL from comm.nccl_id,
    // or the caller's allgather / alltoallv callbacks); the *_sharded calls below exchange
    // through it.  Collective with NCCL.
    Context(int device, const cdx_comm& comm);
    ~Context();
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    cdx_ctx* raw() const { return h_; }
    void set_stream(void* cuda_stream);  // nullptr: legacy default stream
    void sync();                         // waits; surfaces device-side validation errors
    void check(int status) const;        // throws on status != CDX_OK
    uint64_t launches() const;

private:
    cdx_ctx* h_ = nullptr;
};

// Stream-ordered device array of trivially copyable T.
template <class T>
class DeviceArray {
public:
    DeviceArray() = default;
    DeviceArray(Context& cx, size_t n) : cx_(&cx), n_(n) {
        void* p = nullptr;
        cx.check(cdx_alloc(cx.raw(), n * sizeof(T), &p));
        p_ = static_cast<T*>(p);
    }
    DeviceArray(Context& cx, std::span<const T> host) : DeviceArray(cx, host.size()) { upload(host); }
    ~DeviceArray() { reset(); }
    DeviceArray(DeviceArray&& o) noexcept { swap(o); }
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        reset();
        swap(o);
        return *this;
    }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;

    T* data() const { return p_; }
    size_t size() const { return n_; }
    void upload(std::span<const T> host) { cx_->check(cdx_memcpy(cx_->raw(), p_, host.data(), host.size_bytes())); }
    std::vector<T> download() const {  // synchronises the context stream
        std::vector<T> out(n_);
        cx_->check(cdx_memcpy(cx_->raw(), out.data(), p_, n_ * sizeof(T)));
        cx_->sync();
        return out;
    }
    void zero() { cx_->check(cdx_memset(cx_->raw(), p_, 0, n_ * sizeof(T))); }

private:
    void reset() {
        if (p_ && cx_) cdx_free(cx_->raw(), p_);
        p_ = nullptr;
        n_ = 0;
    }
    void swap(DeviceArray& o) noexcept {
        std::swap(cx_, o.cx_);
        std::swap(p_, o.p_);
        std::swap(n_, o.n_);
    }
    Context* cx_ = nullptr;
    T* p_ = nullptr;
    size_t n_ = 0;
};

// ---- K2 + K5: Self-Consistency ---------------------------------------------------------

struct ScShape {
    uint64_t requests = 0;  // R
    uint32_t probes = 0;    // P (knob units)
    uint32_t samples = 0;   // S answers per (request, probe) row
};

// ids u32[R][P][S]; hcert f32[R][P] (nullable); meets u32[R][ceil(P/32)].
void sc_certaindex(Context& cx, const uint32_t* ids, const ScShape& shape,
                   std::span<const metrics::SignalThreshold> thresholds, float* hcert, uint32_t* meets);

// Majority-fraction certaindex (largest cluster / S: the share of the plurality answer,
// runtime.cpp:317-334) thresholds, ANDed with the entropy thresholds above.
struct MajorityThreshold {
    double cutoff = 0.5;
    metrics::ThresholdDir direction = metrics::ThresholdDir::GreaterEq;
};
// The same plus majority f32[R][P] (nullable) and majority thresholds.
void sc_certaindex(Context& cx, const uint32_t* ids, const ScShape& shape,
                   std::span<const metrics::SignalThreshold> thresholds,
                   std::span<const MajorityThreshold> majority_thresholds, float* hcert, float* majority,
                   uint32_t* meets);

struct AllocationOutputs {
    int32_t* exit_knob = nullptr;  // i32[R]
    uint8_t* reason = nullptr;     // u8[R]  CDX_EXIT_CERTAIN | CDX_EXIT_BUDGET
    int32_t* granted = nullptr;    // i32[R]
    int64_t* offsets = nullptr;    // i64[R] global token offsets
    uint32_t* kept = nullptr;      // u32[R] continuing requests (stable)
    uint64_t* n_kept = nullptr;    // device scalars
    int64_t* tokens_saved = nullptr;
    int64_t* total_budget = nullptr;
};

// policy.kind in {Even, StaticThreshold, KStepThreshold}; tokens_per_unit = interval * S.
void allocate_scan(Context& cx, const uint32_t* meets, uint64_t requests, uint32_t probes,
                   const scheduler::AllocationPolicy& policy, int64_t tokens_per_unit, int64_t base_offset,
                   uint32_t kept_base, const AllocationOutputs& out);

// The same over this rank's request shard with GLOBAL offsets, kept indices and totals
// (cdx_allocate_scan_sharded); n_kept is this rank's kept count.
void allocate_scan_sharded(Context& cx, const uint32_t* meets, uint64_t requests, uint32_t probes,
                           const scheduler::AllocationPolicy& policy, int64_t tokens_per_unit,
                           const AllocationOutputs& out, uint64_t* shard_info = nullptr);

// ---- K3: CoT probe window --------------------------------------------------------------

struct CotOutputs {
    int32_t* exit_step = nullptr;  // i32[R], -1 = no exit
    uint8_t* reason = nullptr;     // u8[R]  ExitDecision ordinal
    uint32_t* final_id = nullptr;  // u32[R]
    uint8_t* low_conf = nullptr;   // u8[R]
    float* ck = nullptr;           // f32[R][P] (nullable)
};

// ids u32[R][P], hes u64[R][ceil(P/64)], offsets i64[R][P] (nullable: (p+1)*interval).
void cot_exit(Context& cx, const uint32_t* ids, const uint64_t* hes, const int64_t* offsets, uint64_t requests,
              uint32_t probes, const probe::ProbeConfig& cfg, const CotOutputs& out);

// ---- K4: reward certaindex -------------------------------------------------------------

// rewards f32[G][T][W]; ids u32[G][T][W] (nullable); agg u8[G] (RewardAggregation ordinal).
void reward_certaindex(Context& cx, const float* rewards, const uint32_t* ids, const uint8_t* agg,
                       uint64_t programs, uint32_t steps, uint32_t width,
                       std::span<const metrics::SignalThreshold> thresholds_mean,
                       std::span<const metrics::SignalThreshold> thresholds_max, float* R, float* H,
                       uint32_t* meets);

// ---- K1: canonicalisation + interning ----------------------------------------------------

// arena bytes (device) with offsets u64[n+1] (device); returns the number of unique answers.
uint64_t canon_intern(Context& cx, const char* arena, const uint64_t* offsets, uint64_t n,
                      std::span<const std::string> markers, uint32_t* ids, uint8_t* hesitant,
                      uint64_t* first_index);

// ---- K6: gang-scheduling program order ---------------------------------------------------

// progs: device SoA; returns the number of ordered (live) programs written to order.
uint64_t gang_priority(Context& cx, const cdx_prog_soa& progs, uint64_t n,
                       const scheduler::InterSchedPolicy& policy, double now, uint32_t* order,
                       uint8_t* escalated, uint64_t* keys);

// The GLOBAL order of every rank's live programs (program ids must be global), on every rank
// (cdx_gang_priority_sharded); returns its length.
uint64_t gang_priority_sharded(Context& cx, const cdx_prog_soa& progs, uint64_t n,
                               const scheduler::InterSchedPolicy& policy, double now, uint32_t* order);

// ---- aggregation (runtime.cpp:316-403) ---------------------------------------------------

// SC plurality over each request's exit row (exit_knob i32[R], 1-based) -> answer u32[R]
void sc_aggregate(Context& cx, const uint32_t* ids, const ScShape& shape, const int32_t* exit_knob,
                  uint32_t* answer);
// MCTS first argmax / Rebase exp-weighted plurality at exit step t (0-based); returns the
// number of rewards off the 2^-24 grid (whose exp used the device's exp)
uint64_t reward_aggregate(Context& cx, const float* rewards, const uint32_t* ids, const uint8_t* agg,
                          uint64_t programs, uint32_t steps, uint32_t width, const int32_t* exit_step,
                          uint32_t* answer);

// ---- epsilon-accuracy stop test (probe.cpp:104-120) -----------------------------------------

// eps_step i32[R] = first probe where the test holds (-1 none); state u8[R][P] nullable
void cot_eps_stop(Context& cx, const uint32_t* ids, const uint64_t* hes, uint64_t requests, uint32_t probes,
                  int k, double epsilon, int32_t* eps_step, uint8_t* state);

// ---- JSONL ingestion (probe.cpp:126-165) ----------------------------------------------------

struct JsonlRecords {
    uint32_t* program = nullptr;       // u32[cap] interned program ids (first-seen, dense)
    int32_t* step_index = nullptr;     // i32[cap]
    int64_t* token_offset = nullptr;   // i64[cap]
    uint8_t* hesitant = nullptr;       // u8[cap]
    uint64_t* answer_off = nullptr;    // u64[cap + 1]
    char* answer_arena = nullptr;      // nbytes
    uint64_t* program_off = nullptr;   // u64[cap + 1] (nullable with program_arena)
    char* program_arena = nullptr;     // nbytes
    uint64_t* program_first = nullptr; // u64[cap] (nullable)
};

// text: device bytes; returns {records, programs}; throws std::runtime_error("trace line n: ...")
std::pair<uint64_t, uint64_t> jsonl_parse(Context& cx, const char* text, uint64_t nbytes, uint64_t cap_records,
                                          const JsonlRecords& out);

// ---- CUDA graphs ---------------------------------------------------------------------------

class Graph {
public:
    // Captures the calls fn makes on cx (its stream must not be a default stream).
    template <class F>
    Graph(Context& cx, F&& fn) : cx_(&cx) {
        cx.check(cdx_graph_begin(cx.raw()));
        try {
            fn();
        } catch (...) {
            cdx_graph* g = nullptr;
            cdx_graph_end(cx.raw(), &g);
            cdx_graph_destroy(g);
            throw;
        }
        cx.check(cdx_graph_end(cx.raw(), &g_));
    }
    ~Graph() { cdx_graph_destroy(g_); }
    Graph(const Graph&) = delete;
    Graph& operator=(const Graph&) = delete;
    void launch() { cx_->check(cdx_graph_launch(cx_->raw(), g_)); }

private:
    Context* cx_;
    cdx_graph* g_ = nullptr;
};

}  // namespace cdx::batch
