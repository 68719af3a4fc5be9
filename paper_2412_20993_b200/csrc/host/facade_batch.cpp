// facade_batch.cpp — cdx::batch (include/cdx/batch.hpp): RAII context, error mapping and
// the batched entry points, each a direct call of one C-ABI function of libcdx.so.

#include <cstdlib>
#include <stdexcept>
#include <string>

#include "facade_common.hpp"

namespace cdx::batch {

void raise(int status, const char* message) {
    const std::string msg = message ? message : "";
    switch (status) {
        case CDX_EINVAL: throw std::invalid_argument(msg);
        case CDX_ERANGE: throw std::out_of_range(msg);
        case CDX_ELOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);  // ERUNTIME, ECUDA, ENCCL
    }
}

Context::Context(int device) {
    const int st = cdx_ctx_create(device, &h_);
    if (st != CDX_OK)
        raise(st == CDX_EINVAL ? CDX_EINVAL : CDX_ERUNTIME,
              ("cdx: no usable sm_100 device " + std::to_string(device) +
               " (the Certaindex path runs on the B200 only; there is no CPU fallback)")
                  .c_str());
}

Context::Context(int device, const cdx_comm& comm) {
    const int st = cdx_ctx_create_comm(device, &comm, &h_);
    if (st == CDX_ENCCL) raise(CDX_ERUNTIME, "cdx: NCCL communicator could not be created (libnccl.so.2)");
    if (st != CDX_OK)
        raise(st == CDX_EINVAL ? CDX_EINVAL : CDX_ERUNTIME,
              ("cdx: no usable sm_100 device " + std::to_string(device) + " or a bad communicator").c_str());
}

Context::~Context() {
    if (h_) cdx_ctx_destroy(h_);
}

void Context::set_stream(void* s) { check(cdx_ctx_set_stream(h_, s)); }

void Context::check(int st) const {
    if (st != CDX_OK) raise(st, cdx_last_error(h_));
}

void Context::sync() { check(cdx_sync(h_)); }

uint64_t Context::launches() const { return cdx_launch_count(h_); }

namespace {

struct CThresholds {
    std::vector<cdx_threshold> v;
    explicit CThresholds(std::span<const metrics::SignalThreshold> t) {
        for (const auto& x : t) v.push_back(detail::to_c(x));
    }
    const cdx_threshold* data() const { return v.empty() ? nullptr : v.data(); }
    uint32_t size() const { return static_cast<uint32_t>(v.size()); }
};

uint8_t policy_kind(scheduler::AllocationKind k) {
    switch (k) {
        case scheduler::AllocationKind::Even: return CDX_POL_EVEN;
        case scheduler::AllocationKind::StaticThreshold: return CDX_POL_STATIC_THRESHOLD;
        case scheduler::AllocationKind::KStepThreshold: return CDX_POL_K_STEP_THRESHOLD;
        default: throw std::invalid_argument("allocate: policy kind not supported by the batched path");
    }
}

}  // namespace

void sc_certaindex(Context& cx, const uint32_t* ids, const ScShape& s,
                   std::span<const metrics::SignalThreshold> thresholds, float* hcert, uint32_t* meets) {
    CThresholds th(thresholds);
    cx.check(cdx_sc_certaindex(cx.raw(), ids, s.requests, s.probes, s.samples, th.data(), th.size(), hcert, meets));
}

void sc_certaindex(Context& cx, const uint32_t* ids, const ScShape& s,
                   std::span<const metrics::SignalThreshold> thresholds,
                   std::span<const MajorityThreshold> majority_thresholds, float* hcert, float* majority,
                   uint32_t* meets) {
    CThresholds th(thresholds);
    for (const auto& m : majority_thresholds) {
        cdx_threshold c{};
        c.signal = CDX_SIG_MAJORITY;
        c.dir = m.direction == metrics::ThresholdDir::GreaterEq ? CDX_DIR_GE : CDX_DIR_LE;
        c.cutoff = m.cutoff;
        th.v.push_back(c);
    }
    cx.check(cdx_sc_certaindex_ex(cx.raw(), ids, s.requests, s.probes, s.samples, th.data(), th.size(), hcert,
                                  majority, meets));
}

void allocate_scan(Context& cx, const uint32_t* meets, uint64_t R, uint32_t P,
                   const scheduler::AllocationPolicy& pol, int64_t tokens_per_unit, int64_t base_offset,
                   uint32_t kept_base, const AllocationOutputs& o) {
    cdx_alloc_policy p{};
    p.kind = policy_kind(pol.kind);
    p.detect_at = pol.detect_at_knob;
    p.recheck_every = pol.recheck_every;
    p.resource_cap = pol.resource_cap;
    p.tokens_per_unit = tokens_per_unit;
    cx.check(cdx_allocate_scan(cx.raw(), meets, R, P, &p, base_offset, kept_base, o.exit_knob, o.reason, o.granted,
                               o.offsets, o.kept, o.n_kept, o.tokens_saved, o.total_budget));
}

void allocate_scan_sharded(Context& cx, const uint32_t* meets, uint64_t R, uint32_t P,
                           const scheduler::AllocationPolicy& pol, int64_t tokens_per_unit, const AllocationOutputs& o,
                           uint64_t* shard_info) {
    cdx_alloc_policy p{};
    p.kind = policy_kind(pol.kind);
    p.detect_at = pol.detect_at_knob;
    p.recheck_every = pol.recheck_every;
    p.resource_cap = pol.resource_cap;
    p.tokens_per_unit = tokens_per_unit;
    cx.check(cdx_allocate_scan_sharded(cx.raw(), meets, R, P, &p, o.exit_knob, o.reason, o.granted, o.offsets, o.kept,
                                       o.n_kept, o.tokens_saved, o.total_budget, shard_info));
}

void cot_exit(Context& cx, const uint32_t* ids, const uint64_t* hes, const int64_t* offsets, uint64_t R, uint32_t P,
              const probe::ProbeConfig& cfg, const CotOutputs& o) {
    cfg.validate();
    cdx_probe_cfg c{};
    c.interval_tokens = cfg.interval_tokens;
    c.window = cfg.window;
    c.threshold = cfg.threshold;
    c.max_tokens = cfg.max_tokens;
    cx.check(cdx_cot_exit(cx.raw(), ids, hes, offsets, R, P, &c, o.exit_step, o.reason, o.final_id, o.low_conf, o.ck));
}

void reward_certaindex(Context& cx, const float* rewards, const uint32_t* ids, const uint8_t* agg, uint64_t G,
                       uint32_t T, uint32_t W, std::span<const metrics::SignalThreshold> th_mean,
                       std::span<const metrics::SignalThreshold> th_max, float* R, float* H, uint32_t* meets) {
    CThresholds a(th_mean), b(th_max);
    cx.check(cdx_reward_certaindex(cx.raw(), rewards, ids, agg, G, T, W, a.data(), a.size(), b.data(), b.size(), R, H,
                                   meets));
}

uint64_t canon_intern(Context& cx, const char* arena, const uint64_t* offsets, uint64_t n,
                      std::span<const std::string> markers, uint32_t* ids, uint8_t* hes, uint64_t* first_index) {
    std::vector<const char*> mk;
    for (const auto& m : markers) mk.push_back(m.c_str());
    uint64_t nu = 0;
    cx.check(cdx_canon_intern(cx.raw(), arena, offsets, n, mk.empty() ? nullptr : mk.data(),
                              static_cast<uint32_t>(mk.size()), ids, hes, first_index, &nu));
    return nu;
}

namespace {
cdx_inter_policy inter_policy(const scheduler::InterSchedPolicy& pol) {
    cdx_inter_policy p{};
    p.gang = pol.gang ? 1 : 0;
    switch (pol.order) {
        case scheduler::InterOrder::Fifo: p.order = CDX_ORDER_FIFO; break;
        case scheduler::InterOrder::SjfEstimated: p.order = CDX_ORDER_SJF; break;
        default: throw std::invalid_argument("next_batch: lpm_like_baseline order is not a certaindex policy");
    }
    p.starvation_limit = pol.starvation_limit;
    p.prior_tokens = pol.prior_tokens;
    return p;
}
}  // namespace

uint64_t gang_priority(Context& cx, const cdx_prog_soa& progs, uint64_t n, const scheduler::InterSchedPolicy& pol,
                       double now, uint32_t* order, uint8_t* escalated, uint64_t* keys) {
    const cdx_inter_policy p = inter_policy(pol);
    uint64_t n_out = 0;
    cx.check(cdx_gang_priority(cx.raw(), &progs, n, &p, now, order, &n_out, escalated, keys));
    return n_out;
}

uint64_t gang_priority_sharded(Context& cx, const cdx_prog_soa& progs, uint64_t n,
                               const scheduler::InterSchedPolicy& pol, double now, uint32_t* order) {
    const cdx_inter_policy p = inter_policy(pol);
    uint64_t n_out = 0;
    cx.check(cdx_gang_priority_sharded(cx.raw(), &progs, n, &p, now, order, &n_out));
    return n_out;
}

void sc_aggregate(Context& cx, const uint32_t* ids, const ScShape& s, const int32_t* exit_knob, uint32_t* answer) {
    cx.check(cdx_sc_aggregate(cx.raw(), ids, s.requests, s.probes, s.samples, exit_knob, answer));
}

uint64_t reward_aggregate(Context& cx, const float* rewards, const uint32_t* ids, const uint8_t* agg, uint64_t G,
                          uint32_t T, uint32_t W, const int32_t* exit_step, uint32_t* answer) {
    DeviceArray<uint64_t> inexact(cx, 1);
    cx.check(cdx_reward_aggregate(cx.raw(), rewards, ids, agg, G, T, W, exit_step, answer, inexact.data()));
    return inexact.download()[0];
}

void cot_eps_stop(Context& cx, const uint32_t* ids, const uint64_t* hes, uint64_t R, uint32_t P, int k,
                  double epsilon, int32_t* eps_step, uint8_t* state) {
    cx.check(cdx_cot_eps_stop(cx.raw(), ids, hes, R, P, k, epsilon, eps_step, state));
}

std::pair<uint64_t, uint64_t> jsonl_parse(Context& cx, const char* text, uint64_t nbytes, uint64_t cap,
                                          const JsonlRecords& o) {
    uint64_t nr = 0, np = 0;
    cx.check(cdx_jsonl_parse(cx.raw(), text, nbytes, cap, o.program, o.step_index, o.token_offset, o.hesitant,
                             o.answer_off, o.answer_arena, o.program_off, o.program_arena, o.program_first, &nr, &np));
    return {nr, np};
}

}  // namespace cdx::batch

namespace cdx::detail {

batch::Context& scalar_ctx() {
    thread_local batch::Context cx([] {
        const char* d = std::getenv("CDX_DEVICE");
        return d ? std::atoi(d) : 0;
    }());
    return cx;
}

cdx_threshold to_c(const metrics::SignalThreshold& t) {
    cdx_threshold c{};
    c.signal = static_cast<uint8_t>(t.signal);
    c.dir = static_cast<uint8_t>(t.dir);
    c.cutoff = t.cutoff;
    return c;
}

Interned intern(batch::Context& cx, std::span<const std::string_view> strs, std::span<const std::string> markers,
                bool want_hes, bool want_first) {
    Interned out;
    const uint64_t n = strs.size();
    std::vector<uint64_t> off(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) off[i + 1] = off[i] + strs[i].size();
    std::string arena;
    arena.reserve(off[n]);
    for (auto s : strs) arena.append(s.data(), s.size());
    batch::DeviceArray<char> d_arena(cx, std::span<const char>(arena.data(), arena.size()));
    batch::DeviceArray<uint64_t> d_off(cx, std::span<const uint64_t>(off));
    out.ids = batch::DeviceArray<uint32_t>(cx, n);
    if (want_hes) out.hes = batch::DeviceArray<uint8_t>(cx, n);
    batch::DeviceArray<uint64_t> d_first;
    if (want_first) d_first = batch::DeviceArray<uint64_t>(cx, n);
    out.n_unique = batch::canon_intern(cx, d_arena.data(), d_off.data(), n, markers, out.ids.data(),
                                       want_hes ? out.hes.data() : nullptr, want_first ? d_first.data() : nullptr);
    if (want_first) {
        auto all = d_first.download();
        out.first_index.assign(all.begin(), all.begin() + static_cast<std::ptrdiff_t>(out.n_unique));
    }
    cx.sync();
    return out;
}

}  // namespace cdx::detail
