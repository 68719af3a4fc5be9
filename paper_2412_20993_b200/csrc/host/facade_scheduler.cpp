// facade_scheduler.cpp — cdx::scheduler (include/cdx/scheduler.hpp).
//
//   allocate                   thresholds at the policy's test points on the device
//                              (cdx_meets_thresholds_rows), then K5 cdx_allocate_scan for a
//                              batch of one: the same decision code the batched path runs
//   estimate_iteration_tokens  cdx_iteration_tokens_rows
//   escalate / program_order   K6 cdx_gang_priority
//   next_batch                 program_order, then the ready requests grouped by program

#include <algorithm>
#include <stdexcept>
#include <unordered_map>

#include "cdx/scheduler.hpp"
#include "facade_common.hpp"

namespace cdx::scheduler {

namespace {

void validate(const AllocationPolicy& p, int knob, size_t history) {
    if (p.resource_cap < 1) throw std::invalid_argument("allocate: resource_cap must be >= 1");
    if (p.kind != AllocationKind::Even && p.kind != AllocationKind::StaticThreshold &&
        p.kind != AllocationKind::KStepThreshold)
        throw std::invalid_argument("allocate: policy kind not supported (even, static_threshold, k_step_threshold)");
    if (p.kind != AllocationKind::Even && (p.detect_at_knob < 1 || p.detect_at_knob > p.resource_cap))
        throw std::invalid_argument("allocate: detect_at_knob must be in [1, resource_cap]");
    if (p.kind == AllocationKind::KStepThreshold && p.recheck_every < 1)
        throw std::invalid_argument("allocate: recheck_every must be >= 1");
    if (knob < 0 || knob > p.resource_cap) throw std::invalid_argument("allocate: knob outside [0, resource_cap]");
    if (history < static_cast<size_t>(knob)) throw std::invalid_argument("allocate: history shorter than knob");
}

struct DeviceSoA {
    batch::DeviceArray<double> arrival, last;
    batch::DeviceArray<int64_t> sum;
    batch::DeviceArray<uint32_t> count;
    batch::DeviceArray<int32_t> knob, cap;
    batch::DeviceArray<uint8_t> term;
    batch::DeviceArray<uint32_t> id;
    cdx_prog_soa soa{};
};

// ProgramState list -> device SoA in input order, with the program ids (the last tie-break,
// SPEC.md:470) as an explicit id array.
DeviceSoA upload(batch::Context& cx, std::span<const ProgramState> ps) {
    const size_t n = ps.size();
    std::vector<double> a(n), l(n);
    std::vector<int64_t> s(n);
    std::vector<uint32_t> c(n), id(n);
    std::vector<int32_t> k(n), cap(n);
    std::vector<uint8_t> t(n);
    for (size_t i = 0; i < n; ++i) {
        a[i] = ps[i].arrival;
        l[i] = ps[i].last_service;
        s[i] = ps[i].iteration_token_sum;
        c[i] = ps[i].iteration_count;
        k[i] = ps[i].knob;
        cap[i] = ps[i].resource_cap;
        t[i] = ps[i].terminated ? 1 : 0;
        id[i] = ps[i].program_id;
    }
    DeviceSoA d;
    d.arrival = batch::DeviceArray<double>(cx, std::span<const double>(a));
    d.last = batch::DeviceArray<double>(cx, std::span<const double>(l));
    d.sum = batch::DeviceArray<int64_t>(cx, std::span<const int64_t>(s));
    d.count = batch::DeviceArray<uint32_t>(cx, std::span<const uint32_t>(c));
    d.knob = batch::DeviceArray<int32_t>(cx, std::span<const int32_t>(k));
    d.cap = batch::DeviceArray<int32_t>(cx, std::span<const int32_t>(cap));
    d.term = batch::DeviceArray<uint8_t>(cx, std::span<const uint8_t>(t));
    d.id = batch::DeviceArray<uint32_t>(cx, std::span<const uint32_t>(id));
    d.soa = {d.arrival.data(), d.last.data(), d.sum.data(), d.count.data(), d.knob.data(), d.cap.data(),
             d.term.data(), d.id.data(), 0, 0};
    return d;
}

// order (program ids) and escalation flags from K6
std::pair<std::vector<uint32_t>, std::vector<uint8_t>> order_of(std::span<const ProgramState> ps,
                                                                const InterSchedPolicy& pol, double now,
                                                                bool want_esc) {
    if (ps.empty()) return {};
    auto& cx = detail::scalar_ctx();
    auto d = upload(cx, ps);
    batch::DeviceArray<uint32_t> order(cx, ps.size());
    batch::DeviceArray<uint8_t> esc;
    if (want_esc) esc = batch::DeviceArray<uint8_t>(cx, ps.size());
    const uint64_t n = batch::gang_priority(cx, d.soa, ps.size(), pol, now, order.data(),
                                            want_esc ? esc.data() : nullptr, nullptr);
    auto o = order.download();
    o.resize(n);
    std::vector<uint8_t> e;
    if (want_esc) e = esc.download();
    return {o, e};
}

}  // namespace

AllocationDecision allocate(std::span<const metrics::SignalVector> history, int knob, const AllocationPolicy& p) {
    validate(p, knob, history.size());
    AllocationDecision d;
    if (knob >= p.resource_cap) {  // "always terminate at resource_cap" SPEC.md:407
        d.action = AllocationAction::Terminate;
        d.cause = TerminationCause::ResourceCap;
        return d;
    }
    auto& cx = detail::scalar_ctx();
    const int cap = p.resource_cap;
    // test points reached so far
    std::vector<int> tests;
    if (p.kind != AllocationKind::Even)
        for (int t = p.detect_at_knob; t <= knob;
             t += (p.kind == AllocationKind::KStepThreshold ? p.recheck_every : cap + 1))
            tests.push_back(t);
    const uint32_t words = static_cast<uint32_t>((cap + 31) / 32);
    batch::DeviceArray<uint32_t> meets(cx, words);
    meets.zero();
    if (!tests.empty()) {
        std::vector<double> sig(tests.size() * 4, 0.0);
        std::vector<uint8_t> present(tests.size(), 0);
        for (size_t i = 0; i < tests.size(); ++i)
            for (int k = 0; k < 4; ++k)
                if (auto v = history[static_cast<size_t>(tests[i] - 1)].get(static_cast<metrics::SignalKind>(k))) {
                    sig[i * 4 + static_cast<size_t>(k)] = *v;
                    present[i] |= static_cast<uint8_t>(1u << k);
                }
        if (p.thresholds.size() > 8) throw std::invalid_argument("allocate: at most 8 thresholds per policy");
        std::vector<cdx_threshold> th;
        for (const auto& t : p.thresholds) th.push_back(detail::to_c(t));
        batch::DeviceArray<double> d_sig(cx, std::span<const double>(sig));
        batch::DeviceArray<uint8_t> d_present(cx, std::span<const uint8_t>(present));
        batch::DeviceArray<uint8_t> d_ok(cx, tests.size());
        cx.check(cdx_meets_thresholds_rows(cx.raw(), d_sig.data(), d_present.data(), tests.size(),
                                           th.empty() ? nullptr : th.data(), static_cast<uint32_t>(th.size()),
                                           d_ok.data()));
        const auto ok = d_ok.download();  // surfaces an absent-signal error
        std::vector<uint32_t> bits(words, 0);
        for (size_t i = 0; i < tests.size(); ++i)
            if (ok[i]) bits[static_cast<size_t>(tests[i] - 1) / 32] |= 1u << ((tests[i] - 1) % 32);
        meets.upload(std::span<const uint32_t>(bits));
    }
    batch::DeviceArray<int32_t> exit_knob(cx, 1);
    batch::DeviceArray<uint8_t> reason(cx, 1);
    batch::DeviceArray<uint64_t> n_kept(cx, 1);
    batch::DeviceArray<int64_t> saved(cx, 1);
    batch::AllocationOutputs o;
    o.exit_knob = exit_knob.data();
    o.reason = reason.data();
    o.n_kept = n_kept.data();
    o.tokens_saved = saved.data();
    batch::allocate_scan(cx, meets.data(), 1, static_cast<uint32_t>(cap), p, 1, 0, 0, o);
    const int ek = exit_knob.download()[0];
    const uint8_t why = reason.download()[0];
    if (why == CDX_EXIT_CERTAIN && ek <= knob) {
        d.action = AllocationAction::Terminate;
        d.cause = TerminationCause::Certain;
        return d;
    }
    // grant up to the next decision point
    int next = cap;
    if (p.kind == AllocationKind::StaticThreshold && knob < p.detect_at_knob) next = p.detect_at_knob;
    if (p.kind == AllocationKind::KStepThreshold) {
        next = p.detect_at_knob;
        while (next <= knob) next += p.recheck_every;
        next = std::min(next, cap);
    }
    d.action = AllocationAction::Grant;
    d.grant_units = next - knob;
    return d;
}

double estimate_iteration_tokens(std::span<const long> completed, double prior) {
    auto& cx = detail::scalar_ctx();
    std::vector<int64_t> v(completed.begin(), completed.end());
    const uint64_t off[2] = {0, v.size()};
    batch::DeviceArray<int64_t> d_v(cx, std::span<const int64_t>(v));
    batch::DeviceArray<uint64_t> d_off(cx, std::span<const uint64_t>(off, 2));
    batch::DeviceArray<double> out(cx, 1);
    cx.check(cdx_iteration_tokens_rows(cx.raw(), d_v.data(), d_off.data(), 1, prior, out.data()));
    return out.download()[0];
}

std::vector<bool> escalate(std::span<const ProgramState> programs, double now, double starvation_limit) {
    InterSchedPolicy pol;
    pol.order = InterOrder::Fifo;
    pol.starvation_limit = starvation_limit;
    auto [o, e] = order_of(programs, pol, now, true);
    return std::vector<bool>(e.begin(), e.end());
}

std::vector<uint32_t> program_order(std::span<const ProgramState> programs, const InterSchedPolicy& policy,
                                    double now) {
    return order_of(programs, policy, now, false).first;
}

std::vector<Request> next_batch(std::span<const Request> ready, std::span<const ProgramState> programs,
                                const InterSchedPolicy& policy, double now) {
    if (policy.batch_capacity < 1) throw std::invalid_argument("next_batch: batch_capacity must be >= 1");
    const size_t cap = static_cast<size_t>(policy.batch_capacity);
    std::vector<Request> out;
    if (!policy.gang) {  // request-level order only
        for (size_t i = 0; i < ready.size() && out.size() < cap; ++i) out.push_back(ready[i]);
        return out;
    }
    std::unordered_map<uint32_t, std::vector<Request>> by_prog;
    for (const auto& r : ready) by_prog[r.program_id].push_back(r);
    for (auto& kv : by_prog)
        std::stable_sort(kv.second.begin(), kv.second.end(),
                         [](const Request& a, const Request& b) { return a.branch < b.branch; });
    for (uint32_t pid : program_order(programs, policy, now)) {
        auto it = by_prog.find(pid);
        if (it == by_prog.end()) continue;
        for (const auto& r : it->second) {
            if (out.size() == cap) return out;
            out.push_back(r);
        }
    }
    return out;
}

}  // namespace cdx::scheduler
