// facade_probe.cpp — cdx::probe (include/cdx/probe.hpp) on the B200.
//
//   flag_hesitation  K1 canon_intern's marker scan (ASCII tolower, non-empty markers)
//                                                                     probe.cpp:36-44
//   consistency      K1 ids + cdx_probe_consistency                   probe.cpp:48-75
//   should_exit      K1 ids + cdx_probe_should_exit                   probe.cpp:77-85
//   final_answer     cdx_probe_final_answer (record index), trimmed   probe.cpp:87-102
//   stationary_by_epsilon_test  K1 ids + cdx_probe_eps_stop_rows      probe.cpp:104-120
// ProbeConfig::validate and the enum names are host-side configuration checks with the
// reference's messages.  JSONL trace I/O lives in facade_jsonl.cpp.

#include <climits>
#include <stdexcept>
#include <string>

#include "cdx/metrics.hpp"
#include "cdx/probe.hpp"
#include "facade_common.hpp"

namespace cdx::probe {

void ProbeConfig::validate() const {
    if (interval_tokens < 1) throw std::invalid_argument("probe: interval_tokens must be >= 1");
    if (window < 1) throw std::invalid_argument("probe: window must be >= 1");
    if (threshold <= 0.0 || threshold > 1.0) throw std::invalid_argument("probe: threshold must be in (0,1]");
    if (max_tokens < 1) throw std::invalid_argument("probe: max_tokens must be >= 1");
}

const char* termination_reason_name(TerminationReason r) {
    switch (r) {
        case TerminationReason::Certain: return "certain";
        case TerminationReason::Budget: return "budget";
        case TerminationReason::CriteriaExternal: return "criteria_external";
    }
    return "?";
}

bool flag_hesitation(std::string_view answer, std::span<const std::string> markers) {
    auto& cx = detail::scalar_ctx();
    if (answer.size() <= (1u << 20) && markers.size() <= 16) {  // one round trip (k_scalar.cu)
        std::vector<const char*> mk;
        for (const auto& m : markers) mk.push_back(m.c_str());
        const uint64_t off[2] = {0, answer.size()};
        uint8_t h = 0;
        uint32_t nu = 0;
        cx.check(cdx_cluster_host(cx.raw(), answer.data(), off, 1, mk.data(), static_cast<uint32_t>(mk.size()), nullptr, &h,
                                  nullptr, nullptr, &nu));
        return h != 0;
    }
    const std::string_view one[1] = {answer};
    auto in = detail::intern(cx, one, markers, true, false);
    return in.hes.download()[0] != 0;
}

namespace {

// records -> device ids (interned answers), hesitation flags, step indices, token offsets
struct DeviceTrace {
    detail::Interned in;
    batch::DeviceArray<uint8_t> hes;
    batch::DeviceArray<int32_t> step;
    batch::DeviceArray<int64_t> tok;
    batch::DeviceArray<uint64_t> row_off;
};

DeviceTrace upload(batch::Context& cx, std::span<const AnswerRecord> records, bool want_ids, bool want_tok) {
    DeviceTrace t;
    const size_t n = records.size();
    std::vector<uint8_t> hes(n);
    std::vector<int32_t> step(n);
    std::vector<int64_t> tok(want_tok ? n : 0);
    std::vector<std::string_view> views;
    views.reserve(n);
    for (size_t i = 0; i < n; ++i) {
        hes[i] = records[i].hesitant ? 1 : 0;
        step[i] = records[i].step_index;
        if (want_tok) tok[i] = records[i].token_offset;
        views.push_back(records[i].answer);
    }
    if (want_ids) t.in = detail::intern(cx, views, {}, false, false);
    t.hes = batch::DeviceArray<uint8_t>(cx, std::span<const uint8_t>(hes));
    t.step = batch::DeviceArray<int32_t>(cx, std::span<const int32_t>(step));
    if (want_tok) t.tok = batch::DeviceArray<int64_t>(cx, std::span<const int64_t>(tok));
    const uint64_t off[2] = {0, n};
    t.row_off = batch::DeviceArray<uint64_t>(cx, std::span<const uint64_t>(off, 2));
    return t;
}

}  // namespace

std::optional<double> consistency(std::span<const AnswerRecord> records, int k, int w) {
    if (w < 1) throw std::invalid_argument("consistency: window must be >= 1");
    if (records.empty()) return std::nullopt;  // no usable record can fill a window of w >= 1
    auto& cx = detail::scalar_ctx();
    const auto ar = detail::host_arena(records.begin(), records.end(), [](const AnswerRecord& r) { return std::string_view(r.answer); });
    if (ar.fits) {  // one round trip (k_scalar.cu)
        std::vector<uint8_t> hes;
        std::vector<int32_t> step;
        for (const auto& r : records) {
            hes.push_back(r.hesitant ? 1 : 0);
            step.push_back(r.step_index);
        }
        double c = 0.0;
        uint8_t ready = 0;
        cx.check(cdx_consistency_host(cx.raw(), ar.bytes.data(), ar.off.data(), static_cast<uint32_t>(records.size()),
                                      hes.data(), step.data(), k, w, &c, &ready));
        if (!ready) return std::nullopt;
        return c;
    }
    auto t = upload(cx, records, true, false);
    batch::DeviceArray<int32_t> d_k(cx, std::span<const int32_t>(&k, 1));
    batch::DeviceArray<double> C(cx, 1);
    batch::DeviceArray<uint8_t> ready(cx, 1);
    cx.check(cdx_probe_consistency(cx.raw(), t.in.ids.data(), t.hes.data(), t.step.data(), t.row_off.data(),
                                   d_k.data(), 1, w, C.data(), ready.data()));
    const double c = C.download()[0];
    if (!ready.download()[0]) return std::nullopt;
    return c;
}

ExitDecision should_exit(const ProbeTrace& trace, const ProbeConfig& cfg) {
    cfg.validate();
    if (trace.records.empty()) return ExitDecision::Continue;
    auto& cx = detail::scalar_ctx();
    cdx_probe_cfg c{};
    c.interval_tokens = cfg.interval_tokens;
    c.window = cfg.window;
    c.threshold = cfg.threshold;
    c.max_tokens = cfg.max_tokens;
    uint8_t dec = 0;
    const auto& recs = trace.records;
    const auto ar = detail::host_arena(recs.begin(), recs.end(), [](const AnswerRecord& r) { return std::string_view(r.answer); });
    if (ar.fits) {  // one round trip (k_scalar.cu)
        std::vector<uint8_t> hes;
        std::vector<int32_t> step;
        std::vector<int64_t> tok;
        for (const auto& r : recs) {
            hes.push_back(r.hesitant ? 1 : 0);
            step.push_back(r.step_index);
            tok.push_back(r.token_offset);
        }
        cx.check(cdx_should_exit_host(cx.raw(), ar.bytes.data(), ar.off.data(), static_cast<uint32_t>(recs.size()),
                                      hes.data(), step.data(), tok.data(), &c, &dec));
    } else {
        auto t = upload(cx, trace.records, true, true);
        batch::DeviceArray<uint8_t> d(cx, 1);
        cx.check(cdx_probe_should_exit(cx.raw(), t.in.ids.data(), t.hes.data(), t.step.data(), t.tok.data(),
                                       t.row_off.data(), 1, &c, d.data()));
        dec = d.download()[0];
    }
    switch (dec) {
        case CDX_EXIT_CERTAIN: return ExitDecision::ExitCertain;
        case CDX_EXIT_BUDGET: return ExitDecision::ExitBudget;
        default: return ExitDecision::Continue;
    }
}

FinalAnswer final_answer(const ProbeTrace& trace) {
    if (trace.records.empty()) throw std::invalid_argument("final_answer: empty trace");
    auto& cx = detail::scalar_ctx();
    const int32_t term = trace.terminated_at ? *trace.terminated_at : INT_MIN;
    const uint8_t why = static_cast<uint8_t>(trace.termination_reason);
    if (trace.records.size() <= 0xffffffffull) {  // one round trip (k_scalar.cu)
        std::vector<uint8_t> hes;
        std::vector<int32_t> step;
        for (const auto& r : trace.records) {
            hes.push_back(r.hesitant ? 1 : 0);
            step.push_back(r.step_index);
        }
        uint64_t p = 0;
        uint8_t low = 0;
        cx.check(cdx_final_answer_host(cx.raw(), hes.data(), step.data(), static_cast<uint32_t>(trace.records.size()), term,
                                       why, &p, &low));
        return {std::string(metrics::trim(trace.records[p].answer)), low != 0};
    }
    auto t = upload(cx, trace.records, false, false);
    batch::DeviceArray<int32_t> d_term(cx, std::span<const int32_t>(&term, 1));
    batch::DeviceArray<uint8_t> d_why(cx, std::span<const uint8_t>(&why, 1));
    batch::DeviceArray<uint64_t> pos(cx, 1);
    batch::DeviceArray<uint8_t> low(cx, 1);
    cx.check(cdx_probe_final_answer(cx.raw(), t.hes.data(), t.step.data(), t.row_off.data(), d_term.data(),
                                    d_why.data(), 1, pos.data(), low.data()));
    const uint64_t p = pos.download()[0];
    return {std::string(metrics::trim(trace.records[p].answer)), low.download()[0] != 0};
}

std::optional<bool> stationary_by_epsilon_test(std::span<const AnswerRecord> records, int k, double epsilon) {
    auto& cx = detail::scalar_ctx();
    if (records.empty()) {  // validation first, as theory.cpp:118-119, then "not enough probes"
        cdx_ctx* h = cx.raw();
        batch::DeviceArray<uint64_t> off(cx, 2);
        off.zero();
        batch::DeviceArray<uint8_t> st(cx, 1);
        batch::DeviceArray<uint32_t> ids(cx, 1);
        batch::DeviceArray<uint8_t> hs(cx, 1);
        cx.check(cdx_probe_eps_stop_rows(h, ids.data(), hs.data(), off.data(), 1, k, epsilon, st.data()));
        return std::nullopt;
    }
    auto t = upload(cx, records, true, false);
    batch::DeviceArray<uint8_t> st(cx, 1);
    cx.check(cdx_probe_eps_stop_rows(cx.raw(), t.in.ids.data(), t.hes.data(), t.row_off.data(), 1, k, epsilon,
                                     st.data()));
    const uint8_t v = st.download()[0];
    if (v == 0) return std::nullopt;
    return v == 2;
}

}  // namespace cdx::probe
