// facade_metrics.cpp — cdx::metrics (include/cdx/metrics.hpp) on the B200.
//
//   cluster_exact             K1 canon_intern (trim + exact bytes -> dense first-seen ids)
//                             + cdx_id_histogram (cluster sizes)      metrics.cpp:21-37
//   semantic_entropy /        cdx_entropy_sizes_host: host-libm term (c/n) ln(c/n) per
//   certaindex_entropy        cluster, FP64 device fold in cluster order  metrics.cpp:107-125
//   certaindex_reward         cdx_reward_sets (left fold / first max)  metrics.cpp:127-137
//   combined_meets_thresholds cdx_meets_thresholds_rows               metrics.cpp:159-171
// trim() is the boundary's own view adjustment (it returns a view into the caller's
// string, so it cannot live on the device); which answers are equal is decided by K1.

#include <algorithm>
#include <stdexcept>
#include <string>

#include "cdx/metrics.hpp"
#include "facade_common.hpp"

namespace cdx::metrics {

namespace {
constexpr bool is_ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r' || c == '\f' || c == '\v'; }
}  // namespace

std::string_view trim(std::string_view s) {
    size_t b = 0, e = s.size();
    while (b < e && is_ws(s[b])) ++b;
    while (e > b && is_ws(s[e - 1])) --e;
    return s.substr(b, e - b);
}

Clustering cluster_exact(std::span<const std::string> answers) {
    if (answers.empty()) throw std::invalid_argument("cluster_exact: empty answer set");
    auto& cx = detail::scalar_ctx();
    const auto ar = detail::host_arena(answers.begin(), answers.end(), [](const std::string& s) { return std::string_view(s); });
    if (ar.fits) {  // one round trip (k_scalar.cu)
        const uint32_t n = static_cast<uint32_t>(answers.size());
        std::vector<uint32_t> first(n), sizes(n);
        uint32_t nu = 0;
        cx.check(cdx_cluster_host(cx.raw(), ar.bytes.data(), ar.off.data(), n, nullptr, 0, nullptr, nullptr, first.data(),
                                  sizes.data(), &nu));
        Clustering out;
        out.total = static_cast<int>(n);
        out.clusters.reserve(nu);
        for (uint32_t c = 0; c < nu; ++c)
            out.clusters.push_back({std::string(trim(answers[first[c]])), static_cast<int>(sizes[c])});
        return out;
    }
    std::vector<std::string_view> views(answers.begin(), answers.end());
    auto in = detail::intern(cx, views, {}, false, true);
    batch::DeviceArray<uint32_t> counts(cx, in.n_unique);
    cx.check(cdx_id_histogram(cx.raw(), in.ids.data(), answers.size(), static_cast<uint32_t>(in.n_unique),
                              counts.data()));
    const auto sizes = counts.download();
    Clustering out;
    out.total = static_cast<int>(answers.size());
    out.clusters.reserve(in.n_unique);
    for (uint64_t c = 0; c < in.n_unique; ++c)
        out.clusters.push_back({std::string(trim(answers[in.first_index[c]])), static_cast<int>(sizes[c])});
    return out;
}

namespace {

// (H, H~) of one clustering on the device (any sizes and total, as the reference)
std::pair<double, double> entropy_pair(const Clustering& c) {
    std::vector<int32_t> sizes;
    sizes.reserve(c.clusters.size());
    for (const auto& cl : c.clusters) sizes.push_back(static_cast<int32_t>(cl.size));
    auto& cx = detail::scalar_ctx();
    double h = 0.0, hc = 0.0;
    cx.check(cdx_entropy_host(cx.raw(), sizes.data(), static_cast<uint32_t>(sizes.size()), static_cast<int32_t>(c.total),
                              &h, &hc));
    return {h, hc};
}

}  // namespace

double semantic_entropy(const Clustering& c) { return entropy_pair(c).first; }

double certaindex_entropy(const Clustering& c) {
    if (c.total == 1) return 1.0;  // metrics.cpp:121, ahead of any validation
    return entropy_pair(c).second;
}

double certaindex_reward(const RewardSet& r) {
    if (r.rewards.empty()) throw std::invalid_argument("certaindex_reward: empty reward set");
    auto& cx = detail::scalar_ctx();
    const uint8_t agg = r.aggregation == RewardAggregation::Max ? CDX_AGG_MAX : CDX_AGG_MEAN;
    double out = 0.0;
    cx.check(cdx_reward_host(cx.raw(), r.rewards.data(), r.rewards.size(), agg, &out));
    return out;
}

const char* signal_name(SignalKind kind) {
    switch (kind) {
        case SignalKind::CertaindexEntropy: return "certaindex_entropy";
        case SignalKind::CertaindexReward: return "certaindex_reward";
        case SignalKind::MeanOutputLength: return "mean_output_length";
        case SignalKind::MeanNormLogprob: return "mean_norm_logprob";
    }
    return "?";
}

std::optional<double> SignalVector::get(SignalKind kind) const {
    switch (kind) {
        case SignalKind::CertaindexEntropy: return certaindex_entropy;
        case SignalKind::CertaindexReward: return certaindex_reward;
        case SignalKind::MeanOutputLength: return mean_output_length;
        case SignalKind::MeanNormLogprob: return mean_norm_logprob;
    }
    return std::nullopt;
}

bool combined_meets_thresholds(const SignalVector& s, std::span<const SignalThreshold> thresholds) {
    if (thresholds.empty()) return true;
    auto& cx = detail::scalar_ctx();
    double sig[4] = {0, 0, 0, 0};
    uint8_t present = 0;
    for (int k = 0; k < 4; ++k) {
        if (auto v = s.get(static_cast<SignalKind>(k))) {
            sig[k] = *v;
            present |= static_cast<uint8_t>(1u << k);
        }
    }
    // the device evaluates up to 8 thresholds per call, in order; longer lists continue
    // only while every threshold so far has held (the reference's early return)
    for (size_t i = 0; i < thresholds.size(); i += 8) {
        std::vector<cdx_threshold> th;
        for (size_t j = i; j < std::min(thresholds.size(), i + 8); ++j) th.push_back(detail::to_c(thresholds[j]));
        uint8_t ok = 0;
        cx.check(cdx_meets_host(cx.raw(), sig, present, th.data(), static_cast<uint32_t>(th.size()), &ok));
        if (!ok) return false;
    }
    return true;
}

}  // namespace cdx::metrics
