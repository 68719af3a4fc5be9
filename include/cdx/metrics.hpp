#pragma once
// cdx/metrics.hpp — the reference's certainty-metric API (proj/include/cdx/metrics.hpp),
// re-declared with the same namespace, types, enumerator order and signatures so that a
// caller written against the reference compiles and links unchanged against libcdxhost.so.
//
// Every function that computes a certaindex runs on the B200 through the C-ABI
// (include/cdx_c.h): clustering via K1 canon_intern + id histogram, entropy via the
// host-built term table and an FP64 device fold, reward aggregation and the threshold test
// via device kernels.  Exceptions carry the reference's types and message texts.
//
// Out of scope for this build: trigram_jaccard / cluster_similarity
// (metrics.cpp:39-105, an O(n^2) stand-in for an embedding model no configuration uses) and
// mean_norm_logprob (metrics.cpp:173-181, an appendix ablation signal).  They are not
// declared, so a caller that needs them fails at compile time rather than silently.

#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <vector>

namespace cdx::metrics {

// ---- clustering (metrics.hpp:27-44) --------------------------------------------------

struct AnswerCluster {
    std::string label;  // trimmed text of the cluster's first-seen answer
    int size = 0;       // paths in the cluster
};

struct Clustering {
    std::vector<AnswerCluster> clusters;  // first-seen order
    int total = 0;                        // n = number of answers clustered

    int group_count() const { return static_cast<int>(clusters.size()); }
};

// Drop leading/trailing ' ' '\t' '\n' '\r' '\f' '\v' (metrics.cpp:12-19).  A view into `s`.
std::string_view trim(std::string_view s);

// Exact match of trimmed bytes, clusters in first-seen order (metrics.cpp:21-37).
// Throws std::invalid_argument("cluster_exact: empty answer set") on no answers.
Clustering cluster_exact(std::span<const std::string> answers);

// ---- entropy certaindex (metrics.cpp:107-125) ------------------------------------------

// H = -sum (size/n) ln(size/n) in cluster order, floored at 0.
double semantic_entropy(const Clustering& c);

// (ln n - H) / ln n clamped to [0,1]; n == 1 is 1.0.
double certaindex_entropy(const Clustering& c);

// ---- reward certaindex (metrics.cpp:127-137) -------------------------------------------

enum class RewardAggregation { Mean, Max };

struct RewardSet {
    std::vector<double> rewards;  // every value in [0,1]
    RewardAggregation aggregation = RewardAggregation::Mean;
};

double certaindex_reward(const RewardSet& r);

// ---- signals and thresholds (metrics.cpp:139-171) ---------------------------------------

enum class SignalKind { CertaindexEntropy, CertaindexReward, MeanOutputLength, MeanNormLogprob };

const char* signal_name(SignalKind kind);

// Signals of one program at one knob point; for CoT programs the entropy slot carries the
// probe-window consistency (metrics.hpp:91-92).
struct SignalVector {
    std::optional<double> certaindex_entropy;
    std::optional<double> certaindex_reward;
    std::optional<double> mean_output_length;
    std::optional<double> mean_norm_logprob;

    std::optional<double> get(SignalKind kind) const;
    bool any() const {
        return certaindex_entropy || certaindex_reward || mean_output_length || mean_norm_logprob;
    }
};

enum class ThresholdDir { GreaterEq, LessEq };

struct SignalThreshold {
    SignalKind signal = SignalKind::CertaindexEntropy;
    double cutoff = 0.0;
    ThresholdDir dir = ThresholdDir::GreaterEq;
};

// Inclusive AND over the thresholds in order; empty -> true; a threshold on an absent
// signal throws std::invalid_argument("combined_meets_thresholds: signal '<name>' absent").
bool combined_meets_thresholds(const SignalVector& s, std::span<const SignalThreshold> thresholds);

}  // namespace cdx::metrics
