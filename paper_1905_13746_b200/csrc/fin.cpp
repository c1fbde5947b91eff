// FIN: host-side finalize of the fit -- feature scoring, top-k and the
// smoothed log-parameters -- from the dense per-(group, class, column) sums
// produced by K-FIT.  Tiny ([G, V] work); kept on the host in C++ so the
// logarithm is libm's `log`, the same function CPython's math.log calls, which
// makes the produced bundle bit-identical to the reference's.
//
// Restates, per trainable group (engine.py:166-173):
//   features.class_frequency / score_opcodes   pkg/src/groupnb/features.py:41-75
//   features.select_top_k                      pkg/src/groupnb/features.py:78-86
//   classifier.train_group (priors, log-lik)   pkg/src/groupnb/classifier.py:103-120
//   corpus.trainable_groups                    pkg/src/groupnb/corpus.py:295-307
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../include/gnb.h"

namespace {

constexpr int kBenign = 0, kMalware = 1;

inline uint64_t as_count(double v) { return static_cast<uint64_t>(v); }

}  // namespace

extern "C" int gnb_fin_tables(const double* sums_g, const double* counts_g, int32_t n_classes,
                              int32_t n_cols, const int32_t* features, int32_t n_features,
                              double alpha, double* log_prior, double* log_lik) {
  // classifier.train_group with a class axis (classifier.py:103-120); C = 2
  // is the reference exactly, C > 2 the multi-family generalisation.
  if (!sums_g || !counts_g || !features || !log_prior || !log_lik) return GNB_EINVAL;
  if (n_classes < 2 || n_cols < 1 || n_features < 1 || !(alpha > 0.0) || !std::isfinite(alpha))
    return GNB_EINVAL;
  uint64_t n_tot = 0;
  for (int c = 0; c < n_classes; ++c) n_tot += as_count(counts_g[c]);
  if (n_tot == 0) return GNB_EINVAL;
  for (int c = 0; c < n_classes; ++c)
    log_prior[c] = std::log(static_cast<double>(as_count(counts_g[c])) / static_cast<double>(n_tot));
  // total_c sums each DISTINCT feature once: the reference's per-class count
  // dict is keyed by opcode (classifier.py:91-93, 116), while |F| counts a
  // repeated opcode every time (n_features = len(features.opcodes), :112).
  std::vector<char> seen(static_cast<size_t>(n_cols), 0);
  for (int j = 0; j < n_features; ++j)
    if (features[j] < 0 || features[j] >= n_cols) return GNB_EINVAL;
  for (int c = 0; c < n_classes; ++c) {
    const double* S = sums_g + static_cast<int64_t>(c) * n_cols;
    uint64_t total_c = 0;
    std::fill(seen.begin(), seen.end(), 0);
    for (int j = 0; j < n_features; ++j) {
      if (seen[static_cast<size_t>(features[j])]) continue;
      seen[static_cast<size_t>(features[j])] = 1;
      total_c += as_count(S[features[j]]);
    }
    const double denom = static_cast<double>(total_c) + alpha * static_cast<double>(n_features);
    for (int j = 0; j < n_features; ++j)
      log_lik[static_cast<int64_t>(c) * n_features + j] =
          std::log((static_cast<double>(as_count(S[features[j]])) + alpha) / denom);
  }
  return GNB_OK;
}

extern "C" int gnb_fin_train(const double* sums, const double* counts, int32_t n_groups,
                             int32_t n_cols, int32_t k, double alpha, int32_t min_per_class,
                             int32_t* group_state, int32_t* n_features, int32_t* features,
                             double* log_prior, double* log_lik) {
  if (!sums || !counts || !group_state || !n_features || !features || !log_prior || !log_lik)
    return GNB_EINVAL;
  if (n_groups < 1 || n_cols < 1 || k < 1 || !(alpha > 0.0) || !std::isfinite(alpha) ||
      min_per_class < 1)
    return GNB_EINVAL;
  std::vector<int32_t> cand;
  std::vector<double> score(static_cast<size_t>(n_cols));
  for (int g = 0; g < n_groups; ++g) {
    const double* S = sums + static_cast<int64_t>(g) * 2 * n_cols;  // [2][V]
    const uint64_t n_b = as_count(counts[2 * g + kBenign]);
    const uint64_t n_m = as_count(counts[2 * g + kMalware]);
    n_features[g] = 0;
    std::fill(features + static_cast<int64_t>(g) * k, features + static_cast<int64_t>(g + 1) * k, 0);
    std::fill(log_prior + 2 * g, log_prior + 2 * g + 2, 0.0);
    std::fill(log_lik + static_cast<int64_t>(g) * 2 * k,
              log_lik + static_cast<int64_t>(g + 1) * 2 * k, 0.0);
    if (n_b < static_cast<uint64_t>(min_per_class) || n_m < static_cast<uint64_t>(min_per_class)) {
      group_state[g] = 0;  // not trainable: routed to a neighbour (engine.py:87-103)
      continue;
    }
    // class totals over ALL opcodes (features.py:51-53)
    uint64_t t_b = 0, t_m = 0;
    for (int v = 0; v < n_cols; ++v) {
      t_b += as_count(S[kBenign * n_cols + v]);
      t_m += as_count(S[kMalware * n_cols + v]);
    }
    if (t_m == 0) {  // checked first, as score_opcodes does (features.py:67-68)
      group_state[g] = -1;
      continue;
    }
    if (t_b == 0) {
      group_state[g] = -2;
      continue;
    }
    // candidates: union of nonzero opcodes (features.py:71); |f_m - f_b|
    cand.clear();
    for (int v = 0; v < n_cols; ++v) {
      const uint64_t cb = as_count(S[kBenign * n_cols + v]);
      const uint64_t cm = as_count(S[kMalware * n_cols + v]);
      if (cb == 0 && cm == 0) continue;
      cand.push_back(v);
      const double f_m = static_cast<double>(cm) / static_cast<double>(t_m);
      const double f_b = static_cast<double>(cb) / static_cast<double>(t_b);
      score[v] = std::fabs(f_m - f_b);
    }
    // (-score, mnemonic) with columns in mnemonic order (features.py:85)
    std::sort(cand.begin(), cand.end(), [&](int32_t a, int32_t b) {
      if (score[a] != score[b]) return score[a] > score[b];
      return a < b;
    });
    const int F = static_cast<int>(std::min<size_t>(cand.size(), static_cast<size_t>(k)));
    n_features[g] = F;
    for (int j = 0; j < F; ++j) features[static_cast<int64_t>(g) * k + j] = cand[j];
    // priors ln(n_c / n) and smoothed likelihoods over the selected features
    // only (classifier.py:109-120), written [2][F] then spread to stride k
    double lik_tmp[2 * 4096];
    double* lik = F <= 4096 ? lik_tmp : nullptr;
    std::vector<double> lik_big;
    if (!lik) {
      lik_big.resize(static_cast<size_t>(2) * F);
      lik = lik_big.data();
    }
    const double cnt2[2] = {static_cast<double>(n_b), static_cast<double>(n_m)};
    gnb_fin_tables(S, cnt2, 2, n_cols, features + static_cast<int64_t>(g) * k, F, alpha,
                   log_prior + 2 * g, lik);
    for (int c = 0; c < 2; ++c)
      for (int j = 0; j < F; ++j)
        log_lik[(static_cast<int64_t>(g) * 2 + c) * k + j] = lik[static_cast<int64_t>(c) * F + j];
    group_state[g] = 1;
  }
  return GNB_OK;
}
