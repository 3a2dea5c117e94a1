// include/acs/stats.hpp -- quality metrics and the paper's significance test
// (reference SPEC.md:395-437, module "stats"; PAPER.md Table "Mean distance
// from the optimum": "two-sided nonparametric Wilcoxon rank-sum test").
// Host-side, pure functions; relative_error lives in solver.hpp.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

namespace acs {

// SPEC SampleSummary: mean / min error %, best length, run count, times
struct SampleSummary {
    double mean_error_pct = 0, min_error_pct = 0;  // NaN when no optimum is known
    int64_t best_length = 0;
    double mean_length = 0;
    uint32_t runs = 0;
    double mean_total_ms = 0, mean_construct_ms_per_iter = 0;
};

// Summary of per-run best lengths (optimum <= 0: errors are NaN) and times.
SampleSummary summarize(std::span<const int64_t> lengths, int64_t optimum,
                        std::span<const double> total_ms = {}, std::span<const double> construct_ms = {});

// Two-sided Wilcoxon rank-sum (Mann-Whitney U) p-value, midranks for ties:
// exact enumeration of all rank splits when |xs| + |ys| <= 12, otherwise the
// normal approximation with tie and continuity correction.  p in (0, 1];
// an all-equal pooled sample gives 1.  Requires |xs| >= 3 and |ys| >= 3
// (throws std::invalid_argument otherwise).
double rank_sum_test(std::span<const double> xs, std::span<const double> ys);

// Mann-Whitney U of xs (rank sum of xs minus |xs|(|xs|+1)/2, midranks)
double mann_whitney_u(std::span<const double> xs, std::span<const double> ys);

// Paper table annotation of `candidate` against `baseline` (lower is better):
// '+' significantly better, '-' significantly worse, ' ' otherwise.
char significance_mark(std::span<const double> candidate, std::span<const double> baseline,
                       double alpha = 0.05);

}  // namespace acs
