// stats.cpp -- SPEC "stats" module: SampleSummary,
// Mann-Whitney U / Wilcoxon rank-sum two-sided p-value, table marks.
#include "../../include/acs/stats.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <stdexcept>

#include "../../include/acs_gpu.h"

void acs_set_error(const char *msg);  // capi.cu: thread-local ABI error

namespace acs {

namespace {

// midranks (1-based) of the pooled sample xs ++ ys, plus sum of (t^3 - t)
std::vector<double> midranks(std::span<const double> xs, std::span<const double> ys, double &tie_term) {
    const size_t n = xs.size() + ys.size();
    std::vector<std::pair<double, size_t>> v(n);
    for (size_t i = 0; i < xs.size(); ++i) v[i] = {xs[i], i};
    for (size_t j = 0; j < ys.size(); ++j) v[xs.size() + j] = {ys[j], xs.size() + j};
    std::sort(v.begin(), v.end());
    std::vector<double> r(n);
    tie_term = 0;
    for (size_t i = 0; i < n;) {
        size_t j = i;
        while (j + 1 < n && v[j + 1].first == v[i].first) ++j;
        const double mid = 0.5 * static_cast<double>(i + j) + 1.0;
        for (size_t k = i; k <= j; ++k) r[v[k].second] = mid;
        const double t = static_cast<double>(j - i + 1);
        tie_term += t * t * t - t;
        i = j + 1;
    }
    return r;
}

void check_sizes(std::span<const double> xs, std::span<const double> ys) {
    if (xs.size() < 3 || ys.size() < 3)
        throw std::invalid_argument("rank_sum_test: both samples need at least 3 values");
}

}  // namespace

double mann_whitney_u(std::span<const double> xs, std::span<const double> ys) {
    double tie = 0;
    const std::vector<double> r = midranks(xs, ys, tie);
    double r1 = 0;
    for (size_t i = 0; i < xs.size(); ++i) r1 += r[i];
    const double n1 = static_cast<double>(xs.size());
    return r1 - n1 * (n1 + 1.0) / 2.0;
}

double rank_sum_test(std::span<const double> xs, std::span<const double> ys) {
    check_sizes(xs, ys);
    double tie = 0;
    const std::vector<double> r = midranks(xs, ys, tie);
    const size_t n1 = xs.size(), n2 = ys.size(), N = n1 + n2;
    if (tie == static_cast<double>(N) * N * N - static_cast<double>(N)) return 1.0;  // all equal
    const double base = static_cast<double>(n1) * (n1 + 1) / 2.0;
    double r1 = 0;
    for (size_t i = 0; i < n1; ++i) r1 += r[i];
    const double u = r1 - base;
    if (N <= 12) {
        // exact: every split of the pooled midranks into n1 + n2 is equally likely
        uint64_t total = 0, le = 0, ge = 0;
        const double eps = 1e-9;
        for (uint32_t mask = 0; mask < (1u << N); ++mask) {
            if (static_cast<size_t>(__builtin_popcount(mask)) != n1) continue;
            double s = 0;
            for (size_t i = 0; i < N; ++i)
                if (mask >> i & 1u) s += r[i];
            const double us = s - base;
            ++total;
            le += us <= u + eps;
            ge += us >= u - eps;
        }
        const double p = 2.0 * static_cast<double>(std::min(le, ge)) / static_cast<double>(total);
        return std::min(1.0, p);
    }
    const double dn1 = static_cast<double>(n1), dn2 = static_cast<double>(n2), dN = static_cast<double>(N);
    const double mu = dn1 * dn2 / 2.0;
    const double var = dn1 * dn2 / 12.0 * ((dN + 1.0) - tie / (dN * (dN - 1.0)));
    if (var <= 0) return 1.0;
    const double z = std::max(0.0, std::fabs(u - mu) - 0.5) / std::sqrt(var);
    const double p = std::erfc(z / std::sqrt(2.0));
    return std::min(1.0, std::max(p, std::numeric_limits<double>::min()));
}

char significance_mark(std::span<const double> candidate, std::span<const double> baseline, double alpha) {
    if (candidate.size() < 3 || baseline.size() < 3) return ' ';
    if (rank_sum_test(candidate, baseline) >= alpha) return ' ';
    const double mc = std::accumulate(candidate.begin(), candidate.end(), 0.0) / candidate.size();
    const double mb = std::accumulate(baseline.begin(), baseline.end(), 0.0) / baseline.size();
    return mc < mb ? '+' : (mc > mb ? '-' : ' ');
}

SampleSummary summarize(std::span<const int64_t> lengths, int64_t optimum, std::span<const double> total_ms,
                        std::span<const double> construct_ms) {
    SampleSummary s;
    s.runs = static_cast<uint32_t>(lengths.size());
    if (lengths.empty()) throw std::invalid_argument("summarize: empty sample");
    s.best_length = *std::min_element(lengths.begin(), lengths.end());
    double sum = 0;
    for (int64_t l : lengths) sum += static_cast<double>(l);
    s.mean_length = sum / s.runs;
    if (optimum > 0) {
        s.mean_error_pct = 100.0 * (s.mean_length - optimum) / optimum;
        s.min_error_pct = 100.0 * static_cast<double>(s.best_length - optimum) / optimum;
    } else {
        s.mean_error_pct = s.min_error_pct = std::numeric_limits<double>::quiet_NaN();
    }
    if (!total_ms.empty())
        s.mean_total_ms = std::accumulate(total_ms.begin(), total_ms.end(), 0.0) / total_ms.size();
    if (!construct_ms.empty())
        s.mean_construct_ms_per_iter =
            std::accumulate(construct_ms.begin(), construct_ms.end(), 0.0) / construct_ms.size();
    return s;
}

}  // namespace acs

// ---- C-ABI (host-only) ----
extern "C" int acs_rank_sum_test(const double *xs, uint32_t nx, const double *ys, uint32_t ny, double *p) {
    if (!xs || !ys || !p || nx < 3 || ny < 3) {
        acs_set_error("acs_rank_sum_test: need two samples of at least 3 values and an output");
        return ACS_E_ARG;
    }
    *p = acs::rank_sum_test({xs, nx}, {ys, ny});
    return ACS_OK;
}
