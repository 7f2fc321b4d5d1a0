// facade_memory_model.cpp — fusim memory model (include/fusim/memory_model.hpp).
//
// Behavioural contract: /root/reference/proj/src/memory_model.cpp (fit :76-152,
// predict :154-167, feasible :169-179, greedy packer :181-198, max_packing
// :200-239, warmup_plan :241-259).  Restated here, not copied: the fit solves
// the equilibrated least-squares problem by Gram-Schmidt with
// re-orthogonalisation (same optimum; tests/test_memory_model.py checks it
// against the compiled reference), the packer is the same 0.01 GB subset-sum
// contract with the same first-reach claim order, so ties resolve to the same
// subset.
#include "fusim/memory_model.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <set>

namespace fusim {
namespace {

constexpr int kFeatures = 3;

double feature(const MemSample& s, int c) {
    const double u = static_cast<double>(s.batch_size) * s.seq_len;
    return c == 0 ? 1.0 : c == 1 ? u : u * s.seq_len;
}

// min ||A b - y|| over the columns `cols` of the Eq. 6 design.  Columns are
// scaled to unit norm, orthogonalised twice (CGS2), and b is recovered from the
// triangular factor.  FitError when a column is (numerically) dependent.
std::vector<double> solve_ls(const std::vector<MemSample>& samples, const std::vector<int>& cols) {
    const std::size_t n = samples.size(), p = cols.size();
    std::vector<std::vector<double>> q(p, std::vector<double>(n));
    std::vector<double> scale(p);
    for (std::size_t j = 0; j < p; ++j) {
        double nrm = 0.0;
        for (std::size_t i = 0; i < n; ++i) {
            q[j][i] = feature(samples[i], cols[j]);
            nrm += q[j][i] * q[j][i];
        }
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) throw FitError("fit: zero design column");
        scale[j] = nrm;
        for (double& v : q[j]) v /= nrm;
    }
    std::vector<std::vector<double>> r(p, std::vector<double>(p, 0.0));
    for (std::size_t j = 0; j < p; ++j) {
        for (int pass = 0; pass < 2; ++pass) {
            for (std::size_t m = 0; m < j; ++m) {
                double dot = 0.0;
                for (std::size_t i = 0; i < n; ++i) dot += q[m][i] * q[j][i];
                r[m][j] += dot;
                for (std::size_t i = 0; i < n; ++i) q[j][i] -= dot * q[m][i];
            }
        }
        double nrm = 0.0;
        for (double v : q[j]) nrm += v * v;
        nrm = std::sqrt(nrm);
        if (nrm < 1e-12) throw FitError("fit: rank-deficient design");
        r[j][j] = nrm;
        for (double& v : q[j]) v /= nrm;
    }
    std::vector<double> qty(p, 0.0);
    for (std::size_t j = 0; j < p; ++j)
        for (std::size_t i = 0; i < n; ++i) qty[j] += q[j][i] * samples[i].mem_gb;
    std::vector<double> b(p, 0.0);
    for (std::size_t jj = p; jj-- > 0;) {
        double acc = qty[jj];
        for (std::size_t m = jj + 1; m < p; ++m) acc -= r[jj][m] * b[m];
        b[jj] = acc / r[jj][jj];
    }
    for (std::size_t j = 0; j < p; ++j) b[j] /= scale[j];
    return b;
}

double rmse_of(const std::vector<MemSample>& samples, const double (&beta)[kFeatures]) {
    double ss = 0.0;
    for (const MemSample& s : samples) {
        double pred = 0.0;
        for (int c = 0; c < kFeatures; ++c) pred += beta[c] * feature(s, c);
        ss += (pred - s.mem_gb) * (pred - s.mem_gb);
    }
    return std::sqrt(ss / static_cast<double>(samples.size()));
}

}  // namespace

MemoryModel fit_memory_model(const std::vector<MemSample>& samples, FitConstraint constraint) {
    if (samples.size() < 3) throw FitError("fit: need at least 3 samples");
    std::set<long> products;
    for (const MemSample& s : samples) {
        if (s.batch_size < 1 || s.seq_len < 1 || !(s.mem_gb > 0)) throw FitError("fit: invalid sample");
        products.insert(static_cast<long>(s.batch_size) * s.seq_len);
    }
    if (products.size() < 3) throw FitError("fit: need at least 3 distinct batch_size*seq_len values");

    double beta[kFeatures] = {0.0, 0.0, 0.0};
    if (constraint == FitConstraint::Unconstrained) {
        const std::vector<double> b = solve_ls(samples, {0, 1, 2});
        std::copy(b.begin(), b.end(), beta);
    } else {
        // exact NNLS for three unknowns: every subset of coefficients pinned to
        // zero (bit c of `pinned`), the rest solved freely; keep the feasible
        // candidate with the smallest residual (first found on ties)
        bool have = false;
        double best_rmse = 0.0;
        for (int pinned = 0; pinned < (1 << kFeatures); ++pinned) {
            std::vector<int> free_cols;
            for (int c = 0; c < kFeatures; ++c)
                if (!(pinned >> c & 1)) free_cols.push_back(c);
            double cand[kFeatures] = {0.0, 0.0, 0.0};
            if (!free_cols.empty()) {
                std::vector<double> b;
                try {
                    b = solve_ls(samples, free_cols);
                } catch (const FitError&) {
                    continue;
                }
                if (std::any_of(b.begin(), b.end(), [](double v) { return v < 0.0; })) continue;
                for (std::size_t i = 0; i < free_cols.size(); ++i) cand[free_cols[i]] = b[i];
            }
            const double e = rmse_of(samples, cand);
            if (!have || e < best_rmse) {
                have = true;
                best_rmse = e;
                std::copy(cand, cand + kFeatures, beta);
            }
        }
        if (!have) throw FitError("fit: no feasible nonnegative solution");
    }
    MemoryModel m;
    m.beta0 = beta[0];
    m.beta1 = beta[1];
    m.beta2 = beta[2];
    m.rmse = rmse_of(samples, beta);
    m.sample_count = static_cast<int>(samples.size());
    return m;
}

double predict_memory(const MemoryModel& model, int batch_size, int seq_len) {
    const double tokens = static_cast<double>(batch_size) * seq_len;
    return model.beta0 + tokens * (model.beta1 + model.beta2 * seq_len);
}

double predict_memory_clamped(const MemoryModel& model, int batch_size, int seq_len, double floor_gb,
                              bool* clamped) {
    const double raw = predict_memory(model, batch_size, seq_len);
    if (clamped) *clamped = raw < floor_gb;
    return std::max(raw, floor_gb);
}

bool feasible(const PackingQuery& query, const std::vector<std::size_t>& subset) {
    double sum = 0.0;
    for (std::size_t i : subset) {
        if (i >= query.item_mem_gb.size()) throw UsageError("feasible: index out of range");
        sum += query.item_mem_gb[i];
    }
    return sum <= query.budget_gb + 1e-9;
}

std::vector<std::size_t> max_packing_greedy(const PackingQuery& query) {
    const auto& w = query.item_mem_gb;
    std::vector<std::size_t> order(w.size());
    std::iota(order.begin(), order.end(), std::size_t{0});
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return w[a] > w[b]; });
    std::vector<std::size_t> out;
    double used = 0.0;
    for (std::size_t i : order) {
        if (w[i] < 0) throw UsageError("max_packing: negative item size");
        if (used + w[i] <= query.budget_gb) {
            used += w[i];
            out.push_back(i);
        }
    }
    std::sort(out.begin(), out.end());
    return out;
}

std::vector<std::size_t> max_packing(const PackingQuery& query) {
    const auto& w = query.item_mem_gb;
    if (query.budget_gb < 0) throw UsageError("max_packing: negative budget");
    if (w.size() > 30) return max_packing_greedy(query);
    // centi-GB units: items round up, the budget rounds down (the result is
    // feasible in real GB)
    std::vector<long> units(w.size());
    for (std::size_t i = 0; i < w.size(); ++i) {
        if (w[i] < 0) throw UsageError("max_packing: negative item size");
        units[i] = static_cast<long>(std::ceil(w[i] * 100.0 - 1e-9));
    }
    const long cap = static_cast<long>(std::floor(query.budget_gb * 100.0 + 1e-9));
    if (cap < 0) return {};
    // claim[s]: the item whose addition first made total s reachable (items in
    // index order; -1 = the empty set; kUnreached otherwise)
    constexpr int kUnreached = -2;
    std::vector<int> claim(static_cast<std::size_t>(cap) + 1, kUnreached);
    claim[0] = -1;
    for (std::size_t i = 0; i < units.size(); ++i) {
        const long u = units[i];
        if (u > cap) continue;
        for (long s = cap; s >= u; --s)
            if (claim[s] == kUnreached && claim[s - u] != kUnreached && claim[s - u] != static_cast<int>(i))
                claim[s] = static_cast<int>(i);
    }
    long top = cap;
    while (top > 0 && claim[top] == kUnreached) --top;
    std::vector<std::size_t> out;
    for (long s = top; s > 0; s -= units[claim[s]]) out.push_back(static_cast<std::size_t>(claim[s]));
    std::sort(out.begin(), out.end());
    return out;
}

WarmupPlan warmup_plan(const std::vector<int>& batch_sizes, const std::vector<int>& seq_lens) {
    if (batch_sizes.empty() || seq_lens.empty()) throw UsageError("warmup_plan: empty probe lists");
    WarmupPlan plan;
    std::set<std::pair<int, int>> have;
    std::set<long> products;
    for (int b : batch_sizes)
        for (int l : seq_lens) {
            if (b < 1 || l < 1) throw UsageError("warmup_plan: probes must be >= 1");
            if (!have.emplace(b, l).second) continue;
            plan.probes.emplace_back(b, l);
            products.insert(static_cast<long>(b) * l);
        }
    plan.sufficient = products.size() >= 3;
    return plan;
}

}  // namespace fusim
