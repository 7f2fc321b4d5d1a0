// ref_shim_memory.cpp — extern "C" access to the reference's memory-model fit
// (/root/reference/proj/src/memory_model.cpp, compiled in place by oracle/Makefile).
// TEST INFRASTRUCTURE: used to check that the B200 memory probes
// (tools/memory_probe.py) feed the reference's own Eq. 6 fit.
#include <string>
#include <vector>

#include "fusim/errors.hpp"
#include "fusim/memory_model.hpp"

extern "C" int ref_fit_memory_model(int n, const int* bs, const int* seq, const double* mem, int nonneg,
                                    double* out /* beta0, beta1, beta2, rmse */) {
    try {
        std::vector<fusim::MemSample> s(n);
        for (int i = 0; i < n; ++i) s[i] = fusim::MemSample{bs[i], seq[i], mem[i]};
        const fusim::MemoryModel m = fusim::fit_memory_model(
            s, nonneg ? fusim::FitConstraint::NonNegative : fusim::FitConstraint::Unconstrained);
        out[0] = m.beta0;
        out[1] = m.beta1;
        out[2] = m.beta2;
        out[3] = m.rmse;
        return 0;
    } catch (const fusim::FitError&) {
        return 8;
    } catch (const std::exception&) {
        return 9;
    }
}

// max_packing / max_packing_greedy (memory_model.cpp:181-239): out_idx receives
// the ascending subset, *out_n its size.  Returns 0, 1 on UsageError, 9 otherwise.
extern "C" int ref_max_packing(int n, const double* items, double budget, int greedy, int* out_idx, int* out_n) {
    try {
        fusim::PackingQuery q;
        q.item_mem_gb.assign(items, items + n);
        q.budget_gb = budget;
        const auto r = greedy ? fusim::max_packing_greedy(q) : fusim::max_packing(q);
        for (std::size_t i = 0; i < r.size(); ++i) out_idx[i] = static_cast<int>(r[i]);
        *out_n = static_cast<int>(r.size());
        return 0;
    } catch (const fusim::UsageError&) {
        return 1;
    } catch (const std::exception&) {
        return 9;
    }
}

// warmup_plan (memory_model.cpp:241-259).
extern "C" int ref_warmup_plan(int nb, const int* bs, int nl, const int* ls, int* out_pairs, int* out_n,
                               int* sufficient) {
    try {
        const auto p = fusim::warmup_plan(std::vector<int>(bs, bs + nb), std::vector<int>(ls, ls + nl));
        for (std::size_t i = 0; i < p.probes.size(); ++i) {
            out_pairs[2 * i] = p.probes[i].first;
            out_pairs[2 * i + 1] = p.probes[i].second;
        }
        *out_n = static_cast<int>(p.probes.size());
        *sufficient = p.sufficient ? 1 : 0;
        return 0;
    } catch (const fusim::UsageError&) {
        return 1;
    } catch (const std::exception&) {
        return 9;
    }
}
