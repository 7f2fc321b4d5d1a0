// facade_capi.cpp — extern "C" wrappers (include/fusim_c.h) over the façade's
// host packer so the Python executor runs the same C++ MinPad code.
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "fusim/batch_select.hpp"
#include "fusim/memory_model.hpp"
#include "fusim/workload.hpp"
#include "fusim_c.h"

namespace {
thread_local std::string g_err;

int32_t code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const fusim::UsageError*>(&e)) return 1;
    if (dynamic_cast<const fusim::ConfigError*>(&e)) return 7;
    if (dynamic_cast<const fusim::FitError*>(&e)) return 8;
    return 9;
}
}  // namespace

extern "C" {

const char* fusim_c_last_error(void) { return g_err.c_str(); }

int32_t fusim_c_select(int32_t strategy, int32_t n, const int32_t* counts, const int32_t* lengths,
                       const int32_t* priority, const double* submit, int32_t m, int32_t* chosen_idx,
                       int64_t* meta) {
    return fusim_c_select_ids(strategy, n, nullptr, counts, lengths, priority, submit, m, chosen_idx, meta);
}

int32_t fusim_c_select_ids(int32_t strategy, int32_t n, const char* const* ids, const int32_t* counts,
                           const int32_t* lengths, const int32_t* priority, const double* submit, int32_t m,
                           int32_t* chosen_idx, int64_t* meta) {
    try {
        std::vector<fusim::BatchCandidate> cs(static_cast<std::size_t>(n));
        std::vector<std::string> names(static_cast<std::size_t>(n));
        int off = 0;
        for (int i = 0; i < n; ++i) {
            names[i] = ids ? std::string(ids[i]) : "c" + std::to_string(i);
            cs[i].job_id = names[i];
            cs[i].item_lengths.assign(lengths + off, lengths + off + counts[i]);
            off += counts[i];
            cs[i].priority = priority[i];
            cs[i].submit_time = submit[i];
        }
        fusim::SelectionResult r;
        switch (strategy) {
            case 0: r = fusim::select_fifo(cs, m); break;
            case 1: r = fusim::select_priority(cs, m); break;
            case 2: r = fusim::select_minpad(cs, m); break;
            default: r = fusim::brute_force_min_padding(cs, m); break;
        }
        meta[0] = static_cast<int64_t>(r.chosen.size());
        meta[1] = r.fused_max_len;
        meta[2] = r.total_sequences;
        meta[3] = r.padding_tokens;
        for (std::size_t i = 0; i < r.chosen.size(); ++i)
            chosen_idx[i] = static_cast<int32_t>(std::find(names.begin(), names.end(), r.chosen[i]) - names.begin());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int32_t fusim_c_sample_lengths(int32_t family, int32_t min_len, int32_t max_len, double mean, double stddev,
                               int32_t nhist, const int32_t* hist_len, const int32_t* hist_count,
                               int32_t count, uint64_t seed, int32_t* out) {
    try {
        fusim::LengthDistribution d;
        d.family = family == 0 ? fusim::LengthFamily::Uniform
                 : family == 1 ? fusim::LengthFamily::NormalTruncated
                               : fusim::LengthFamily::EmpiricalHistogram;
        d.min_len = min_len;
        d.max_len = max_len;
        d.mean = mean;
        d.stddev = stddev;
        for (int i = 0; i < nhist; ++i) d.histogram[hist_len[i]] = hist_count[i];
        std::mt19937_64 rng(seed);
        const std::vector<int> v = fusim::sample_lengths(d, count, rng);
        std::memcpy(out, v.data(), sizeof(int32_t) * v.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// ------------------------------------------------------------------ memory model
int32_t fusim_c_fit_memory_model(int32_t n, const int32_t* bs, const int32_t* seq, const double* mem,
                                 int32_t nonneg, double* out) {
    try {
        std::vector<fusim::MemSample> s(static_cast<std::size_t>(std::max(n, 0)));
        for (int i = 0; i < n; ++i) s[i] = fusim::MemSample{bs[i], seq[i], mem[i]};
        const fusim::MemoryModel m = fusim::fit_memory_model(
            s, nonneg ? fusim::FitConstraint::NonNegative : fusim::FitConstraint::Unconstrained);
        out[0] = m.beta0;
        out[1] = m.beta1;
        out[2] = m.beta2;
        out[3] = m.rmse;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int32_t fusim_c_max_packing(int32_t n, const double* item_gb, double budget_gb, int32_t greedy, int32_t* out_idx,
                            int32_t* out_n) {
    try {
        fusim::PackingQuery q;
        q.item_mem_gb.assign(item_gb, item_gb + std::max(n, 0));
        q.budget_gb = budget_gb;
        const auto r = greedy ? fusim::max_packing_greedy(q) : fusim::max_packing(q);
        for (std::size_t i = 0; i < r.size(); ++i) out_idx[i] = static_cast<int32_t>(r[i]);
        *out_n = static_cast<int32_t>(r.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

int32_t fusim_c_warmup_plan(int32_t nb, const int32_t* batch_sizes, int32_t nl, const int32_t* seq_lens,
                            int32_t* out_pairs, int32_t* out_n, int32_t* sufficient) {
    try {
        const fusim::WarmupPlan p = fusim::warmup_plan(std::vector<int>(batch_sizes, batch_sizes + std::max(nb, 0)),
                                                       std::vector<int>(seq_lens, seq_lens + std::max(nl, 0)));
        for (std::size_t i = 0; i < p.probes.size(); ++i) {
            out_pairs[2 * i] = p.probes[i].first;
            out_pairs[2 * i + 1] = p.probes[i].second;
        }
        *out_n = static_cast<int32_t>(p.probes.size());
        *sufficient = p.sufficient ? 1 : 0;
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

}  // extern "C"
