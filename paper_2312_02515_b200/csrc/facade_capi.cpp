// facade_capi.cpp — extern "C" wrappers (include/fusim_c.h) over the façade's
// host packer so the Python executor runs the same C++ MinPad code.
#include <cstring>
#include <string>
#include <vector>

#include "fusim/batch_select.hpp"
#include "fusim/workload.hpp"
#include "fusim_c.h"

namespace {
thread_local std::string g_err;

int32_t code_of(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const fusim::UsageError*>(&e)) return 1;
    if (dynamic_cast<const fusim::ConfigError*>(&e)) return 7;
    return 9;
}
}  // namespace

extern "C" {

const char* fusim_c_last_error(void) { return g_err.c_str(); }

int32_t fusim_c_select(int32_t strategy, int32_t n, const int32_t* counts, const int32_t* lengths,
                       const int32_t* priority, const double* submit, int32_t m, int32_t* chosen_idx,
                       int64_t* meta) {
    try {
        std::vector<fusim::BatchCandidate> cs(static_cast<std::size_t>(n));
        int off = 0;
        for (int i = 0; i < n; ++i) {
            cs[i].job_id = "c" + std::to_string(i);
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
        for (std::size_t i = 0; i < r.chosen.size(); ++i) chosen_idx[i] = std::stoi(r.chosen[i].substr(1));
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

}  // extern "C"
