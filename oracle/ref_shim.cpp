// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference sources
// (/root/reference/proj/src/{lora,batch_select,workload}.cpp, compiled in place
// by oracle/Makefile into oracle/_ref/libfusim_ref.so).  TEST INFRASTRUCTURE:
// used only to pin the oracle (golden fixtures), by tests, and as the timed CPU
// baseline (`cpu_baseline.kind = "reference"`).  Nothing here is reference code;
// it only marshals plain arrays into the reference's own types and calls it.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <random>
#include <string>
#include <vector>

#include "fusim/batch_select.hpp"
#include "fusim/errors.hpp"
#include "fusim/lora.hpp"
#include "fusim/workload.hpp"

using namespace fusim;

namespace {
thread_local std::string g_err;

int code_of(const std::exception& e) {
    if (dynamic_cast<const UsageError*>(&e)) return 1;
    if (dynamic_cast<const ShapeError*>(&e)) return 2;
    if (dynamic_cast<const RoutingError*>(&e)) return 3;
    if (dynamic_cast<const NumericError*>(&e)) return 4;
    if (dynamic_cast<const StateError*>(&e)) return 5;
    if (dynamic_cast<const ConfigError*>(&e)) return 7;
    return 9;
}

#define GUARD_BEGIN try {
#define GUARD_END                  \
    }                              \
    catch (const std::exception& e) { \
        g_err = e.what();          \
        return code_of(e);         \
    }

Matrix mat(const double* p, int r, int c) {
    Matrix m(r, c);
    if (p) std::memcpy(m.data.data(), p, sizeof(double) * r * c);
    return m;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// fused_shape over a flattened (group_sizes, lengths) description
int ref_fused_shape(int ngroups, const int* group_sizes, const int* lengths, int* max_len,
                    int64_t* sequences, int64_t* total, int64_t* padding, double* ratio) {
    GUARD_BEGIN
    std::vector<std::vector<int>> g(ngroups);
    int off = 0;
    for (int i = 0; i < ngroups; ++i)
        for (int j = 0; j < group_sizes[i]; ++j) g[i].push_back(lengths[off++]);
    const FusedShape s = fused_shape(g);
    *max_len = s.max_len;
    *sequences = s.sequences;
    *total = s.total_tokens;
    *padding = s.padding_tokens;
    *ratio = s.padding_ratio();
    return 0;
    GUARD_END
}

// Build a FusedBatch from (job, sequence) descriptions and run fused_forward.
//   W0 d x k; per job j: rank[j], A_j (rank x k) at A_all + aoff, B_j (d x rank) at B_all + boff
//   (jobs with has_adapter[j] == 0 are omitted from the adapter map -> RoutingError)
//   sequences: seq_job[s], seq_len[s], rows concatenated in X_all (sum len x k)
//   outputs: out (nseq * max_len * d), mask (nseq * max_len), meta[4] = {max_len, S, total, padding}
static int fused_forward_impl(const Matrix& W0, int njobs, const int* ranks, const int* has_adapter,
                              const double* A_all, const double* B_all, int nseq, const int* seq_job,
                              const int* seq_len, const double* X_all, double* out, uint8_t* mask,
                              int64_t* meta);

int ref_fused_forward_w(const double* W0p, int d, int k, int njobs, const int* ranks,
                        const int* has_adapter, const double* A_all, const double* B_all, int nseq,
                        const int* seq_job, const int* seq_len, const double* X_all, double* out,
                        uint8_t* mask, int64_t* meta) {
    GUARD_BEGIN
    const Matrix W0 = mat(W0p, d, k);
    return fused_forward_impl(W0, njobs, ranks, has_adapter, A_all, B_all, nseq, seq_job, seq_len, X_all,
                              out, mask, meta);
    GUARD_END
}

// Weight handle: the frozen W0 marshalled once into a reference Matrix so the
// timed baseline measures fused_forward itself, not the array copy.
void* ref_weights_create(const double* W0p, int d, int k) { return new Matrix(mat(W0p, d, k)); }
void ref_weights_destroy(void* h) { delete static_cast<Matrix*>(h); }

int ref_fused_forward_h(void* W0h, int njobs, const int* ranks, const int* has_adapter,
                        const double* A_all, const double* B_all, int nseq, const int* seq_job,
                        const int* seq_len, const double* X_all, double* out, uint8_t* mask,
                        int64_t* meta) {
    GUARD_BEGIN
    return fused_forward_impl(*static_cast<Matrix*>(W0h), njobs, ranks, has_adapter, A_all, B_all, nseq,
                              seq_job, seq_len, X_all, out, mask, meta);
    GUARD_END
}

}  // extern "C"

static int fused_forward_impl(const Matrix& W0, int njobs, const int* ranks, const int* has_adapter,
                              const double* A_all, const double* B_all, int nseq, const int* seq_job,
                              const int* seq_len, const double* X_all, double* out, uint8_t* mask,
                              int64_t* meta) {
    const int d = W0.rows, k = W0.cols;
    std::map<std::string, AdapterWeights> adapters;
    size_t ao = 0, bo = 0;
    for (int j = 0; j < njobs; ++j) {
        const int r = ranks[j];
        if (has_adapter[j]) {
            AdapterWeights a;
            a.job_id = "j" + std::to_string(j);
            a.rank = r;
            a.A = mat(A_all + ao, r, k);
            a.B = mat(B_all + bo, d, r);
            adapters[a.job_id] = std::move(a);
        }
        ao += static_cast<size_t>(r) * k;
        bo += static_cast<size_t>(d) * r;
    }
    std::vector<JobBatch> batches;
    size_t xo = 0;
    for (int s = 0; s < nseq; ++s) {
        const std::string id = "j" + std::to_string(seq_job[s]);
        if (batches.empty() || batches.back().job_id != id) {
            JobBatch b;
            b.job_id = id;
            batches.push_back(std::move(b));
        }
        batches.back().sequences.push_back(mat(X_all + xo, seq_len[s], k));
        xo += static_cast<size_t>(seq_len[s]) * k;
    }
    const FusedBatch fb = fuse(batches);
    const auto outs = fused_forward(W0, adapters, fb);
    meta[0] = fb.max_len;
    meta[1] = fb.num_sequences;
    meta[2] = fb.total_tokens;
    meta[3] = fb.padding_tokens;
    if (mask) std::memcpy(mask, fb.mask.data(), fb.mask.size());
    if (out)
        for (size_t s = 0; s < outs.size(); ++s)
            std::memcpy(out + s * static_cast<size_t>(fb.max_len) * d, outs[s].data.data(),
                        sizeof(double) * outs[s].data.size());
    return 0;
}

extern "C" {

// lora_forward (column convention): h (d x m) = W0 x + B (A x)
int ref_lora_forward(const double* W0p, int d, int k, int rank, const double* Ap, int arows,
                     int acols, const double* Bp, int brows, int bcols, const double* xp, int xrows,
                     int m, double* out) {
    GUARD_BEGIN
    AdapterWeights a;
    a.rank = rank;
    a.A = mat(Ap, arows, acols);
    a.B = mat(Bp, brows, bcols);
    const Matrix h = lora_forward(mat(W0p, d, k), a, mat(xp, xrows, m));
    std::memcpy(out, h.data.data(), sizeof(double) * h.data.size());
    return 0;
    GUARD_END
}

int ref_matmul(const double* a, int ar, int ac, const double* b, int br, int bc, double* out) {
    GUARD_BEGIN
    const Matrix c = matmul(mat(a, ar, ac), mat(b, br, bc));
    std::memcpy(out, c.data.data(), sizeof(double) * c.data.size());
    return 0;
    GUARD_END
}

int ref_count_launches(int num_jobs, int fused, int64_t* small, int64_t* large) {
    GUARD_BEGIN
    const LaunchCount c = count_launches(num_jobs, fused ? LaunchMode::Fused : LaunchMode::PerJob);
    *small = c.small_launches;
    *large = c.large_launches;
    return 0;
    GUARD_END
}

// select_minpad / fifo / priority / brute force.  strategy: 0 fifo, 1 priority, 2 minpad, 3 brute
// candidates: n, item counts, lengths flattened, priority, submit.  chosen_idx receives
// indices (into the candidate list) in result order; meta = {count, max_len, sequences, padding}.
int ref_select(int strategy, int n, const int* counts, const int* lengths, const int* priority,
               const double* submit, int m, int* chosen_idx, int64_t* meta, double* ratio) {
    GUARD_BEGIN
    std::vector<BatchCandidate> cs(n);
    int off = 0;
    for (int i = 0; i < n; ++i) {
        cs[i].job_id = "c" + std::to_string(i);
        for (int j = 0; j < counts[i]; ++j) cs[i].item_lengths.push_back(lengths[off++]);
        cs[i].priority = priority[i];
        cs[i].submit_time = submit[i];
    }
    SelectionResult r;
    switch (strategy) {
        case 0: r = select_fifo(cs, m); break;
        case 1: r = select_priority(cs, m); break;
        case 2: r = select_minpad(cs, m); break;
        default: r = brute_force_min_padding(cs, m); break;
    }
    meta[0] = static_cast<int64_t>(r.chosen.size());
    meta[1] = r.fused_max_len;
    meta[2] = r.total_sequences;
    meta[3] = r.padding_tokens;
    *ratio = r.padding_ratio;
    for (size_t i = 0; i < r.chosen.size(); ++i) chosen_idx[i] = std::stoi(r.chosen[i].substr(1));
    return 0;
    GUARD_END
}

// sample_lengths with the reference's own std::mt19937_64 + libstdc++ distributions.
// family: 0 uniform, 1 normal-truncated, 2 histogram (hist_len/hist_count pairs)
int ref_sample_lengths(int family, int min_len, int max_len, double mean, double stddev, int nhist,
                       const int* hist_len, const int* hist_count, int count, uint64_t seed, int* out) {
    GUARD_BEGIN
    LengthDistribution d;
    d.family = family == 0 ? LengthFamily::Uniform
             : family == 1 ? LengthFamily::NormalTruncated
                           : LengthFamily::EmpiricalHistogram;
    d.min_len = min_len;
    d.max_len = max_len;
    d.mean = mean;
    d.stddev = stddev;
    for (int i = 0; i < nhist; ++i) d.histogram[hist_len[i]] = hist_count[i];
    std::mt19937_64 rng(seed);
    const auto v = sample_lengths(d, count, rng);
    std::memcpy(out, v.data(), sizeof(int) * v.size());
    return 0;
    GUARD_END
}

// JobState peek/commit trace: runs `rounds` peek+commit cycles over `items`,
// writing each peeked batch's size to sizes[r] and lengths flattened to out.
int ref_batch_trace(int nitems, const int* items, int batch_size, int rounds, int* sizes, int* out,
                    int64_t* final_cursor) {
    GUARD_BEGIN
    JobSpec spec;
    spec.id = "j";
    spec.batch_size = batch_size;
    spec.true_iterations = 1;
    for (int i = 0; i < nitems; ++i) spec.dataset.items.push_back(DataItem{items[i]});
    JobState js(spec);
    int o = 0;
    for (int r = 0; r < rounds; ++r) {
        const auto b = js.next_candidate_batch();
        sizes[r] = static_cast<int>(b.size());
        for (const auto& it : b) out[o++] = it.length;
        js.commit_batch(b.size());
    }
    *final_cursor = static_cast<int64_t>(js.cursor);
    return 0;
    GUARD_END
}

}  // extern "C"
