/*
 * fusim_c.h — C entry points of the host packer in libfusim_b200.so.
 *
 * The MinPad / FIFO / priority selection (fusim::select_*, façade of
 * /root/reference/proj/src/batch_select.cpp:56-128) and the seeded length
 * generators (fusim::sample_lengths, workload.cpp:88-125) are host C++; these
 * extern "C" wrappers let non-C++ executors (the Python trainer) use exactly
 * the same code instead of re-implementing it.  Integer-exact with the
 * reference (tests/test_packer.py).
 */
#ifndef FUSIM_C_H_
#define FUSIM_C_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* strategy: 0 fifo, 1 priority, 2 minpad, 3 brute force.
 * Candidate i has counts[i] item lengths (flattened in `lengths`), priority[i],
 * submit[i]; candidate ids are "c<i>".  chosen_idx receives the selected
 * candidate indices in result order; meta = {count, fused_max_len,
 * total_sequences, padding_tokens}.  Returns 0, or 1 (UsageError) / 9 (other)
 * with the message in fusim_c_last_error(). */
int32_t fusim_c_select(int32_t strategy, int32_t n, const int32_t* counts, const int32_t* lengths,
                       const int32_t* priority, const double* submit, int32_t m, int32_t* chosen_idx,
                       int64_t* meta);

/* family: 0 uniform [min,max], 1 normal(mean, stddev) rounded + clamped, 2 histogram. */
int32_t fusim_c_sample_lengths(int32_t family, int32_t min_len, int32_t max_len, double mean, double stddev,
                               int32_t nhist, const int32_t* hist_len, const int32_t* hist_count,
                               int32_t count, uint64_t seed, int32_t* out);

/* As fusim_c_select with the candidates' real ids (ids[i], NUL-terminated): the
 * reference's tie-breaks compare job ids (batch_select.cpp:10-15). */
int32_t fusim_c_select_ids(int32_t strategy, int32_t n, const char* const* ids, const int32_t* counts,
                           const int32_t* lengths, const int32_t* priority, const double* submit, int32_t m,
                           int32_t* chosen_idx, int64_t* meta);

/* Memory model (fusim/memory_model.hpp; reference memory_model.cpp:76-259).
 * fit: out = {beta0, beta1, beta2, rmse}; returns 8 on FitError.
 * max_packing: out_idx (n entries) receives the ascending subset, out_n its size;
 * greedy != 0 forces the largest-first packer.
 * warmup_plan: out_pairs (2 * nb * nl) receives (batch_size, seq_len) probes. */
int32_t fusim_c_fit_memory_model(int32_t n, const int32_t* bs, const int32_t* seq, const double* mem,
                                 int32_t nonneg, double* out);
int32_t fusim_c_max_packing(int32_t n, const double* item_gb, double budget_gb, int32_t greedy, int32_t* out_idx,
                            int32_t* out_n);
int32_t fusim_c_warmup_plan(int32_t nb, const int32_t* batch_sizes, int32_t nl, const int32_t* seq_lens,
                            int32_t* out_pairs, int32_t* out_n, int32_t* sufficient);

const char* fusim_c_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* FUSIM_C_H_ */
