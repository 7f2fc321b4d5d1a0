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

const char* fusim_c_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* FUSIM_C_H_ */
