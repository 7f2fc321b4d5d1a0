/*
 * mlora.h — C ABI of the B200-native BatchFusion multi-LoRA linear layer.
 *
 * This is the drop-in boundary for the hot path of ASPEN (arXiv 2312.02515)
 * whose CPU reference lives in /root/reference/proj/include/fusim/lora.hpp and
 * /root/reference/proj/src/lora.cpp.  Every entry point names the reference
 * interface it replaces (file:line).  The reference is a C++ library; its C++
 * API is reproduced on top of this ABI by include/fusim/lora.hpp (the façade,
 * paper_2312_02515_b200/csrc/facade_lora.cpp), and Python binds it through
 * ctypes (paper_2312_02515_b200/_native.py).
 *
 * Conventions:
 *   - Plain pointers and sizes only.  Device pointers are caller-owned CUDA
 *     device memory; host pointers are marked `host`.  Nothing allocates on a
 *     hot call except the context's grow-only workspace.
 *   - Errors are returned as mlora_status, never thrown across the boundary.
 *     The status values mirror the reference exception taxonomy
 *     (/root/reference/proj/include/fusim/errors.hpp:13-23) and every
 *     precondition is checked on the host BEFORE any device work, exactly where
 *     the reference checks it (lora.cpp:20-23, 62-70, 106-109, 115-131, 163-167).
 *   - Calls on one context are ordered on the stream passed in; use one
 *     context per GPU/thread (the reference is single-threaded and reentrant,
 *     /root/reference/SPEC.md:161-162).
 *   - Storage convention is the reference's: W0 is d x k (out x in), A_j is
 *     r_j x k, B_j is d x r_j, all row-major (lora.hpp:16,36-37).  Fused rows
 *     follow FusedBatch order: job order, then sequence order (lora.cpp:143-156).
 *   - Device dtype: bf16 operands, fp32 accumulation, fp32 gradients/optimizer
 *     state.  The reference has no scale; s_j = 1 reproduces it.
 *
 * Packed adapter layout ("cat" layout), owned by the caller:
 *   R_pad = sum_j roundup(r_j, 16); job j owns columns [roff[j], roff[j+1]).
 *   A_cat  : R_pad x k   (rows of job j = A_j, zero rows up to the padded rank)
 *   B_cat  : d x R_pad   (cols of job j = B_j, zero cols up to the padded rank)
 *   H_cat  : rows x R_pad, block-diagonal: H[t, roff[j]:roff[j]+r_j] = s_j X_t A_j^T
 *            for t in job j's segment, 0 elsewhere (saved by fwd for bwd).
 */
#ifndef MLORA_H_
#define MLORA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors fusim::Error subclasses (errors.hpp:13-23). */
typedef enum mlora_status {
    MLORA_OK = 0,
    MLORA_USAGE = 1,   /* fusim::UsageError   — precondition violated       */
    MLORA_SHAPE = 2,   /* fusim::ShapeError   — dimension mismatch          */
    MLORA_ROUTING = 3, /* fusim::RoutingError — batch routed to no adapter  */
    MLORA_NUMERIC = 4, /* fusim::NumericError — non-finite input            */
    MLORA_STATE = 5,   /* fusim::StateError   — object in the wrong state   */
    MLORA_CUDA = 6     /* device/runtime failure (no reference analogue)    */
} mlora_status;

typedef struct mlora_ctx mlora_ctx;
typedef struct mlora_plan mlora_plan;

/* Replaces fusim::FusedShape (lora.hpp:51-61). */
typedef struct mlora_fused_shape {
    int32_t max_len;
    int64_t sequences;
    int64_t total_tokens;   /* sequences * max_len  (ξ)   */
    int64_t padding_tokens; /* Σ (max_len - len)    (ξ_p) */
} mlora_fused_shape;

const char* mlora_status_string(mlora_status s);
/* Human-readable text of the last failing call on this context (or thread, for ctx==NULL). */
const char* mlora_last_error(const mlora_ctx* ctx);
/* ABI version, bumped on any signature change. */
int32_t mlora_abi_version(void);

/* ---------------------------------------------------------------- context */
mlora_status mlora_ctx_create(int32_t device, mlora_ctx** out);
mlora_status mlora_ctx_destroy(mlora_ctx* ctx);
/* Number of SMs of the context's device (148 on B200). */
int32_t mlora_ctx_num_sms(const mlora_ctx* ctx);
/* Kernels launched through this context since creation (telemetry). */
int64_t mlora_ctx_launch_count(const mlora_ctx* ctx);
/* Kernels launched by the context-free entry points (model / decoder kernels:
 * masked CE, norms, RoPE, SwiGLU, attention, ...) in this process (telemetry). */
int64_t mlora_free_launch_count(void);
/* Live per-kernel timing: while enabled, every launch is bracketed by CUDA
 * events on its own stream.  profile_read synchronises on the recorded events
 * and returns the accumulated launch count / device milliseconds of one kernel
 * kind: 0 base GEMM (forward), 1 base GEMM (dX), 2 rank-r down-projection (H/G),
 * 3 segmented dA/dB reduction, 4 split-reduce / pack / loss, 5 AdamW. */
mlora_status mlora_ctx_set_profiling(mlora_ctx* ctx, int32_t enable);
mlora_status mlora_ctx_profile_read(mlora_ctx* ctx, int32_t kind, int64_t* count, double* total_ms,
                                    int32_t reset);
/* A device interval on `stream`: timer_stop records the end event, waits for it
 * and returns the milliseconds since timer_start (one interval per context). */
mlora_status mlora_ctx_timer_start(mlora_ctx* ctx, void* stream);
mlora_status mlora_ctx_timer_stop(mlora_ctx* ctx, void* stream, double* ms);

/* ---------------------------------------------------------------- accounting
 * Replaces fusim::fused_shape (lora.hpp:63, lora.cpp:72-85).  Integer-exact.
 * `lengths` (host) is the flattened per-group length list; groups do not
 * matter for the result. */
mlora_status mlora_fused_shape_of(const int32_t* lengths, int64_t n, mlora_fused_shape* out);

/* Replaces fusim::count_launches (lora.hpp:97-106, lora.cpp:184-189):
 * mode 0 = PerJob -> (4k, 0), mode 1 = Fused -> (2k, 2).  USAGE if k < 1. */
mlora_status mlora_count_launches(int32_t num_jobs, int32_t mode, int64_t* small_launches,
                                  int64_t* large_launches);

/* ---------------------------------------------------------------- plan
 * The segment layout of one fused batch: which rows belong to which job.
 * Replaces the routing/mask role of fusim::FusedBatch (lora.hpp:65-82) for the
 * kernels.  seg_offsets (host, J+1, non-decreasing, seg[0]=0) partitions the
 * `rows = seg[J]` fused rows; ranks/scales (host, J) give r_j >= 1 and s_j.
 * Builds the device tables (segment offsets, padded rank offsets, per-m-tile
 * LoRA k-block ranges, per-chunk token ranges) with one H2D copy on `stream`.
 * 1 <= num_jobs <= 128 per plan (USAGE otherwise); more jobs than that go to
 * further plans / GPUs (adapter-parallel, see the multi-GPU section). */
mlora_status mlora_plan_create(mlora_ctx* ctx, int32_t num_jobs, const int64_t* seg_offsets,
                               const int32_t* ranks, const float* scales, void* stream,
                               mlora_plan** out);
/* Re-point an existing plan (same jobs, ranks and scales) at the next fused
 * batch's segment layout.  Stream-ordered and non-blocking: the tables go up
 * through pinned staging on `stream`, so kernels already enqueued there still
 * read the previous layout and the host can pack step t+1 while step t runs. */
mlora_status mlora_plan_update(mlora_plan* plan, const int64_t* seg_offsets, void* stream);
mlora_status mlora_plan_destroy(mlora_plan* plan);
int64_t mlora_plan_rows(const mlora_plan* plan);
int32_t mlora_plan_num_jobs(const mlora_plan* plan);
int32_t mlora_plan_rank_padded(const mlora_plan* plan);
/* host, J+1 entries */
mlora_status mlora_plan_rank_offsets(const mlora_plan* plan, int32_t* roff_out);

/* ---------------------------------------------------------------- forward
 * Replaces fusim::fused_forward (lora.hpp:93-95, lora.cpp:160-182):
 *   Y[rows, d] = X[rows, k] W0[d, k]^T + H_cat B_cat^T,  H_cat = s_j X_j A_j^T.
 * Two tcgen05 launches: the rank-r down-projection (H, saved for backward)
 * and the frozen-base GEMM whose LoRA k-blocks accumulate H B^T into the same
 * TMEM tile.  SHAPE if d, k are not positive multiples of 8.
 * X, W0, A_cat, B_cat, Y, H: bf16 device pointers (layouts above). */
mlora_status mlora_linear_fwd(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                              const void* X, const void* W0, const void* A_cat, const void* B_cat,
                              void* Y, void* H, void* stream);

/* As mlora_linear_fwd, and (row_sq != NULL) the forward GEMM's epilogue also
 * writes, per 256-column block nb of Y, row_sq[nb * rows + t] = sum over the
 * block's columns of bf16(Y[t, c])^2 — the layer loss without re-reading Y.
 * row_sq holds mlora_rowsq_blocks(d) * rows floats. */
mlora_status mlora_linear_fwd_ex(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                                 const void* X, const void* W0, const void* A_cat, const void* B_cat,
                                 void* Y, void* H, float* row_sq, void* stream);
int32_t mlora_rowsq_blocks(int32_t d);
/* loss[j] = 1/2 sum over tensors t, blocks and job j's rows of row_sq[t] (fixed order). */
mlora_status mlora_loss_from_rowsq(mlora_ctx* ctx, const mlora_plan* plan, const float* const* row_sq,
                                   const int32_t* d, int32_t num_tensors, float* loss, void* stream);

/* Backward of mlora_linear_fwd (no reference function; pinned by composing
 * the reference primitives):
 *   G_cat = s_j dY_j B_j          (rows x R_pad, bf16 scratch, caller-owned)
 *   dX    = dY W0 + G_cat A_cat   (bf16, skipped when dX == NULL)
 *   dA_cat = G_cat^T X            (fp32, R_pad x k, segmented over job rows)
 *   dB_cat = dY^T H_cat           (fp32, d x R_pad, segmented over job rows) */
mlora_status mlora_linear_bwd(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                              const void* dY, const void* X, const void* H, const void* W0,
                              const void* A_cat, const void* B_cat, void* G, void* dX,
                              float* dA_cat, float* dB_cat, void* stream);

/* ---------------------------------------------------------------- layer-level building blocks
 * The same kernels as mlora_linear_fwd/bwd, exposed per op so a layer issues
 * each HBM-bound op ONCE for all of its projections (grouped launch: one
 * problem per projection, up to 8 per launch) — launch count per layer step is
 * independent of the number of projections as well as of the number of jobs.
 *
 * down_group, forward (backward = 0):  out_i = H_i = s_j in_i A_cat_i^T  (in_i: X_i [rows, width_i],
 *                                      adapter_i: A_cat_i [R_pad, width_i])
 * down_group, backward (backward = 1): out_i = G_i = s_j in_i B_cat_i    (in_i: dY_i [rows, width_i = d_i],
 *                                      adapter_i: B_cat_i [d_i, R_pad]) */
mlora_status mlora_down_group(mlora_ctx* ctx, const mlora_plan* plan, int32_t n, int32_t backward,
                              const int32_t* width, const void* const* in, const void* const* adapter,
                              void* const* out, void* stream);
/* Y = X W0^T + H B_cat^T (CTA-pair tcgen05 GEMM; optional fused row sums, see _ex).
 * H == B_cat == NULL: the plain frozen GEMM Y = X W0^T (e.g. a model's LM head). */
mlora_status mlora_base_fwd(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k, const void* X,
                            const void* W0, const void* H, const void* B_cat, void* Y, float* row_sq,
                            void* stream);
/* dX = dY W0 + G A_cat  (G == A_cat == NULL: dX = dY W0). */
mlora_status mlora_base_dx(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k, const void* dY,
                           const void* W0, const void* G, const void* A_cat, void* dX, void* stream);
/* dA_cat_i = G_i^T X_i and dB_cat_i = dY_i^T H_i for n projections (two grouped launches + at most one
 * grouped fixed-order split reduction). */
mlora_status mlora_grad_group(mlora_ctx* ctx, const mlora_plan* plan, int32_t n, const int32_t* d,
                              const int32_t* k, const void* const* X, const void* const* dY,
                              const void* const* H, const void* const* G, float* const* dA_cat,
                              float* const* dB_cat, void* stream);

/* ---------------------------------------------------------------- adapters
 * Pack per-job reference-layout adapters (device fp32: A_j r_j x k, B_j d x r_j)
 * into the cat layout (fp32 master and bf16 operand copies; either output
 * pointer may be NULL).  RoutingError semantics: a NULL A_j/B_j is ROUTING. */
mlora_status mlora_pack_adapters(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                                 const float* const* A_ptrs, const float* const* B_ptrs,
                                 float* A_cat_f32, float* B_cat_f32, void* A_cat_bf16,
                                 void* B_cat_bf16, void* stream);

/* One fused AdamW step over every adapter tensor of every projection
 * (no reference function; parity unpinned).  Each group is a
 * cat-layout tensor whose job of element (i, c) is given by its rows
 * (layout 0, A_cat: row i in [roff[j], roff[j+1])) or columns (layout 1, B_cat).
 * lr/step are per job (host arrays of J entries: the paper trains jobs with
 * different learning rates); step[j] = 0 marks a job that was
 * not in this fused batch — its p, m, v are left untouched.  Writes the fp32 master and, when
 * p_bf16 != NULL, the bf16 operand copy used by the GEMMs. */
typedef struct mlora_adam_group {
    float* p;
    const float* g;
    float* m;
    float* v;
    void* p_bf16;
    int64_t rows;
    int64_t cols;
    int32_t layout; /* 0: rows by job (A_cat), 1: cols by job (B_cat) */
    int32_t _pad;
} mlora_adam_group;

mlora_status mlora_adam_step(mlora_ctx* ctx, const mlora_plan* plan, const mlora_adam_group* groups,
                             int32_t num_groups, const float* lr, const int32_t* step, float beta1,
                             float beta2, float eps, float weight_decay, void* stream);
/* As mlora_adam_step; loss_gate (device fp32 [J], may be NULL) skips every job
 * whose loss is not finite this step, without a host sync: its p, m, v stay
 * untouched (skip-on-overflow), so a diverged job's NaN gradient never reaches
 * its adapter — which the next step's fused tiles share with the other jobs. */
mlora_status mlora_adam_step_ex(mlora_ctx* ctx, const mlora_plan* plan, const mlora_adam_group* groups,
                                int32_t num_groups, const float* lr, const int32_t* step, float beta1,
                                float beta2, float eps, float weight_decay, const float* loss_gate,
                                void* stream);

/* ---------------------------------------------------------------- fp64 path
 * Device fp64 GEMM with the reference's exact per-element operation order
 * (lora.cpp:19-34: k ascending, a_ik == 0 terms skipped, product and sum
 * rounded separately), so results are bitwise equal to fusim::matmul.
 * C[M,N] = op(A)[M,K] op(B)[K,N]; op(A)(i,k) = transA ? A[k*lda+i] : A[i*lda+k].
 * All pointers device fp64.  Used by the fusim::* C++ façade (fp64 API). */
mlora_status mlora_f64_gemm(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int32_t transA,
                            const double* B, int64_t ldb, int32_t transB, double* C, int64_t ldc,
                            void* stream);
/* c = a + b elementwise (lora.cpp:36-42), device fp64. */
mlora_status mlora_f64_add(int64_t n, const double* a, const double* b, double* c, void* stream);

/* Device fuse — replaces the data / mask half of fusim::fuse (lora.hpp:88,
 * lora.cpp:114-158) for bf16 hidden states that already live in HBM.
 * Sequence i (FusedBatch order: job order, then sequence order) is copied
 * from src[i] (device, lens[i] rows, row stride ld_src[i] elements, or dim
 * when ld_src == NULL) into the fused matrix dst (bf16, dim columns):
 *   padded = 1: the reference layout — every sequence in a max_len slot,
 *               max_len = max lens, the slot's tail rows zero-filled;
 *   padded = 0: packed — real rows back to back.
 * mask (device uint8, may be NULL) gets 1 on copied rows and 0 on pad rows;
 * row_offsets (host, num_seqs + 1, may be NULL) receives each sequence's first
 * row.  USAGE on no sequences / an empty sequence (lora.cpp:115, 131), as the
 * reference.  A pure copy: bit-exact.  Routing and ξ accounting stay on the
 * host (mlora_fused_shape_of). */
mlora_status mlora_fuse_rows(mlora_ctx* ctx, int32_t num_seqs, const void* const* src, const int64_t* ld_src,
                             const int32_t* lens, int64_t dim, int32_t padded, void* dst, uint8_t* mask,
                             int64_t* row_offsets, void* stream);

/* Non-finite guard, between the loss and the backward.  For every job j with a
 * non-finite loss[j] (device fp32 [J]), zero its rows seg[j]..seg[j+1] of each
 * bf16 row-major tensor (rows x cols[t]), normally the backward's dY.  The fused
 * reductions multiply a job's dY rows by the exact zeros the other jobs' columns
 * of H_cat hold (dB = dY^T H), and 0 * inf = NaN: without the guard a job whose
 * activations overflow would poison every co-scheduled job.  The reference
 * computes each sequence separately (lora.cpp:168-181), so this is what keeps
 * the jobs independent, as it requires.  The diverged job keeps its non-finite
 * loss, which is what detect_stop (progress.cpp:90-124) consumes; its gradient
 * for this step is zero (skip-on-overflow, as in loss-scaled mixed precision).
 * Pass every tensor the backward reads (dY, the saved H_cat, each projection's
 * input X; up to 32): a NaN left in any of them meets the structural zeros of
 * the other jobs' columns.  One launch; in the all-finite case it reads J floats. */
mlora_status mlora_zero_nonfinite_rows(mlora_ctx* ctx, const mlora_plan* plan, const float* loss,
                                       void* const* tensors, const int32_t* cols, int32_t num_tensors,
                                       void* stream);

/* ---------------------------------------------------------------- model kernels (K4, K5)
 * No reference counterpart (the reference model is analytic): parity unpinned,
 * checked against fp64 restatements.  All device pointers; deterministic.
 *
 * Padding-masked cross-entropy over the fused batch (C4: V = 65024):
 *   row_loss[t] = logsumexp(logits[t]) - logits[t, labels[t]]   (0 where mask[t] == 0)
 *   loss[j]     = mean of row_loss over job j's real rows (seg_dev: device J+1 offsets)
 *   dlogits[t]  = (softmax(logits[t]) - onehot(labels[t])) / n_j  (0 on pad rows), optional
 * mask may be NULL (every row real).  row_loss: rows floats, inv_count: J floats (scratch). */
mlora_status mlora_masked_ce(int32_t num_jobs, const int32_t* seg_dev, int64_t rows, int32_t V, const void* logits,
                             const int32_t* labels, const uint8_t* mask, float* row_loss, float* loss,
                             float* inv_count, void* dlogits, void* stream);
/* RMSNorm: y = x * rstd * w, rstd = 1 / sqrt(mean(x^2) + eps) (bf16 x, w, y; fp32 rstd). */
mlora_status mlora_rmsnorm_fwd(int64_t rows, int32_t h, const void* x, const void* w, float eps, void* y,
                               float* rstd, void* stream);
/* dx = rstd (g - xhat mean(g xhat)), g = dy w; dw = sum_rows dy xhat (fp32, fixed-order
 * reduction through workspace[ceil(rows / rows_per_block) * h]). */
mlora_status mlora_rmsnorm_bwd(int64_t rows, int32_t h, const void* dy, const void* x, const void* w,
                               const float* rstd, void* dx, float* dw, float* workspace, int32_t rows_per_block,
                               void* stream);
/* Rotary embedding on [rows, heads, head_dim] bf16 (rotate-half pairing), angle
 * pos[row] * base^(-2i/head_dim); inverse = 1 applies the transpose (backward). */
mlora_status mlora_rope(int64_t rows, int32_t heads, int32_t head_dim, const void* x, void* y, const int32_t* pos,
                        float base, int32_t inverse, void* stream);

/* Per-job synthetic layer loss L_j = 1/2 sum_p sum_{t in job j} ||Y_p[t]||^2 over
 * `num_tensors` bf16 tensors Y[p] (rows x cols[p]); loss: device fp32 [J].
 * Deterministic (fixed-order two-level reduction).  Unfused form of the loss the
 * trainer step takes from the forward GEMM epilogues (mlora_linear_fwd_ex +
 * mlora_loss_from_rowsq); the reference's only runtime loss consumer is
 * detect_stop (progress.cpp:90-124). */
mlora_status mlora_segment_sumsq_loss(mlora_ctx* ctx, const mlora_plan* plan, const void* const* Y,
                                      const int32_t* cols, int32_t num_tensors, float* loss, void* stream);

/* ---------------------------------------------------------------- decoder-layer kernels (configs C1, C4)
 * The kernels around the LoRA linears that a whole LLaMA / ChatGLM2-shaped
 * decoder needs to be fine-tuned on the fused batch end to end
 * (paper_2312_02515_b200/model.py).  No reference counterpart (the reference
 * has no model: SURVEY.md App. A), parity unpinned: checked against a PyTorch
 * fp32 restatement of the same model.  Deterministic; bf16 tensors, fp32 math.
 *
 * Frozen token embedding: x[t] = E[tokens[t]] (E bf16 [V, h], h % 8 == 0;
 * tokens device int32, caller-validated to [0, V)). */
mlora_status mlora_embed(int64_t rows, int32_t h, int32_t V, const int32_t* tokens, const void* E, void* x,
                         void* stream);
/* Residual add fused into RMSNorm: x_out = bf16(x + delta) (skipped when delta == NULL),
 * y = x_out * rstd * w, rstd = 1 / sqrt(mean(x_out^2) + eps).  x_out must not alias x. */
mlora_status mlora_add_rmsnorm(int64_t rows, int32_t h, const void* x, const void* delta, const void* w, float eps,
                               void* x_out, void* y, float* rstd, void* stream);
/* RMSNorm backward for a frozen weight, summing the n_dy <= 4 gradients that
 * reach y (e.g. the dX of q, k, v) and adding the residual gradient dres
 * (may be NULL): dx = dres + rstd (g - xhat mean(g xhat)), g = w sum_i dy_i. */
mlora_status mlora_rmsnorm_bwd_sum(int64_t rows, int32_t h, int32_t n_dy, const void* const* dy, const void* dres,
                                   const void* x, const void* w, const float* rstd, void* dx, void* stream);
/* SwiGLU: out[t, c] = silu(gate[t, c]) * up[t, c] (out is rows x f, contiguous; gate / up
 * are column slices with row strides ld_*, e.g. the two halves of ChatGLM2's h_to_4h). */
mlora_status mlora_swiglu_fwd(int64_t rows, int32_t f, const void* gate, int64_t ld_gate, const void* up,
                              int64_t ld_up, void* out, void* stream);
mlora_status mlora_swiglu_bwd(int64_t rows, int32_t f, const void* gate, int64_t ld_gate, const void* up,
                              int64_t ld_up, const void* dout, void* dgate, int64_t ld_dgate, void* dup,
                              int64_t ld_dup, void* stream);

/* Causal attention over the fused row layout.  Sequence s owns rows
 * seq_offsets[s] .. seq_offsets[s+1] (device int32, S + 1 entries); its real
 * tokens are the first seq_lens[s] rows (device int32 [S]; NULL: all), the
 * rest are padding (output 0, no gradient).  Grouped-query: query head h reads
 * K/V head h / (heads / kv_heads) (ChatGLM2 multi-query: kv_heads = 2).
 * head_dim 64 or 128.  RoPE (rotate-half, the angle of mlora_rope with
 * pos = row - seq start) is applied to Q and K inside the kernel when
 * rope_base > 0.  lse: fp32 [heads, rows] (natural log), saved for backward.
 * flags & MLORA_ATTN_PREROTATED: q and k were already rotated by
 * mlora_attn_rope (saved once per step, so no tile re-rotates them); the
 * backward still returns dq / dk with respect to the UNROTATED q and k. */
#define MLORA_ATTN_PREROTATED 1
typedef struct mlora_attn_desc {
    const int32_t* seq_offsets;
    const int32_t* seq_lens;
    int64_t rows;
    int32_t num_seqs;
    int32_t max_len;  /* >= the longest slot (host-side bound for the grid) */
    int32_t heads;
    int32_t kv_heads;
    int32_t head_dim;
    float rope_base;
    float softmax_scale;
    int32_t flags;
} mlora_attn_desc;

/* q: rows x ldq (head h at column h * head_dim), k / v: rows x ld (K/V head g at g * head_dim). */
mlora_status mlora_attn_fwd(const mlora_attn_desc* desc, const void* q, int64_t ldq, const void* k, int64_t ldk,
                            const void* v, int64_t ldv, void* o, int64_t ldo, float* lse, void* stream);
/* dst = RoPE(src) for n_heads heads per row (pos = row - sequence start; padding rows -> 0). */
mlora_status mlora_attn_rope(const mlora_attn_desc* desc, const void* src, int64_t ld_src, int32_t n_heads, void* dst,
                             int64_t ld_dst, void* stream);
/* dq, dk, dv (bf16, written, same column layout as q, k, v); dsum: fp32 [heads, rows] scratch. */
mlora_status mlora_attn_bwd(const mlora_attn_desc* desc, const void* q, int64_t ldq, const void* k, int64_t ldk,
                            const void* v, int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                            const float* lse, float* dsum, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                            int64_t lddv, void* stream);

/* ---------------------------------------------------------------- one fused layer step (the trainer hook)
 * The whole BatchFusion training iteration of one transformer layer's LoRA'd
 * projections, as ONE call: the runtime counterpart of the reference
 * simulator's fused iteration (/root/reference/proj/src/sim.cpp:163-191, whose
 * duration the reference charges analytically at :177-179).  Per call, on
 * `stream`, in this order (launch count independent of the number of jobs):
 *   forward, in dependency waves: every projection whose input is ready gets
 *     its rank-r down-projection in one grouped launch (projections sharing an
 *     input go through the shared-input kernel), then its base GEMM
 *     Y = X W0^T + H B_cat^T with the fused per-row sum of bf16(Y)^2;
 *   loss[j] = 1/2 sum_p ||Y_p[rows of j]||^2 (so dL/dY_p = Y_p, input detached)
 *     fused with the non-finite guard (as mlora_zero_nonfinite_rows, over every
 *     tensor the backward reads: each Y, H and input — a diverged job's rows, x
 *     included): one row-sum launch + one loss / guard launch;
 *   backward: G = s dY B_cat for every projection (one grouped launch), dX per
 *     projection (reverse order), dA / dB for every projection (grouped);
 *   and, in mlora_layer_step, one AdamW over all 2n adapter tensors (per-job lr,
 *     step[j] = 0 leaves job j untouched, loss-gated: a job whose loss is not
 *     finite keeps p, m, v).
 * Every tensor is caller-owned device memory, described once at creation (the
 * layer object holds only the descriptors); rows = mlora_plan_rows(plan), set
 * by mlora_plan_update before the call, must not exceed `capacity`. */
typedef struct mlora_layer_proj {
    int32_t d;          /* output width (rows of W0) */
    int32_t k;          /* input width (cols of W0) */
    int32_t src;        /* -1: the layer input x (rows x k); p >= 0: projection p's Y (p != self, acyclic) */
    int32_t src_col0;   /* first column of the source's Y that this input starts at */
    const void* W0;     /* bf16 d x k, frozen */
    float* A;           /* fp32 master A_cat, R_pad x k */
    float* B;           /* fp32 master B_cat, d x R_pad */
    float* mA;          /* AdamW moments, same shapes */
    float* vA;
    float* mB;
    float* vB;
    void* A_bf16;       /* bf16 operand copies (written by AdamW) */
    void* B_bf16;
    float* dA;          /* fp32 gradients */
    float* dB;
    void* Y;            /* bf16 capacity x d */
    void* H;            /* bf16 capacity x R_pad (saved s X A^T) */
    void* G;            /* bf16 capacity x R_pad (s dY B) */
    void* dX;           /* bf16 capacity x k */
    float* row_sq;      /* mlora_rowsq_blocks(d) * capacity floats */
    void* in_scratch;   /* bf16 capacity x k; needed only when the input is a column slice of a
                           wider source (src_col0 != 0 or the source's d != k), else NULL */
} mlora_layer_proj;

typedef struct mlora_adam_hparams {
    float beta1, beta2, eps, weight_decay;
} mlora_adam_hparams;

typedef struct mlora_layer mlora_layer;
/* USAGE on a bad source index / cycle / null tensor, SHAPE on widths that do
 * not chain (k != the source's d without a scratch buffer); at most 16 projections. */
mlora_status mlora_layer_create(mlora_ctx* ctx, mlora_plan* plan, int32_t n, const mlora_layer_proj* proj,
                                int64_t capacity, mlora_layer** out);
mlora_status mlora_layer_destroy(mlora_layer* layer);
/* forward + loss + guard + backward (no optimizer); x: bf16 rows x proj[first x-fed].k; loss: device fp32 [J]. */
mlora_status mlora_layer_forward_backward(mlora_layer* layer, void* x, float* loss, void* stream);
/* forward_backward + AdamW (lr, step: host arrays of J entries; hp NULL: 0.9, 0.999, 1e-8, 0). */
mlora_status mlora_layer_step(mlora_layer* layer, void* x, const float* lr, const int32_t* step,
                              const mlora_adam_hparams* hp, float* loss, void* stream);
/* mlora_layer_step bracketed by CUDA events on `stream`, then synchronised: returns the step's
 * device milliseconds and copies the per-job losses to loss_host (J floats) — the measured
 * duration an executor charges in place of the reference's analytic IterationTimeModel. */
mlora_status mlora_layer_step_timed(mlora_layer* layer, void* x, const float* lr, const int32_t* step,
                                    const mlora_adam_hparams* hp, float* loss, float* loss_host,
                                    double* device_ms, void* stream);

/* ---------------------------------------------------------------- device memory / init helpers
 * For hosts that do not link the CUDA runtime themselves (the C++ façade, C
 * programs): everything goes through this library's one runtime instance.
 * kind: 0 host->device, 1 device->host, 2 device->device. */
mlora_status mlora_malloc(mlora_ctx* ctx, size_t bytes, void** out);
mlora_status mlora_free(mlora_ctx* ctx, void* ptr);
mlora_status mlora_memcpy(mlora_ctx* ctx, void* dst, const void* src, size_t bytes, int32_t kind, void* stream);
mlora_status mlora_memset(mlora_ctx* ctx, void* dst, int32_t value, size_t bytes, void* stream);
mlora_status mlora_stream_sync(mlora_ctx* ctx, void* stream);
/* Free / total device memory of the context's GPU (cudaMemGetInfo): the live
 * warm-up probes of the memory model (memory_model.cpp:241-259 plans them). */
mlora_status mlora_mem_info(mlora_ctx* ctx, size_t* free_bytes, size_t* total_bytes);
/* Deterministic counter-based uniform fill: dst[i] = lo + (hi - lo) * u(seed, i),
 * u in [0, 1) from a 64-bit mix of (seed, i) — the same values on any device,
 * launch shape or host language (used to initialise synthetic weights and data
 * identically from Python and C++).  dtype: 0 fp32, 1 bf16 (round to nearest). */
mlora_status mlora_fill_uniform(void* dst, int64_t n, int32_t dtype, uint64_t seed, float lo, float hi,
                                void* stream);

/* ---------------------------------------------------------------- multi-GPU
 * Adapter-parallel: jobs are partitioned across GPUs (one process and one
 * context per GPU); the frozen base weights are replicated ONCE at start-up and
 * the steady-state step has no collective.  The reference has no multi-GPU
 * runtime (its simulator models one device, sim.hpp:16-31; its batches are
 * routed per job, lora.cpp:165-167, which is what makes the job partition
 * exact).  NCCL is loaded at first use (dlopen "libnccl.so.2", override with
 * MLORA_NCCL_LIBRARY); without it these calls return MLORA_CUDA and every other
 * entry point is unaffected.
 *
 * Start-up: rank 0 calls mlora_comm_unique_id and ships the id bytes to the
 * other ranks over any out-of-band channel; every rank then calls
 * mlora_comm_create with its own context (the communicator is bound to the
 * context's device). */
typedef struct mlora_comm mlora_comm;
int32_t mlora_comm_id_bytes(void); /* 128 */
mlora_status mlora_comm_nccl_version(int32_t* version /* host */);
mlora_status mlora_comm_unique_id(uint8_t* id /* host, mlora_comm_id_bytes() bytes */);
mlora_status mlora_comm_create(mlora_ctx* ctx, const uint8_t* id /* host */, int32_t nranks, int32_t rank,
                               mlora_comm** out);
mlora_status mlora_comm_destroy(mlora_comm* comm);
int32_t mlora_comm_rank(const mlora_comm* comm);
int32_t mlora_comm_size(const mlora_comm* comm);
/* Replicate n device buffers (e.g. every W0 of the model) from `root` to all
 * ranks in place, as ONE NCCL group (pipelined over NVLink/NVSwitch).
 * Stream-ordered on `stream`; USAGE on a bad root / null buffer / negative size. */
mlora_status mlora_broadcast_base(mlora_comm* comm, int32_t n, void* const* ptrs, const int64_t* bytes,
                                  int32_t root, void* stream);
/* In-place fp32 sum over ranks (per-job metric aggregation; not on the step path). */
mlora_status mlora_comm_sum_f32(mlora_comm* comm, float* buf, int64_t count, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MLORA_H_ */
