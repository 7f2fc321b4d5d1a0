/*
 * train_step.c — a plain C11 host program driving the C ABI (include/mlora.h)
 * through one fused multi-LoRA training step, with no Python or torch anywhere:
 *
 *   plan (2 jobs, ranks 8 and 16, scales 2 and 0.5, uneven segments)
 *   -> mlora_pack_adapters    reference-layout A_j, B_j  -> cat layout (fp32 + bf16)
 *   -> mlora_linear_fwd       Y = X W0^T + s_j (X A_j^T) B_j^T      (lora.cpp:160-182)
 *   -> mlora_linear_bwd       dX, dA_j, dB_j for dY = Y
 *   -> mlora_adam_step        per-job lr
 *
 * Every result is checked against an fp64 CPU computation in this file on the
 * same bf16-rounded inputs (rel-L2 per job <= 1e-2; AdamW to fp32 rounding).
 * It is what a C or C++ host runtime (or a cgo / JNI stub) would write.
 * Exit status 0 and a final "OK" line on success.
 *
 * Build: gcc -std=c11 -O2 -I include train_step.c -L <pkg> -lmlora -L <cuda>/lib64 -lcudart -lm
 */
#include <cuda_runtime_api.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "mlora.h"

#define J 2
#define M 96   /* fused rows: job 0 rows [0, 40), job 1 rows [40, 96) */
#define K 64   /* in features  */
#define D 128  /* out features */

static int failures = 0;

#define CHECK_ML(call)                                                                       \
    do {                                                                                     \
        mlora_status st_ = (call);                                                           \
        if (st_ != MLORA_OK) {                                                               \
            fprintf(stderr, "%s:%d %s -> %s: %s\n", __FILE__, __LINE__, #call,               \
                    mlora_status_string(st_), mlora_last_error(ctx));                        \
            return 1;                                                                        \
        }                                                                                    \
    } while (0)
#define CHECK_CUDA(call)                                                                     \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess) {                                                             \
            fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #call, cudaGetErrorString(e_)); \
            return 1;                                                                        \
        }                                                                                    \
    } while (0)

/* bf16 <-> fp32, round to nearest even (finite inputs only) */
static uint16_t to_bf16(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return (uint16_t)(u >> 16);
}
static float from_bf16(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

static uint64_t rng_state = 0x2312025150ULL;
static float urand(void) { /* U(-1, 1), xorshift64* */
    rng_state ^= rng_state >> 12;
    rng_state ^= rng_state << 25;
    rng_state ^= rng_state >> 27;
    uint64_t r = rng_state * 0x2545F4914F6CDD1DULL;
    return (float)((r >> 11) * (1.0 / 9007199254740992.0)) * 2.f - 1.f;
}

static void expect_close(const char* what, int job, const double* got, const double* want, int n, double tol) {
    double num = 0, den = 0;
    for (int i = 0; i < n; ++i) {
        num += (got[i] - want[i]) * (got[i] - want[i]);
        den += want[i] * want[i];
    }
    const double rel = sqrt(num / (den > 0 ? den : 1));
    const int ok = rel <= tol && isfinite(rel);
    printf("%-6s job %d: rel-L2 %.2e (tol %.0e) %s\n", what, job, rel, tol, ok ? "ok" : "FAIL");
    if (!ok) ++failures;
}

int main(void) {
    mlora_ctx* ctx = NULL;
    CHECK_ML(mlora_ctx_create(0, &ctx));
    const int64_t seg[J + 1] = {0, 40, M};
    const int32_t rank[J] = {8, 16};
    const float scale[J] = {2.0f, 0.5f};
    mlora_plan* plan = NULL;
    CHECK_ML(mlora_plan_create(ctx, J, seg, rank, scale, NULL, &plan));
    const int R = mlora_plan_rank_padded(plan);
    int32_t roff[J + 1];
    CHECK_ML(mlora_plan_rank_offsets(plan, roff));

    /* ---- host data: bf16 X, W0; fp32 adapters in the reference layout (A_j r x K, B_j D x r) */
    static uint16_t hX[M * K], hW[D * K], hY[M * D], hH[M * 64], hdX[M * K];
    static float hA[J][16 * K], hB[J][D * 16];
    for (int i = 0; i < M * K; ++i) hX[i] = to_bf16(urand());
    for (int i = 0; i < D * K; ++i) hW[i] = to_bf16(urand() / 8.f);
    for (int j = 0; j < J; ++j) {
        for (int i = 0; i < rank[j] * K; ++i) hA[j][i] = urand() / 8.f;
        for (int i = 0; i < D * rank[j]; ++i) hB[j][i] = urand() / 4.f;
    }

    void *dX_, *dW, *dY, *dH, *dG, *ddX, *dAcat16, *dBcat16;
    float *dA[J], *dB[J], *dAcat, *dBcat, *ddA, *ddB, *mA, *vA, *mB, *vB;
    CHECK_CUDA(cudaMalloc(&dX_, sizeof hX));
    CHECK_CUDA(cudaMalloc(&dW, sizeof hW));
    CHECK_CUDA(cudaMalloc(&dY, sizeof hY));
    CHECK_CUDA(cudaMalloc(&dH, (size_t)M * R * 2));
    CHECK_CUDA(cudaMalloc(&dG, (size_t)M * R * 2));
    CHECK_CUDA(cudaMalloc(&ddX, sizeof hdX));
    CHECK_CUDA(cudaMalloc(&dAcat16, (size_t)R * K * 2));
    CHECK_CUDA(cudaMalloc(&dBcat16, (size_t)D * R * 2));
    CHECK_CUDA(cudaMalloc((void**)&dAcat, (size_t)R * K * 4));
    CHECK_CUDA(cudaMalloc((void**)&dBcat, (size_t)D * R * 4));
    CHECK_CUDA(cudaMalloc((void**)&ddA, (size_t)R * K * 4));
    CHECK_CUDA(cudaMalloc((void**)&ddB, (size_t)D * R * 4));
    CHECK_CUDA(cudaMalloc((void**)&mA, (size_t)R * K * 4));
    CHECK_CUDA(cudaMalloc((void**)&vA, (size_t)R * K * 4));
    CHECK_CUDA(cudaMalloc((void**)&mB, (size_t)D * R * 4));
    CHECK_CUDA(cudaMalloc((void**)&vB, (size_t)D * R * 4));
    CHECK_CUDA(cudaMemset(mA, 0, (size_t)R * K * 4));
    CHECK_CUDA(cudaMemset(vA, 0, (size_t)R * K * 4));
    CHECK_CUDA(cudaMemset(mB, 0, (size_t)D * R * 4));
    CHECK_CUDA(cudaMemset(vB, 0, (size_t)D * R * 4));
    for (int j = 0; j < J; ++j) {
        CHECK_CUDA(cudaMalloc((void**)&dA[j], sizeof hA[j]));
        CHECK_CUDA(cudaMalloc((void**)&dB[j], sizeof hB[j]));
        CHECK_CUDA(cudaMemcpy(dA[j], hA[j], sizeof hA[j], cudaMemcpyHostToDevice));
        CHECK_CUDA(cudaMemcpy(dB[j], hB[j], sizeof hB[j], cudaMemcpyHostToDevice));
    }
    CHECK_CUDA(cudaMemcpy(dX_, hX, sizeof hX, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(dW, hW, sizeof hW, cudaMemcpyHostToDevice));

    /* ---- the step, all on the default stream */
    const float* Ap[J] = {dA[0], dA[1]};
    const float* Bp[J] = {dB[0], dB[1]};
    CHECK_ML(mlora_pack_adapters(ctx, plan, D, K, Ap, Bp, dAcat, dBcat, dAcat16, dBcat16, NULL));
    CHECK_ML(mlora_linear_fwd(ctx, plan, D, K, dX_, dW, dAcat16, dBcat16, dY, dH, NULL));
    CHECK_ML(mlora_linear_bwd(ctx, plan, D, K, /*dY=*/dY, dX_, dH, dW, dAcat16, dBcat16, dG, ddX, ddA, ddB, NULL));
    static float gA[64 * K], gB[D * 64], pA0[64 * K], pB0[D * 64];
    CHECK_CUDA(cudaDeviceSynchronize());
    CHECK_CUDA(cudaMemcpy(gA, ddA, (size_t)R * K * 4, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(gB, ddB, (size_t)D * R * 4, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(pA0, dAcat, (size_t)R * K * 4, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(pB0, dBcat, (size_t)D * R * 4, cudaMemcpyDeviceToHost));
    const float lr[J] = {1e-3f, 5e-3f};
    const int32_t step[J] = {1, 1};
    mlora_adam_group groups[2] = {{dAcat, ddA, mA, vA, dAcat16, R, K, 0, 0}, {dBcat, ddB, mB, vB, dBcat16, D, R, 1, 0}};
    CHECK_ML(mlora_adam_step(ctx, plan, groups, 2, lr, step, 0.9f, 0.999f, 1e-8f, 0.0f, NULL));
    static float pA1[64 * K], pB1[D * 64];
    CHECK_CUDA(cudaDeviceSynchronize());
    CHECK_CUDA(cudaMemcpy(hY, dY, sizeof hY, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(hH, dH, (size_t)M * R * 2, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(hdX, ddX, sizeof hdX, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(pA1, dAcat, (size_t)R * K * 4, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(pB1, dBcat, (size_t)D * R * 4, cudaMemcpyDeviceToHost));

    /* ---- fp64 CPU check on the same bf16 operands */
    static double Ab[J][16 * K], Bb[J][D * 16], y_ref[M * D], y_got[M * D], h[M * 16], g[M * 16];
    static double dx_ref[M * K], dx_got[M * K], da_ref[16 * K], da_got[16 * K], db_ref[D * 16], db_got[D * 16];
    for (int j = 0; j < J; ++j) {
        for (int i = 0; i < rank[j] * K; ++i) Ab[j][i] = from_bf16(to_bf16(hA[j][i]));
        for (int i = 0; i < D * rank[j]; ++i) Bb[j][i] = from_bf16(to_bf16(hB[j][i]));
    }
    for (int j = 0; j < J; ++j) {
        const int r = rank[j], t0 = (int)seg[j], t1 = (int)seg[j + 1], n = t1 - t0;
        /* forward: h = s X A^T; y = X W0^T + h B^T */
        for (int t = t0; t < t1; ++t)
            for (int c = 0; c < r; ++c) {
                double acc = 0;
                for (int q = 0; q < K; ++q) acc += from_bf16(hX[t * K + q]) * Ab[j][c * K + q];
                h[(t - t0) * r + c] = scale[j] * acc;
            }
        for (int t = t0; t < t1; ++t)
            for (int o = 0; o < D; ++o) {
                double acc = 0;
                for (int q = 0; q < K; ++q) acc += from_bf16(hX[t * K + q]) * from_bf16(hW[o * K + q]);
                for (int c = 0; c < r; ++c) acc += h[(t - t0) * r + c] * Bb[j][o * r + c];
                y_ref[(t - t0) * D + o] = acc;
                y_got[(t - t0) * D + o] = from_bf16(hY[t * D + o]);
            }
        expect_close("Y", j, y_got, y_ref, n * D, 1e-2);
        /* backward with dY = the device's Y (bf16), H = the device's saved H */
        for (int t = t0; t < t1; ++t)
            for (int c = 0; c < r; ++c) {
                double acc = 0;
                for (int o = 0; o < D; ++o) acc += from_bf16(hY[t * D + o]) * Bb[j][o * r + c];
                g[(t - t0) * r + c] = scale[j] * acc;
            }
        for (int t = t0; t < t1; ++t)
            for (int q = 0; q < K; ++q) {
                double acc = 0;
                for (int o = 0; o < D; ++o) acc += from_bf16(hY[t * D + o]) * from_bf16(hW[o * K + q]);
                for (int c = 0; c < r; ++c) acc += g[(t - t0) * r + c] * Ab[j][c * K + q];
                dx_ref[(t - t0) * K + q] = acc;
                dx_got[(t - t0) * K + q] = from_bf16(hdX[t * K + q]);
            }
        expect_close("dX", j, dx_got, dx_ref, n * K, 1e-2);
        for (int c = 0; c < r; ++c)
            for (int q = 0; q < K; ++q) {
                double acc = 0;
                for (int t = t0; t < t1; ++t) acc += g[(t - t0) * r + c] * from_bf16(hX[t * K + q]);
                da_ref[c * K + q] = acc;
                da_got[c * K + q] = gA[(roff[j] + c) * K + q];
            }
        expect_close("dA", j, da_got, da_ref, r * K, 1e-2);
        for (int o = 0; o < D; ++o)
            for (int c = 0; c < r; ++c) {
                double acc = 0;
                for (int t = t0; t < t1; ++t) acc += from_bf16(hY[t * D + o]) * from_bf16(hH[t * R + roff[j] + c]);
                db_ref[o * r + c] = acc;
                db_got[o * r + c] = gB[o * R + roff[j] + c];
            }
        expect_close("dB", j, db_got, db_ref, D * r, 1e-2);
    }
    /* AdamW step 1 (m = (1-b1) g, v = (1-b2) g^2, bias-corrected), from the device's own gradients */
    double worst = 0;
    for (int i = 0; i < R * K + D * R; ++i) {
        const int isA = i < R * K;
        const int e = isA ? i : i - R * K;
        const int col = isA ? e / K : e % R; /* rank column of the element */
        int j = 0;
        while (j + 1 < J && roff[j + 1] <= col) ++j;
        const float gr = isA ? gA[e] : gB[e];
        const float p0 = isA ? pA0[e] : pB0[e];
        const float p1 = isA ? pA1[e] : pB1[e];
        const float m = (1.f - 0.9f) * gr, v = (1.f - 0.999f) * gr * gr;
        const float mh = m / (1.f - 0.9f), vh = v / (1.f - 0.999f);
        const float want = p0 - lr[j] * (mh / (sqrtf(vh) + 1e-8f));
        const double err = fabs((double)p1 - want) / (fabs(want) + 1e-6);
        if (err > worst) worst = err;
    }
    printf("AdamW  max rel err %.2e %s\n", worst, worst <= 1e-5 ? "ok" : "FAIL");
    if (worst > 1e-5) ++failures;

    /* errors come back as status codes, never exceptions or aborts */
    if (mlora_linear_fwd(ctx, plan, D, 60, dX_, dW, dAcat16, dBcat16, dY, dH, NULL) != MLORA_SHAPE) {
        printf("expected MLORA_SHAPE for k = 60\n");
        ++failures;
    }
    mlora_plan_destroy(plan);
    mlora_ctx_destroy(ctx);
    printf(failures ? "FAILED (%d)\n" : "OK\n", failures);
    return failures ? 1 : 0;
}
