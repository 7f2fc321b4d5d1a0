// mlora_aux.cuh — the HBM-bound helpers around the tcgen05 GEMMs:
//   * split-partial reduction of the segmented dA/dB reductions,
//   * packing of per-job reference-layout adapters into the cat layout,
//   * one fused AdamW step over every adapter tensor with per-job lr/step.
// All are grid-stride, float4-vectorised streaming kernels; their roofline is
// HBM bandwidth (bytes per element stated next to each kernel).
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

namespace mlora {

constexpr int kMaxJobs = 128;
constexpr int kMaxAdamGroups = 32;

// out[i] = sum_s part[s * stride + i]   (fixed order: deterministic)
// bytes/elem = 4 * nsplit (read) + 4 (write)
__global__ void reduce_splits_kernel(const float4* __restrict__ part, float4* __restrict__ out,
                                     long long n4, long long stride4, int nsplit) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
         i += (long long)gridDim.x * blockDim.x) {
        float4 a = part[i];
        for (int s = 1; s < nsplit; ++s) {
            const float4 b = part[s * stride4 + i];
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        out[i] = a;
    }
}

// Grouped version: several gradients' split partials in one launch.
// part_i = [nsplit][n4_i] float4; out_i[e] = sum_s part_i[s][e] (fixed order).
struct ReduceGroupArgs {
    struct Item {
        const float4* part;
        float4* out;
        long long n4;
        long long start4;  // first element of this item in the flattened index space
    } item[8];
    int n;
    int nsplit;
    long long total4;
};

__global__ void reduce_splits_group_kernel(const __grid_constant__ ReduceGroupArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.total4;
         i += (long long)gridDim.x * blockDim.x) {
        int g = 0;
        while (g + 1 < a.n && a.item[g + 1].start4 <= i) ++g;
        const ReduceGroupArgs::Item& it = a.item[g];
        const long long e = i - it.start4;
        float4 acc = it.part[e];
        for (int s = 1; s < a.nsplit; ++s) {
            const float4 b = it.part[s * it.n4 + e];
            acc.x += b.x; acc.y += b.y; acc.z += b.z; acc.w += b.w;
        }
        it.out[e] = acc;
    }
}

struct PackArgs {
    const float* A[kMaxJobs];
    const float* B[kMaxJobs];
    int roff[kMaxJobs + 1];
    int rank[kMaxJobs];
    int J, d, k, R_pad;
    float* A_f32;
    float* B_f32;
    __nv_bfloat16* A_bf16;
    __nv_bfloat16* B_bf16;
};

__device__ __forceinline__ int job_of_col(const int* roff, int J, int c) {
    int lo = 0, hi = J - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (roff[mid] <= c) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// A_cat (R_pad x k) then B_cat (d x R_pad), one element per thread-iteration.
__global__ void pack_adapters_kernel(const __grid_constant__ PackArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const long long nA = (long long)a.R_pad * a.k;
    const long long nB = (long long)a.d * a.R_pad;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nA + nB;
         e += (long long)gridDim.x * blockDim.x) {
        float val;
        if (e < nA) {
            const int i = static_cast<int>(e / a.k);
            const int c = static_cast<int>(e % a.k);
            const int j = job_of_col(a.roff, a.J, i);
            const int li = i - a.roff[j];
            val = li < a.rank[j] ? a.A[j][(long long)li * a.k + c] : 0.f;
            if (a.A_f32) a.A_f32[e] = val;
            if (a.A_bf16) a.A_bf16[e] = __float2bfloat16_rn(val);
        } else {
            const long long f = e - nA;
            const int row = static_cast<int>(f / a.R_pad);
            const int c = static_cast<int>(f % a.R_pad);
            const int j = job_of_col(a.roff, a.J, c);
            const int lc = c - a.roff[j];
            val = lc < a.rank[j] ? a.B[j][(long long)row * a.rank[j] + lc] : 0.f;
            if (a.B_f32) a.B_f32[f] = val;
            if (a.B_bf16) a.B_bf16[f] = __float2bfloat16_rn(val);
        }
    }
}

struct AdamGroupDev {
    float* p;
    const float* g;
    float* m;
    float* v;
    __nv_bfloat16* pb;
    long long rows, cols;
    long long start4;  // first float4 index of this group in the flattened stream
    int layout;
};

struct AdamArgs {
    AdamGroupDev grp[kMaxAdamGroups];
    int ngroups;
    long long total4;
    int roff[kMaxJobs + 1];
    int J;
    float lr[kMaxJobs];
    float bc1[kMaxJobs];   // 1 / (1 - beta1^t_j); 0: job absent this step
    float bc2[kMaxJobs];   // 1 / (1 - beta2^t_j)
    float beta1, beta2, eps, wd;
    const float* loss_gate;  // device [J] or NULL: a job whose loss is not finite is skipped
};

// AdamW over all groups.  bytes/param: read p,g,m,v (16) + write p,m,v (12)
// (+2 for the bf16 operand copy) = 30 B.
__global__ void adam_kernel(const __grid_constant__ AdamArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    for (long long i4 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i4 < a.total4;
         i4 += (long long)gridDim.x * blockDim.x) {
        int gi = 0;
        while (gi + 1 < a.ngroups && a.grp[gi + 1].start4 <= i4) ++gi;
        const AdamGroupDev& G = a.grp[gi];
        // element index within the group (< 2^31): 32-bit index arithmetic
        const int e = static_cast<int>(i4 - G.start4) * 4;
        const int cols = static_cast<int>(G.cols);
        const int row = e / cols;
        const int col = e - row * cols;
        const int j = job_of_col(a.roff, a.J, G.layout == 0 ? row : col);
        const float lr = a.lr[j], ibc1 = a.bc1[j], ibc2 = a.bc2[j];
        if (ibc1 == 0.f) continue;  // step 0: job not in this fused batch -> p, m, v untouched
        if (a.loss_gate && !isfinite(__ldg(a.loss_gate + j))) continue;  // skip-on-overflow (diverged job)
        float4 p = reinterpret_cast<float4*>(G.p)[e / 4];
        const float4 g = reinterpret_cast<const float4*>(G.g)[e / 4];
        float4 m = reinterpret_cast<float4*>(G.m)[e / 4];
        float4 v = reinterpret_cast<float4*>(G.v)[e / 4];
        float* pp = &p.x; const float* gg = &g.x; float* mm = &m.x; float* vv = &v.x;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            mm[u] = a.beta1 * mm[u] + (1.f - a.beta1) * gg[u];
            vv[u] = a.beta2 * vv[u] + (1.f - a.beta2) * gg[u] * gg[u];
            const float mh = mm[u] * ibc1;  // bias corrections as reciprocals (host, per job)
            const float vh = vv[u] * ibc2;
            pp[u] -= lr * (mh / (sqrtf(vh) + a.eps) + a.wd * pp[u]);
        }
        reinterpret_cast<float4*>(G.p)[e / 4] = p;
        reinterpret_cast<float4*>(G.m)[e / 4] = m;
        reinterpret_cast<float4*>(G.v)[e / 4] = v;
        if (G.pb) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(p.x, p.y);
            __nv_bfloat162 hi = __floats2bfloat162_rn(p.z, p.w);
            uint2 w;
            w.x = *reinterpret_cast<uint32_t*>(&lo);
            w.y = *reinterpret_cast<uint32_t*>(&hi);
            reinterpret_cast<uint2*>(G.pb)[e / 4] = w;
        }
    }
}

// ---------------------------------------------------------------- per-job loss
// Synthetic layer loss used by the bench/trainer step: L_j = 1/2 sum over the
// projection outputs Y_p and job j's rows of ||y||^2 (so dL/dY_p = Y_p).
// Deterministic two-level reduction: row sums (one warp per row), then a
// fixed-order per-job block sum.  bytes/elem = 2 (bf16 read).
constexpr int kMaxLossTensors = 16;
struct SumsqArgs {
    const __nv_bfloat16* y[kMaxLossTensors];
    int cols[kMaxLossTensors];
    int ntensors;
    int rows;
    float* row_acc;  // [rows]
};

__global__ void row_sumsq_kernel(const __grid_constant__ SumsqArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int warps = blockDim.x / 32;
    const int lane = threadIdx.x & 31;
    for (int row = blockIdx.x * warps + threadIdx.x / 32; row < a.rows; row += gridDim.x * warps) {
        float acc = 0.f;
        for (int t = 0; t < a.ntensors; ++t) {
            const uint4* p = reinterpret_cast<const uint4*>(a.y[t] + (long long)row * a.cols[t]);
            const int n8 = a.cols[t] / 8;
            for (int i = lane; i < n8; i += 32) {
                const uint4 w = p[i];
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(h[e]);
                    acc = fmaf(f.x, f.x, acc);
                    acc = fmaf(f.y, f.y, acc);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) a.row_acc[row] = acc;
    }
}

// Non-finite guard: every job whose loss is not finite gets its rows of each
// tensor zeroed (the backward's dY), so no inf/NaN reaches the structural
// zeros the fused reductions multiply it by (other jobs' columns of H_cat in
// dB = dY^T H) — 0 * inf would poison co-scheduled jobs.  Grid (J, ysplit);
// the common all-finite case reads J floats and exits.
constexpr int kMaxGuardTensors = 32;
struct GuardArgs {
    __nv_bfloat16* t[kMaxGuardTensors];
    int cols[kMaxGuardTensors];
    int ntensors;
    const int* seg;     // device, J+1
    const float* loss;  // device, J
};

__global__ void zero_nonfinite_rows_kernel(const __grid_constant__ GuardArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int j = blockIdx.x;
    if (isfinite(a.loss[j])) return;
    const int r0 = a.seg[j], r1 = a.seg[j + 1];
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (int t = 0; t < a.ntensors; ++t) {
        const int n8 = a.cols[t] / 8;
        const long long total = (long long)(r1 - r0) * n8;
        uint4* base = reinterpret_cast<uint4*>(a.t[t] + (long long)r0 * a.cols[t]);
        for (long long i = (long long)blockIdx.y * blockDim.x + threadIdx.x; i < total;
             i += (long long)gridDim.y * blockDim.x)
            base[i] = z;
    }
}

// ---------------------------------------------------------------- device fuse
// fusim::fuse (lora.cpp:114-158) for bf16 hidden states on the device:
// sequence s of the fused batch (job order, then sequence order) is copied from
// its own buffer to rows off[s] .. off[s] + len[s] of the fused matrix; in the
// padded layout the slot's remaining rows (to off[s+1]) are zero-filled, and
// mask[row] = 1 exactly on copied rows.  One CTA per (32-row chunk of a slot,
// sequence), 16-byte copies.  A pure copy: bit-exact.
constexpr int kFuseMaxSeqs = 256;  // per launch (kernel parameter table)
struct FuseArgs {
    const __nv_bfloat16* src[kFuseMaxSeqs];
    long long ld[kFuseMaxSeqs];   // source row stride (elements)
    long long off[kFuseMaxSeqs + 1];
    int len[kFuseMaxSeqs];
    int nseq;
    long long dim;                // elements per row (multiple of 8)
    __nv_bfloat16* dst;
    uint8_t* mask;
};

__global__ void fuse_rows_kernel(const __grid_constant__ FuseArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int s = blockIdx.y;
    const long long slot = a.off[s + 1] - a.off[s];
    const int r0 = blockIdx.x * 32;
    if (r0 >= slot) return;
    const int r1 = static_cast<int>(slot < r0 + 32 ? slot : r0 + 32);
    const int n8 = static_cast<int>(a.dim / 8);
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (int e = threadIdx.x; e < (r1 - r0) * n8; e += blockDim.x) {
        const int r = r0 + e / n8, c = e % n8;
        uint4* d = reinterpret_cast<uint4*>(a.dst + (a.off[s] + r) * a.dim) + c;
        *d = r < a.len[s] ? reinterpret_cast<const uint4*>(a.src[s] + r * a.ld[s])[c] : z;
    }
    if (a.mask)
        for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) a.mask[a.off[s] + r] = r < a.len[s] ? 1 : 0;
}

__global__ void segment_loss_kernel(const float* __restrict__ row_acc, const int* __restrict__ seg,
                                    float* __restrict__ loss) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ float red[32];
    const int j = blockIdx.x;
    const int r0 = seg[j], r1 = seg[j + 1];
    float acc = 0.f;
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) acc += row_acc[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
        acc = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (threadIdx.x == 0) loss[j] = 0.5f * acc;
    }
}

// Per-job loss from the row partials the forward GEMM epilogue wrote:
// loss[j] = 1/2 sum_t sum_nb sum_{rows of j} row_sq_t[nb][row], fixed order.
struct RowSqArgs {
    const float* part[kMaxLossTensors];
    int nblk[kMaxLossTensors];
    int ntensors;
    int rows;
};

// step 1: row_acc[r] = sum_t sum_nb row_sq_t[nb][r].  Block (32, kRowSqSlices):
// x = one of 32 consecutive rows (128-byte coalesced loads), y = a fixed slice
// of the (tensor, column-block) list; the slices are combined in a fixed order
// (deterministic).  One thread per row summing all ~170 partials serially left
// the launch latency-bound (22 us at C2 for 5.4 MB); 8 slices: 12.1 us; 32 slices
// (~5 loads per thread, one round of memory latency): 8.6 us.
constexpr int kRowSqSlices = 32;
__global__ void __launch_bounds__(32 * kRowSqSlices)
rowsq_rows_kernel(const __grid_constant__ RowSqArgs a, float* __restrict__ row_acc) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ float red[kRowSqSlices][33];
    const int r = blockIdx.x * 32 + threadIdx.x;
    float rs = 0.f;
    if (r < a.rows) {
        int i = 0;
        for (int t = 0; t < a.ntensors; ++t) {
            const float* part = a.part[t];
            const int nblk = a.nblk[t];
            int nb = (static_cast<int>(threadIdx.y) - i) % kRowSqSlices;
            if (nb < 0) nb += kRowSqSlices;
#pragma unroll 4
            for (; nb < nblk; nb += kRowSqSlices) rs += __ldg(part + (long long)nb * a.rows + r);
            i += nblk;
        }
    }
    red[threadIdx.y][threadIdx.x] = rs;
    __syncthreads();
    if (threadIdx.y == 0 && r < a.rows) {
        float s = 0.f;
#pragma unroll
        for (int y = 0; y < kRowSqSlices; ++y) s += red[y][threadIdx.x];
        row_acc[r] = s;
    }
}
// step 2: segment_loss_kernel (fixed-order per-job block sum of row_acc)

// The layer step's step 2 fused with the non-finite guard: grid (J, ysplit).
// Every CTA of job j sums the job's row_acc in the same fixed order (8 KB per
// job at C2: the redundancy is cheaper than a cross-CTA hand-over), CTA y = 0
// stores loss[j], and when the loss is not finite all ysplit CTAs zero the
// job's rows of the guarded tensors (as zero_nonfinite_rows_kernel).  One
// launch instead of two between the forward and the backward.
__global__ void __launch_bounds__(256) loss_guard_kernel(const float* __restrict__ row_acc,
                                                          float* __restrict__ loss, const __grid_constant__ GuardArgs a) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    __shared__ float red[8];
    __shared__ float total;
    const int j = blockIdx.x;
    const int r0 = a.seg[j], r1 = a.seg[j + 1];
    float acc = 0.f;
    for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) acc += row_acc[r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < static_cast<int>(blockDim.x / 32); ++w) t += red[w];
        total = 0.5f * t;
        if (blockIdx.y == 0) loss[j] = total;
    }
    __syncthreads();
    if (isfinite(total)) return;
    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
    for (int t = 0; t < a.ntensors; ++t) {
        const int n8 = a.cols[t] / 8;
        const long long cnt = (long long)(r1 - r0) * n8;
        uint4* base = reinterpret_cast<uint4*>(a.t[t] + (long long)r0 * a.cols[t]);
        for (long long i = (long long)blockIdx.y * blockDim.x + threadIdx.x; i < cnt;
             i += (long long)gridDim.y * blockDim.x)
            base[i] = z;
    }
}

}  // namespace mlora
