// mlora_model.cu — the small HBM-bound kernels around the LoRA linears
// (north star item 4): padding-masked cross-entropy with
// per-job mean loss, RMSNorm forward/backward, rotary embedding.
//
// The reference has none of these (its model is analytic), so their semantics
// are "parity unpinned": they are checked against fp64 numpy restatements in
// tests/test_gpu_model.py.  All reductions are deterministic (fixed order, no
// float atomics).  Roofline: HBM bandwidth; bytes per row are stated per kernel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "../../include/mlora.h"
#include "sm100.cuh"

namespace {

__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <typename T>
__device__ __forceinline__ T block_reduce(T v, T* red, bool is_max) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T u = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? (u > v ? u : v) : v + u;
    }
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < (int)(blockDim.x >> 5) ? red[lane] : (is_max ? -INFINITY : T(0));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const T u = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? (u > v ? u : v) : v + u;
        }
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

// ---------------------------------------------------------------- masked CE
// Three launches: per-job real-row counts (inv_count, needed by the row pass),
// the row pass, and the per-job mean.  Row pass: a persistent grid, one row per
// CTA at a time; pass 1 streams the row from HBM with 16-byte loads and an
// online (max, sum-exp), marking it L2 evict_last; pass 2 re-reads it from L2
// (evict_first) and writes dlogits = (softmax - onehot) / n_j (0 on pad rows,
// rounded once) as an evict_first stream.  bytes/row: 2V read + 2V write
// (ncu at C4: 1.97 GB read for 1.6 GB of logits; 3.04 GB without the hints).
__global__ void ce_count_kernel(const uint8_t* __restrict__ mask, const int* __restrict__ seg,
                                float* __restrict__ inv_count) {
    pdl_prologue();
    __shared__ float red[32];
    const int j = blockIdx.x;
    float cnt = 0.f;
    for (int r = seg[j] + threadIdx.x; r < seg[j + 1]; r += blockDim.x) cnt += (mask == nullptr || mask[r]) ? 1.f : 0.f;
    cnt = block_reduce(cnt, red, false);
    if (threadIdx.x == 0) inv_count[j] = cnt > 0.f ? 1.f / cnt : 0.f;
}

__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
    const float mn = fmaxf(m, m2);
    if (mn == -INFINITY) return;
    s = (m == -INFINITY ? 0.f : s * __expf(m - mn)) + (m2 == -INFINITY ? 0.f : s2 * __expf(m2 - mn));
    m = mn;
}

// L2 cache-policy hints: the row pass keeps each logits row L2-resident
// between its two reads (evict_last), and lets the dlogits stream and the
// second read go first (evict_first).
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_hint(const uint4* ptr, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(ptr), "l"(pol));
    return r;
}
__device__ __forceinline__ void st_hint(uint4* ptr, uint4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w), "l"(pol)
                 : "memory");
}

__global__ void __launch_bounds__(256) ce_rows_kernel(const __nv_bfloat16* __restrict__ logits, int V,
                                                      const int* __restrict__ labels, const uint8_t* __restrict__ mask,
                                                      const int* __restrict__ seg, int J,
                                                      const float* __restrict__ inv_count, long long rows,
                                                      float* __restrict__ row_loss, __nv_bfloat16* __restrict__ dlogits) {
    pdl_prologue();
    __shared__ float rm[8], rs[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool vec = (V & 7) == 0;
    const uint64_t keep = l2_policy_last(), stream_out = l2_policy_first();
    for (long long row = blockIdx.x; row < rows; row += gridDim.x) {
        const __nv_bfloat16* src = logits + row * V;
        float m = -INFINITY, sum = 0.f;
        if (vec) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll 4
            for (int i = threadIdx.x; i < V / 8; i += blockDim.x) {
                const uint4 u = ld_hint(s4 + i, keep);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
                float f[8];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 x = __bfloat1622float2(h[e]);
                    f[2 * e] = x.x, f[2 * e + 1] = x.y;
                }
                float cm = f[0];
#pragma unroll
                for (int e = 1; e < 8; ++e) cm = fmaxf(cm, f[e]);
                float cs = 0.f;
#pragma unroll
                for (int e = 0; e < 8; ++e) cs += __expf(f[e] - cm);
                ms_merge(m, sum, cm, cs);
            }
        } else {
            for (int i = threadIdx.x; i < V; i += blockDim.x) ms_merge(m, sum, __bfloat162float(src[i]), 1.f);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float m2 = __shfl_xor_sync(0xffffffffu, m, o), s2 = __shfl_xor_sync(0xffffffffu, sum, o);
            ms_merge(m, sum, m2, s2);
        }
        if (lane == 0) rm[w] = m, rs[w] = sum;
        __syncthreads();
        m = rm[0], sum = rs[0];
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) ms_merge(m, sum, rm[k], rs[k]);
        __syncthreads();  // rm / rs are reused by the next row
        const float lse = m + __logf(sum);
        const bool real = mask == nullptr || mask[row] != 0;
        const int label = labels[row];
        if (threadIdx.x == 0) row_loss[row] = real ? lse - __bfloat162float(src[label]) : 0.f;
        if (!dlogits) continue;
        int j = 0;
        for (int t = 1; t < J; ++t)
            if (seg[t] <= row) j = t;
        const float sc = real ? inv_count[j] : 0.f;
        __nv_bfloat16* dst = dlogits + row * V;
        if (vec) {
            const uint4* s4 = reinterpret_cast<const uint4*>(src);
            uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll 4
            for (int i = threadIdx.x; i < V / 8; i += blockDim.x) {
                const uint4 u = ld_hint(s4 + i, stream_out);
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
                uint4 o;
                uint32_t* ow = &o.x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float2 x = __bfloat1622float2(h[e]);
                    const int c = i * 8 + 2 * e;
                    const float g0 = sc * (__expf(x.x - lse) - (c == label ? 1.f : 0.f));
                    const float g1 = sc * (__expf(x.y - lse) - (c + 1 == label ? 1.f : 0.f));
                    const __nv_bfloat162 r = __floats2bfloat162_rn(g0, g1);
                    ow[e] = *reinterpret_cast<const uint32_t*>(&r);
                }
                st_hint(d4 + i, o, stream_out);
            }
        } else {
            for (int i = threadIdx.x; i < V; i += blockDim.x)
                dst[i] = __float2bfloat16_rn(sc * (__expf(__bfloat162float(src[i]) - lse) - (i == label ? 1.f : 0.f)));
        }
    }
}

// Row pass on a cluster of kCeCl CTAs (V % 8 == 0, 32 <= V <= kCeClusterMaxV): CTA r of
// the cluster owns a quarter of every row it visits.  The quarter row (32.5 KB at
// V = 65024) arrives in shared memory by ONE bulk TMA copy, double-buffered (the next
// row's copy is in flight while this one is reduced), so the row is read from HBM once
// and re-read from shared memory, never from L2.  Three clusters' CTAs share an SM, so
// one CTA's reductions overlap another's loads (the grid is as many clusters as are
// co-resident: a second wave would double the time).  Each CTA reduces its quarter to
// (max, sum 2^((x - max) log2 e)); the partials go to every CTA of the cluster by
// st.async into their shared memory, completing on their mbarrier (no per-row cluster
// barrier, whose release would wait for the previous row's dlogits stores to drain),
// and are merged in rank order (all CTAs compute the same lse: deterministic).  The
// dlogits pass re-reads the quarter from shared memory.  C4 (12 288 rows x V = 65 024):
// 1.07 ms -> 0.78 ms, DRAM 3.57 -> 3.15 GB.  Pad rows (mask 0)
// are never loaded: their dlogits are written as zeros.  DRAM: 2V read (real rows)
// + 2V written per row.
constexpr int kCeCl = 4;
constexpr int kCeThreads = 256;
constexpr int kCeClusterMaxV = 74 * 1024;
constexpr float kLog2e = 1.4426950408889634f;
__host__ __device__ __forceinline__ int ce_part(int V) { return (V / (8 * kCeCl)) * 8; }  // ranks 0..CL-2
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__global__ void __cluster_dims__(kCeCl, 1, 1) __launch_bounds__(kCeThreads, 3)
ce_rows_cluster_kernel(const __nv_bfloat16* __restrict__ logits, int V, const int* __restrict__ labels,
                       const uint8_t* __restrict__ mask, const int* __restrict__ seg, int J,
                       const float* __restrict__ inv_count, long long rows, float* __restrict__ row_loss,
                       __nv_bfloat16* __restrict__ dlogits) {
    using namespace mlora::sm100;
    extern __shared__ __align__(128) uint8_t ce_smem[];
    __shared__ float red[kCeThreads / 32];
    __shared__ float2 xch[2][kCeCl];   // every rank's (max, sum) of the row, by iteration parity
    __shared__ float lse_s;
    __shared__ __align__(8) uint64_t full[2];
    __shared__ __align__(8) uint64_t xbar[2];  // the other ranks' partials of the row have landed
    const uint32_t rank = cluster_ctarank();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int part = ce_part(V);
    const int off = static_cast<int>(rank) * part;
    const int n = rank + 1 == kCeCl ? V - (kCeCl - 1) * part : part;   // this CTA's columns [off, off + n)
    const int slot_bytes = ((((V - (kCeCl - 1) * part) > part ? V - (kCeCl - 1) * part : part) * 2 + 127) / 128) * 128;
    const long long cl = blockIdx.x / kCeCl, ncl = gridDim.x / kCeCl;
    if (threadIdx.x == 0) {
        mbar_init(&full[0], 1);
        mbar_init(&full[1], 1);
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        fence_barrier_init();
    }
    cluster_sync();  // barriers initialised, every CTA of the cluster running (DSMEM targets exist)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint64_t read_once = l2_policy_first(), stream_out = l2_policy_first();
    auto is_real = [&](long long row) { return mask == nullptr || mask[row] != 0; };
    auto issue = [&](int it, long long row) {
        if (threadIdx.x == 0 && is_real(row)) {
            mbar_arrive_expect_tx(&full[it & 1], static_cast<uint32_t>(2 * n));
            bulk_load_hint(smem_u32(ce_smem + (it & 1) * slot_bytes), logits + row * V + off,
                           static_cast<uint32_t>(2 * n), &full[it & 1], read_once);
        }
    };
    if (cl < rows) issue(0, cl);
    int it = 0;
    uint32_t phase[2] = {0u, 0u};  // completed loads / exchanges per slot (pad rows do neither)
    for (long long row = cl; row < rows; row += ncl, ++it) {
        if (row + ncl < rows) issue(it + 1, row + ncl);  // its slot was released by iteration it - 1
        const bool real = is_real(row);
        const uint4* buf = reinterpret_cast<const uint4*>(ce_smem + (it & 1) * slot_bytes);
        if (real) {
            mbar_wait(&full[it & 1], phase[it & 1] & 1u);
            // the quarter row is in shared memory: a packed-bf16 max pass, then one exp2
            // per element against that max (no online rescaling)
            __nv_bfloat162 mx2 = __float2bfloat162_rn(-INFINITY);
            for (int i = threadIdx.x; i < n / 8; i += kCeThreads) {
                const uint4 u = buf[i];
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
                mx2 = __hmax2(mx2, __hmax2(__hmax2(h[0], h[1]), __hmax2(h[2], h[3])));
            }
            float m = fmaxf(__low2float(mx2), __high2float(mx2));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            if (lane == 0) red[w] = m;
            __syncthreads();
            m = red[0];
#pragma unroll
            for (int k = 1; k < kCeThreads / 32; ++k) m = fmaxf(m, red[k]);
            const float mb = m * kLog2e;
            float sum = 0.f;
            for (int i = threadIdx.x; i < n / 8; i += kCeThreads) {
                const uint4 u = buf[i];
                const uint32_t* q = &u.x;
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    sum += ex2_approx(fmaf(__uint_as_float(q[e] << 16), kLog2e, -mb));
                    sum += ex2_approx(fmaf(__uint_as_float(q[e] & 0xffff0000u), kLog2e, -mb));
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            __syncthreads();  // every thread has read red[] (the max) before it is reused
            if (lane == 0) red[w] = sum;
            __syncthreads();
            if (threadIdx.x == 0) {
                sum = red[0];
                for (int k = 1; k < kCeThreads / 32; ++k) sum += red[k];
                // this rank's partial to every other rank (st.async + their xbar), own slot locally
                mbar_arrive_expect_tx(&xbar[it & 1], 8u * (kCeCl - 1));
#pragma unroll
                for (int r = 0; r < kCeCl; ++r)
                    if (r != static_cast<int>(rank))
                        st_async_v2(mapa_shared(smem_u32(&xch[it & 1][rank]), r), m, sum,
                                    mapa_shared(smem_u32(&xbar[it & 1]), r));
                xch[it & 1][rank] = make_float2(m, sum);
                mbar_wait_cluster(&xbar[it & 1], phase[it & 1] & 1u);
                float mm = xch[it & 1][0].x, ss = xch[it & 1][0].y;  // fixed order: rank 0, 1, ...
#pragma unroll
                for (int r = 1; r < kCeCl; ++r) ms_merge(mm, ss, xch[it & 1][r].x, xch[it & 1][r].y);
                lse_s = mm + __logf(ss);
            }
            ++phase[it & 1];
        }
        __syncthreads();
        const float lse = lse_s;
        const int label = labels[row];
        if (threadIdx.x == 0) {
            if (!real) {
                if (rank == 0) row_loss[row] = 0.f;
            } else if (label >= off && label < off + n) {
                row_loss[row] = lse - __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(buf)[label - off]);
            }
        }
        if (dlogits) {
            int j = 0;
            for (int t = 1; t < J; ++t)
                if (seg[t] <= row) j = t;
            const float sc = real ? inv_count[j] : 0.f;
            const float lb = lse * kLog2e;
            const int li = label - off;  // the label's column in this part (may be outside)
            uint4* d4 = reinterpret_cast<uint4*>(dlogits + row * V + off);
            for (int i = threadIdx.x; i < n / 8; i += kCeThreads) {
                uint4 o = make_uint4(0u, 0u, 0u, 0u);
                if (real) {
                    const uint4 u = buf[i];
                    const uint32_t* q = &u.x;
                    uint32_t* ow = &o.x;
                    float g[8];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        g[2 * e] = sc * ex2_approx(fmaf(__uint_as_float(q[e] << 16), kLog2e, -lb));
                        g[2 * e + 1] = sc * ex2_approx(fmaf(__uint_as_float(q[e] & 0xffff0000u), kLog2e, -lb));
                    }
                    if (li >= 8 * i && li < 8 * i + 8) {  // the one-hot term, once per row
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            if (8 * i + e == li) g[e] -= sc;
                    }
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const __nv_bfloat162 r = __floats2bfloat162_rn(g[2 * e], g[2 * e + 1]);
                        ow[e] = *reinterpret_cast<const uint32_t*>(&r);
                    }
                }
                st_hint(d4 + i, o, stream_out);
            }
        }
        __syncthreads();  // this slot's reads and lse_s are done before their reuse
    }
    cluster_sync();  // no DSMEM write may target an exited CTA
}

// loss[j] = (sum of row_loss over job j's rows) * inv_count[j]: fixed order.
__global__ void ce_loss_kernel(const float* __restrict__ row_loss, const int* __restrict__ seg,
                               const float* __restrict__ inv_count, float* __restrict__ loss) {
    pdl_prologue();
    __shared__ float red[32];
    const int j = blockIdx.x;
    float acc = 0.f;
    for (int r = seg[j] + threadIdx.x; r < seg[j + 1]; r += blockDim.x) acc += row_loss[r];
    acc = block_reduce(acc, red, false);
    if (threadIdx.x == 0) loss[j] = acc * inv_count[j];
}

// ---------------------------------------------------------------- RMSNorm
// y = x * rstd * w, rstd = 1/sqrt(mean(x^2) + eps).  One CTA per row.
// bytes/row: 2h read + 2h write (+ w from L2).
__global__ void rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w, int h,
                                   float eps, __nv_bfloat16* __restrict__ y, float* __restrict__ rstd) {
    pdl_prologue();
    __shared__ float red[32];
    const __nv_bfloat16* xr = x + (long long)blockIdx.x * h;
    float ss = 0.f;
    for (int i = threadIdx.x; i < h; i += blockDim.x) {
        const float v = __bfloat162float(xr[i]);
        ss = fmaf(v, v, ss);
    }
    ss = block_reduce(ss, red, false);
    const float r = rsqrtf(ss / h + eps);
    if (threadIdx.x == 0) rstd[blockIdx.x] = r;
    __nv_bfloat16* yr = y + (long long)blockIdx.x * h;
    for (int i = threadIdx.x; i < h; i += blockDim.x)
        yr[i] = __float2bfloat16_rn(__bfloat162float(xr[i]) * r * __bfloat162float(w[i]));
}

// dx = rstd * (g - xhat * mean(g * xhat)), g = dy * w; dw partials per row block (deterministic).
__global__ void rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                                   const __nv_bfloat16* __restrict__ w, const float* __restrict__ rstd, int rows,
                                   int h, __nv_bfloat16* __restrict__ dx, float* __restrict__ dw_part,
                                   int rows_per_block) {
    pdl_prologue();
    __shared__ float red[32];
    const int r0 = blockIdx.x * rows_per_block;
    const int r1 = min(rows, r0 + rows_per_block);
    // dw partial for this block's rows: each thread owns columns i, i + blockDim, ...
    for (int i = threadIdx.x; i < h; i += blockDim.x) dw_part[(long long)blockIdx.x * h + i] = 0.f;
    for (int row = r0; row < r1; ++row) {
        const __nv_bfloat16* xr = x + (long long)row * h;
        const __nv_bfloat16* gr = dy + (long long)row * h;
        const float r = rstd[row];
        float dot = 0.f;
        for (int i = threadIdx.x; i < h; i += blockDim.x)
            dot += __bfloat162float(gr[i]) * __bfloat162float(w[i]) * __bfloat162float(xr[i]) * r;
        dot = block_reduce(dot, red, false) / h;
        for (int i = threadIdx.x; i < h; i += blockDim.x) {
            const float xh = __bfloat162float(xr[i]) * r;
            const float g = __bfloat162float(gr[i]) * __bfloat162float(w[i]);
            dx[(long long)row * h + i] = __float2bfloat16_rn(r * (g - xh * dot));
            dw_part[(long long)blockIdx.x * h + i] += __bfloat162float(gr[i]) * xh;
        }
    }
}

__global__ void column_sum_kernel(const float* __restrict__ part, int nblk, int h, float* __restrict__ out) {
    pdl_prologue();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < h; i += gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int b = 0; b < nblk; ++b) s += part[(long long)b * h + i];
        out[i] = s;
    }
}

// ---------------------------------------------------------------- RoPE
// x, y: [rows, heads, head_dim] bf16; rotate-half pairing (i, i + head_dim/2)
// by angle pos * base^(-2i/head_dim); inverse = 1 rotates by -angle (backward).
__global__ void rope_kernel(const __nv_bfloat16* __restrict__ x, __nv_bfloat16* __restrict__ y,
                            const int* __restrict__ pos, int heads, int hd, float base, int inverse) {
    pdl_prologue();
    const int row = blockIdx.x;
    const int half = hd / 2;
    const float p = static_cast<float>(pos[row]);
    for (int e = threadIdx.x; e < heads * half; e += blockDim.x) {
        const int hh = e / half, i = e % half;
        const float inv_freq = exp2f(-(2.f * i / hd) * log2f(base));
        float sn, cs;
        sincosf(p * inv_freq, &sn, &cs);
        if (inverse) sn = -sn;
        const long long o = ((long long)row * heads + hh) * hd;
        const float a = __bfloat162float(x[o + i]), b = __bfloat162float(x[o + i + half]);
        y[o + i] = __float2bfloat16_rn(a * cs - b * sn);
        y[o + i + half] = __float2bfloat16_rn(b * cs + a * sn);
    }
}

}  // namespace
void mlora_count_free_launch();  // mlora_decoder.cu
namespace {

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*k)(KArgs...), dim3 g, dim3 b, size_t smem, void* stream, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k, args...);
    if (e == cudaSuccess) mlora_count_free_launch();
    return e;
}

}  // namespace

extern "C" {

mlora_status mlora_masked_ce(int32_t num_jobs, const int32_t* seg_dev, int64_t rows, int32_t V, const void* logits,
                             const int32_t* labels, const uint8_t* mask, float* row_loss, float* loss,
                             float* inv_count, void* dlogits, void* stream) {
    if (rows < 1 || V < 1 || num_jobs < 1 || !seg_dev || !logits || !labels || !row_loss || !loss || !inv_count)
        return MLORA_USAGE;
    if ((reinterpret_cast<uintptr_t>(logits) & 15) || (reinterpret_cast<uintptr_t>(dlogits) & 15))
        return MLORA_USAGE;  // 16-byte aligned rows (V % 8 == 0 takes the vector path)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int* seg = static_cast<const int*>(seg_dev);
    if (launch(ce_count_kernel, dim3(num_jobs), dim3(1024), 0, stream, mask, seg, inv_count) != cudaSuccess)
        return MLORA_CUDA;
    if (V % 8 == 0 && V >= 8 * kCeCl && V <= kCeClusterMaxV) {
        // cluster row pass: each quarter row by one bulk copy into shared memory
        const int part = ce_part(V);
        const size_t slot = ((static_cast<size_t>(std::max(part, V - (kCeCl - 1) * part)) * 2 + 127) / 128) * 128;
        const size_t smem = 2 * slot;
        if (cudaFuncSetAttribute(ce_rows_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)) != cudaSuccess)
            return MLORA_CUDA;
        // as many clusters as can be co-resident (a persistent grid: a second wave would
        // double the time), from the occupancy calculator, not from smem arithmetic
        int max_clusters = 0;
        {
            cudaLaunchConfig_t oc{};
            oc.gridDim = dim3(kCeCl * 1024);
            oc.blockDim = dim3(kCeThreads);
            oc.dynamicSmemBytes = smem;
            cudaLaunchAttribute ca;
            ca.id = cudaLaunchAttributeClusterDimension;
            ca.val.clusterDim.x = kCeCl;
            ca.val.clusterDim.y = 1;
            ca.val.clusterDim.z = 1;
            oc.attrs = &ca;
            oc.numAttrs = 1;
            if (cudaOccupancyMaxActiveClusters(&max_clusters, ce_rows_cluster_kernel, &oc) != cudaSuccess ||
                max_clusters < 1)
                max_clusters = sms / kCeCl;
        }
        const unsigned clusters = static_cast<unsigned>(std::min<long long>(rows, max_clusters));
        if (launch(ce_rows_cluster_kernel, dim3(kCeCl * clusters), dim3(kCeThreads), smem, stream,
                   static_cast<const __nv_bfloat16*>(logits), static_cast<int>(V), labels, mask, seg,
                   static_cast<int>(num_jobs), static_cast<const float*>(inv_count), static_cast<long long>(rows),
                   row_loss, static_cast<__nv_bfloat16*>(dlogits)) != cudaSuccess)
            return MLORA_CUDA;
    } else {
        const unsigned grid = static_cast<unsigned>(std::min<long long>(rows, 4LL * sms));
        if (launch(ce_rows_kernel, dim3(grid), dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(logits),
                   static_cast<int>(V), labels, mask, seg, static_cast<int>(num_jobs),
                   static_cast<const float*>(inv_count), static_cast<long long>(rows), row_loss,
                   static_cast<__nv_bfloat16*>(dlogits)) != cudaSuccess)
            return MLORA_CUDA;
    }
    if (launch(ce_loss_kernel, dim3(num_jobs), dim3(1024), 0, stream, static_cast<const float*>(row_loss), seg,
               static_cast<const float*>(inv_count), loss) != cudaSuccess)
        return MLORA_CUDA;
    return MLORA_OK;
}

mlora_status mlora_rmsnorm_fwd(int64_t rows, int32_t h, const void* x, const void* w, float eps, void* y,
                               float* rstd, void* stream) {
    if (rows < 1 || h < 1 || !x || !w || !y || !rstd) return MLORA_USAGE;
    if (!(eps > 0.f)) return MLORA_USAGE;
    return launch(rmsnorm_fwd_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, stream,
                  static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w), static_cast<int>(h),
                  eps, static_cast<__nv_bfloat16*>(y), rstd) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

mlora_status mlora_rmsnorm_bwd(int64_t rows, int32_t h, const void* dy, const void* x, const void* w,
                               const float* rstd, void* dx, float* dw, float* workspace, int32_t rows_per_block,
                               void* stream) {
    if (rows < 1 || h < 1 || !dy || !x || !w || !rstd || !dx || !dw || !workspace || rows_per_block < 1)
        return MLORA_USAGE;
    const int nblk = static_cast<int>((rows + rows_per_block - 1) / rows_per_block);
    if (launch(rmsnorm_bwd_kernel, dim3(nblk), dim3(256), 0, stream, static_cast<const __nv_bfloat16*>(dy),
               static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(w), rstd,
               static_cast<int>(rows), static_cast<int>(h), static_cast<__nv_bfloat16*>(dx), workspace,
               static_cast<int>(rows_per_block)) != cudaSuccess)
        return MLORA_CUDA;
    return launch(column_sum_kernel, dim3((h + 255) / 256), dim3(256), 0, stream, static_cast<const float*>(workspace),
                  nblk, static_cast<int>(h), dw) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

mlora_status mlora_rope(int64_t rows, int32_t heads, int32_t head_dim, const void* x, void* y, const int32_t* pos,
                        float base, int32_t inverse, void* stream) {
    if (rows < 1 || heads < 1 || head_dim < 2 || (head_dim & 1) || !x || !y || !pos || !(base > 1.f))
        return MLORA_USAGE;
    return launch(rope_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, stream,
                  static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), pos, static_cast<int>(heads),
                  static_cast<int>(head_dim), base, static_cast<int>(inverse)) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

}  // extern "C"
