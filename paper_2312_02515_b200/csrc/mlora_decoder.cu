// mlora_decoder.cu — the decoder-layer kernels around the fused multi-LoRA
// linears, so a whole LLaMA / ChatGLM2-shaped model can be LoRA-fine-tuned on
// the fused batch end to end (BASELINE configs C1 and C4: token embedding,
// RMSNorm with the residual add fused in, causal attention over the packed
// sequences with RoPE fused into its Q/K loads, SwiGLU, and their backwards).
//
// The reference has no model arithmetic at all ("no trainer,
// no model"), so these are "parity unpinned": tests/test_gpu_decoder.py checks
// them against a plain PyTorch fp32 restatement of the same model.  All
// reductions are deterministic (fixed order, no float atomics).
//
// Attention works on the fused row layout directly: sequence s owns rows
// seq_offsets[s] .. seq_offsets[s+1] (packed: back to back; padded: one
// max_len slot per sequence with the real tokens first), so no gather /
// transpose to a [batch, heads, len, head_dim] tensor is ever materialised.
// Q/K/V are column slices of the projection outputs (row stride ld), which
// covers ChatGLM2's fused qkv output (multi-query: 2 K/V groups) as well as
// LLaMA's separate q, k, v.  Attention is not on the BatchFusion hot path; the
// tiles run on the CUDA cores in fp32 (64 x 64 tiles, 4 x 4 register blocking)
// — correct and deterministic, not a tensor-core kernel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "../../include/mlora.h"

namespace {

constexpr int kBM = 64;  // rows (queries or keys) per attention tile
constexpr int kThreads = 256;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ void pdl_prologue() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ float block_sum(float v, float* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < static_cast<int>(blockDim.x >> 5) ? red[lane] : 0.f;
        v = warp_sum(v);
        if (lane == 0) red[0] = v;
    }
    __syncthreads();
    return red[0];
}

__host__ __device__ __forceinline__ const __nv_bfloat16* bf(const void* p) { return static_cast<const __nv_bfloat16*>(p); }
__host__ __device__ __forceinline__ __nv_bfloat16* bfw(void* p) { return static_cast<__nv_bfloat16*>(p); }

// ---------------------------------------------------------------- embedding
// x[t, :] = E[tokens[t], :]; one CTA per row, 16-byte vectors (h % 8 == 0).
__global__ void embed_kernel(const int* __restrict__ tokens, const uint4* __restrict__ E, int h8,
                             uint4* __restrict__ x) {
    pdl_prologue();
    const long long t = blockIdx.x;
    const long long tok = tokens[t];
    for (int i = threadIdx.x; i < h8; i += blockDim.x) x[t * h8 + i] = E[tok * h8 + i];
}

// ---------------------------------------------------------------- residual add + RMSNorm
// xo = bf16(x + delta) (the residual stream, when delta != NULL), y = xo * rstd * w.
// bytes/row: 2h (x) + 2h (delta) + 2h (xo) + 2h (y).
__global__ void add_rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ delta,
                                   const __nv_bfloat16* __restrict__ w, int h, float eps,
                                   __nv_bfloat16* __restrict__ xo, __nv_bfloat16* __restrict__ y,
                                   float* __restrict__ rstd) {
    pdl_prologue();
    __shared__ float red[32];
    const long long o = (long long)blockIdx.x * h;
    const __nv_bfloat16* src = delta ? xo : x;
    float ss = 0.f;
    for (int i = threadIdx.x; i < h; i += blockDim.x) {
        float v = __bfloat162float(x[o + i]);
        if (delta) {
            const __nv_bfloat16 s = __float2bfloat16_rn(v + __bfloat162float(delta[o + i]));
            xo[o + i] = s;
            v = __bfloat162float(s);
        }
        ss = fmaf(v, v, ss);
    }
    ss = block_sum(ss, red);  // (its __syncthreads also orders the xo writes before the re-read)
    const float r = rsqrtf(ss / h + eps);
    if (threadIdx.x == 0) rstd[blockIdx.x] = r;
    for (int i = threadIdx.x; i < h; i += blockDim.x)
        y[o + i] = __float2bfloat16_rn(__bfloat162float(src[o + i]) * r * __bfloat162float(w[i]));
}

// dx = dres + rstd (g - xhat mean(g xhat)), g = w * sum_k dy_k  (frozen w: no dw).
struct SumArgs {
    const __nv_bfloat16* dy[4];
    int n;
};

__global__ void rmsnorm_bwd_sum_kernel(SumArgs a, const __nv_bfloat16* __restrict__ dres,
                                       const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                                       const float* __restrict__ rstd, int h, __nv_bfloat16* __restrict__ dx) {
    pdl_prologue();
    __shared__ float red[32];
    const long long o = (long long)blockIdx.x * h;
    const float r = rstd[blockIdx.x];
    auto g_at = [&](int i) {
        float s = 0.f;
        for (int k = 0; k < a.n; ++k) s += __bfloat162float(a.dy[k][o + i]);
        return s * __bfloat162float(w[i]);
    };
    float dot = 0.f;
    for (int i = threadIdx.x; i < h; i += blockDim.x) dot = fmaf(g_at(i), __bfloat162float(x[o + i]) * r, dot);
    dot = block_sum(dot, red) / h;
    for (int i = threadIdx.x; i < h; i += blockDim.x) {
        const float xh = __bfloat162float(x[o + i]) * r;
        float v = r * (g_at(i) - xh * dot);
        if (dres) v += __bfloat162float(dres[o + i]);
        dx[o + i] = __float2bfloat16_rn(v);
    }
}

// ---------------------------------------------------------------- SwiGLU
__device__ __forceinline__ float sigmoidf_(float g) { return 1.f / (1.f + __expf(-g)); }

__global__ void swiglu_fwd_kernel(long long n, int f, const __nv_bfloat16* __restrict__ g, long long ldg,
                                  const __nv_bfloat16* __restrict__ u, long long ldu, __nv_bfloat16* __restrict__ out) {
    pdl_prologue();
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const long long t = e / f, c = e % f;
        const float gv = __bfloat162float(g[t * ldg + c]);
        out[e] = __float2bfloat16_rn(gv * sigmoidf_(gv) * __bfloat162float(u[t * ldu + c]));
    }
}

__global__ void swiglu_bwd_kernel(long long n, int f, const __nv_bfloat16* __restrict__ g, long long ldg,
                                  const __nv_bfloat16* __restrict__ u, long long ldu,
                                  const __nv_bfloat16* __restrict__ dout, __nv_bfloat16* __restrict__ dg,
                                  long long lddg, __nv_bfloat16* __restrict__ du, long long lddu) {
    pdl_prologue();
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const long long t = e / f, c = e % f;
        const float gv = __bfloat162float(g[t * ldg + c]);
        const float uv = __bfloat162float(u[t * ldu + c]);
        const float d = __bfloat162float(dout[e]);
        const float sg = sigmoidf_(gv);
        dg[t * lddg + c] = __float2bfloat16_rn(d * uv * sg * (1.f + gv * (1.f - sg)));
        du[t * lddu + c] = __float2bfloat16_rn(d * gv * sg);
    }
}

// ---------------------------------------------------------------- attention
struct AttnArgs {
    const int* seq_off;  // [S + 1] slot starts
    const int* seq_len;  // [S] real lengths (NULL: slot size)
    int heads, kv_heads;
    float rope_base;     // 0: no rotary
    float scale;         // softmax scale (1/sqrt(head_dim) normally)
    long long rows;
    const __nv_bfloat16 *q, *k, *v, *o, *dO;
    long long ldq, ldk, ldv, ldo, lddo;
    __nv_bfloat16 *out, *dq, *dk, *dv;
    long long ldout, lddq, lddk, lddv;
    float* lse;          // [heads][rows], natural log
    float* dsum;         // [heads][rows], sum_d dO * O
};

template <int HD>
struct Tile {
    static constexpr int LD = HD + 4;     // fp32 row stride of Q/K/V/dO tiles
    static constexpr int PLD = kBM + 4;   // fp32 row stride of P / dS tiles
    static constexpr int DV = HD / 64;    // float4 column groups per thread: d = tx*4 + 64c + e
};

__device__ __forceinline__ void seq_range(const AttnArgs& a, int s, int& start, int& len) {
    start = a.seq_off[s];
    const int slot = a.seq_off[s + 1] - start;
    len = a.seq_len ? min(a.seq_len[s], slot) : slot;
}

// Load rows [r0, r0 + 64) of one head (column offset col) into a fp32 tile,
// rotating pairs (i, i + HD/2) by pos * base^(-2i/HD) (the same angle as
// mlora_rope) when rope != 0; rows at or beyond `len` are zero.
template <int HD>
__device__ void load_tile(float* dst, const __nv_bfloat16* src, long long ld, int start, int r0, int len, int col,
                          float rope_base, bool rope) {
    constexpr int half = HD / 2, LD = Tile<HD>::LD;
    for (int e = threadIdx.x; e < kBM * (half / 2); e += blockDim.x) {
        const int r = e / (half / 2), i = (e % (half / 2)) * 2;
        const int pos = r0 + r;
        float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
        if (pos < len) {
            const __nv_bfloat16* p = src + (long long)(start + pos) * ld + col;
            const float2 A = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p + i));
            const float2 B = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(p + i + half));
            a0 = A.x, a1 = A.y, b0 = B.x, b1 = B.y;
            if (rope) {
                const float lb = log2f(rope_base);
                float s0, c0, s1, c1;
                sincosf(pos * exp2f(-(2.f * i / HD) * lb), &s0, &c0);
                sincosf(pos * exp2f(-(2.f * (i + 1) / HD) * lb), &s1, &c1);
                const float ra0 = a0 * c0 - b0 * s0, rb0 = b0 * c0 + a0 * s0;
                const float ra1 = a1 * c1 - b1 * s1, rb1 = b1 * c1 + a1 * s1;
                a0 = ra0, b0 = rb0, a1 = ra1, b1 = rb1;
            }
        }
        float* d = dst + r * LD;
        *reinterpret_cast<float2*>(d + i) = make_float2(a0, a1);
        *reinterpret_cast<float2*>(d + i + half) = make_float2(b0, b1);
    }
}

// Store a fp32 tile [64][LD] (already scaled) as bf16 rows of one head, applying
// the inverse rotation when rope != 0; rows at or beyond len are written as 0.
template <int HD>
__device__ void store_tile(const float* srcs, __nv_bfloat16* dst, long long ld, int start, int r0, int len, int col,
                           int slot, float rope_base, bool rope) {
    constexpr int half = HD / 2, LD = Tile<HD>::LD;
    for (int e = threadIdx.x; e < kBM * (half / 2); e += blockDim.x) {
        const int r = e / (half / 2), i = (e % (half / 2)) * 2;
        const int pos = r0 + r;
        if (pos >= slot) continue;
        const float* s = srcs + r * LD;
        float a0 = s[i], a1 = s[i + 1], b0 = s[i + half], b1 = s[i + half + 1];
        if (pos >= len) {
            a0 = a1 = b0 = b1 = 0.f;
        } else if (rope) {
            const float lb = log2f(rope_base);
            float s0, c0, s1, c1;
            sincosf(pos * exp2f(-(2.f * i / HD) * lb), &s0, &c0);
            sincosf(pos * exp2f(-(2.f * (i + 1) / HD) * lb), &s1, &c1);
            const float ra0 = a0 * c0 + b0 * s0, rb0 = b0 * c0 - a0 * s0;  // R(-theta)
            const float ra1 = a1 * c1 + b1 * s1, rb1 = b1 * c1 - a1 * s1;
            a0 = ra0, b0 = rb0, a1 = ra1, b1 = rb1;
        }
        __nv_bfloat16* p = dst + (long long)(start + pos) * ld + col;
        *reinterpret_cast<__nv_bfloat162*>(p + i) = __floats2bfloat162_rn(a0, a1);
        *reinterpret_cast<__nv_bfloat162*>(p + i + half) = __floats2bfloat162_rn(b0, b1);
    }
}

// acc[a][b] = sum_d X[ty*4 + a][d] * Y[tx + 16 b][d] over one 64 x 64 tile pair.
template <int HD>
__device__ __forceinline__ void tile_dot(const float* X, const float* Y, int ty, int tx, float acc[4][4]) {
    constexpr int LD = Tile<HD>::LD;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = 0.f;
#pragma unroll 4
    for (int d = 0; d < HD; d += 4) {
        float4 x[4], y[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) x[a] = *reinterpret_cast<const float4*>(X + (ty * 4 + a) * LD + d);
#pragma unroll
        for (int b = 0; b < 4; ++b) y[b] = *reinterpret_cast<const float4*>(Y + (tx + 16 * b) * LD + d);
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
                acc[a][b] += x[a].x * y[b].x + x[a].y * y[b].y + x[a].z * y[b].z + x[a].w * y[b].w;
    }
}

// acc[a][c*4+e] += sum_i P[i][ty*4 + a] * Z[i][tx*4 + 64c + e]   (transposed-P product; P row stride PLD)
template <int HD, bool TRANS>
__device__ __forceinline__ void tile_pz(const float* P, const float* Z, int ty, int tx, float acc[4][HD / 16]) {
    constexpr int LD = Tile<HD>::LD, PLD = Tile<HD>::PLD, DV = Tile<HD>::DV;
#pragma unroll 2
    for (int i = 0; i < kBM; ++i) {
        float p[4];
        if constexpr (TRANS) {
            const float4 q = *reinterpret_cast<const float4*>(P + i * PLD + ty * 4);
            p[0] = q.x, p[1] = q.y, p[2] = q.z, p[3] = q.w;
        } else {
#pragma unroll
            for (int a = 0; a < 4; ++a) p[a] = P[(ty * 4 + a) * PLD + i];
        }
#pragma unroll
        for (int c = 0; c < DV; ++c) {
            const float4 z = *reinterpret_cast<const float4*>(Z + i * LD + tx * 4 + 64 * c);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                acc[a][c * 4 + 0] = fmaf(p[a], z.x, acc[a][c * 4 + 0]);
                acc[a][c * 4 + 1] = fmaf(p[a], z.y, acc[a][c * 4 + 1]);
                acc[a][c * 4 + 2] = fmaf(p[a], z.z, acc[a][c * 4 + 2]);
                acc[a][c * 4 + 3] = fmaf(p[a], z.w, acc[a][c * 4 + 3]);
            }
        }
    }
}

template <int HD>
__device__ __forceinline__ void acc_to_smem(float* dst, const float acc[4][HD / 16], int ty, int tx, float s) {
    constexpr int LD = Tile<HD>::LD, DV = Tile<HD>::DV;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < DV; ++c)
            *reinterpret_cast<float4*>(dst + (ty * 4 + a) * LD + tx * 4 + 64 * c) =
                make_float4(s * acc[a][c * 4 + 0], s * acc[a][c * 4 + 1], s * acc[a][c * 4 + 2],
                            s * acc[a][c * 4 + 3]);
}

template <int HD>
constexpr size_t attn_smem_fwd() {
    return sizeof(float) * (3 * kBM * Tile<HD>::LD + kBM * Tile<HD>::PLD);
}
template <int HD>
constexpr size_t attn_smem_bwd() {
    return sizeof(float) * (4 * kBM * Tile<HD>::LD + 2 * kBM * Tile<HD>::PLD + 2 * kBM);
}

// Forward: one CTA per (query tile, sequence, head).  Online softmax in the
// log2 domain; O = softmax(scale Q K^T, causal) V; lse in natural log.
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_fwd_kernel(AttnArgs a) {
    pdl_prologue();
    int start, len;
    seq_range(a, blockIdx.y, start, len);
    const int slot = a.seq_off[blockIdx.y + 1] - start;
    const int q0 = blockIdx.x * kBM;
    if (q0 >= slot) return;
    const int h = blockIdx.z, kvh = h / (a.heads / a.kv_heads);
    constexpr int LD = Tile<HD>::LD, PLD = Tile<HD>::PLD, DV = Tile<HD>::DV;
    extern __shared__ __align__(16) float sm[];
    float* Qs = sm;
    float* Ks = Qs + kBM * LD;
    float* Vs = Ks + kBM * LD;
    float* Ps = Vs + kBM * LD;
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const bool rope = a.rope_base > 0.f;
    const float c2 = a.scale * kLog2e;

    load_tile<HD>(Qs, a.q, a.ldq, start, q0, len, h * HD, a.rope_base, rope);
    float m[4], l[4], o[4][HD / 16];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        m[i] = -INFINITY;
        l[i] = 0.f;
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) o[i][c] = 0.f;
    }
    const int nkt = q0 < len ? (min(q0 + kBM, len) + kBM - 1) / kBM : 0;
    for (int kt = 0; kt < nkt; ++kt) {
        __syncthreads();
        load_tile<HD>(Ks, a.k, a.ldk, start, kt * kBM, len, kvh * HD, a.rope_base, rope);
        load_tile<HD>(Vs, a.v, a.ldv, start, kt * kBM, len, kvh * HD, a.rope_base, false);
        __syncthreads();
        float s[4][4];
        tile_dot<HD>(Qs, Ks, ty, tx, s);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int qi = q0 + ty * 4 + i;
            float mx = -INFINITY;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int kj = kt * kBM + tx + 16 * b;
                s[i][b] = (kj <= qi && qi < len) ? s[i][b] * c2 : -INFINITY;
                mx = fmaxf(mx, s[i][b]);
            }
#pragma unroll
            for (int off = 8; off > 0; off >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
            const float mn = fmaxf(m[i], mx);
            const float alpha = mn == -INFINITY ? 1.f : exp2f(m[i] - mn);
            float ps = 0.f;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const float p = mn == -INFINITY ? 0.f : exp2f(s[i][b] - mn);
                Ps[(ty * 4 + i) * PLD + tx + 16 * b] = p;
                ps += p;
            }
            l[i] = l[i] * alpha + ps;
            m[i] = mn;
#pragma unroll
            for (int c = 0; c < HD / 16; ++c) o[i][c] *= alpha;
        }
        __syncwarp();  // P rows of this thread group are written by the same half-warp
        tile_pz<HD, false>(Ps, Vs, ty, tx, o);
    }
    // epilogue
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        float lt = l[i];
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) lt += __shfl_xor_sync(0xffffffffu, lt, off);
        const int qi = q0 + ty * 4 + i;
        if (qi >= slot) continue;
        const bool ok = qi < len && lt > 0.f;
        const float inv = ok ? 1.f / lt : 0.f;
        __nv_bfloat16* dst = a.out + (long long)(start + qi) * a.ldout + h * HD;
#pragma unroll
        for (int c = 0; c < DV; ++c) {
            const __nv_bfloat162 v0 = __floats2bfloat162_rn(o[i][c * 4 + 0] * inv, o[i][c * 4 + 1] * inv);
            const __nv_bfloat162 v1 = __floats2bfloat162_rn(o[i][c * 4 + 2] * inv, o[i][c * 4 + 3] * inv);
            uint2 pk;
            pk.x = *reinterpret_cast<const uint32_t*>(&v0);
            pk.y = *reinterpret_cast<const uint32_t*>(&v1);
            *reinterpret_cast<uint2*>(dst + tx * 4 + 64 * c) = pk;
        }
        if (tx == 0) a.lse[(long long)h * a.rows + start + qi] = ok ? (m[i] + log2f(lt)) * kLn2 : 0.f;
    }
}

// dsum[h][t] = sum_d dO[t, h*HD + d] * O[t, h*HD + d]   (one warp per (row, head))
__global__ void attn_dsum_kernel(AttnArgs a, int hd) {
    pdl_prologue();
    const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (wid >= a.rows * a.heads) return;
    const long long t = wid / a.heads;
    const int h = static_cast<int>(wid % a.heads);
    const __nv_bfloat16* o = a.o + t * a.ldo + (long long)h * hd;
    const __nv_bfloat16* d = a.dO + t * a.lddo + (long long)h * hd;
    float s = 0.f;
    for (int i = lane; i < hd; i += 32) s = fmaf(__bfloat162float(o[i]), __bfloat162float(d[i]), s);
    s = warp_sum(s);
    if (lane == 0) a.dsum[(long long)h * a.rows + t] = s;
}

// P and dS of one (query tile, key tile): P = exp(scale Q K^T - lse) (causal,
// masked to 0), dS = P (dO V^T - dsum).  Written to Ps / dSs [64][PLD] (rows = queries).
template <int HD>
__device__ __forceinline__ void p_ds_tile(const float* Qs, const float* Ks, const float* dOs, const float* Vs,
                                          const float* lse2, const float* dsm, int q0, int k0, int len, float c2,
                                          float* Ps, float* dSs, int ty, int tx) {
    constexpr int PLD = Tile<HD>::PLD;
    float s[4][4], dp[4][4];
    tile_dot<HD>(Qs, Ks, ty, tx, s);
    tile_dot<HD>(dOs, Vs, ty, tx, dp);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = ty * 4 + i, qi = q0 + r;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int c = tx + 16 * b, kj = k0 + c;
            const float p = (kj <= qi && qi < len) ? exp2f(s[i][b] * c2 - lse2[r]) : 0.f;
            Ps[r * PLD + c] = p;
            dSs[r * PLD + c] = p * (dp[i][b] - dsm[r]);
        }
    }
}

// dK, dV: one CTA per (key tile, sequence, K/V head); loops over the query
// heads of its group and the query tiles at or after the key tile (causal), so
// the GQA / MQA head sum is a fixed-order register accumulation.
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_bwd_dkv_kernel(AttnArgs a) {
    pdl_prologue();
    int start, len;
    seq_range(a, blockIdx.y, start, len);
    const int slot = a.seq_off[blockIdx.y + 1] - start;
    const int k0 = blockIdx.x * kBM;
    if (k0 >= slot) return;
    const int kvh = blockIdx.z, group = a.heads / a.kv_heads;
    constexpr int LD = Tile<HD>::LD, PLD = Tile<HD>::PLD;
    extern __shared__ __align__(16) float sm[];
    float* Ks = sm;
    float* Vs = Ks + kBM * LD;
    float* Qs = Vs + kBM * LD;
    float* dOs = Qs + kBM * LD;
    float* Ps = dOs + kBM * LD;
    float* dSs = Ps + kBM * PLD;
    float* lse2 = dSs + kBM * PLD;
    float* dsm = lse2 + kBM;
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const bool rope = a.rope_base > 0.f;
    const float c2 = a.scale * kLog2e;

    load_tile<HD>(Ks, a.k, a.ldk, start, k0, len, kvh * HD, a.rope_base, rope);
    load_tile<HD>(Vs, a.v, a.ldv, start, k0, len, kvh * HD, a.rope_base, false);
    float dk[4][HD / 16], dv[4][HD / 16];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) dk[i][c] = dv[i][c] = 0.f;
    const int nqt = (len + kBM - 1) / kBM;
    for (int hh = 0; hh < group; ++hh) {
        const int h = kvh * group + hh;
        for (int qt = k0 / kBM; qt < nqt; ++qt) {
            const int q0 = qt * kBM;
            __syncthreads();
            load_tile<HD>(Qs, a.q, a.ldq, start, q0, len, h * HD, a.rope_base, rope);
            load_tile<HD>(dOs, a.dO, a.lddo, start, q0, len, h * HD, a.rope_base, false);
            for (int r = tid; r < kBM; r += blockDim.x) {
                const bool ok = q0 + r < len;
                lse2[r] = ok ? a.lse[(long long)h * a.rows + start + q0 + r] * kLog2e : 0.f;
                dsm[r] = ok ? a.dsum[(long long)h * a.rows + start + q0 + r] : 0.f;
            }
            __syncthreads();
            p_ds_tile<HD>(Qs, Ks, dOs, Vs, lse2, dsm, q0, k0, len, c2, Ps, dSs, ty, tx);
            __syncthreads();
            tile_pz<HD, true>(Ps, dOs, ty, tx, dv);   // dV[j] += sum_i P[i][j] dO[i]
            tile_pz<HD, true>(dSs, Qs, ty, tx, dk);   // dK[j] += sum_i dS[i][j] Q[i]
        }
    }
    __syncthreads();
    acc_to_smem<HD>(Ks, dk, ty, tx, a.scale);
    acc_to_smem<HD>(Vs, dv, ty, tx, 1.f);
    __syncthreads();
    store_tile<HD>(Ks, a.dk, a.lddk, start, k0, len, kvh * HD, slot, a.rope_base, rope);
    store_tile<HD>(Vs, a.dv, a.lddv, start, k0, len, kvh * HD, slot, a.rope_base, false);
}

// dQ: one CTA per (query tile, sequence, head); loops over key tiles 0..qt.
template <int HD>
__global__ void __launch_bounds__(kThreads) attn_bwd_dq_kernel(AttnArgs a) {
    pdl_prologue();
    int start, len;
    seq_range(a, blockIdx.y, start, len);
    const int slot = a.seq_off[blockIdx.y + 1] - start;
    const int q0 = blockIdx.x * kBM;
    if (q0 >= slot) return;
    const int h = blockIdx.z, kvh = h / (a.heads / a.kv_heads);
    constexpr int LD = Tile<HD>::LD, PLD = Tile<HD>::PLD;
    extern __shared__ __align__(16) float sm[];
    float* Qs = sm;
    float* dOs = Qs + kBM * LD;
    float* Ks = dOs + kBM * LD;
    float* Vs = Ks + kBM * LD;
    float* Ps = Vs + kBM * LD;
    float* dSs = Ps + kBM * PLD;
    float* lse2 = dSs + kBM * PLD;
    float* dsm = lse2 + kBM;
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const bool rope = a.rope_base > 0.f;
    const float c2 = a.scale * kLog2e;

    load_tile<HD>(Qs, a.q, a.ldq, start, q0, len, h * HD, a.rope_base, rope);
    load_tile<HD>(dOs, a.dO, a.lddo, start, q0, len, h * HD, a.rope_base, false);
    for (int r = tid; r < kBM; r += blockDim.x) {
        const bool ok = q0 + r < len;
        lse2[r] = ok ? a.lse[(long long)h * a.rows + start + q0 + r] * kLog2e : 0.f;
        dsm[r] = ok ? a.dsum[(long long)h * a.rows + start + q0 + r] : 0.f;
    }
    float dq[4][HD / 16];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int c = 0; c < HD / 16; ++c) dq[i][c] = 0.f;
    const int nkt = q0 < len ? (min(q0 + kBM, len) + kBM - 1) / kBM : 0;
    for (int kt = 0; kt < nkt; ++kt) {
        __syncthreads();
        load_tile<HD>(Ks, a.k, a.ldk, start, kt * kBM, len, kvh * HD, a.rope_base, rope);
        load_tile<HD>(Vs, a.v, a.ldv, start, kt * kBM, len, kvh * HD, a.rope_base, false);
        __syncthreads();
        p_ds_tile<HD>(Qs, Ks, dOs, Vs, lse2, dsm, q0, kt * kBM, len, c2, Ps, dSs, ty, tx);
        __syncwarp();  // dS rows of this thread group are written by the same half-warp
        tile_pz<HD, false>(dSs, Ks, ty, tx, dq);  // dQ[i] += sum_j dS[i][j] K[j]
    }
    __syncthreads();
    acc_to_smem<HD>(Qs, dq, ty, tx, a.scale);
    __syncthreads();
    store_tile<HD>(Qs, a.dq, a.lddq, start, q0, len, h * HD, slot, a.rope_base, rope);
}

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
    return cudaLaunchKernelEx(&cfg, k, args...);
}

mlora_status check_attn(const mlora_attn_desc* d) {
    if (!d || !d->seq_offsets || d->num_seqs < 1 || d->max_len < 1 || d->rows < 1) return MLORA_USAGE;
    if (d->heads < 1 || d->kv_heads < 1 || d->heads % d->kv_heads != 0) return MLORA_SHAPE;
    if (d->head_dim != 64 && d->head_dim != 128) return MLORA_SHAPE;
    if (d->rope_base != 0.f && !(d->rope_base > 1.f)) return MLORA_USAGE;
    if (!(d->softmax_scale > 0.f)) return MLORA_USAGE;
    return MLORA_OK;
}

bool ld_ok(long long ld, int cols) { return ld >= cols && (ld % 2) == 0; }

AttnArgs attn_args(const mlora_attn_desc* d) {
    AttnArgs a{};
    a.seq_off = d->seq_offsets;
    a.seq_len = d->seq_lens;
    a.heads = d->heads;
    a.kv_heads = d->kv_heads;
    a.rope_base = d->rope_base;
    a.scale = d->softmax_scale;
    a.rows = d->rows;
    return a;
}

template <typename K>
cudaError_t launch_attn(K kernel, const mlora_attn_desc* d, int heads_z, size_t smem, void* stream,
                        const AttnArgs& a) {
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) !=
        cudaSuccess)
        return cudaErrorInvalidValue;
    const dim3 grid((d->max_len + kBM - 1) / kBM, d->num_seqs, heads_z);
    return launch(kernel, grid, dim3(kThreads), smem, stream, a);
}

}  // namespace

extern "C" {

mlora_status mlora_embed(int64_t rows, int32_t h, int32_t V, const int32_t* tokens, const void* E, void* x,
                         void* stream) {
    if (rows < 1 || h < 8 || (h % 8) || V < 1 || !tokens || !E || !x) return MLORA_USAGE;
    return launch(embed_kernel, dim3(static_cast<unsigned>(rows)), dim3(128), 0, stream, tokens,
                  static_cast<const uint4*>(E), static_cast<int>(h / 8), static_cast<uint4*>(x)) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

mlora_status mlora_add_rmsnorm(int64_t rows, int32_t h, const void* x, const void* delta, const void* w, float eps,
                               void* x_out, void* y, float* rstd, void* stream) {
    if (rows < 1 || h < 1 || !x || !w || !y || !rstd || (delta && !x_out) || !(eps > 0.f)) return MLORA_USAGE;
    return launch(add_rmsnorm_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, stream, bf(x), bf(delta), bf(w),
                  static_cast<int>(h), eps, bfw(x_out), bfw(y), rstd) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

mlora_status mlora_rmsnorm_bwd_sum(int64_t rows, int32_t h, int32_t n_dy, const void* const* dy, const void* dres,
                                   const void* x, const void* w, const float* rstd, void* dx, void* stream) {
    if (rows < 1 || h < 1 || n_dy < 1 || n_dy > 4 || !dy || !x || !w || !rstd || !dx) return MLORA_USAGE;
    SumArgs a{};
    for (int i = 0; i < n_dy; ++i) {
        if (!dy[i]) return MLORA_USAGE;
        a.dy[i] = bf(dy[i]);
    }
    a.n = n_dy;
    return launch(rmsnorm_bwd_sum_kernel, dim3(static_cast<unsigned>(rows)), dim3(256), 0, stream, a, bf(dres), bf(x),
                  bf(w), rstd, static_cast<int>(h), bfw(dx)) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

mlora_status mlora_swiglu_fwd(int64_t rows, int32_t f, const void* gate, int64_t ld_gate, const void* up,
                              int64_t ld_up, void* out, void* stream) {
    if (rows < 1 || f < 1 || !gate || !up || !out || ld_gate < f || ld_up < f) return MLORA_USAGE;
    const long long n = rows * (long long)f;
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148LL * 16));
    return launch(swiglu_fwd_kernel, dim3(blocks), dim3(256), 0, stream, n, static_cast<int>(f), bf(gate),
                  static_cast<long long>(ld_gate), bf(up), static_cast<long long>(ld_up), bfw(out)) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

mlora_status mlora_swiglu_bwd(int64_t rows, int32_t f, const void* gate, int64_t ld_gate, const void* up,
                              int64_t ld_up, const void* dout, void* dgate, int64_t ld_dgate, void* dup,
                              int64_t ld_dup, void* stream) {
    if (rows < 1 || f < 1 || !gate || !up || !dout || !dgate || !dup || ld_gate < f || ld_up < f || ld_dgate < f ||
        ld_dup < f)
        return MLORA_USAGE;
    const long long n = rows * (long long)f;
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148LL * 16));
    return launch(swiglu_bwd_kernel, dim3(blocks), dim3(256), 0, stream, n, static_cast<int>(f), bf(gate),
                  static_cast<long long>(ld_gate), bf(up), static_cast<long long>(ld_up), bf(dout), bfw(dgate),
                  static_cast<long long>(ld_dgate), bfw(dup), static_cast<long long>(ld_dup)) == cudaSuccess
               ? MLORA_OK
               : MLORA_CUDA;
}

mlora_status mlora_attn_fwd(const mlora_attn_desc* d, const void* q, int64_t ldq, const void* k, int64_t ldk,
                            const void* v, int64_t ldv, void* o, int64_t ldo, float* lse, void* stream) {
    mlora_status st = check_attn(d);
    if (st != MLORA_OK) return st;
    if (!q || !k || !v || !o || !lse) return MLORA_USAGE;
    const int hd = d->head_dim;
    if (!ld_ok(ldq, d->heads * hd) || !ld_ok(ldk, d->kv_heads * hd) || !ld_ok(ldv, d->kv_heads * hd) ||
        !ld_ok(ldo, d->heads * hd))
        return MLORA_SHAPE;
    AttnArgs a = attn_args(d);
    a.q = bf(q), a.k = bf(k), a.v = bf(v), a.out = bfw(o);
    a.ldq = ldq, a.ldk = ldk, a.ldv = ldv, a.ldout = ldo;
    a.lse = lse;
    const cudaError_t e = hd == 64 ? launch_attn(attn_fwd_kernel<64>, d, d->heads, attn_smem_fwd<64>(), stream, a)
                                   : launch_attn(attn_fwd_kernel<128>, d, d->heads, attn_smem_fwd<128>(), stream, a);
    return e == cudaSuccess ? MLORA_OK : MLORA_CUDA;
}

mlora_status mlora_attn_bwd(const mlora_attn_desc* d, const void* q, int64_t ldq, const void* k, int64_t ldk,
                            const void* v, int64_t ldv, const void* o, int64_t ldo, const void* dout, int64_t lddo,
                            const float* lse, float* dsum, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                            int64_t lddv, void* stream) {
    mlora_status st = check_attn(d);
    if (st != MLORA_OK) return st;
    if (!q || !k || !v || !o || !dout || !lse || !dsum || !dq || !dk || !dv) return MLORA_USAGE;
    const int hd = d->head_dim, qc = d->heads * hd, kc = d->kv_heads * hd;
    if (!ld_ok(ldq, qc) || !ld_ok(ldk, kc) || !ld_ok(ldv, kc) || !ld_ok(ldo, qc) || !ld_ok(lddo, qc) ||
        !ld_ok(lddq, qc) || !ld_ok(lddk, kc) || !ld_ok(lddv, kc))
        return MLORA_SHAPE;
    AttnArgs a = attn_args(d);
    a.q = bf(q), a.k = bf(k), a.v = bf(v), a.o = bf(o), a.dO = bf(dout);
    a.ldq = ldq, a.ldk = ldk, a.ldv = ldv, a.ldo = ldo, a.lddo = lddo;
    a.dq = bfw(dq), a.dk = bfw(dk), a.dv = bfw(dv);
    a.lddq = lddq, a.lddk = lddk, a.lddv = lddv;
    a.lse = const_cast<float*>(lse);
    a.dsum = dsum;
    const long long warps = d->rows * d->heads;
    if (launch(attn_dsum_kernel, dim3(static_cast<unsigned>((warps * 32 + 255) / 256)), dim3(256), 0, stream, a,
               hd) != cudaSuccess)
        return MLORA_CUDA;
    cudaError_t e;
    if (hd == 64) {
        e = launch_attn(attn_bwd_dkv_kernel<64>, d, d->kv_heads, attn_smem_bwd<64>(), stream, a);
        if (e == cudaSuccess) e = launch_attn(attn_bwd_dq_kernel<64>, d, d->heads, attn_smem_bwd<64>(), stream, a);
    } else {
        e = launch_attn(attn_bwd_dkv_kernel<128>, d, d->kv_heads, attn_smem_bwd<128>(), stream, a);
        if (e == cudaSuccess) e = launch_attn(attn_bwd_dq_kernel<128>, d, d->heads, attn_smem_bwd<128>(), stream, a);
    }
    return e == cudaSuccess ? MLORA_OK : MLORA_CUDA;
}

}  // extern "C"
