// mlora_capi.cu — host side of the C ABI declared in include/mlora.h.
//
// Owns: the per-device context (TMA descriptor cache, grow-only workspace,
// launch telemetry), the fused-batch plan (segment tables uploaded once per
// step), and the launch logic of the tcgen05 kernels in mlora_gemm.cuh.
// Every reference precondition is validated here, on the host, before any
// device work.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/mlora.h"
#include <nvtx3/nvToolsExt.h>

#include "mlora_aux.cuh"
#include "mlora_gemm.cuh"
#include "mlora_down_multi.cuh"

using namespace mlora;

namespace {

thread_local std::string g_last_error;

constexpr int kMaxSplit = 8;
constexpr int kBaseStages = 4;
constexpr int kSmallStages = 4;

using GemmLayoutBase = GemmSmem<256, kBaseStages>;
using GemmLayoutSmall = GemmSmem<64, kSmallStages>;

}  // namespace

struct mlora_ctx {
    int device = 0;
    int num_sms = 0;
    PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    std::map<std::tuple<const void*, uint64_t, uint64_t, uint64_t, uint32_t, uint32_t>, CUtensorMap> tmaps;
    void* workspace = nullptr;
    size_t workspace_bytes = 0;
    long long launches = 0;
    std::string last_error;
    // optional live per-kernel timing: (kind, start, stop) event pairs recorded on
    // the launch stream around every launch while profiling is on
    bool profiling = false;
    std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> prof_pending;
    std::vector<cudaEvent_t> event_pool;
    double prof_ms[8] = {0};
    long long prof_count[8] = {0};
    cudaEvent_t timer[2] = {nullptr, nullptr};  // mlora_ctx_timer_start / _stop
};

struct mlora_plan {
    mlora_ctx* ctx = nullptr;
    int J = 0;
    int rows = 0;
    int R_pad = 0;
    int n_mblk = 0;
    int n_chunks = 0;
    std::vector<int> seg, roff, rank;
    std::vector<float> scale;
    std::vector<int> ext;                 // [n_mblk][2]   (128-row m-blocks)
    std::vector<int> ext256;              // [n_mblk256][2] (256-row m-blocks of the CTA-pair kernel)
    std::vector<int> grp256;              // [n_mblk256][2] 16-column rank groups [lo, hi) of the jobs present
    int n_mblk256 = 0;
    std::vector<int> down;                // [n_down][3]
    int n_down = 0;
    int down_groups_max = 1;              // widest down tile, in 16-row rank groups
    std::vector<int> chunk_kb;            // [n_chunks][2] token k-block range
    int grad_off[kMaxSplit + 1] = {0};    // offset (ints) of the split-ns table
    // device copies (one allocation, grow-only) and the pinned staging of their upload
    void* dev = nullptr;
    size_t dev_bytes = 0;
    void* staging = nullptr;
    size_t staging_bytes = 0;
    cudaEvent_t staging_done = nullptr;
    int* d_seg = nullptr;
    int* d_roff = nullptr;
    float* d_scale = nullptr;
    int* d_ext = nullptr;
    int* d_ext256 = nullptr;
    int* d_grp256 = nullptr;
    int* d_down = nullptr;
    int* d_grad = nullptr;
};

namespace {

mlora_status fail(mlora_ctx* ctx, mlora_status st, const std::string& msg) {
    g_last_error = msg;
    if (ctx) ctx->last_error = msg;
    return st;
}

#define MLORA_CUDA_TRY(ctx, expr)                                                       \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            return fail(ctx, MLORA_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

inline int cdiv(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// 2-D bf16 tensor map, SWIZZLE_128B, OOB -> zero fill.
mlora_status get_tmap(mlora_ctx* ctx, const void* ptr, uint64_t inner, uint64_t outer,
                      uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer, CUtensorMap* out) {
    auto key = std::make_tuple(ptr, inner, outer, ld_elems, box_inner, box_outer);
    auto it = ctx->tmaps.find(key);
    if (it != ctx->tmaps.end()) {
        *out = it->second;
        return MLORA_OK;
    }
    if (reinterpret_cast<uintptr_t>(ptr) % 16 != 0)
        return fail(ctx, MLORA_USAGE, "tensor base pointer must be 16-byte aligned");
    CUtensorMap m;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {ld_elems * 2};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = ctx->encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return fail(ctx, MLORA_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    if (ctx->tmaps.size() > 4096) ctx->tmaps.clear();
    ctx->tmaps.emplace(key, m);
    *out = m;
    return MLORA_OK;
}

mlora_status ensure_workspace(mlora_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->workspace_bytes) return MLORA_OK;
    if (ctx->workspace) {
        cudaDeviceSynchronize();
        cudaFree(ctx->workspace);
        ctx->workspace = nullptr;
        ctx->workspace_bytes = 0;
    }
    MLORA_CUDA_TRY(ctx, cudaMalloc(&ctx->workspace, bytes));
    ctx->workspace_bytes = bytes;
    return MLORA_OK;
}

// Every kernel goes through cudaLaunchKernelEx with programmatic stream
// serialisation (PDL): the next kernel's prologue overlaps this one's tail; the
// kernels themselves griddepcontrol.wait before their first global access.
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     unsigned cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    unsigned n = 0;
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = cluster_x;
        attr[n].val.clusterDim.y = 1;
        attr[n].val.clusterDim.z = 1;
        ++n;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

cudaEvent_t pool_event(mlora_ctx* ctx) {
    if (!ctx->event_pool.empty()) {
        cudaEvent_t e = ctx->event_pool.back();
        ctx->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Kernel kinds for the live profile: 0 base fwd, 1 base dX, 2 down (H/G), 3 grad (dA/dB),
// 4 aux (reduce/pack/adam/loss).
// Every launch site opens one: an NVTX range named after the kernel kind (free
// unless a profiler is attached — nsys/ncu timelines then group the launches
// per op), plus, while live profiling is on, a CUDA-event pair on the stream.
struct ProfScope {
    mlora_ctx* ctx;
    int kind;
    cudaStream_t stream;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(mlora_ctx* c, int k, cudaStream_t s) : ctx(c), kind(k), stream(s) {
        static const char* const kNames[] = {"mlora.base_fwd", "mlora.base_dx", "mlora.down",
                                             "mlora.grad",     "mlora.aux",     "mlora.adam"};
        nvtxRangePushA(kind >= 0 && kind < 6 ? kNames[kind] : "mlora");
        if (ctx->profiling) {
            a = pool_event(ctx);
            b = pool_event(ctx);
            cudaEventRecord(a, stream);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEventRecord(b, stream);
            ctx->prof_pending.emplace_back(kind, a, b);
        }
        nvtxRangePop();
    }
};

// cudaFuncAttributeMaxDynamicSharedMemorySize is per (kernel, device): opt in
// once per pair, under a lock (contexts on several devices / threads share the
// process's kernels).
mlora_status ensure_smem_attr(mlora_ctx* ctx, const void* kern, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({kern, ctx->device})) return MLORA_OK;
    MLORA_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.insert({kern, ctx->device});
    return MLORA_OK;
}

constexpr int kGroupMax = 8;  // problems per grouped launch (a transformer layer has <= 7 LoRA'd projections)

// Accumulates the problems of one (possibly grouped) launch.
template <int NP>
struct ProblemSet {
    GemmProblemSet<NP> ps{};
    bool add(const CUtensorMap& a0, const CUtensorMap& b0, const CUtensorMap& a1, const CUtensorMap& b1,
             const GemmParams& p) {
        if (ps.nprobs >= NP) return false;
        GemmProblem& g = ps.prob[ps.nprobs++];
        g.tmA0 = a0;
        g.tmB0 = b0;
        g.tmA1 = a1;
        g.tmB1 = b1;
        g.p = p;
        g.tile_begin = ps.total_tiles;
        ps.total_tiles += p.num_tiles;
        return true;
    }
};

// One launch of the 1-CTA (KSPLIT=1) or K-split-pair (KSPLIT=2) tcgen05 kernel over a problem set.
template <int MODE, int BN, int STAGES, bool A_MN, bool B_MN, int KSPLIT, int NP>
mlora_status launch_gemm(mlora_ctx* ctx, const ProblemSet<NP>& set, int ctas_per_sm, cudaStream_t stream) {
    if (set.ps.total_tiles <= 0) return MLORA_OK;
    using L = GemmSmem<BN, STAGES, KSPLIT>;
    auto kern = mlora_gemm_kernel<MODE, BN, STAGES, A_MN, B_MN, KSPLIT, NP>;
    mlora_status st = ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), L::kDynBytes);
    if (st != MLORA_OK) return st;
    // a persistent grid with the same number of tiles per unit: ceil(tiles / units) rounds
    // either way, but no final round with a few units streaming alone (C2: the dB group's
    // 332 tiles on 166 CTAs instead of 296, 124.3 -> 111.5 us; the G group's 448 tiles on
    // 64 pairs instead of 74, 119.7 -> 117.0 us)
    const int max_units = ctx->num_sms * ctas_per_sm / KSPLIT;
    const int rounds = (set.ps.total_tiles + max_units - 1) / max_units;
    const int units = (set.ps.total_tiles + rounds - 1) / rounds;
    ProfScope ps(ctx, MODE == MODE_DOWN ? 2 : 3, stream);
    MLORA_CUDA_TRY(ctx, launch_k(kern, dim3(units * KSPLIT), dim3(kNumThreads), L::kDynBytes, stream, KSPLIT,
                                 set.ps));
    ++ctx->launches;
    return MLORA_OK;
}

constexpr int kPairStages = 6;

template <bool B_MN>
mlora_status launch_base_pair(mlora_ctx* ctx, const CUtensorMap& a0, const CUtensorMap& b0,
                              const CUtensorMap& a1, const CUtensorMap& b1, const CUtensorMap& o,
                              const GemmParams& p, cudaStream_t stream) {
    if (p.num_tiles <= 0) return MLORA_OK;
    using L = PairSmem<kPairStages>;
    auto kern = mlora_base_pair_kernel<kPairStages, B_MN>;
    mlora_status st = ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), L::kDynBytes);
    if (st != MLORA_OK) return st;
    const int clusters = std::min(p.num_tiles, ctx->num_sms / 2);
    ProfScope ps(ctx, B_MN ? 1 : 0, stream);
    MLORA_CUDA_TRY(ctx, launch_k(kern, dim3(2 * clusters), dim3(kNumThreads), L::kDynBytes, stream, 1, a0, b0,
                                 a1, b1, o, p));
    ++ctx->launches;
    return MLORA_OK;
}

// Frozen-base GEMM + LoRA k-blocks (forward: B_MN=false; dX: B_MN=true), on
// the CTA-pair kernel.
template <bool B_MN>
mlora_status run_base(mlora_ctx* ctx, const mlora_plan* plan, const void* A0, int64_t lda0, int K0,
                      const void* B0, const void* A1, const void* B1, int R, int N, void* out,
                      cudaStream_t s, float* row_sq = nullptr) {
    const int M = plan->rows;
    constexpr uint32_t bbox = 128;  // K-major B rows staged per TMA box (one CTA's half of the pair's 256)
    // A1 == B1 == NULL: no LoRA term (frozen GEMM, e.g. an LM head): no extra
    // k-blocks (ext_tab == NULL), tA1/tB1 are never read.
    const bool lora = A1 != nullptr;
    CUtensorMap tA0, tB0, tA1, tB1;
    mlora_status st;
    if ((st = get_tmap(ctx, A0, K0, M, lda0, 64, 128, &tA0)) != MLORA_OK) return st;
    if (lora && (st = get_tmap(ctx, A1, R, M, R, 64, 128, &tA1)) != MLORA_OK) return st;
    if (!B_MN) {
        // B0 = W0 [N=d, K0=k], B1 = B_cat [N=d, R]
        if ((st = get_tmap(ctx, B0, K0, N, K0, 64, bbox, &tB0)) != MLORA_OK) return st;
        if (lora && (st = get_tmap(ctx, B1, R, N, R, 64, bbox, &tB1)) != MLORA_OK) return st;
    } else {
        // B0 = W0 [K0=d, N=k] (n contiguous), B1 = A_cat [R, N=k]
        if ((st = get_tmap(ctx, B0, N, K0, N, 64, 64, &tB0)) != MLORA_OK) return st;
        if (lora && (st = get_tmap(ctx, B1, N, R, N, 64, 64, &tB1)) != MLORA_OK) return st;
    }
    if (!lora) {
        tA1 = tA0;
        tB1 = tB0;
    }
    CUtensorMap tOut;  // the epilogue's TMA store: 64-column x 32-row boxes of C [M, N]
    if ((st = get_tmap(ctx, out, N, M, N, 64, 32, &tOut)) != MLORA_OK) return st;
    GemmParams pb{};
    pb.M = M;
    pb.N = N;
    pb.num_kb = cdiv(K0, kBK);
    pb.out = out;
    pb.ldo = N;
    pb.seg = plan->d_seg;
    pb.roff = plan->d_roff;
    pb.scale = plan->d_scale;
    pb.num_jobs = plan->J;
    pb.row_sq = row_sq;
    // Raster.  K <= 8192: super-rows of m-blocks whose A slab (~32 MB) stays L2-resident
    // while all of B streams past it, at least a square wave (8 m-blocks x ~9 n-blocks for
    // the 74 concurrent tiles).  K > 8192 (5.6 MB slabs at K = 11008: the 74 tiles in
    // flight span ~100 MB): super-columns of 8 n-blocks, n fastest — the W0 slabs (kept
    // with evict_last) stay resident while the A slabs stream past them, which cuts the
    // launch's DRAM reads 839 -> 740 MB (ncu sweeps, profiles/r02_raster_k11008.md)
    const long long slab = (long long)kPairBM * K0 * 2;
    pb.raster_group = K0 > 8192 ? -8 : static_cast<int>(std::max<long long>(8, (32LL << 20) / slab));
    // W0 with an L2 evict_last policy: measured on one B200 (profiles/r02_l2_policy.md,
    // tools/step_probe.py, interleaved A/B): C2 step 4.93 -> 4.79 ms rested, 5.23 -> 5.07
    // ms in a 20-step burst, 5.69 -> 5.42 J per step sustained
    pb.keep_b_in_l2 = 1;
    pb.n_mblk = plan->n_mblk256;
    pb.n_nblk = cdiv(N, kPairBN);
    pb.num_tiles = pb.n_mblk * pb.n_nblk;
    pb.ext_tab = lora ? plan->d_ext256 : nullptr;
    pb.ext_grp = lora ? plan->d_grp256 : nullptr;
    return launch_base_pair<B_MN>(ctx, tA0, tB0, tA1, tB1, tOut, pb, s);
}

constexpr int kDownStages = 6;

template <int NB>
mlora_status launch_down_multi(mlora_ctx* ctx, const mlora_plan* plan, int K, const void* x,
                               const void* const* bop, void* const* out, cudaStream_t s) {
    using L = DownMultiSmem;
    static_assert(L::kDynBytes <= 232448, "shared memory budget");
    const int M = plan->rows, R = plan->R_pad;
    DownMultiArgs<NB> a{};
    mlora_status st;
    if ((st = get_tmap(ctx, x, K, M, K, 64, 128, &a.tmA)) != MLORA_OK) return st;
    for (int b = 0; b < NB; ++b) {
        if ((st = get_tmap(ctx, bop[b], K, R, K, 64, 16, &a.tmB[b])) != MLORA_OK) return st;
        a.out[b] = out[b];
    }
    // ring sized for the plan's widest tile (16-row rank groups of the jobs present)
    a.stage_bytes = L::stage_bytes(NB, plan->down_groups_max);
    a.stages = L::stages_for(a.stage_bytes);
    GemmParams& p = a.p;
    p.M = M;
    p.N = R;
    p.num_kb = cdiv(K, kBK);
    p.n_mblk = plan->n_mblk;
    p.num_tiles = plan->n_down;
    p.ldo = R;
    p.ext_tab = plan->d_ext;
    p.down_tab = plan->d_down;
    p.seg = plan->d_seg;
    p.roff = plan->d_roff;
    p.scale = plan->d_scale;
    p.num_jobs = plan->J;
    if (p.num_tiles <= 0) return MLORA_OK;
    auto kern = mlora_down_multi_kernel<NB>;
    if ((st = ensure_smem_attr(ctx, reinterpret_cast<const void*>(kern), L::kDynBytes)) != MLORA_OK) return st;
    const int clusters = std::min(p.num_tiles, ctx->num_sms / 2);
    ProfScope ps(ctx, 2, s);
    MLORA_CUDA_TRY(ctx, launch_k(kern, dim3(2 * clusters), dim3(kNumThreads), L::kDynBytes, s, 2, a));
    ++ctx->launches;
    return MLORA_OK;
}

mlora_status launch_down_multi_n(mlora_ctx* ctx, const mlora_plan* plan, int nb, int K, const void* x,
                                 const void* const* bop, void* const* out, cudaStream_t s) {
    switch (nb) {
        case 2: return launch_down_multi<2>(ctx, plan, K, x, bop, out, s);
        case 3: return launch_down_multi<3>(ctx, plan, K, x, bop, out, s);
        case 4: return launch_down_multi<4>(ctx, plan, K, x, bop, out, s);
        case 5: return launch_down_multi<5>(ctx, plan, K, x, bop, out, s);
        default: return fail(ctx, MLORA_USAGE, "shared-input group size out of range");
    }
}

// Rank-r down-projections of n projections in ONE launch (K split across CTA
// pairs, DSMEM reduction):  out_i = s_j in_i Bop_i^T, block-diagonal.
//   forward (B_MN=false): in = X_i [rows, K_i], Bop = A_cat_i [R, K_i]  -> H_i
//   backward (B_MN=true): in = dY_i [rows, K_i = d_i], Bop = B_cat_i [K_i, R] -> G_i
template <bool B_MN>
mlora_status run_down_group(mlora_ctx* ctx, const mlora_plan* plan, int n, const int32_t* K,
                            const void* const* in, const void* const* bop, void* const* out, cudaStream_t s) {
    const int M = plan->rows, R = plan->R_pad;
    for (int i = 0; i < n; ++i) {
        if (!in[i] || !bop[i] || !out[i]) return fail(ctx, MLORA_USAGE, "null tensor pointer");
        if (K[i] <= 0 || K[i] % 8) return fail(ctx, MLORA_SHAPE, "down-projection width must be a positive multiple of 8");
    }
    // Forward: projections reading the same input (q, k, v, gate, up <- x) go
    // through the shared-input kernel, up to 5 per launch — x enters the SMs once
    // per rank chunk instead of once per projection.
    std::vector<int> order;
    std::vector<bool> taken(n, false);
    for (int i = 0; i < n; ++i) {
        if (taken[i]) continue;
        std::vector<int> same{i};
        if (!B_MN)
            for (int j = i + 1; j < n; ++j)
                if (!taken[j] && in[j] == in[i] && K[j] == K[i]) same.push_back(j);
        if (same.size() < 2) {
            order.push_back(i);
            continue;
        }
        for (size_t c0 = 0; c0 < same.size(); c0 += kDownMultiMax) {
            const int nb = static_cast<int>(std::min<size_t>(kDownMultiMax, same.size() - c0));
            if (nb == 1) {
                order.push_back(same[c0]);
                continue;
            }
            const void* bops[kDownMultiMax];
            void* outs[kDownMultiMax];
            for (int b = 0; b < nb; ++b) {
                bops[b] = bop[same[c0 + b]];
                outs[b] = out[same[c0 + b]];
            }
            mlora_status st = launch_down_multi_n(ctx, plan, nb, K[i], in[i], bops, outs, s);
            if (st != MLORA_OK) return st;
        }
        for (int j : same) taken[j] = true;
    }
    // Everything else: one grouped launch, one problem per projection.  Tile
    // order: equal widths interleave the problems tile by tile (projections fed
    // by one hidden state stream it concurrently and share L2); mixed widths
    // run back to back, widest first — interleaving would hand each cluster
    // tiles of a single problem whenever the cluster count is a multiple of the
    // problem count (74 clusters, 2 problems: one half of the grid gets every
    // 11008-wide tile), a 2.7x load imbalance.
    const int nrest = static_cast<int>(order.size());
    bool same_k = true;
    for (int oi = 1; oi < nrest; ++oi) same_k = same_k && K[order[oi]] == K[order[0]];
    if (!same_k) std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return K[x] > K[y]; });
    for (int i0 = 0; i0 < nrest; i0 += kGroupMax) {
        ProblemSet<kGroupMax> set;
        for (int oi = i0; oi < std::min(nrest, i0 + kGroupMax); ++oi) {
            const int i = order[oi];
            CUtensorMap tA, tB, tB16;
            mlora_status st;
            if ((st = get_tmap(ctx, in[i], K[i], M, K[i], 64, 128, &tA)) != MLORA_OK) return st;
            if (!B_MN) st = get_tmap(ctx, bop[i], K[i], R, K[i], 64, 64, &tB);   // A_cat [R, K] K-major
            else st = get_tmap(ctx, bop[i], R, K[i], R, 64, 64, &tB);            // B_cat [K, R] MN-major
            if (st != MLORA_OK) return st;
            // forward: A_cat loaded by 16-row rank groups (only the m-block's jobs', down_group_lo/hi)
            tB16 = tB;
            if (!B_MN && (st = get_tmap(ctx, bop[i], K[i], R, K[i], 64, 16, &tB16)) != MLORA_OK) return st;
            GemmParams p{};
            p.M = M;
            p.N = R;
            p.num_kb = cdiv(K[i], kBK);
            p.n_mblk = plan->n_mblk;
            p.num_tiles = plan->n_down;
            p.out = out[i];
            p.ldo = R;
            p.ext_tab = plan->d_ext;
            p.down_tab = plan->d_down;
            p.seg = plan->d_seg;
            p.roff = plan->d_roff;
            p.scale = plan->d_scale;
            p.num_jobs = plan->J;
            set.add(tA, tB, tA, tB16, p);
        }
        set.ps.interleave = same_k ? 1 : 0;
        mlora_status st = launch_gemm<MODE_DOWN, 64, kDownStages, false, B_MN, 2, kGroupMax>(ctx, set, 1, s);
        if (st != MLORA_OK) return st;
    }
    return MLORA_OK;
}

mlora_status check_dims(mlora_ctx* ctx, const mlora_plan* plan, int d, int k) {
    if (!ctx || !plan) return fail(ctx, MLORA_USAGE, "null context or plan");
    if (plan->ctx != ctx) return fail(ctx, MLORA_USAGE, "plan belongs to another context");
    if (d <= 0 || k <= 0 || d % 8 != 0 || k % 8 != 0)
        return fail(ctx, MLORA_SHAPE, "d and k must be positive multiples of 8 (TMA 16-byte rows), got d=" +
                                          std::to_string(d) + " k=" + std::to_string(k));
    return MLORA_OK;
}

// Segmented gradient reductions of n projections in one launch:
//   MODE_GRADT: dA_cat_i [R, F_i=k_i] = G_i^T X_i   (a = X_i, b = G_i)
//   MODE_GRAD : dB_cat_i [F_i=d_i, R] = dY_i^T H_i  (a = dY_i, b = H_i)
// each 64-column rank chunk reduced over its jobs' token range only.  The token
// range is split (same split count for the whole group) only as far as needed
// to give ~1 tile per SM; split partials are summed in a fixed order by one
// grouped reduce launch (deterministic, no atomics).
template <int MODE>
mlora_status run_grad_group(mlora_ctx* ctx, const mlora_plan* plan, int n, const int32_t* F,
                            const void* const* a, const void* const* b, float* const* out, cudaStream_t s) {
    const int M = plan->rows, R = plan->R_pad;
    long long base = 0;
    for (int i = 0; i < n; ++i) {
        if (!a[i] || !b[i] || !out[i]) return fail(ctx, MLORA_USAGE, "null tensor pointer");
        if (F[i] <= 0 || F[i] % 8) return fail(ctx, MLORA_SHAPE, "gradient width must be a positive multiple of 8");
        base += (long long)cdiv(F[i], kBM) * plan->n_chunks;
    }
    // split only below one tile per SM: at C2 the dA group (278 tiles) unsplit runs in
    // 59.7 us reading 322 MB, split in two 71.1 us + a 9.3 us reduce reading 389 MB (ncu)
    const long long want = ctx->num_sms;
    int ns = static_cast<int>(std::max<long long>(1, (want + base - 1) / std::max<long long>(base, 1)));
    int max_len = 1;
    for (int c = 0; c < plan->n_chunks; ++c)
        max_len = std::max(max_len, plan->chunk_kb[2 * c + 1] - plan->chunk_kb[2 * c]);
    ns = std::min({ns, std::max(1, max_len / 4), kMaxSplit});
    std::vector<long long> part_off(n + 1, 0);
    for (int i = 0; i < n; ++i) part_off[i + 1] = part_off[i] + (ns > 1 ? (long long)ns * F[i] * R : 0);
    if (ns > 1) {
        mlora_status st = ensure_workspace(ctx, sizeof(float) * part_off[n]);
        if (st != MLORA_OK) return st;
    }
    float* ws = static_cast<float*>(ctx->workspace);
    for (int i0 = 0; i0 < n; i0 += kGroupMax) {
        ProblemSet<kGroupMax> set;
        ReduceGroupArgs red{};
        for (int i = i0; i < std::min(n, i0 + kGroupMax); ++i) {
            CUtensorMap tA, tB;
            mlora_status st;
            if ((st = get_tmap(ctx, a[i], F[i], M, F[i], 64, 64, &tA)) != MLORA_OK) return st;  // MN-major
            if ((st = get_tmap(ctx, b[i], R, M, R, 64, 64, &tB)) != MLORA_OK) return st;        // MN-major
            const long long nelem = (long long)F[i] * R;
            GemmParams p{};
            p.M = F[i];
            p.N = R;
            p.n_mblk = cdiv(F[i], kBM);
            p.nsplit = ns;
            p.num_tiles = p.n_mblk * plan->n_chunks * ns;
            p.out = ns > 1 ? static_cast<void*>(ws + part_off[i]) : static_cast<void*>(out[i]);
            p.ldo = (MODE == MODE_GRADT) ? F[i] : R;
            p.split_stride = nelem;
            p.grad_tab = plan->d_grad + plan->grad_off[ns];
            p.seg = plan->d_seg;
            p.roff = plan->d_roff;
            p.scale = plan->d_scale;
            p.num_jobs = plan->J;
            set.add(tA, tB, tA, tB, p);
            ReduceGroupArgs::Item& it = red.item[red.n++];
            it.part = reinterpret_cast<const float4*>(ws + part_off[i]);
            it.out = reinterpret_cast<float4*>(out[i]);
            it.n4 = nelem / 4;
            it.start4 = red.total4;
            red.total4 += it.n4;
        }
        mlora_status st = launch_gemm<MODE, 64, kSmallStages, true, true, 1, kGroupMax>(ctx, set, 2, s);
        if (st != MLORA_OK) return st;
        if (ns > 1) {
            red.nsplit = ns;
            const int blocks = static_cast<int>(std::min<long long>(cdiv(red.total4, 256), 8LL * ctx->num_sms));
            ProfScope ps(ctx, 4, s);
            MLORA_CUDA_TRY(ctx, launch_k(reduce_splits_group_kernel, dim3(blocks), dim3(256), 0, s, 1, red));
            ++ctx->launches;
        }
    }
    return MLORA_OK;
}

}  // namespace

// Bridge for the other translation units of libmlora.so (mlora_comm.cpp).
namespace mlora_internal {
mlora_status set_error(mlora_ctx* ctx, mlora_status st, const std::string& msg) { return fail(ctx, st, msg); }
int ctx_device(const mlora_ctx* ctx) { return ctx->device; }
}  // namespace mlora_internal

extern "C" {

int32_t mlora_abi_version(void) { return 1; }

const char* mlora_status_string(mlora_status s) {
    switch (s) {
        case MLORA_OK: return "ok";
        case MLORA_USAGE: return "usage error";
        case MLORA_SHAPE: return "shape error";
        case MLORA_ROUTING: return "routing error";
        case MLORA_NUMERIC: return "numeric error";
        case MLORA_STATE: return "state error";
        case MLORA_CUDA: return "cuda error";
    }
    return "unknown status";
}

const char* mlora_last_error(const mlora_ctx* ctx) {
    return ctx ? ctx->last_error.c_str() : g_last_error.c_str();
}

mlora_status mlora_ctx_create(int32_t device, mlora_ctx** out) {
    if (!out) return fail(nullptr, MLORA_USAGE, "out is null");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(nullptr, MLORA_CUDA, "no CUDA device available");
    if (device < 0 || device >= ndev) return fail(nullptr, MLORA_USAGE, "device index out of range");
    DeviceGuard g(device);
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess)
        return fail(nullptr, MLORA_CUDA, "cudaGetDeviceProperties failed");
    if (prop.major != 10)
        return fail(nullptr, MLORA_CUDA, "mlora kernels are built for sm_100a (B200); device is sm_" +
                                             std::to_string(prop.major) + std::to_string(prop.minor));
    auto* ctx = new mlora_ctx();
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn) {
        delete ctx;
        return fail(nullptr, MLORA_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
    }
    ctx->encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    *out = ctx;
    return MLORA_OK;
}

mlora_status mlora_ctx_destroy(mlora_ctx* ctx) {
    if (!ctx) return MLORA_OK;
    DeviceGuard g(ctx->device);
    if (ctx->workspace) {
        cudaDeviceSynchronize();
        cudaFree(ctx->workspace);
    }
    for (auto& t : ctx->prof_pending) {
        cudaEventDestroy(std::get<1>(t));
        cudaEventDestroy(std::get<2>(t));
    }
    for (auto e : ctx->event_pool) cudaEventDestroy(e);
    for (auto e : ctx->timer)
        if (e) cudaEventDestroy(e);
    delete ctx;
    return MLORA_OK;
}

int32_t mlora_ctx_num_sms(const mlora_ctx* ctx) { return ctx ? ctx->num_sms : 0; }

mlora_status mlora_ctx_set_profiling(mlora_ctx* ctx, int32_t enable) {
    if (!ctx) return fail(nullptr, MLORA_USAGE, "null context");
    ctx->profiling = enable != 0;
    return MLORA_OK;
}

mlora_status mlora_ctx_profile_read(mlora_ctx* ctx, int32_t kind, int64_t* count, double* total_ms,
                                    int32_t reset) {
    if (!ctx || !count || !total_ms || kind < 0 || kind >= 8) return fail(ctx, MLORA_USAGE, "bad argument");
    DeviceGuard g(ctx->device);
    for (auto& t : ctx->prof_pending) {
        cudaEvent_t a = std::get<1>(t), b = std::get<2>(t);
        MLORA_CUDA_TRY(ctx, cudaEventSynchronize(b));
        float ms = 0.f;
        MLORA_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, a, b));
        ctx->prof_ms[std::get<0>(t)] += ms;
        ctx->prof_count[std::get<0>(t)] += 1;
        ctx->event_pool.push_back(a);
        ctx->event_pool.push_back(b);
    }
    ctx->prof_pending.clear();
    *count = ctx->prof_count[kind];
    *total_ms = ctx->prof_ms[kind];
    if (reset)
        for (int i = 0; i < 8; ++i) ctx->prof_ms[i] = 0, ctx->prof_count[i] = 0;
    return MLORA_OK;
}
int64_t mlora_ctx_launch_count(const mlora_ctx* ctx) { return ctx ? ctx->launches : 0; }

mlora_status mlora_ctx_timer_start(mlora_ctx* ctx, void* stream) {
    if (!ctx) return fail(nullptr, MLORA_USAGE, "null context");
    DeviceGuard g(ctx->device);
    if (!ctx->timer[0]) {
        MLORA_CUDA_TRY(ctx, cudaEventCreate(&ctx->timer[0]));
        MLORA_CUDA_TRY(ctx, cudaEventCreate(&ctx->timer[1]));
    }
    MLORA_CUDA_TRY(ctx, cudaEventRecord(ctx->timer[0], static_cast<cudaStream_t>(stream)));
    return MLORA_OK;
}

mlora_status mlora_ctx_timer_stop(mlora_ctx* ctx, void* stream, double* ms) {
    if (!ctx || !ms) return fail(ctx, MLORA_USAGE, "null argument");
    if (!ctx->timer[0]) return fail(ctx, MLORA_STATE, "timer not started");
    DeviceGuard g(ctx->device);
    MLORA_CUDA_TRY(ctx, cudaEventRecord(ctx->timer[1], static_cast<cudaStream_t>(stream)));
    MLORA_CUDA_TRY(ctx, cudaEventSynchronize(ctx->timer[1]));
    float f = 0.f;
    MLORA_CUDA_TRY(ctx, cudaEventElapsedTime(&f, ctx->timer[0], ctx->timer[1]));
    *ms = f;
    return MLORA_OK;
}

// lora.cpp:72-85: max_len over all lengths, sequences = count,
// total = sequences * max_len, padding = total - Σ len.
mlora_status mlora_fused_shape_of(const int32_t* lengths, int64_t n, mlora_fused_shape* out) {
    if (!out || (n > 0 && !lengths)) return fail(nullptr, MLORA_USAGE, "null argument");
    mlora_fused_shape s{0, 0, 0, 0};
    long long real = 0;
    for (int64_t i = 0; i < n; ++i) {
        s.max_len = std::max<int32_t>(s.max_len, lengths[i]);
        ++s.sequences;
        real += lengths[i];
    }
    s.total_tokens = s.sequences * s.max_len;
    s.padding_tokens = s.total_tokens - real;
    *out = s;
    return MLORA_OK;
}

// lora.cpp:184-189
mlora_status mlora_count_launches(int32_t num_jobs, int32_t mode, int64_t* small_launches,
                                  int64_t* large_launches) {
    if (num_jobs < 1) return fail(nullptr, MLORA_USAGE, "count_launches: need at least one job");
    if (!small_launches || !large_launches) return fail(nullptr, MLORA_USAGE, "null argument");
    if (mode != 0 && mode != 1) return fail(nullptr, MLORA_USAGE, "count_launches: bad mode");
    const int64_t k = num_jobs;
    *small_launches = mode == 0 ? 4 * k : 2 * k;
    *large_launches = mode == 0 ? 0 : 2;
    return MLORA_OK;
}

}  // extern "C"

namespace {

mlora_status check_segments(mlora_ctx* ctx, int32_t num_jobs, const int64_t* seg_offsets) {
    if (!seg_offsets) return fail(ctx, MLORA_USAGE, "null argument");
    if (seg_offsets[0] != 0) return fail(ctx, MLORA_USAGE, "seg_offsets[0] must be 0");
    for (int j = 0; j < num_jobs; ++j)
        if (seg_offsets[j + 1] < seg_offsets[j]) return fail(ctx, MLORA_USAGE, "seg_offsets must be non-decreasing");
    if (seg_offsets[num_jobs] < 1) return fail(ctx, MLORA_USAGE, "fused batch has no rows");
    if (seg_offsets[num_jobs] > (1LL << 30)) return fail(ctx, MLORA_USAGE, "too many rows");
    return MLORA_OK;
}

// Host tables of a segment layout (ranks/roff/scale already set) -> one blob:
// seg | roff | scale | ext | ext256 | down | grad, with the section offsets.
std::vector<int> build_tables(mlora_plan* p, const int64_t* seg_offsets, size_t off[8]) {
    const int J = p->J;
    const long long rows = seg_offsets[J];
    p->rows = static_cast<int>(rows);
    p->seg.assign(J + 1, 0);
    for (int j = 0; j <= J; ++j) p->seg[j] = static_cast<int>(seg_offsets[j]);
    p->n_mblk = cdiv(rows, kBM);
    p->n_chunks = cdiv(p->R_pad, kBK);
    auto job_of_row = [&](int r) {
        int j = static_cast<int>(std::upper_bound(p->seg.begin(), p->seg.end(), r) - p->seg.begin()) - 1;
        return std::min(std::max(j, 0), J - 1);
    };
    // per m-block: the 64-col chunks (LoRA k-blocks) of the jobs present
    p->ext.assign(2 * p->n_mblk, 0);
    p->down.clear();
    for (int mb = 0; mb < p->n_mblk; ++mb) {
        const int r0 = mb * kBM;
        const int r1 = std::min<int>(r0 + kBM, p->rows) - 1;
        const int ja = job_of_row(r0), jb = job_of_row(r1);
        p->ext[2 * mb] = p->roff[ja] / kBK;
        p->ext[2 * mb + 1] = cdiv(p->roff[jb + 1], kBK);
        // flags: bit 0 = first chunk (zero-fill duty), bits 1-3 / 4-6 = the chunk's 16-row rank
        // groups [lo, hi) held by the jobs present (roff is a multiple of 16: exact)
        const int c_lo = p->roff[ja], c_hi = p->roff[jb + 1];
        for (int c = p->ext[2 * mb]; c < p->ext[2 * mb + 1]; ++c) {
            const int lo = (std::max(c_lo, c * kBK) - c * kBK) / 16;
            const int hi = (std::min(c_hi, (c + 1) * kBK) - c * kBK + 15) / 16;
            p->down.push_back(mb);
            p->down.push_back(c);
            p->down.push_back((c == p->ext[2 * mb] ? 1 : 0) | (lo << 1) | (hi << 4));
        }
    }
    p->n_down = static_cast<int>(p->down.size() / 3);
    p->down_groups_max = 1;
    for (int t = 0; t < p->n_down; ++t)
        p->down_groups_max = std::max(p->down_groups_max, down_group_hi(p->down[3 * t + 2]) - down_group_lo(p->down[3 * t + 2]));
    p->n_mblk256 = cdiv(rows, kPairBM);
    p->ext256.assign(2 * p->n_mblk256, 0);
    p->grp256.assign(2 * p->n_mblk256, 0);
    for (int mb = 0; mb < p->n_mblk256; ++mb) {
        const int r0 = mb * kPairBM;
        const int r1 = std::min<int>(r0 + kPairBM, p->rows) - 1;
        const int ja = job_of_row(r0), jb = job_of_row(r1);
        p->ext256[2 * mb] = p->roff[ja] / kBK;
        p->ext256[2 * mb + 1] = cdiv(p->roff[jb + 1], kBK);
        p->grp256[2 * mb] = p->roff[ja] / 16;       // roff is a multiple of 16: exact
        p->grp256[2 * mb + 1] = p->roff[jb + 1] / 16;
    }
    // per chunk: union of the token segments of the jobs owning its columns
    p->chunk_kb.assign(2 * p->n_chunks, 0);
    for (int c = 0; c < p->n_chunks; ++c) {
        const int c0 = c * kBK, c1 = c0 + kBK;
        int ja = -1, jb = -1;
        for (int j = 0; j < J; ++j)
            if (p->roff[j + 1] > c0 && p->roff[j] < c1) {
                if (ja < 0) ja = j;
                jb = j;
            }
        const int t0 = p->seg[ja], t1 = p->seg[jb + 1];
        p->chunk_kb[2 * c] = t0 / kBK;
        p->chunk_kb[2 * c + 1] = t1 > t0 ? cdiv(t1, kBK) : t0 / kBK;
    }
    std::vector<int> grad;
    for (int ns = 1; ns <= kMaxSplit; ++ns) {
        p->grad_off[ns] = static_cast<int>(grad.size());
        for (int c = 0; c < p->n_chunks; ++c) {
            const int a = p->chunk_kb[2 * c], b = p->chunk_kb[2 * c + 1];
            const int len = b - a;
            for (int s = 0; s < ns; ++s) {
                grad.push_back(a + static_cast<int>((long long)len * s / ns));
                grad.push_back(a + static_cast<int>((long long)len * (s + 1) / ns));
            }
        }
    }
    std::vector<int> blob;
    auto append = [&](const std::vector<int>& v) {
        const size_t o = blob.size();
        blob.insert(blob.end(), v.begin(), v.end());
        while (blob.size() % 4) blob.push_back(0);
        return o;
    };
    std::vector<int> scale_bits(J);
    std::memcpy(scale_bits.data(), p->scale.data(), sizeof(float) * J);
    off[0] = append(p->seg);
    off[1] = append(p->roff);
    off[2] = append(scale_bits);
    off[3] = append(p->ext);
    off[4] = append(p->ext256);
    off[5] = append(p->down);
    off[6] = append(grad);
    off[7] = append(p->grp256);
    return blob;
}

// Stream-ordered upload: pinned staging + cudaMemcpyAsync, device buffer grown with
// cudaMallocAsync/cudaFreeAsync.  Kernels already enqueued on `stream` still see the
// old tables (the copy runs after them); nothing blocks the host.
mlora_status upload_tables(mlora_plan* p, const std::vector<int>& blob, const size_t off[8], cudaStream_t s) {
    mlora_ctx* ctx = p->ctx;
    const size_t bytes = blob.size() * sizeof(int);
    if (p->staging_done) MLORA_CUDA_TRY(ctx, cudaEventSynchronize(p->staging_done));  // staging reusable
    if (bytes > p->staging_bytes) {
        if (p->staging) cudaFreeHost(p->staging);
        p->staging = nullptr;
        MLORA_CUDA_TRY(ctx, cudaMallocHost(&p->staging, 2 * bytes));
        p->staging_bytes = 2 * bytes;
    }
    if (bytes > p->dev_bytes) {
        if (p->dev) MLORA_CUDA_TRY(ctx, cudaFreeAsync(p->dev, s));
        p->dev = nullptr;
        MLORA_CUDA_TRY(ctx, cudaMallocAsync(&p->dev, 2 * bytes, s));
        p->dev_bytes = 2 * bytes;
    }
    std::memcpy(p->staging, blob.data(), bytes);
    MLORA_CUDA_TRY(ctx, cudaMemcpyAsync(p->dev, p->staging, bytes, cudaMemcpyHostToDevice, s));
    if (!p->staging_done) MLORA_CUDA_TRY(ctx, cudaEventCreateWithFlags(&p->staging_done, cudaEventDisableTiming));
    MLORA_CUDA_TRY(ctx, cudaEventRecord(p->staging_done, s));
    int* base = static_cast<int*>(p->dev);
    p->d_seg = base + off[0];
    p->d_roff = base + off[1];
    p->d_scale = reinterpret_cast<float*>(base + off[2]);
    p->d_ext = base + off[3];
    p->d_ext256 = base + off[4];
    p->d_down = base + off[5];
    p->d_grad = base + off[6];
    p->d_grp256 = base + off[7];
    return MLORA_OK;
}

void release_plan(mlora_plan* p) {
    if (p->dev) {
        cudaDeviceSynchronize();
        cudaFree(p->dev);
    }
    if (p->staging_done) cudaEventDestroy(p->staging_done);
    if (p->staging) cudaFreeHost(p->staging);
    delete p;
}

}  // namespace

extern "C" {

mlora_status mlora_plan_create(mlora_ctx* ctx, int32_t num_jobs, const int64_t* seg_offsets,
                               const int32_t* ranks, const float* scales, void* stream,
                               mlora_plan** out) {
    if (!ctx || !out || !seg_offsets || !ranks) return fail(ctx, MLORA_USAGE, "null argument");
    *out = nullptr;
    if (num_jobs < 1 || num_jobs > kMaxJobs)
        return fail(ctx, MLORA_USAGE, "num_jobs must be in [1, " + std::to_string(kMaxJobs) + "]");
    mlora_status st = check_segments(ctx, num_jobs, seg_offsets);
    if (st != MLORA_OK) return st;
    for (int j = 0; j < num_jobs; ++j) {
        if (ranks[j] < 1) return fail(ctx, MLORA_USAGE, "adapter rank must be >= 1");
        if (scales && !std::isfinite(scales[j])) return fail(ctx, MLORA_NUMERIC, "non-finite scale");
    }
    DeviceGuard g(ctx->device);
    auto* p = new mlora_plan();
    p->ctx = ctx;
    p->J = num_jobs;
    p->roff.assign(num_jobs + 1, 0);
    p->rank.assign(ranks, ranks + num_jobs);
    p->scale.resize(num_jobs);
    for (int j = 0; j < num_jobs; ++j) {
        p->roff[j + 1] = p->roff[j] + ((ranks[j] + 15) / 16) * 16;
        p->scale[j] = scales ? scales[j] : 1.0f;
    }
    p->R_pad = p->roff[num_jobs];
    size_t off[8];
    const std::vector<int> blob = build_tables(p, seg_offsets, off);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    st = upload_tables(p, blob, off, s);
    if (st == MLORA_OK && cudaStreamSynchronize(s) != cudaSuccess) st = fail(ctx, MLORA_CUDA, "plan upload failed");
    if (st != MLORA_OK) {
        release_plan(p);
        return st;
    }
    *out = p;
    return MLORA_OK;
}

mlora_status mlora_plan_update(mlora_plan* plan, const int64_t* seg_offsets, void* stream) {
    if (!plan) return fail(nullptr, MLORA_USAGE, "null plan");
    mlora_ctx* ctx = plan->ctx;
    mlora_status st = check_segments(ctx, plan->J, seg_offsets);
    if (st != MLORA_OK) return st;
    DeviceGuard g(ctx->device);
    size_t off[8];
    const std::vector<int> blob = build_tables(plan, seg_offsets, off);
    return upload_tables(plan, blob, off, static_cast<cudaStream_t>(stream));
}

mlora_status mlora_plan_destroy(mlora_plan* plan) {
    if (!plan) return MLORA_OK;
    DeviceGuard g(plan->ctx->device);
    release_plan(plan);
    return MLORA_OK;
}

int64_t mlora_plan_rows(const mlora_plan* plan) { return plan ? plan->rows : 0; }
int32_t mlora_plan_num_jobs(const mlora_plan* plan) { return plan ? plan->J : 0; }
int32_t mlora_plan_rank_padded(const mlora_plan* plan) { return plan ? plan->R_pad : 0; }
mlora_status mlora_plan_rank_offsets(const mlora_plan* plan, int32_t* roff_out) {
    if (!plan || !roff_out) return fail(nullptr, MLORA_USAGE, "null argument");
    std::copy(plan->roff.begin(), plan->roff.end(), roff_out);
    return MLORA_OK;
}

mlora_status mlora_linear_fwd_ex(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                                 const void* X, const void* W0, const void* A_cat, const void* B_cat,
                                 void* Y, void* H, float* row_sq, void* stream) {
    mlora_status st = check_dims(ctx, plan, d, k);
    if (st != MLORA_OK) return st;
    if (!X || !W0 || !A_cat || !B_cat || !Y || !H) return fail(ctx, MLORA_USAGE, "null tensor pointer");
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // (1) H = s_j X A_j^T, block-diagonal, bf16
    const int32_t kk = k;
    void* hh = H;
    st = run_down_group<false>(ctx, plan, 1, &kk, &X, &A_cat, &hh, s);
    if (st != MLORA_OK) return st;
    // (2) Y = X W0^T + H B_cat^T
    return run_base<false>(ctx, plan, X, k, k, W0, H, B_cat, plan->R_pad, d, Y, s, row_sq);
}

mlora_status mlora_linear_fwd(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                              const void* X, const void* W0, const void* A_cat, const void* B_cat,
                              void* Y, void* H, void* stream) {
    return mlora_linear_fwd_ex(ctx, plan, d, k, X, W0, A_cat, B_cat, Y, H, nullptr, stream);
}

int32_t mlora_rowsq_blocks(int32_t d) { return cdiv(d, kPairBN); }

mlora_status mlora_loss_from_rowsq(mlora_ctx* ctx, const mlora_plan* plan, const float* const* row_sq,
                                   const int32_t* d, int32_t num_tensors, float* loss, void* stream) {
    if (!ctx || !plan || !row_sq || !d || !loss) return fail(ctx, MLORA_USAGE, "null argument");
    if (num_tensors < 1 || num_tensors > kMaxLossTensors) return fail(ctx, MLORA_USAGE, "num_tensors out of range");
    RowSqArgs a{};
    for (int t = 0; t < num_tensors; ++t) {
        if (!row_sq[t] || d[t] <= 0) return fail(ctx, MLORA_USAGE, "bad row-sum tensor");
        a.part[t] = row_sq[t];
        a.nblk[t] = cdiv(d[t], kPairBN);
    }
    a.ntensors = num_tensors;
    a.rows = plan->rows;
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    mlora_status st = ensure_workspace(ctx, sizeof(float) * plan->rows);
    if (st != MLORA_OK) return st;
    float* row_acc = static_cast<float*>(ctx->workspace);
    ProfScope ps(ctx, 4, s);
    MLORA_CUDA_TRY(ctx, launch_k(rowsq_rows_kernel, dim3(cdiv(plan->rows, 32)), dim3(32, kRowSqSlices), 0, s, 1, a,
                                 row_acc));
    MLORA_CUDA_TRY(ctx, launch_k(segment_loss_kernel, dim3(plan->J), dim3(1024), 0, s, 1,
                                 static_cast<const float*>(row_acc), static_cast<const int*>(plan->d_seg), loss));
    ctx->launches += 2;
    return MLORA_OK;
}

mlora_status mlora_linear_bwd(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                              const void* dY, const void* X, const void* H, const void* W0,
                              const void* A_cat, const void* B_cat, void* G, void* dX,
                              float* dA_cat, float* dB_cat, void* stream) {
    mlora_status st = check_dims(ctx, plan, d, k);
    if (st != MLORA_OK) return st;
    if (!dY || !X || !H || !W0 || !A_cat || !B_cat || !G)
        return fail(ctx, MLORA_USAGE, "null tensor pointer");
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int32_t dd = d, kk = k;
    void* gg = G;
    // (1) G = s_j dY B_j   (B operand B_cat viewed MN-major: n = rank col, k = d)
    st = run_down_group<true>(ctx, plan, 1, &dd, &dY, &B_cat, &gg, s);
    if (st != MLORA_OK) return st;
    // (2) dX = dY W0 + G A_cat   (W0 and A_cat as MN-major B operands)
    if (dX) {
        st = run_base<true>(ctx, plan, dY, d, d, W0, G, A_cat, plan->R_pad, k, dX, s);
        if (st != MLORA_OK) return st;
    }
    // (3) dA_cat = G^T X over each chunk's token range  (stored R_pad x k)
    if (dA_cat) {
        const void* gc = G;
        st = run_grad_group<MODE_GRADT>(ctx, plan, 1, &kk, &X, &gc, &dA_cat, s);
        if (st != MLORA_OK) return st;
    }
    // (4) dB_cat = dY^T H over each chunk's token range  (stored d x R_pad)
    if (dB_cat) {
        st = run_grad_group<MODE_GRAD>(ctx, plan, 1, &dd, &dY, &H, &dB_cat, s);
        if (st != MLORA_OK) return st;
    }
    return MLORA_OK;
}

// ---------------------------------------------------------------- layer-level grouped entry points
mlora_status mlora_down_group(mlora_ctx* ctx, const mlora_plan* plan, int32_t n, int32_t backward,
                              const int32_t* width, const void* const* in, const void* const* adapter,
                              void* const* out, void* stream) {
    if (!ctx || !plan || n < 0 || (n > 0 && (!width || !in || !adapter || !out)))
        return fail(ctx, MLORA_USAGE, "null argument");
    if (plan->ctx != ctx) return fail(ctx, MLORA_USAGE, "plan belongs to another context");
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    return backward ? run_down_group<true>(ctx, plan, n, width, in, adapter, out, s)
                    : run_down_group<false>(ctx, plan, n, width, in, adapter, out, s);
}

mlora_status mlora_base_fwd(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k, const void* X,
                            const void* W0, const void* H, const void* B_cat, void* Y, float* row_sq,
                            void* stream) {
    mlora_status st = check_dims(ctx, plan, d, k);
    if (st != MLORA_OK) return st;
    if (!X || !W0 || !Y || (!H != !B_cat)) return fail(ctx, MLORA_USAGE, "null tensor pointer");
    DeviceGuard g(ctx->device);
    return run_base<false>(ctx, plan, X, k, k, W0, H, B_cat, plan->R_pad, d, Y, static_cast<cudaStream_t>(stream),
                           row_sq);
}

mlora_status mlora_base_dx(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k, const void* dY,
                           const void* W0, const void* G, const void* A_cat, void* dX, void* stream) {
    mlora_status st = check_dims(ctx, plan, d, k);
    if (st != MLORA_OK) return st;
    if (!dY || !W0 || !dX || (!G != !A_cat)) return fail(ctx, MLORA_USAGE, "null tensor pointer");
    DeviceGuard g(ctx->device);
    return run_base<true>(ctx, plan, dY, d, d, W0, G, A_cat, plan->R_pad, k, dX, static_cast<cudaStream_t>(stream));
}

mlora_status mlora_grad_group(mlora_ctx* ctx, const mlora_plan* plan, int32_t n, const int32_t* d,
                              const int32_t* k, const void* const* X, const void* const* dY,
                              const void* const* H, const void* const* G, float* const* dA_cat,
                              float* const* dB_cat, void* stream) {
    if (!ctx || !plan || n < 0 || (n > 0 && (!d || !k || !X || !dY || !H || !G || !dA_cat || !dB_cat)))
        return fail(ctx, MLORA_USAGE, "null argument");
    if (plan->ctx != ctx) return fail(ctx, MLORA_USAGE, "plan belongs to another context");
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    mlora_status st = run_grad_group<MODE_GRADT>(ctx, plan, n, k, X, G, dA_cat, s);
    if (st != MLORA_OK) return st;
    return run_grad_group<MODE_GRAD>(ctx, plan, n, d, dY, H, dB_cat, s);
}

mlora_status mlora_pack_adapters(mlora_ctx* ctx, const mlora_plan* plan, int32_t d, int32_t k,
                                 const float* const* A_ptrs, const float* const* B_ptrs,
                                 float* A_cat_f32, float* B_cat_f32, void* A_cat_bf16,
                                 void* B_cat_bf16, void* stream) {
    mlora_status st = check_dims(ctx, plan, d, k);
    if (st != MLORA_OK) return st;
    if (!A_ptrs || !B_ptrs) return fail(ctx, MLORA_USAGE, "null pointer array");
    PackArgs a{};
    for (int j = 0; j < plan->J; ++j) {
        if (!A_ptrs[j] || !B_ptrs[j])
            return fail(ctx, MLORA_ROUTING, "no adapter for job " + std::to_string(j));
        if (plan->rank[j] > std::min(d, k)) return fail(ctx, MLORA_USAGE, "adapter rank exceeds min(d, k)");
        a.A[j] = A_ptrs[j];
        a.B[j] = B_ptrs[j];
        a.rank[j] = plan->rank[j];
        a.roff[j] = plan->roff[j];
    }
    a.roff[plan->J] = plan->roff[plan->J];
    a.J = plan->J;
    a.d = d;
    a.k = k;
    a.R_pad = plan->R_pad;
    a.A_f32 = A_cat_f32;
    a.B_f32 = B_cat_f32;
    a.A_bf16 = static_cast<__nv_bfloat16*>(A_cat_bf16);
    a.B_bf16 = static_cast<__nv_bfloat16*>(B_cat_bf16);
    DeviceGuard g(ctx->device);
    const long long n = (long long)plan->R_pad * k + (long long)d * plan->R_pad;
    const int blocks = static_cast<int>(std::min<long long>(cdiv(n, 256), 8LL * ctx->num_sms));
    ProfScope ps(ctx, 4, static_cast<cudaStream_t>(stream));
    MLORA_CUDA_TRY(ctx, launch_k(pack_adapters_kernel, dim3(blocks), dim3(256), 0,
                                 static_cast<cudaStream_t>(stream), 1, a));
    ++ctx->launches;
    return MLORA_OK;
}

mlora_status mlora_adam_step(mlora_ctx* ctx, const mlora_plan* plan, const mlora_adam_group* groups,
                             int32_t num_groups, const float* lr, const int32_t* step, float beta1,
                             float beta2, float eps, float weight_decay, void* stream) {
    return mlora_adam_step_ex(ctx, plan, groups, num_groups, lr, step, beta1, beta2, eps, weight_decay, nullptr,
                              stream);
}

mlora_status mlora_adam_step_ex(mlora_ctx* ctx, const mlora_plan* plan, const mlora_adam_group* groups,
                                int32_t num_groups, const float* lr, const int32_t* step, float beta1,
                                float beta2, float eps, float weight_decay, const float* loss_gate,
                                void* stream) {
    if (!ctx || !plan || (num_groups > 0 && !groups) || !lr || !step)
        return fail(ctx, MLORA_USAGE, "null argument");
    if (!(beta1 >= 0.f && beta1 < 1.f && beta2 >= 0.f && beta2 < 1.f && eps > 0.f))
        return fail(ctx, MLORA_USAGE, "bad Adam hyper-parameters");
    DeviceGuard g(ctx->device);
    AdamArgs a{};
    a.J = plan->J;
    for (int j = 0; j <= plan->J; ++j) a.roff[j] = plan->roff[j];
    for (int j = 0; j < plan->J; ++j) {
        if (step[j] < 0) return fail(ctx, MLORA_USAGE, "Adam step must be >= 0 (0 = job inactive this step)");
        if (!std::isfinite(lr[j])) return fail(ctx, MLORA_NUMERIC, "non-finite learning rate");
        a.lr[j] = lr[j];
        // reciprocal bias corrections (0 marks a job absent from this step)
        a.bc1[j] = step[j] == 0 ? 0.f : static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(beta1), step[j])));
        a.bc2[j] = step[j] == 0 ? 0.f : static_cast<float>(1.0 / (1.0 - std::pow(static_cast<double>(beta2), step[j])));
    }
    a.beta1 = beta1;
    a.beta2 = beta2;
    a.eps = eps;
    a.wd = weight_decay;
    a.loss_gate = loss_gate;
    for (int g0 = 0; g0 < num_groups; g0 += kMaxAdamGroups) {
        const int ng = std::min(kMaxAdamGroups, num_groups - g0);
        long long start4 = 0;
        for (int i = 0; i < ng; ++i) {
            const mlora_adam_group& G = groups[g0 + i];
            if (!G.p || !G.g || !G.m || !G.v) return fail(ctx, MLORA_USAGE, "null Adam tensor");
            if (G.cols % 4 != 0) return fail(ctx, MLORA_SHAPE, "Adam group cols must be a multiple of 4");
            const long long bound = G.layout == 0 ? G.rows : G.cols;
            if (bound != plan->R_pad) return fail(ctx, MLORA_SHAPE, "Adam group job axis must have R_pad entries");
            a.grp[i] = AdamGroupDev{G.p, G.g, G.m, G.v, static_cast<__nv_bfloat16*>(G.p_bf16),
                                    G.rows, G.cols, start4, G.layout};
            start4 += G.rows * G.cols / 4;
        }
        a.ngroups = ng;
        a.total4 = start4;
        if (start4 == 0) continue;
        const int blocks = static_cast<int>(std::min<long long>(cdiv(start4, 256), 8LL * ctx->num_sms));
        ProfScope ps(ctx, 5, static_cast<cudaStream_t>(stream));
        MLORA_CUDA_TRY(ctx, launch_k(adam_kernel, dim3(blocks), dim3(256), 0, static_cast<cudaStream_t>(stream), 1,
                                     a));
        ++ctx->launches;
    }
    return MLORA_OK;
}

mlora_status mlora_segment_sumsq_loss(mlora_ctx* ctx, const mlora_plan* plan, const void* const* Y,
                                      const int32_t* cols, int32_t num_tensors, float* loss, void* stream) {
    if (!ctx || !plan || !Y || !cols || !loss) return fail(ctx, MLORA_USAGE, "null argument");
    if (num_tensors < 1 || num_tensors > kMaxLossTensors)
        return fail(ctx, MLORA_USAGE, "num_tensors out of range");
    SumsqArgs a{};
    for (int t = 0; t < num_tensors; ++t) {
        if (!Y[t] || cols[t] <= 0 || cols[t] % 8 != 0)
            return fail(ctx, MLORA_SHAPE, "loss tensors need cols that are positive multiples of 8");
        a.y[t] = static_cast<const __nv_bfloat16*>(Y[t]);
        a.cols[t] = cols[t];
    }
    a.ntensors = num_tensors;
    a.rows = plan->rows;
    DeviceGuard g(ctx->device);
    mlora_status st = ensure_workspace(ctx, sizeof(float) * plan->rows);
    if (st != MLORA_OK) return st;
    a.row_acc = static_cast<float*>(ctx->workspace);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int blocks = std::min(cdiv(plan->rows, 8), 8 * ctx->num_sms);
    ProfScope ps(ctx, 4, s);
    MLORA_CUDA_TRY(ctx, launch_k(row_sumsq_kernel, dim3(blocks), dim3(256), 0, s, 1, a));
    MLORA_CUDA_TRY(ctx, launch_k(segment_loss_kernel, dim3(plan->J), dim3(1024), 0, s, 1,
                                 static_cast<const float*>(a.row_acc), static_cast<const int*>(plan->d_seg), loss));
    ctx->launches += 2;
    return MLORA_OK;
}

mlora_status mlora_fuse_rows(mlora_ctx* ctx, int32_t num_seqs, const void* const* src, const int64_t* ld_src,
                             const int32_t* lens, int64_t dim, int32_t padded, void* dst, uint8_t* mask,
                             int64_t* row_offsets, void* stream) {
    if (!ctx || !src || !lens || !dst) return fail(ctx, MLORA_USAGE, "null argument");
    if (num_seqs < 1) return fail(ctx, MLORA_USAGE, "fuse: no sequences");  // lora.cpp:115
    if (dim < 8 || dim % 8) return fail(ctx, MLORA_SHAPE, "fuse: row width must be a positive multiple of 8");
    if (reinterpret_cast<uintptr_t>(dst) % 16) return fail(ctx, MLORA_USAGE, "tensor base pointer must be 16-byte aligned");
    int max_len = 0;
    for (int i = 0; i < num_seqs; ++i) {
        if (lens[i] < 1) return fail(ctx, MLORA_USAGE, "fuse: empty sequence");  // lora.cpp:131
        if (!src[i] || reinterpret_cast<uintptr_t>(src[i]) % 16)
            return fail(ctx, MLORA_USAGE, "fuse: null or misaligned sequence buffer");
        const long long ld = ld_src ? ld_src[i] : dim;
        if (ld < dim || ld % 8) return fail(ctx, MLORA_SHAPE, "fuse: source row stride must be >= dim, multiple of 8");
        max_len = std::max(max_len, lens[i]);
    }
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    long long base = 0;
    for (int s0 = 0; s0 < num_seqs; s0 += kFuseMaxSeqs) {
        FuseArgs a{};
        a.nseq = std::min(kFuseMaxSeqs, num_seqs - s0);
        a.dim = dim;
        a.dst = static_cast<__nv_bfloat16*>(dst);
        a.mask = mask;
        a.off[0] = base;
        int chunk_max = 0;
        for (int i = 0; i < a.nseq; ++i) {
            a.src[i] = static_cast<const __nv_bfloat16*>(src[s0 + i]);
            a.ld[i] = ld_src ? ld_src[s0 + i] : dim;
            a.len[i] = lens[s0 + i];
            a.off[i + 1] = a.off[i] + (padded ? max_len : lens[s0 + i]);
            if (row_offsets) row_offsets[s0 + i] = a.off[i];
            chunk_max = std::max<int>(chunk_max, static_cast<int>(a.off[i + 1] - a.off[i]));
        }
        base = a.off[a.nseq];
        MLORA_CUDA_TRY(ctx, launch_k(fuse_rows_kernel, dim3(cdiv(chunk_max, 32), a.nseq), dim3(256), 0, s, 1, a));
        ++ctx->launches;
    }
    if (row_offsets) row_offsets[num_seqs] = base;
    return MLORA_OK;
}

}  // extern "C"

namespace mlora {
// Internal (layer step): per-job loss from the forward epilogues' row sums fused with
// the non-finite guard over `tensors` — rowsq_rows_kernel + loss_guard_kernel.
mlora_status layer_loss_guard(mlora_ctx* ctx, const mlora_plan* plan, const float* const* row_sq, const int32_t* d,
                              int32_t num_rowsq, float* loss, void* const* tensors, const int32_t* cols,
                              int32_t num_tensors, cudaStream_t s) {
    if (num_rowsq < 1 || num_rowsq > kMaxLossTensors) return fail(ctx, MLORA_USAGE, "num_tensors out of range");
    if (num_tensors < 1 || num_tensors > kMaxGuardTensors) return fail(ctx, MLORA_USAGE, "too many guarded tensors");
    RowSqArgs ra{};
    for (int t = 0; t < num_rowsq; ++t) {
        if (!row_sq[t] || d[t] <= 0) return fail(ctx, MLORA_USAGE, "bad row-sum tensor");
        ra.part[t] = row_sq[t];
        ra.nblk[t] = cdiv(d[t], kPairBN);
    }
    ra.ntensors = num_rowsq;
    ra.rows = plan->rows;
    GuardArgs ga{};
    for (int t = 0; t < num_tensors; ++t) {
        if (!tensors[t] || cols[t] <= 0 || cols[t] % 8 != 0 || reinterpret_cast<uintptr_t>(tensors[t]) % 16 != 0)
            return fail(ctx, MLORA_SHAPE, "guarded tensors need 16-byte aligned rows of a multiple of 8 columns");
        ga.t[t] = static_cast<__nv_bfloat16*>(tensors[t]);
        ga.cols[t] = cols[t];
    }
    ga.ntensors = num_tensors;
    ga.seg = plan->d_seg;
    ga.loss = loss;
    DeviceGuard g(ctx->device);
    mlora_status st = ensure_workspace(ctx, sizeof(float) * plan->rows);
    if (st != MLORA_OK) return st;
    float* row_acc = static_cast<float*>(ctx->workspace);
    ProfScope ps(ctx, 4, s);
    MLORA_CUDA_TRY(ctx, launch_k(rowsq_rows_kernel, dim3(cdiv(plan->rows, 32)), dim3(32, kRowSqSlices), 0, s, 1, ra,
                                 row_acc));
    MLORA_CUDA_TRY(ctx, launch_k(loss_guard_kernel, dim3(plan->J, 16), dim3(256), 0, s, 1,
                                 static_cast<const float*>(row_acc), loss, ga));
    ctx->launches += 2;
    return MLORA_OK;
}
}  // namespace mlora

extern "C" {

mlora_status mlora_zero_nonfinite_rows(mlora_ctx* ctx, const mlora_plan* plan, const float* loss,
                                       void* const* tensors, const int32_t* cols, int32_t num_tensors,
                                       void* stream) {
    if (!ctx || !plan || !loss || !tensors || !cols) return fail(ctx, MLORA_USAGE, "null argument");
    if (num_tensors < 1 || num_tensors > kMaxGuardTensors) return fail(ctx, MLORA_USAGE, "num_tensors out of range");
    GuardArgs a{};
    for (int t = 0; t < num_tensors; ++t) {
        if (!tensors[t] || cols[t] <= 0 || cols[t] % 8 != 0)
            return fail(ctx, MLORA_SHAPE, "guarded tensors need cols that are positive multiples of 8");
        if (reinterpret_cast<uintptr_t>(tensors[t]) % 16 != 0)
            return fail(ctx, MLORA_USAGE, "tensor base pointer must be 16-byte aligned");
        a.t[t] = static_cast<__nv_bfloat16*>(tensors[t]);
        a.cols[t] = cols[t];
    }
    a.ntensors = num_tensors;
    a.seg = plan->d_seg;
    a.loss = loss;
    DeviceGuard g(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ProfScope ps(ctx, 4, s);
    MLORA_CUDA_TRY(ctx, launch_k(zero_nonfinite_rows_kernel, dim3(plan->J, 16), dim3(256), 0, s, 1, a));
    ++ctx->launches;
    return MLORA_OK;
}

}  // extern "C"
