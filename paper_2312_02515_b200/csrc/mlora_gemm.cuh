// mlora_gemm.cuh — the one tcgen05 GEMM engine behind every multi-LoRA product.
//
// BatchFusion (ASPEN, arXiv 2312.02515, Eq. 1; reference fp64 loop in
// /root/reference/proj/src/lora.cpp:160-182) computes, per job row-segment j,
//     Y_j = X_j W0^T + (X_j A_j^T) B_j^T .
// On B200 every term of the forward and backward is one of four tile programs
// of the same persistent, warp-specialised kernel:
//
//   MODE_BASE : C[M,N]  = A0[M,K] B0[N,K]^T  (+ A1[M,R] B1[N,R]^T on the
//               k-blocks of the jobs present in the m-tile)       -> bf16 C
//               forward:  A0=X,  B0=W0 (K-major), A1=H_cat, B1=B_cat
//               dX:       A0=dY, B0=W0 (MN-major), A1=G_cat, B1=A_cat (MN)
//               — on a CTA pair, mlora_base_pair_kernel (below)
//   MODE_DOWN : H_cat[M, 64-col chunk] = s_j * A0 B0^T, masked block-diagonal
//               H = s X A_cat^T  (B0 = A_cat K-major)
//               G = s dY B_cat   (B0 = B_cat MN-major)
//   MODE_GRADT: dA_cat^T partials  [F, 64-col chunk] = X^T G_cat over the
//               chunk's token range, stored transposed ([R_pad, F], fp32)
//   MODE_GRAD : dB_cat partials    [F, 64-col chunk] = dY^T H_cat  ([F, R_pad])
//
// mlora_gemm_kernel runs DOWN / GRADT / GRAD.
// Roles (192 threads): warp 0 = TMA producer,
// warp 1 = TMEM allocator + single-thread tcgen05.mma issuer, warps 2..5 =
// epilogue (TMEM -> registers -> HBM).  Accumulators are double-buffered in
// TMEM so the epilogue of tile i overlaps the MMAs of tile i+1.  Operands are
// staged by TMA with 128-byte swizzle in a STAGES-deep mbarrier ring.
#pragma once

#include "sm100.cuh"

namespace mlora {

enum GemmMode : int { MODE_BASE = 0, MODE_DOWN = 1, MODE_GRADT = 2, MODE_GRAD = 3 };

constexpr int kBM = 128;        // UMMA M (rows of the output tile)
constexpr int kBK = 64;         // 64 bf16 = one 128 B swizzle row
constexpr int kUmmaK = 16;      // K per tcgen05.mma kind::f16
constexpr int kNumThreads = 192;


struct GemmParams {
    int M;             // valid output rows (tokens for BASE/DOWN, features for GRAD*)
    int N;             // valid output cols (d for BASE, R_pad for DOWN/GRAD*)
    int num_kb;        // main-segment k-blocks (BASE/DOWN)
    int n_mblk;        // number of 128-row blocks
    int n_nblk;        // number of BN-col blocks (BASE)
    int num_tiles;
    int nsplit;        // token splits (GRAD*)
    void* out;         // output base
    long long ldo;     // output leading dimension (elements)
    long long split_stride;  // elements between split partials (GRAD*)
    const int* ext_tab;   // [n_mblk][2]  extra (LoRA) k-block range per m-block
    const int* ext_grp;   // BASE (pair): [n_mblk][2] 16-column rank groups [lo, hi) of the m-block's jobs
    const int* down_tab;  // [num_tiles][3] (m_blk, chunk, flags) for MODE_DOWN (flags: down_group_lo/hi)
    const int* grad_tab;  // [nchunks*nsplit][2] token k-block range
    float* row_sq;        // BASE (pair) optional: [n_nblk][M] sum over the tile's columns of bf16(Y)^2
    int raster_group;     // BASE (pair): > 0 m-blocks per super-row (m fastest); < 0 n-blocks per super-column (n fastest); 0 plain m-fastest
    int keep_b_in_l2;     // BASE (pair): load the main B operand (W0) with an L2 evict_last policy
    const int* seg;       // [J+1] row offsets of job segments
    const int* roff;      // [J+1] padded rank column offsets
    const float* scale;   // [J] per-job LoRA scale s_j
    int num_jobs;
};

struct TileInfo {
    int m0, n0;
    int kb0, kb1;   // main segment k-blocks
    int xb0, xb1;   // extra segment k-blocks
    int aux;        // DOWN: flags; GRAD*: split index
};

template <int MODE, int BN>
__device__ __forceinline__ TileInfo decode_tile(const GemmParams& p, int t) {
    static_assert(MODE != MODE_BASE, "the base GEMM runs on the CTA-pair kernel");
    TileInfo ti;
    if constexpr (MODE == MODE_DOWN) {
        const int mb = __ldg(p.down_tab + 3 * t);
        const int c = __ldg(p.down_tab + 3 * t + 1);
        ti.aux = __ldg(p.down_tab + 3 * t + 2);
        ti.m0 = mb * kBM;
        ti.n0 = c * BN;
        ti.kb0 = 0;
        ti.kb1 = p.num_kb;
        ti.xb0 = ti.xb1 = 0;
    } else {
        const int fb = t % p.n_mblk;
        const int cs = t / p.n_mblk;  // chunk * nsplit + split
        ti.m0 = fb * kBM;
        ti.n0 = (cs / p.nsplit) * BN;
        ti.kb0 = __ldg(p.grad_tab + 2 * cs);
        ti.kb1 = __ldg(p.grad_tab + 2 * cs + 1);
        ti.xb0 = ti.xb1 = 0;
        ti.aux = cs % p.nsplit;
    }
    return ti;
}

// MODE_DOWN tile flags: bit 0 = first chunk of the m-block (zero-fill duty);
// bits 1-3 / 4-6 = [lo, hi) of the 16-row rank groups of the chunk that belong
// to the jobs present in the m-block (mlora_capi.cu build_tables).  Only those
// rank rows of the K-major adapter operand are loaded and multiplied.
__host__ __device__ __forceinline__ int down_group_lo(int flags) { return (flags >> 1) & 7; }
__host__ __device__ __forceinline__ int down_group_hi(int flags) { return (flags >> 4) & 7; }

__device__ __forceinline__ int job_of_row(const int* seg, int num_jobs, int row) {
    // largest j with seg[j] <= row (segments partition [0, M))
    int lo = 0, hi = num_jobs - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (__ldg(seg + mid) <= row) lo = mid; else hi = mid - 1;
    }
    return lo;
}

// MODE_DOWN epilogue for one row of a 64-column chunk tile: H/G = s_j * acc on
// the columns of the row's own job, exactly 0 on every other column (a select,
// not a multiply, so a non-finite acc of another job's columns never leaks).
// The first chunk tile of an m-block (aux & 1) also zero-fills the row's
// columns outside the m-block's LoRA k-block range, so H/G are fully
// block-diagonal in HBM.
//
// The row's job lookup (a dependent chain of table loads) is split off into
// down_row_info so the epilogue can issue it before it waits for the
// mainloop, and a multi-projection epilogue does it once per row, not once
// per projection.
struct DownRow {
    int c_lo, c_hi;  // the row's job's columns
    float s;         // its scale
    int z0, z1;      // first chunk tile: columns kept (LoRA k-block range); z0 = z1 = -1 otherwise
};

__device__ __forceinline__ DownRow down_row_info(const GemmParams& p, int row, int m0, int aux) {
    DownRow r;
    const int jr = job_of_row(p.seg, p.num_jobs, row < p.M ? row : p.M - 1);
    r.c_lo = __ldg(p.roff + jr);
    r.c_hi = __ldg(p.roff + jr + 1);
    r.s = __ldg(p.scale + jr);
    r.z0 = r.z1 = -1;
    if (aux & 1) {
        const int mb = m0 / kBM;
        r.z0 = __ldg(p.ext_tab + 2 * mb) * kBK;
        r.z1 = __ldg(p.ext_tab + 2 * mb + 1) * kBK;
    }
    return r;
}

// First chunk tile of an m-block: zero the row's columns outside its LoRA k-block range.
__device__ __forceinline__ void down_zero_outside(const GemmParams& p, const DownRow& r, __nv_bfloat16* out, int row) {
    uint4* rowp = reinterpret_cast<uint4*>(out + (long long)row * p.ldo);
    const uint4 zero = make_uint4(0, 0, 0, 0);
    for (int cc = 0; cc < p.N; cc += 8)
        if (cc < r.z0 || cc >= r.z1) rowp[cc / 8] = zero;
}

template <int BN>
__device__ __forceinline__ void down_store_row(const GemmParams& p, const DownRow& r, __nv_bfloat16* out, int row,
                                               int n0, const float* accv) {
    uint4* dst = reinterpret_cast<uint4*>(out + (long long)row * p.ldo + n0);
#pragma unroll
    for (int g = 0; g < BN / 8; ++g) {
        if (n0 + 8 * g + 8 > p.N) break;
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int cc = n0 + 8 * g + e;
            f[e] = (cc >= r.c_lo && cc < r.c_hi) ? r.s * accv[8 * g + e] : 0.f;
        }
        uint4 w;
        w.x = sm100::pack_bf16x2(f[0], f[1]);
        w.y = sm100::pack_bf16x2(f[2], f[3]);
        w.z = sm100::pack_bf16x2(f[4], f[5]);
        w.w = sm100::pack_bf16x2(f[6], f[7]);
        dst[g] = w;
    }
    if (r.z0 >= 0) down_zero_outside(p, r, out, row);
}

template <int BN, int STAGES, int KSPLIT = 1>
struct GemmSmem {
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    // K-split across a CTA pair: the follower's fp32 partial tile lands here (DSMEM)
    static constexpr int kPartOffset = STAGES * kStageBytes;
    static constexpr int kPartBytes = KSPLIT == 2 ? kBM * BN * 4 : 0;
    static constexpr int kBarOffset = kPartOffset + kPartBytes;
    // full[S], empty[S], tmem_full[2], tmem_empty[2], part_full, part_empty, tmem base slot
    static constexpr int kBytes = kBarOffset + (2 * STAGES + 6) * 8 + 16;
    static constexpr int kDynBytes = kBytes + 1024;  // manual 1 KB alignment slack
};


// One GEMM problem of a (possibly grouped) launch: its operand tensor maps, its
// parameters and the global index of its first tile.  A launch carries up to NP
// problems by value in the kernel's parameter space (__grid_constant__), so one
// launch serves e.g. the rank-r down-projections of every projection of a layer:
// the ~12 us fixed cost of an HBM-bound launch (pipeline fill, TMEM/barrier
// setup, tail) is paid once per layer instead of once per projection.
struct alignas(64) GemmProblem {
    CUtensorMap tmA0, tmB0, tmA1, tmB1;
    GemmParams p;
    int tile_begin;
};

template <int NP>
struct GemmProblemSet {
    GemmProblem prob[NP];
    int nprobs;
    int total_tiles;
    // 1: all problems have the same tile count and tile t is tile t / nprobs of
    // problem t % nprobs, so problems reading the same operand rows (e.g. the
    // projections fed by one hidden state) run them concurrently and share L2.
    int interleave;
};

// KSPLIT = 2 (MODE_DOWN): launched in clusters of 2; CTA r of the pair reduces
// the r-th half of the K range into its own TMEM, the follower ships its fp32
// partial tile to the leader's smem over DSMEM and the leader adds it in a fixed
// order (deterministic) before the masked/scaled store.  Doubles the CTAs that
// stream the HBM-bound operand and halves the bytes each must keep in flight.
template <int MODE, int BN, int STAGES, bool A_MN, bool B_MN, int KSPLIT = 1, int NP = 1>
__global__ void __launch_bounds__(kNumThreads, 1)
mlora_gemm_kernel(const __grid_constant__ GemmProblemSet<NP> ps) {
    using namespace sm100;
    using L = GemmSmem<BN, STAGES, KSPLIT>;
    static_assert(KSPLIT == 1 || (KSPLIT == 2 && MODE == MODE_DOWN && BN == 64), "K split: DOWN, BN=64 only");
    static_assert(BN % 64 == 0 && BN >= 64 && BN <= 256, "BN must be a multiple of 64 in [64,256]");
    constexpr uint32_t kTmemCols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128
                                 : (2 * BN <= 256) ? 256 : 512;
    constexpr uint32_t kIdesc = idesc_bf16_f32(kBM, BN, A_MN, B_MN);

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_addr - raw_addr);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint64_t* pfull_bar = tempty_bar + 2;
    uint64_t* pempty_bar = pfull_bar + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty_bar + 1);

    const uint32_t warp = warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t krank = KSPLIT == 2 ? cluster_ctarank() : 0u;
    const int t_first = static_cast<int>(blockIdx.x) / KSPLIT;
    const int t_step = static_cast<int>(gridDim.x) / KSPLIT;
    // problem owning global tile t (problems are few and tiles visited in order)
    auto find = [&](int t) {
        if (ps.interleave) return t % ps.nprobs;
        int pi = 0;
        while (pi + 1 < ps.nprobs && ps.prob[pi + 1].tile_begin <= t) ++pi;
        return pi;
    };
    // this CTA's tile program: for a K-split pair, its half of the main k-blocks
    auto tile_of = [&](int pi, int t) {
        const int local_t = ps.interleave ? t / ps.nprobs : t - ps.prob[pi].tile_begin;
        TileInfo ti = decode_tile<MODE, BN>(ps.prob[pi].p, local_t);
        if constexpr (KSPLIT == 2) {
            const int mid = ti.kb0 + (ti.kb1 - ti.kb0) / 2;
            if (krank == 0) ti.kb1 = mid; else ti.kb0 = mid;
        }
        return ti;
    };
    const int num_tiles = ps.total_tiles;

    if (warp == 0 && elect_one()) {
        for (int pi = 0; pi < ps.nprobs; ++pi) {
            tma_prefetch_desc(&ps.prob[pi].tmA0);
            tma_prefetch_desc(&ps.prob[pi].tmB0);
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar + a, 1);
            mbar_init(tempty_bar + a, 128);
        }
        mbar_init(pfull_bar, 4);   // follower's 4 epilogue warps (K split)
        mbar_init(pempty_bar, 4);  // leader's 4 epilogue warps (K split)
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    if constexpr (KSPLIT == 2) cluster_sync(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_launch_dependents();
    griddep_wait();  // predecessor's results visible; everything above overlapped its tail

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = t_first; t < num_tiles; t += t_step) {
                const int pi = find(t);
                const GemmProblem& P = ps.prob[pi];
                const TileInfo ti = tile_of(pi, t);
                const int nmain = ti.kb1 - ti.kb0;
                const int nk = nmain + (ti.xb1 - ti.xb0);
                // forward down-projection: only the present jobs' 16-row rank groups of A_cat
                // (tmB1 = the same tensor, 16-row box); everything else loads whole tiles
                constexpr bool kNarrow = MODE == MODE_DOWN && !B_MN;
                const int glo = kNarrow ? down_group_lo(ti.aux) : 0, ghi = kNarrow ? down_group_hi(ti.aux) : 0;
                const uint32_t tx = kNarrow ? static_cast<uint32_t>(L::kABytes + (ghi - glo) * 16 * kBK * 2)
                                            : static_cast<uint32_t>(L::kStageBytes);
                for (int it = 0; it < nk; ++it) {
                    mbar_wait(empty_bar + stage, phase ^ 1u);
                    const bool ext = it >= nmain;
                    const CUtensorMap* mA = ext ? &P.tmA1 : &P.tmA0;
                    const CUtensorMap* mB = ext ? &P.tmB1 : &P.tmB0;
                    const int kc = (ext ? (ti.xb0 + it - nmain) : (ti.kb0 + it)) * kBK;
                    const uint32_t sA = base_addr + stage * L::kStageBytes;
                    const uint32_t sB = sA + L::kABytes;
                    uint64_t* bar = full_bar + stage;
                    mbar_arrive_expect_tx(bar, tx);
                    if constexpr (!A_MN) {
                        tma_load_2d(sA, mA, bar, kc, ti.m0);
                    } else {
#pragma unroll
                        for (int h = 0; h < kBM / 64; ++h)
                            tma_load_2d(sA + h * 8192, mA, bar, ti.m0 + 64 * h, kc);
                    }
                    if constexpr (kNarrow) {
                        for (int g = glo; g < ghi; ++g)
                            tma_load_2d(sB + g * 16 * kBK * 2, &P.tmB1, bar, kc, ti.n0 + 16 * g);
                    } else if constexpr (!B_MN) {
                        tma_load_2d(sB, mB, bar, kc, ti.n0);
                    } else {
#pragma unroll
                        for (int h = 0; h < BN / 64; ++h)
                            tma_load_2d(sB + h * 8192, mB, bar, ti.n0 + 64 * h, kc);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        int stage = 0;
        uint32_t phase = 0;
        int local = 0;
        for (int t = t_first; t < num_tiles; t += t_step, ++local) {
            const TileInfo ti = tile_of(find(t), t);
            const int nk = (ti.kb1 - ti.kb0) + (ti.xb1 - ti.xb0);
            const int acc = local & 1;
            const uint32_t use = static_cast<uint32_t>(local >> 1);
            mbar_wait(tempty_bar + acc, (use & 1u) ^ 1u);
            tc_fence_after();
            uint32_t d_tmem = tmem_base + acc * BN;
            uint32_t idesc = kIdesc;
            uint32_t b_off = 0;
            if constexpr (MODE == MODE_DOWN && !B_MN) {
                const int glo = down_group_lo(ti.aux), ghi = down_group_hi(ti.aux);
                idesc = idesc_bf16_f32(kBM, 16 * (ghi - glo), A_MN, B_MN);
                d_tmem += 16 * glo;
                b_off = glo * 16 * kBK * 2;
            }
            for (int it = 0; it < nk; ++it) {
                mbar_wait(full_bar + stage, phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sA = base_addr + stage * L::kStageBytes;
                    const uint32_t sB = sA + L::kABytes;
#pragma unroll
                    for (int j = 0; j < kBK / kUmmaK; ++j) {
                        const uint64_t ad = A_MN ? sdesc_sw128(sA + j * 2048, 8192, 1024)
                                                 : sdesc_sw128(sA + j * 32, 16, 1024);
                        const uint64_t bd = B_MN ? sdesc_sw128(sB + j * 2048, 8192, 1024)
                                                 : sdesc_sw128(sB + b_off + j * 32, 16, 1024);
                        mma_bf16(d_tmem, ad, bd, idesc, (it | j) != 0 ? 1u : 0u);
                    }
                    tc_commit(empty_bar + stage);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            }
            if (elect_one()) tc_commit(tfull_bar + acc);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2..5)
        const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
        const int rloc = static_cast<int>(q * 32 + lane);
        int local = 0;
        for (int t = t_first; t < num_tiles; t += t_step, ++local) {
            const int pi = find(t);
            const GemmParams& p = ps.prob[pi].p;
            const TileInfo ti = tile_of(pi, t);
            const bool empty = (ti.kb1 - ti.kb0) + (ti.xb1 - ti.xb0) == 0;
            const int acc = local & 1;
            const uint32_t use = static_cast<uint32_t>(local >> 1);
            const int row = ti.m0 + rloc;
            const bool row_ok = row < p.M;
            DownRow dr{};
            if constexpr (MODE == MODE_DOWN) dr = down_row_info(p, row, ti.m0, ti.aux);  // overlaps the mainloop
            mbar_wait(tfull_bar + acc, use & 1u);
            tc_fence_after();
            const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * BN;

            if constexpr (MODE == MODE_DOWN) {
                __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
                // 16-column groups holding written accumulators (narrowed forward: the present jobs')
                const int glo = B_MN ? 0 : down_group_lo(ti.aux), ghi = B_MN ? BN / 16 : down_group_hi(ti.aux);
                float accv[BN];
#pragma unroll
                for (int c = 0; c < BN / 32; ++c) {
                    const bool live = !empty && 2 * c < ghi && 2 * c + 2 > glo;
                    uint32_t v[32];
                    if (live) { tmem_ld32(t_row + c * 32, v); tmem_wait_ld(); }
#pragma unroll
                    for (int e = 0; e < 32; ++e) accv[c * 32 + e] = live ? __uint_as_float(v[e]) : 0.f;
                }
                bool store = true;
                if constexpr (KSPLIT == 2) {
                    // partial tile layout [BN/4][128 rows][4]: a warp moves 512 contiguous bytes per float4
                    float4* part = reinterpret_cast<float4*>(smem + L::kPartOffset);
                    if (krank == 1) {
                        mbar_wait(pempty_bar, (static_cast<uint32_t>(local) & 1u) ^ 1u);
#pragma unroll
                        for (int g = 0; g < BN / 4; ++g)
                            if (g >= 4 * glo && g < 4 * ghi)
                                st_cluster_v4(mapa_shared(smem_u32(part + g * kBM + rloc), 0),
                                              make_float4(accv[4 * g], accv[4 * g + 1], accv[4 * g + 2], accv[4 * g + 3]));
                        // every lane orders its DSMEM stores at cluster scope before lane 0's release-arrive
                        asm volatile("fence.acq_rel.cluster;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(pfull_bar), 0));
                        store = false;
                    } else {
                        mbar_wait_cluster(pfull_bar, static_cast<uint32_t>(local) & 1u);
#pragma unroll
                        for (int g = 0; g < BN / 4; ++g) {
                            if (g < 4 * glo || g >= 4 * ghi) continue;
                            const float4 q4 = part[g * kBM + rloc];
                            accv[4 * g] += q4.x;
                            accv[4 * g + 1] += q4.y;
                            accv[4 * g + 2] += q4.z;
                            accv[4 * g + 3] += q4.w;
                        }
                        // reads of the partial buffer complete before the follower may overwrite it
                        asm volatile("fence.acq_rel.cluster;" ::: "memory");
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(pempty_bar), 1));
                    }
                }
                if (store && row_ok) down_store_row<BN>(p, dr, out, row, ti.n0, accv);
            } else if constexpr (MODE == MODE_GRADT) {
                float* out = static_cast<float*>(p.out) + (long long)ti.aux * p.split_stride;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t v[32];
                    if (!empty) { tmem_ld32(t_row + c * 32, v); tmem_wait_ld(); }
                    if (row_ok) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const int col = ti.n0 + c * 32 + e;
                            if (col < p.N) out[(long long)col * p.ldo + row] = empty ? 0.f : __uint_as_float(v[e]);
                        }
                    }
                }
            } else {  // MODE_GRAD
                float* out = static_cast<float*>(p.out) + (long long)ti.aux * p.split_stride;
#pragma unroll 1
                for (int c = 0; c < BN / 32; ++c) {
                    uint32_t v[32];
                    if (!empty) { tmem_ld32(t_row + c * 32, v); tmem_wait_ld(); }
                    const int col = ti.n0 + c * 32;
                    if (row_ok && col < p.N) {
                        float4* dst = reinterpret_cast<float4*>(out + (long long)row * p.ldo + col);
#pragma unroll
                        for (int g = 0; g < 8; ++g) {
                            if (col + 4 * g + 4 <= p.N) {
                                float4 w;
                                w.x = empty ? 0.f : __uint_as_float(v[4 * g + 0]);
                                w.y = empty ? 0.f : __uint_as_float(v[4 * g + 1]);
                                w.z = empty ? 0.f : __uint_as_float(v[4 * g + 2]);
                                w.w = empty ? 0.f : __uint_as_float(v[4 * g + 3]);
                                dst[g] = w;
                            }
                        }
                    }
                }
            }
            tc_fence_before();
            mbar_arrive(tempty_bar + acc);
        }
    }

    __syncthreads();
    if constexpr (KSPLIT == 2) cluster_sync();  // no DSMEM traffic may target an exited CTA
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ============================================================================
// MODE_BASE on a CTA pair (cta_group::2): one 256 x 256 output tile per
// cluster, UMMA M=256 N=256.  CTA r of the pair stages A rows [m0+128r, +128)
// and B rows [n0+128r, +128) (half of the N tile) in its own smem; the leader
// CTA issues every tcgen05.mma for the pair, each CTA's TMEM holds its own 128
// accumulator rows.  Per SM this halves the B-operand TMA/L2 traffic of the
// 1-CTA kernel (32 KB per 64-deep k-block instead of 48 KB) and leaves room for
// a 6-stage ring, i.e. ~2.5k cycles of load lookahead.
// ============================================================================
constexpr int kPairBM = 256;
constexpr int kPairBN = 256;

// Grouped raster: tiles walk super-rows of `group_m` m-blocks (m fastest inside a
// super-row) so the A rows of a super-row stay L2-resident while every n-block
// of B streams past them; group_m <= 0 means plain m-fastest order.
__device__ __forceinline__ void pair_tile_coords(const GemmParams& p, int t, int& mb, int& nb) {
    if (p.raster_group < 0) {
        // super-columns of -raster_group n-blocks: n fastest inside, m walks
        const int gn = -p.raster_group;
        const int per_group = gn * p.n_mblk;
        const int g = t / per_group, r = t - g * per_group;
        const int cols_in_group = min(gn, p.n_nblk - g * gn);
        nb = g * gn + r % cols_in_group;
        mb = r / cols_in_group;
        return;
    }
    const int gm = p.raster_group > 0 ? p.raster_group : p.n_mblk;
    const int per_group = gm * p.n_nblk;
    const int g = t / per_group, r = t - g * per_group;
    const int rows_in_group = min(gm, p.n_mblk - g * gm);
    mb = g * gm + r % rows_in_group;
    nb = r / rows_in_group;
}

template <int STAGES>
struct PairSmem {
    static constexpr int kABytes = 128 * kBK * 2;   // this CTA's A rows
    static constexpr int kBBytes = 128 * kBK * 2;   // this CTA's half of the B tile
    static constexpr int kStageBytes = kABytes + kBBytes;
    // output staging of the TMA-store epilogue: per epilogue warp two 32-row x
    // 64-column bf16 boxes (128-byte swizzled rows), written by the warp and stored
    // by one TMA each while the warp converts the next 64 columns
    static constexpr int kOutBufBytes = 32 * 64 * 2;
    static constexpr int kOutOffset = STAGES * kStageBytes;
    static constexpr int kBarOffset = kOutOffset + 4 * 2 * kOutBufBytes;
    static constexpr int kBytes = kBarOffset + (2 * STAGES + 4) * 8 + 16;
    static constexpr int kDynBytes = kBytes + 1024;
};

template <int STAGES, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kNumThreads, 1)
mlora_base_pair_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                       const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                       const __grid_constant__ CUtensorMap tmOut, const GemmParams p) {
    using namespace sm100;
    using L = PairSmem<STAGES>;
    constexpr uint32_t kTmemCols = 512;  // 2 x 256 fp32 accumulator columns
    constexpr uint32_t kIdesc = idesc_bf16_f32(kPairBM, kPairBN, false, B_MN);

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_addr - raw_addr);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;
    uint64_t* tempty_bar = tfull_bar + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

    const uint32_t warp = warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t cta = cluster_ctarank();
    const bool leader = cta == 0;
    const int cluster_id = blockIdx.x >> 1;
    const int nclusters = gridDim.x >> 1;

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&tmA0);
        tma_prefetch_desc(&tmB0);
        tma_prefetch_desc(&tmA1);
        tma_prefetch_desc(&tmB1);
        tma_prefetch_desc(&tmOut);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar + s, 1);    // leader producer's arrive.expect_tx
            mbar_init(empty_bar + s, 1);   // leader MMA's multicast commit
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar + a, 1);   // leader MMA's multicast commit
            mbar_init(tempty_bar + a, 8);  // 4 epilogue warps x 2 CTAs (leader copy used)
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc_2cta(tmem_slot, kTmemCols);
        tmem_relinquish_2cta();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_launch_dependents();
    griddep_wait();  // predecessor's results visible; everything above overlapped its tail

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (both CTAs)
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            // W0 is re-read by every super-row of m-blocks; when asked, its lines are
            // kept in L2 (evict_last) while the streamed A rows age out normally
            const uint64_t pol_b = p.keep_b_in_l2 ? l2_policy_evict_last() : l2_policy_evict_normal();
            for (int t = cluster_id; t < p.num_tiles; t += nclusters) {
                int mb, nb;
                pair_tile_coords(p, t, mb, nb);
                const int m0 = mb * kPairBM + static_cast<int>(cta) * 128;
                const int n0 = nb * kPairBN + static_cast<int>(cta) * 128;
                const int xb0 = p.ext_tab ? __ldg(p.ext_tab + 2 * mb) : 0;
                const int xb1 = p.ext_tab ? __ldg(p.ext_tab + 2 * mb + 1) : 0;
                const int nmain = p.num_kb;
                const int nk = nmain + (xb1 - xb0);
                for (int it = 0; it < nk; ++it) {
                    mbar_wait(empty_bar + stage, phase ^ 1u);
                    const bool ext = it >= nmain;
                    const CUtensorMap* mA = ext ? &tmA1 : &tmA0;
                    const CUtensorMap* mB = ext ? &tmB1 : &tmB0;
                    const int kc = (ext ? (xb0 + it - nmain) : it) * kBK;
                    const uint32_t sA = base_addr + stage * L::kStageBytes;
                    const uint32_t sB = sA + L::kABytes;
                    const uint32_t lbar = smem_u32(full_bar + stage) & kPeerBitMask;
                    if (leader) mbar_arrive_expect_tx(full_bar + stage, 2 * L::kStageBytes);
                    tma_load_2d_2sm(sA, mA, lbar, kc, m0);
                    if constexpr (!B_MN) {
                        tma_load_2d_2sm_hint(sB, mB, lbar, kc, n0, pol_b);
                    } else {
                        tma_load_2d_2sm_hint(sB, mB, lbar, n0, kc, pol_b);
                        tma_load_2d_2sm_hint(sB + 8192, mB, lbar, n0 + 64, kc, pol_b);
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (leader CTA only)
        if (leader) {
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = cluster_id; t < p.num_tiles; t += nclusters, ++local) {
                int mb, nb;
                pair_tile_coords(p, t, mb, nb);
                const int xb0 = p.ext_tab ? __ldg(p.ext_tab + 2 * mb) : 0;
                const int nk = p.num_kb + (p.ext_tab ? __ldg(p.ext_tab + 2 * mb + 1) - xb0 : 0);
                // LoRA k-blocks: only the UMMA k-steps of the rank groups of the jobs present
                // (H / G are block-diagonal: the other groups' columns are exact zeros there)
                const int glo = p.ext_grp ? __ldg(p.ext_grp + 2 * mb) : 0;
                const int ghi = p.ext_grp ? __ldg(p.ext_grp + 2 * mb + 1) : 0x7fffffff;
                const int acc = local & 1;
                const uint32_t use = static_cast<uint32_t>(local >> 1);
                mbar_wait(tempty_bar + acc, (use & 1u) ^ 1u);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kPairBN;
                for (int it = 0; it < nk; ++it) {
                    mbar_wait(full_bar + stage, phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t sA = base_addr + stage * L::kStageBytes;
                        const uint32_t sB = sA + L::kABytes;
#pragma unroll
                        for (int j = 0; j < kBK / kUmmaK; ++j) {
                            if (it >= p.num_kb) {
                                const int g = (xb0 + it - p.num_kb) * (kBK / kUmmaK) + j;
                                if (g < glo || g >= ghi) continue;
                            }
                            const uint64_t ad = sdesc_sw128(sA + j * 32, 16, 1024);
                            const uint64_t bd = B_MN ? sdesc_sw128(sB + j * 2048, 8192, 1024)
                                                     : sdesc_sw128(sB + j * 32, 16, 1024);
                            mma_bf16_2cta(d_tmem, ad, bd, kIdesc, (it | j) != 0 ? 1u : 0u);
                        }
                        tc_commit_2cta_mc(empty_bar + stage, 0x3);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                }
                if (elect_one()) tc_commit_2cta_mc(tfull_bar + acc, 0x3);
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2..5, both CTAs)
        // TMEM -> registers -> bf16 -> a 128-byte-swizzled staging box -> TMA store:
        // each warp owns 32 rows (its TMEM lane quarter) and stores them 64 columns at
        // a time, double-buffered, so the stores run under the next chunk's loads
        const uint32_t q = warp & 3;
        const int rloc = static_cast<int>(cta * 128 + q * 32 + lane);
        const uint32_t out_stage = base_addr + L::kOutOffset + q * 2 * L::kOutBufBytes;
        int local = 0, nstore = 0;
        for (int t = cluster_id; t < p.num_tiles; t += nclusters, ++local) {
            int mb, nb;
            pair_tile_coords(p, t, mb, nb);
            const int acc = local & 1;
            const uint32_t use = static_cast<uint32_t>(local >> 1);
            mbar_wait(tfull_bar + acc, use & 1u);
            tc_fence_after();
            const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * kPairBN;
            const int row = mb * kPairBM + rloc;
            const int row0 = mb * kPairBM + static_cast<int>(cta * 128 + q * 32);
            const bool row_ok = row < p.M;
            float sq = 0.f;  // fused loss: sum of squares of the stored (bf16-rounded) outputs
#pragma unroll 1
            for (int c = 0; c < kPairBN / 64; ++c) {
                const int col0 = nb * kPairBN + c * 64;
                if (col0 >= p.N) break;
                uint32_t v[64];
                tmem_ld32(t_row + c * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
                tmem_ld32(t_row + c * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
                tmem_wait_ld();
                const uint32_t buf = out_stage + static_cast<uint32_t>(nstore & 1) * L::kOutBufBytes;
                if (lane == 0) bulk_wait_group_read<1>();  // the store issued from `buf` two chunks ago has read it
                __syncwarp();
#pragma unroll
                for (int j = 0; j < 8; ++j) {  // 16-byte chunk j: columns col0 + 8j .. col0 + 8j + 7
                    uint32_t w[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        w[h] = pack_bf16x2(__uint_as_float(v[8 * j + 2 * h]), __uint_as_float(v[8 * j + 2 * h + 1]));
                        const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
                        if (col0 + 8 * j < p.N) {
                            sq = fmaf(f.x, f.x, sq);
                            sq = fmaf(f.y, f.y, sq);
                        }
                    }
                    const uint32_t dst = buf + lane * 128u + ((static_cast<uint32_t>(j) ^ (lane & 7u)) << 4);
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(w[0]), "r"(w[1]),
                                 "r"(w[2]), "r"(w[3])
                                 : "memory");
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmOut, buf, col0, row0);  // rows past M / columns past N are clipped
                    bulk_commit_group();
                }
                ++nstore;
            }
            if (p.row_sq && row_ok) p.row_sq[(long long)nb * p.M + row] = sq;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty_bar + acc), 0));
        }
        if (lane == 0) bulk_wait_group_read<0>();  // the staging must outlive every store's read
    }

    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2cta(tmem_base, kTmemCols);
    }
}

}  // namespace mlora
