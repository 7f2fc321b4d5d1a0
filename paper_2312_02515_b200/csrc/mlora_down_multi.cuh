// mlora_down_multi.cuh — the forward rank-r down-projection of NB projections
// that read the SAME input (q, k, v, gate, up all read the layer's hidden
// state x):  H_p = s_j x A_cat_p^T  for p = 0..NB-1, one launch.
//
// The grouped MODE_DOWN launch gives every projection its own tiles: x enters
// the SMs NB times (5 x 64 MiB at C2).  Here a tile is (m-block, 64-column
// rank chunk) for ALL NB projections: a k-block stage holds ONE x tile
// (128 x 64) and the adapter rows of the NB projections, and one x tile feeds
// all of them.
//
// Only the rank rows of the jobs present in the m-block are loaded and
// multiplied: H is block-diagonal, so of a 64-column chunk a 128-row m-block
// needs just the 16-row rank groups [lo, hi) of its own jobs' columns (the
// down table's flags, down_group_lo/hi).  At C2 an m-block lies inside one
// rank-16 job: 16 of the 64 adapter rows per projection.  The NB projections'
// groups sit back to back in the stage (one K-major operand of NB (hi - lo)
// 16-row groups), so a k-step is ONE UMMA 128 x 16 NB (hi - lo) while that is
// <= 256 (C2: N = 80), and its accumulators are adjacent in TMEM.  The stage
// size follows the plan's widest tile (host: `stage_bytes`, `stages`), so a
// narrow plan gets a deeper ring (C2: 8 stages of 26 KB instead of 4 of 56 KB).
//
// As in the grouped kernel (mlora_gemm.cuh, KSPLIT = 2) a CTA pair splits the
// K range.  Once both mainloops are over the pair splits the epilogue too: CTA r
// finalises the projections b with b % 2 == r, so each CTA ships its fp32
// partials of the partner's projections (only the live 16-column groups) over
// DSMEM into the partner's then idle stage ring in one go, then adds the
// partner's partials of its own projections (one IEEE addition: deterministic,
// bitwise equal to the grouped kernel) and applies the per-job select/scale
// store (down_store_row).  Both CTAs' epilogue warps work, so the exposed
// epilogue of a tile is about half of a one-sided hand-over.  Accumulator
// columns outside [lo, hi) do not exist; the epilogue feeds zeros there and the
// per-row job select (a select, not a multiply) keeps them out of every stored
// value.  One TMEM buffer: at C2 every cluster owns at most one tile, so there
// is nothing to double-buffer.
#pragma once

#include "mlora_gemm.cuh"

namespace mlora {

constexpr int kDownMultiMax = 5;

template <int NB>
struct DownMultiArgs {
    CUtensorMap tmA;       // x  [M, K]  K-major, box 64 x 128
    CUtensorMap tmB[NB];   // A_cat_p [R, K] K-major, box 64 x 16 (one 16-row rank group)
    void* out[NB];         // H_p [M, R] bf16
    GemmParams p;          // M, N = R, num_kb, num_tiles (= down tiles), ldo, tables
    int stage_bytes;       // x tile + NB x (widest tile's rank groups) x 2 KB, a multiple of 2 KB
    int stages;            // ring depth (<= kDownMultiMaxStages)
};

constexpr int kDownMultiMaxStages = 12;

struct DownMultiSmem {
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kGroupBytes = 16 * kBK * 2;  // one 16-row rank group (two 1 KB swizzle atoms)
    static constexpr int kRingBytes = 225 * 1024;     // stage ring (runtime stage size and depth)
    // The partner's partials land in this CTA's ring once its mainloop is over:
    // projection b's 16-column group g at (4 b + g) * kPartGroupBytes.
    static constexpr int kPartGroupBytes = kBM * 16 * 4;
    static_assert(kDownMultiMax * 4 * kPartGroupBytes <= kRingBytes, "ring too small for the partials");
    static constexpr int kBarOffset = kRingBytes;
    // full[S], empty[S], tmem_full, tmem_empty, part_full, ring_ready, ring_free, tmem slot
    static constexpr int kBytes = kBarOffset + (2 * kDownMultiMaxStages + 5) * 8 + 16;
    static constexpr int kDynBytes = kBytes + 1024;
    static constexpr int stage_bytes(int nb, int groups) { return kABytes + nb * groups * kGroupBytes; }
    static constexpr int stages_for(int stage_bytes) {
        return kRingBytes / stage_bytes < kDownMultiMaxStages ? kRingBytes / stage_bytes : kDownMultiMaxStages;
    }
};

template <int NB>
__global__ void __launch_bounds__(kNumThreads, 1)
mlora_down_multi_kernel(const __grid_constant__ DownMultiArgs<NB> a) {
    using namespace sm100;
    using L = DownMultiSmem;
    static_assert(NB >= 1 && NB <= kDownMultiMax, "NB out of range");
    constexpr uint32_t kTmemCols = NB * 64 <= 64 ? 64 : NB * 64 <= 128 ? 128 : NB * 64 <= 256 ? 256 : 512;
    const GemmParams& p = a.p;
    const int STAGES = a.stages;
    const uint32_t stage_bytes = static_cast<uint32_t>(a.stage_bytes);

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_addr - raw_addr);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
    uint64_t* empty_bar = full_bar + kDownMultiMaxStages;
    uint64_t* tfull_bar = empty_bar + kDownMultiMaxStages;
    uint64_t* tempty_bar = tfull_bar + 1;
    uint64_t* pfull_bar = tempty_bar + 1;   // the partner's partials have landed in this CTA's ring
    uint64_t* ready_bar = pfull_bar + 1;    // the partner's ring may take this CTA's partials
    uint64_t* free_bar = ready_bar + 1;     // partials consumed, this CTA's ring reusable by TMA
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(free_bar + 1);

    const uint32_t warp = warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t krank = cluster_ctarank();
    const int t_first = static_cast<int>(blockIdx.x) / 2;
    const int t_step = static_cast<int>(gridDim.x) / 2;
    // this CTA's half of the K range
    const int kmid = p.num_kb / 2;
    const int kb0 = krank == 0 ? 0 : kmid, kb1 = krank == 0 ? kmid : p.num_kb;

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&a.tmA);
#pragma unroll
        for (int b = 0; b < NB; ++b) {
            tma_prefetch_desc(&a.tmB[b]);
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, 1);
        }
        mbar_init(tfull_bar, 1);
        mbar_init(tempty_bar, 128);
        mbar_init(pfull_bar, 4);  // the partner's 4 epilogue warps (remote)
        mbar_init(ready_bar, 4);  // the partner's 4 epilogue warps (remote)
        mbar_init(free_bar, 4);   // this CTA's 4 epilogue warps
        fence_barrier_init();
    }
    if (warp == 1) {
        tmem_alloc(tmem_slot, kTmemCols);
        tmem_relinquish();
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_launch_dependents();
    griddep_wait();

    if (warp == 0) {
        // ------------------------------------------------ TMA producer
        if (elect_one()) {
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = t_first; t < p.num_tiles; t += t_step, ++local) {
                const int m0 = __ldg(p.down_tab + 3 * t) * kBM;
                const int n0 = __ldg(p.down_tab + 3 * t + 1) * 64;
                const int fl = __ldg(p.down_tab + 3 * t + 2);
                const int glo = down_group_lo(fl), ng = down_group_hi(fl) - glo;
                const uint32_t tx = L::kABytes + static_cast<uint32_t>(NB * ng * L::kGroupBytes);
                // the ring held the previous tile's partials until this CTA's epilogue read them
                if (local > 0) mbar_wait(free_bar, static_cast<uint32_t>(local - 1) & 1u);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(empty_bar + stage, phase ^ 1u);
                    const uint32_t sA = base_addr + stage * stage_bytes;
                    uint64_t* bar = full_bar + stage;
                    mbar_arrive_expect_tx(bar, tx);
                    tma_load_2d(sA, &a.tmA, bar, kb * kBK, m0);
                    uint32_t sB = sA + L::kABytes;
#pragma unroll
                    for (int b = 0; b < NB; ++b)
                        for (int g = 0; g < ng; ++g, sB += L::kGroupBytes)
                            tma_load_2d(sB, &a.tmB[b], bar, kb * kBK, n0 + 16 * (glo + g));
                    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer
        int stage = 0;
        uint32_t phase = 0;
        int local = 0;
        for (int t = t_first; t < p.num_tiles; t += t_step, ++local) {
            const int fl = __ldg(p.down_tab + 3 * t + 2);
            const int rows = 16 * NB * (down_group_hi(fl) - down_group_lo(fl));  // B operand rows (N)
            mbar_wait(tempty_bar, (static_cast<uint32_t>(local) & 1u) ^ 1u);
            tc_fence_after();
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(full_bar + stage, phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sA = base_addr + stage * stage_bytes;
#pragma unroll
                    for (int j = 0; j < kBK / kUmmaK; ++j) {
                        const uint64_t ad = sdesc_sw128(sA + j * 32, 16, 1024);
                        // the NB projections' rank groups are one K-major operand: N <= 256 per UMMA
                        for (int r0 = 0; r0 < rows; r0 += 256) {
                            const int n = rows - r0 < 256 ? rows - r0 : 256;
                            const uint64_t bd = sdesc_sw128(sA + L::kABytes + r0 * 128 + j * 32, 16, 1024);
                            mma_bf16(tmem_base + r0, ad, bd, idesc_bf16_f32(kBM, n, false, false),
                                     (kb > kb0 || j) ? 1u : 0u);
                        }
                    }
                    tc_commit(empty_bar + stage);
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1u; }
            }
            if (elect_one()) tc_commit(tfull_bar);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2..5)
        const uint32_t q = warp & 3;
        const int rloc = static_cast<int>(q * 32 + lane);
        // partial of projection b, column group g: [4 float4][128 rows] at (4 b + g) * kPartGroupBytes
        float4* part = reinterpret_cast<float4*>(smem);
        const bool empty_k = kb1 == kb0;  // K shorter than two k-blocks: this half adds nothing
        int local = 0;
        for (int t = t_first; t < p.num_tiles; t += t_step, ++local) {
            const uint32_t par = static_cast<uint32_t>(local) & 1u;
            const int m0 = __ldg(p.down_tab + 3 * t) * kBM;
            const int n0 = __ldg(p.down_tab + 3 * t + 1) * 64;
            const int aux = __ldg(p.down_tab + 3 * t + 2);
            const int glo = down_group_lo(aux), ghi = down_group_hi(aux), ng = ghi - glo;
            const int row = m0 + rloc;
            const bool row_ok = row < p.M;
            // the row's job lookup, once for all NB projections, under the mainloop
            const DownRow dr = down_row_info(p, row, m0, aux);
            mbar_wait(tfull_bar, par);  // this CTA's MMAs are done: its ring is idle
            tc_fence_after();
            // projection b's group g (glo <= g < ghi) sits at TMEM column 16 (b ng + g - glo)
            auto load_acc = [&](int b, float* accv) {
                uint32_t v[4][16];
#pragma unroll
                for (int g = 0; g < 4; ++g)
                    if (!empty_k && g >= glo && g < ghi)
                        tmem_ld16(tmem_base + ((q * 32u) << 16) + 16 * (b * ng + g - glo), v[g]);
                tmem_wait_ld();  // one wait for all of the projection's live groups
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    const bool live = !empty_k && g >= glo && g < ghi;
#pragma unroll
                    for (int e = 0; e < 16; ++e) accv[16 * g + e] = live ? __uint_as_float(v[g][e]) : 0.f;
                }
            };
            auto part_at = [&](int b, int g, int f) { return part + ((4 * b + g) * 4 + f) * kBM + rloc; };
            // Symmetric hand-over: CTA r finalises the projections b with b % 2 == r and ships
            // its partials of the others into the partner's ring, so both CTAs' epilogue warps
            // share the work (the partner's ring must be idle first: `ready`).
            const uint32_t partner = krank ^ 1u;
            // this CTA's ring: its TMA data were all consumed by the MMAs behind tfull
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(ready_bar), partner));
            mbar_wait_cluster(ready_bar, par);  // the partner's ring may take this CTA's partials
            for (int b = 0; b < NB; ++b) {
                if ((b & 1) == static_cast<int>(krank)) continue;
                float accv[64];
                load_acc(b, accv);
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    if (g < glo || g >= ghi) continue;
#pragma unroll
                    for (int f = 0; f < 4; ++f) {
                        const float* v = accv + 16 * g + 4 * f;
                        st_cluster_v4(mapa_shared(smem_u32(part_at(b, g, f)), partner), make_float4(v[0], v[1], v[2], v[3]));
                    }
                }
            }
            // every lane orders its DSMEM stores at cluster scope before lane 0's release-arrive
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(pfull_bar), partner));
            mbar_wait_cluster(pfull_bar, par);  // the partner's partials of this CTA's projections
            for (int b = 0; b < NB; ++b) {
                if ((b & 1) != static_cast<int>(krank)) continue;
                float accv[64];
                load_acc(b, accv);
                // K-half 0 + K-half 1: one IEEE addition, commutative, so the result is the
                // same bits whichever CTA finalises (bitwise equal to the grouped kernel)
#pragma unroll
                for (int g = 0; g < 4; ++g) {
                    if (g < glo || g >= ghi) continue;
#pragma unroll
                    for (int f = 0; f < 4; ++f) {
                        const float4 q4 = *part_at(b, g, f);
                        float* v = accv + 16 * g + 4 * f;
                        v[0] += q4.x;
                        v[1] += q4.y;
                        v[2] += q4.z;
                        v[3] += q4.w;
                    }
                }
                if (row_ok)
                    down_store_row<64>(p, dr, static_cast<__nv_bfloat16*>(a.out[b]), row, n0, accv);
            }
            // partial reads complete before this CTA's producer may refill its ring
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(free_bar);
            tc_fence_before();
            mbar_arrive(tempty_bar);
        }
    }

    __syncthreads();
    cluster_sync();  // no DSMEM traffic may target an exited CTA
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem_base, kTmemCols);
    }
}

}  // namespace mlora
