// mlora_down_multi.cuh — the forward rank-r down-projection of NB projections
// that read the SAME input (q, k, v, gate, up all read the layer's hidden
// state x):  H_p = s_j x A_cat_p^T  for p = 0..NB-1, one launch.
//
// The grouped MODE_DOWN launch gives every projection its own tiles: x enters
// the SMs NB times (5 x 64 MiB at C2) and every k-step is a narrow N = 64 MMA.
// Here a tile is (m-block, 64-column rank chunk) for ALL NB projections: a
// k-block stage holds ONE x tile (128 x 64) and the NB adapter tiles (64 x 64
// each, back to back = one K-major operand of NB x 64 rows), and the MMA warp
// issues UMMA 128 x 256 (four projections) plus one 128 x 64(NB-4) per k-step
// into NB adjacent 64-column TMEM accumulators.
//
// As in the grouped kernel (mlora_gemm.cuh, KSPLIT = 2) a CTA pair splits the
// K range.  Once both mainloops are over, the follower ships all NB fp32
// partial tiles over DSMEM into the leader's then idle stage ring in one go
// (one handshake and one cluster fence per tile, not one per projection); the
// leader adds them in a fixed order (deterministic) and applies the per-job
// select/scale store (down_store_row).  One TMEM buffer (NB x 64 <= 512
// columns): at C2 every cluster owns at most one tile, so there is nothing to
// double-buffer.
#pragma once

#include "mlora_gemm.cuh"

namespace mlora {

constexpr int kDownMultiMax = 5;

template <int NB>
struct DownMultiArgs {
    CUtensorMap tmA;       // x  [M, K]  K-major, box 64 x 128
    CUtensorMap tmB[NB];   // A_cat_p [R, K] K-major, box 64 x 64
    void* out[NB];         // H_p [M, R] bf16
    GemmParams p;          // M, N = R, num_kb, num_tiles (= down tiles), ldo, tables
};

template <int NB, int STAGES>
struct DownMultiSmem {
    static constexpr int kABytes = kBM * kBK * 2;
    static constexpr int kBBytes = 64 * kBK * 2;
    static constexpr int kStageBytes = kABytes + NB * kBBytes;
    // The follower's NB fp32 partial tiles land in the leader's stage ring once
    // its mainloop is over (no dedicated buffer: the ring is idle then).
    static constexpr int kPartTileBytes = kBM * 64 * 4;
    static constexpr int kBarOffset = STAGES * kStageBytes;
    static_assert(NB * kPartTileBytes <= kBarOffset, "stage ring too small for the partials");
    // full[S], empty[S], tmem_full, tmem_empty, part_full, ring_ready, ring_free, tmem slot
    static constexpr int kBytes = kBarOffset + (2 * STAGES + 5) * 8 + 16;
    static constexpr int kDynBytes = kBytes + 1024;
};

template <int NB, int STAGES>
__global__ void __launch_bounds__(kNumThreads, 1)
mlora_down_multi_kernel(const __grid_constant__ DownMultiArgs<NB> a) {
    using namespace sm100;
    using L = DownMultiSmem<NB, STAGES>;
    static_assert(NB >= 1 && NB <= kDownMultiMax, "NB out of range");
    constexpr uint32_t kTmemCols = NB * 64 <= 64 ? 64 : NB * 64 <= 128 ? 128 : NB * 64 <= 256 ? 256 : 512;
    constexpr uint32_t kIdesc256 = idesc_bf16_f32(kBM, 256, false, false);
    constexpr uint32_t kIdescRem = idesc_bf16_f32(kBM, (NB % 4 ? NB % 4 : 4) * 64, false, false);
    const GemmParams& p = a.p;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    const uint32_t base_addr = (raw_addr + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (base_addr - raw_addr);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
    uint64_t* empty_bar = full_bar + STAGES;
    uint64_t* tfull_bar = empty_bar + STAGES;
    uint64_t* tempty_bar = tfull_bar + 1;
    uint64_t* pfull_bar = tempty_bar + 1;   // leader: the follower's partials have landed
    uint64_t* ready_bar = pfull_bar + 1;    // follower: the leader's ring may take them
    uint64_t* free_bar = ready_bar + 1;     // leader: partials consumed, ring reusable by TMA
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
        for (int b = 0; b < NB; ++b) tma_prefetch_desc(&a.tmB[b]);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar + s, 1);
            mbar_init(empty_bar + s, 1);
        }
        mbar_init(tfull_bar, 1);
        mbar_init(tempty_bar, 128);
        mbar_init(pfull_bar, 4);  // follower's 4 epilogue warps (remote)
        mbar_init(ready_bar, 4);  // leader's 4 epilogue warps (remote)
        mbar_init(free_bar, 4);   // leader's 4 epilogue warps
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
                // the leader's ring held the previous tile's partials until its epilogue read them
                if (krank == 0 && local > 0) mbar_wait(free_bar, static_cast<uint32_t>(local - 1) & 1u);
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(empty_bar + stage, phase ^ 1u);
                    const uint32_t sA = base_addr + stage * L::kStageBytes;
                    uint64_t* bar = full_bar + stage;
                    mbar_arrive_expect_tx(bar, L::kStageBytes);
                    tma_load_2d(sA, &a.tmA, bar, kb * kBK, m0);
#pragma unroll
                    for (int b = 0; b < NB; ++b)
                        tma_load_2d(sA + L::kABytes + b * L::kBBytes, &a.tmB[b], bar, kb * kBK, n0);
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
            mbar_wait(tempty_bar, (static_cast<uint32_t>(local) & 1u) ^ 1u);
            tc_fence_after();
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(full_bar + stage, phase);
                tc_fence_after();
                if (elect_one()) {
                    const uint32_t sA = base_addr + stage * L::kStageBytes;
#pragma unroll
                    for (int j = 0; j < kBK / kUmmaK; ++j) {
                        const uint64_t ad = sdesc_sw128(sA + j * 32, 16, 1024);
                        // the NB adapter tiles sit back to back: one K-major operand of
                        // NB x 64 rows, issued as N = 256 (4 projections) + remainder
#pragma unroll
                        for (int b0 = 0; b0 < NB; b0 += 4) {
                            const uint64_t bd = sdesc_sw128(sA + L::kABytes + b0 * L::kBBytes + j * 32, 16, 1024);
                            const uint32_t idesc = NB - b0 >= 4 ? kIdesc256 : kIdescRem;
                            mma_bf16(tmem_base + b0 * 64, ad, bd, idesc, (kb > kb0 || j) ? 1u : 0u);
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
        // partial tile b: [16 float4 column groups][128 rows] at b * kPartTileBytes
        float4* part = reinterpret_cast<float4*>(smem);
        const bool empty_k = kb1 == kb0;  // K shorter than two k-blocks: this half adds nothing
        int local = 0;
        for (int t = t_first; t < p.num_tiles; t += t_step, ++local) {
            const uint32_t par = static_cast<uint32_t>(local) & 1u;
            const int m0 = __ldg(p.down_tab + 3 * t) * kBM;
            const int n0 = __ldg(p.down_tab + 3 * t + 1) * 64;
            const int aux = __ldg(p.down_tab + 3 * t + 2);
            mbar_wait(tfull_bar, par);  // this CTA's MMAs are done: its ring is idle
            tc_fence_after();
            const int row = m0 + rloc;
            const bool row_ok = row < p.M;
            auto load_acc = [&](int b, float* accv) {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    uint32_t v[32];
                    if (!empty_k) {
                        tmem_ld32(tmem_base + ((q * 32u) << 16) + b * 64 + c * 32, v);
                        tmem_wait_ld();
                    }
#pragma unroll
                    for (int e = 0; e < 32; ++e) accv[c * 32 + e] = empty_k ? 0.f : __uint_as_float(v[e]);
                }
            };
            if (krank == 1) {
                // ship all NB partials into the leader's ring in one go
                mbar_wait_cluster(ready_bar, par);
                for (int b = 0; b < NB; ++b) {
                    float accv[64];
                    load_acc(b, accv);
                    float4* dst = part + b * (L::kPartTileBytes / 16);
#pragma unroll
                    for (int g = 0; g < 16; ++g)
                        st_cluster_v4(mapa_shared(smem_u32(dst + g * kBM + rloc), 0),
                                      make_float4(accv[4 * g], accv[4 * g + 1], accv[4 * g + 2], accv[4 * g + 3]));
                }
                // every lane orders its DSMEM stores at cluster scope before lane 0's release-arrive
                asm volatile("fence.acq_rel.cluster;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(pfull_bar), 0));
            } else {
                // the ring's TMA data were all consumed by the MMAs behind tfull
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(ready_bar), 1));
                mbar_wait_cluster(pfull_bar, par);
                for (int b = 0; b < NB; ++b) {
                    float accv[64];
                    load_acc(b, accv);
                    const float4* src = part + b * (L::kPartTileBytes / 16);
#pragma unroll
                    for (int g = 0; g < 16; ++g) {
                        const float4 q4 = src[g * kBM + rloc];
                        accv[4 * g] += q4.x;
                        accv[4 * g + 1] += q4.y;
                        accv[4 * g + 2] += q4.z;
                        accv[4 * g + 3] += q4.w;
                    }
                    if (row_ok)
                        down_store_row<64>(p, static_cast<__nv_bfloat16*>(a.out[b]), row, m0, n0, aux, accv);
                }
                // partial reads complete before the producer's TMA may refill the ring
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(free_bar);
            }
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
