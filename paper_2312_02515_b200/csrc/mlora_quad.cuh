// mlora_quad.cuh — MODE_BASE on a cluster of 4 CTAs = two CTA pairs sharing the
// weight tile through TMA multicast.
//
// Cluster tile: 512 rows x 256 cols.  Pair p (CTAs 2p, 2p+1) computes rows
// [512 mb + 256 p, +256) with UMMA M=256 N=256 (cta_group::2) exactly as the
// pair kernel; both pairs consume the same B tile (W0 rows n0..n0+255), so each
// B half-tile (128 rows, per CTA rank r) is loaded ONCE from L2 and multicast to
// CTAs r and r+2: CTA (p, r) issues the 64-row box p of half r.  Per SM this
// removes half of the B-operand L2->SM traffic (a quarter of all operand
// traffic) at identical MMA work — less data-movement energy under the 1 kW cap.
//
// Synchronisation differences from the pair kernel:
//   * a stage's smem is written by the other pair's multicast too, so a stage is
//     free only after BOTH pairs' MMAs consumed it: each pair leader commits to
//     the empty barriers of all 4 CTAs (mask 0xF) and empty barriers count 2;
//   * the LoRA k-blocks are the union over the cluster's 512 rows (ext512), so
//     both pairs walk the same k-block sequence (block-diagonal H makes the
//     extra products exactly zero).
#pragma once

#include "mlora_gemm.cuh"

namespace mlora {

constexpr int kQuadBM = 512;

__device__ __forceinline__ void tma_load_2d_2sm_mc(uint32_t smem_dst, const CUtensorMap* map, uint32_t leader_bar,
                                                   int c0, int c1, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        ".multicast::cluster [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "h"(mask)
        : "memory");
}

template <int STAGES, bool B_MN>
__global__ void __launch_bounds__(kNumThreads, 1)
mlora_base_quad_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                       const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                       const GemmParams p) {
    using namespace sm100;
    using L = PairSmem<STAGES>;
    constexpr uint32_t kTmemCols = 512;
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
    const uint32_t cta = cluster_ctarank();   // 0..3
    const uint32_t pair = cta >> 1, r = cta & 1;
    const bool leader = r == 0;
    const int cluster_id = blockIdx.x >> 2;
    const int nclusters = gridDim.x >> 2;

    if (warp == 0 && elect_one()) {
        tma_prefetch_desc(&tmA0);
        tma_prefetch_desc(&tmB0);
        tma_prefetch_desc(&tmA1);
        tma_prefetch_desc(&tmB1);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full_bar + s, 1);    // pair leader's arrive.expect_tx
            mbar_init(empty_bar + s, 2);   // both pair leaders' multicast commits
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(tfull_bar + a, 1);
            mbar_init(tempty_bar + a, 8);
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
    griddep_wait();

    if (warp == 0) {
        // ------------------------------------------------ TMA producer (all 4 CTAs)
        if (elect_one()) {
            const uint16_t bmask = static_cast<uint16_t>((1u << r) | (1u << (r + 2)));
            int stage = 0;
            uint32_t phase = 0;
            for (int t = cluster_id; t < p.num_tiles; t += nclusters) {
                int mb, nb;
                pair_tile_coords(p, t, mb, nb);
                const int m0 = mb * kQuadBM + static_cast<int>(pair) * kPairBM + static_cast<int>(r) * 128;
                const int nh = nb * kPairBN + static_cast<int>(r) * 128;  // this CTA's B half
                const int xb0 = __ldg(p.ext_tab + 2 * mb), xb1 = __ldg(p.ext_tab + 2 * mb + 1);
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
                    // box `pair` (64 rows / 64 cols) of this CTA's B half, multicast to CTA r of both pairs
                    if constexpr (!B_MN)
                        tma_load_2d_2sm_mc(sB + pair * 8192, mB, lbar, kc, nh + 64 * static_cast<int>(pair), bmask);
                    else
                        tma_load_2d_2sm_mc(sB + pair * 8192, mB, lbar, nh + 64 * static_cast<int>(pair), kc, bmask);
                    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (pair leaders)
        if (leader) {
            const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pair));
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = cluster_id; t < p.num_tiles; t += nclusters, ++local) {
                int mb, nb;
                pair_tile_coords(p, t, mb, nb);
                const int nk = p.num_kb + (__ldg(p.ext_tab + 2 * mb + 1) - __ldg(p.ext_tab + 2 * mb));
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
                            const uint64_t ad = sdesc_sw128(sA + j * 32, 16, 1024);
                            const uint64_t bd = B_MN ? sdesc_sw128(sB + j * 2048, 8192, 1024)
                                                     : sdesc_sw128(sB + j * 32, 16, 1024);
                            mma_bf16_2cta(d_tmem, ad, bd, kIdesc, (it | j) != 0 ? 1u : 0u);
                        }
                        tc_commit_2cta_mc(empty_bar + stage, 0xF);  // the stage is shared by both pairs
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1u; }
                }
                if (elect_one()) tc_commit_2cta_mc(tfull_bar + acc, pair_mask);
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------ epilogue (warps 2..5, all 4 CTAs)
        const uint32_t q = warp & 3;
        const int rloc = static_cast<int>(pair * kPairBM + r * 128 + q * 32 + lane);
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(p.out);
        int local = 0;
        for (int t = cluster_id; t < p.num_tiles; t += nclusters, ++local) {
            int mb, nb;
            pair_tile_coords(p, t, mb, nb);
            const int acc = local & 1;
            const uint32_t use = static_cast<uint32_t>(local >> 1);
            mbar_wait(tfull_bar + acc, use & 1u);
            tc_fence_after();
            const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * kPairBN;
            const int row = mb * kQuadBM + rloc;
            const bool row_ok = row < p.M;
            float sq = 0.f;
#pragma unroll 1
            for (int c = 0; c < kPairBN / 32; ++c) {
                uint32_t v[32];
                tmem_ld32(t_row + c * 32, v);
                tmem_wait_ld();
                const int col = nb * kPairBN + c * 32;
                if (row_ok && col < p.N) {
                    uint4* dst = reinterpret_cast<uint4*>(out + (long long)row * p.ldo + col);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (col + 8 * g + 8 <= p.N) {
                            uint32_t w[4];
#pragma unroll
                            for (int h = 0; h < 4; ++h) {
                                w[h] = pack_bf16x2(__uint_as_float(v[8 * g + 2 * h]), __uint_as_float(v[8 * g + 2 * h + 1]));
                                const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[h]));
                                sq = fmaf(f.x, f.x, sq);
                                sq = fmaf(f.y, f.y, sq);
                            }
                            dst[g] = make_uint4(w[0], w[1], w[2], w[3]);
                        }
                    }
                }
            }
            if (p.row_sq && row_ok) p.row_sq[(long long)nb * p.M + row] = sq;
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(mapa_shared(smem_u32(tempty_bar + acc), 2 * pair));
        }
    }

    __syncthreads();
    cluster_sync();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_2cta(tmem_base, kTmemCols);
    }
}

}  // namespace mlora
