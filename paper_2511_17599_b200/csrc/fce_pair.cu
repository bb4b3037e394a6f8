// CTA-pair (cta_group::2) variant of the tile kernel's generic contraction:
// one 256 x 256 output tile per pair, each CTA loading its 128 rows of A and
// its 128 columns of B per 64-deep K stage (32 KB / stage / CTA, 6 stages),
// the even CTA issuing tcgen05.mma.cta_group::2 (M=256, N=256, K=16) for both.
// Used by fce_gemm_bf16 (pair = 1) and as the building block the persistent
// kernels follow.
#include <cmath>
#include <cstdio>

#include "fce_internal.h"
#include "sm100_ptx.cuh"

namespace fce {

using namespace ptx;

constexpr int kPairStages = 6;
constexpr int kPairStageA = 128 * kBK * 2;  // this CTA's 128 rows of A
constexpr int kPairStageB = 128 * kBK * 2;  // this CTA's 128 columns of B
constexpr int kPairSmem = kPairStages * (kPairStageA + kPairStageB) + 1024 + 256;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    fce_pair_gemm_kernel(const __grid_constant__ GemmProblem q, const __grid_constant__ TensorMaps maps) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kPairStages * kPairStageA;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kPairStages * kPairStageB);
    uint64_t* full = bars;
    uint64_t* empty = bars + kPairStages;
    uint64_t* tfull = bars + 2 * kPairStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1;
    const int n_pairs = gridDim.x >> 1;
    const int m_tiles = (q.m + 255) / 256;
    const int n_tiles = (q.n + 255) / 256;
    const int units = m_tiles * n_tiles;
    // L2 raster: groups of kGroupM row tiles, row tile fastest inside a group
    constexpr int kGroupM = 8;
    auto tile_of = [&](int u, int& mt, int& nt) {
        const int per_group = kGroupM * n_tiles;
        const int g = u / per_group;
        const int gsize = min(kGroupM, m_tiles - g * kGroupM);
        const int l = u - g * per_group;
        nt = l / gsize;
        mt = g * kGroupM + (l - nt * gsize);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPairStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&maps.a0);
        tma_prefetch_desc(&maps.b0);
    }
    if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t leader_full0 = mapa_shared(&full[0], 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int u = pair; u < units; u += n_pairs) {
                int mt, nt;
                tile_of(u, mt, nt);
                const int a_row = mt * 256 + rank * 128;
                const int b_row = nt * 256 + rank * 128;
                for (int kb = 0; kb < q.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0)
                        mbar_arrive_expect_tx(&full[stage], 2 * (kPairStageA + kPairStageB));
                    const uint32_t fb = leader_full0 + stage * 8;
                    uint8_t* a_dst = sA + stage * kPairStageA;
                    uint8_t* b_dst = sB + stage * kPairStageB;
                    if (!q.a_mn) {
                        tma_load_2d_pair(a_dst, &maps.a0, fb, kb * kBK, a_row, kEvictNormal);
                    } else {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            tma_load_2d_pair(a_dst + j * 8192, &maps.a0, fb, a_row + 64 * j, kb * kBK,
                                             kEvictNormal);
                    }
                    if (!q.b_mn) {
                        tma_load_2d_pair(b_dst, &maps.b0, fb, kb * kBK, b_row, kEvictNormal);
                    } else {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            tma_load_2d_pair(b_dst + j * 8192, &maps.b0, fb, b_row + 64 * j, kb * kBK,
                                             kEvictNormal);
                    }
                    if (++stage == kPairStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            const uint32_t idesc = make_idesc_bf16(256, 256, q.a_mn, q.b_mn);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int u = pair; u < units; u += n_pairs) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kBN;
                for (int kb = 0; kb < q.k_blocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + stage * kPairStageA);
                    const uint32_t b_base = smem_u32(sB + stage * kPairStageB);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k) {
                        const uint64_t ad = q.a_mn ? make_sdesc_sw128(a_base + k * 2048, 8192, 1024)
                                                   : make_sdesc_sw128(a_base + k * 32, 16, 1024);
                        const uint64_t bd = q.b_mn ? make_sdesc_sw128(b_base + k * 2048, 8192, 1024)
                                                   : make_sdesc_sw128(b_base + k * 32, 16, 1024);
                        umma_bf16_pair(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
                    }
                    umma_commit_pair(&empty[stage], 0x3);
                    if (++stage == kPairStages) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_pair(&tfull[acc], 0x3);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        const int qw = warp & 3;
        const int r = qw * 32 + lane;
        const uint32_t leader_tempty0 = mapa_shared(&tempty[0], 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = pair; u < units; u += n_pairs) {
            int mt, nt;
            tile_of(u, mt, nt);
            const int64_t row = static_cast<int64_t>(mt) * 256 + rank * 128 + r;
            mbar_wait(&tfull[acc], acc_phase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(qw * 32) << 16) +
                                   static_cast<uint32_t>(acc * kBN);
#pragma unroll 1
            for (int c = 0; c < kBN / 32; ++c) {
                float v[32];
                tmem_ld32(taddr + c * 32, v);
                const int col0 = nt * 256 + c * 32;
                if (row < q.m && q.accumulate != 2) {
                    float* dst = q.c + row * q.ldc + col0;
                    const bool vec = (col0 + 32 <= q.n) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                    if (vec) {
                        if (q.accumulate) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4) red_add_v4(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; j += 4) st_v4(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
                        }
                    } else {
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < q.n) {
                                if (q.accumulate)
                                    atomicAdd(dst + j, v[j]);
                                else
                                    dst[j] = v[j];
                            }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(leader_tempty0 + acc * 8);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
        }
    }

    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 2) tmem_dealloc_pair<512>(tmem_base);
}

cudaError_t launch_pair_gemm(const GemmProblem& q, const TensorMaps& maps, int sms,
                             cudaStream_t stream) {
    {
        cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fce_pair_gemm_kernel), kPairSmem);
        if (e != cudaSuccess) return e;
    }
    const int units = ((q.m + 255) / 256) * ((q.n + 255) / 256);
    int pairs = sms / 2;
    if (pairs > units) pairs = units;
    fce_pair_gemm_kernel<<<2 * pairs, kThreads, kPairSmem, stream>>>(q, maps);
    return cudaGetLastError();
}

}  // namespace fce
