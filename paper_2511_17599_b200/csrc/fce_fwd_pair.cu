// CTA-pair forward: the fce_tile_kernel<kEpiForward> schedule on
// tcgen05.mma.cta_group::2 (M = 256, N = 256, K = 16).
//
// A pair owns 256 rows of H; per 64-deep K stage each CTA loads its own 128
// rows of H and its 128-row half of the 256-wide W tile (32 KB / stage / CTA
// instead of 48 KB), and the even CTA issues one MMA for both.  Each CTA's
// TMEM then holds S = H_rows . W_tile^T for its 128 rows x all 256 columns,
// so the epilogue (online max / sum-exp + target gather, Alg. 1,
// reference proj/include/fusedce/fused_forward.hpp:47-73) is the 1-CTA one
// unchanged.  Halving the W bytes staged per flop cuts L2->SMEM traffic and
// SMEM reads, which is what the power-capped clock pays for.
//
// Roles (256 threads, 1 CTA / SM, cluster of 2): warp 0 TMA (both CTAs),
// warp 1 MMA (even CTA), warp 2 TMEM allocation, warps 4-7 epilogue.
#include <cmath>

#include "fce_internal.h"
#include "sm100_ptx.cuh"

namespace fce {

using namespace ptx;

namespace {
constexpr int kFS = 6;                       // smem ring depth
constexpr int kFA = 128 * kBK * 2;           // this CTA's 128 rows of H per stage
constexpr int kFB = 128 * kBK * 2;           // this CTA's 128 rows of the W tile per stage
constexpr int kFwdPairSmem = kFS * (kFA + kFB) + 1024 + 256;
constexpr float kL2e = 1.4426950408889634f;

struct FUnit {
    int m_pair, split, t0, nt;
};

// L2 raster as the 1-CTA forward (get_unit): groups of m_group row pairs,
// split slow and row pair fast inside a group.
__device__ __forceinline__ FUnit fwd_unit(const TileParams& p, int u) {
    FUnit r;
    const int per_group = p.m_group * p.splits;
    const int g = u / per_group;
    const int gsize = min(p.m_group, p.m_blocks - g * p.m_group);
    const int local = u - g * per_group;
    const int s = local / gsize;
    r.m_pair = g * p.m_group + (local - s * gsize);
    r.split = s;
    r.t0 = static_cast<int>(static_cast<long long>(s) * p.v_tiles / p.splits);
    r.nt = static_cast<int>(static_cast<long long>(s + 1) * p.v_tiles / p.splits) - r.t0;
    return r;
}
}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    fce_fwd_pair_kernel(const __grid_constant__ TileParams p, const __grid_constant__ TensorMaps maps) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kFS * kFA;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kFS * kFB);
    uint64_t* full = bars;
    uint64_t* empty = bars + kFS;
    uint64_t* tfull = bars + 2 * kFS;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = blockIdx.x >> 1;
    const int n_pairs = gridDim.x >> 1;
    // compacted forward: row pairs past the device count of live rows are skipped
    const int n_eff = p.n_valid ? static_cast<int>(min(static_cast<unsigned long long>(p.n_rows), *p.n_valid))
                                : p.n_rows;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kFS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 8);  // 4 epilogue warps x 2 CTAs, on the even CTA
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
        // ------------------------------------------------ TMA producer (both CTAs)
        const uint32_t leader_full0 = mapa_shared(&full[0], 0);
        const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
        const uint64_t pol = policy_evict_normal();
        int stage = 0;
        uint32_t phase = 0;
        for (int u = pair; u < p.units; u += n_pairs) {
            const FUnit un = fwd_unit(p, u);
            if (un.m_pair * 256 >= n_eff) continue;
            const int a_row = un.m_pair * 256 + rank * 128;
            for (int t = 0; t < un.nt; ++t) {
                const int b_row = (un.t0 + t) * kBN + rank * 128;
                for (int kb = 0; kb < p.k_blocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx_w(&full[stage], 2 * (kFA + kFB));
                    const uint32_t fb = leader_full0 + stage * 8;
                    tma_load_2d_pair_w(sa0 + stage * kFA, &maps.a0, fb, kb * kBK, a_row, pol);
                    tma_load_2d_pair_w(sb0 + stage * kFB, &maps.b0, fb, kb * kBK, b_row, pol);
                    if (++stage == kFS) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------ MMA issuer (even CTA)
        if (rank == 0) {
            const uint32_t idesc = make_idesc_bf16(256, kBN, 0, 0);
            const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
            const uint64_t ad0 = make_sdesc_sw128(sa0, 16, 1024);
            const uint64_t bd0 = make_sdesc_sw128(sb0, 16, 1024);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int u = pair; u < p.units; u += n_pairs) {
                const FUnit un = fwd_unit(p, u);
                if (un.m_pair * 256 >= n_eff) continue;
                for (int t = 0; t < un.nt; ++t) {
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * kBN;
                    for (int kb = 0; kb < p.k_blocks; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint64_t ads = ad0 + static_cast<uint64_t>((stage * kFA) >> 4);
                        const uint64_t bds = bd0 + static_cast<uint64_t>((stage * kFB) >> 4);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k)
                            umma_bf16_pair_w(d_tmem, ads + 2 * k, bds + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
                        umma_commit_pair_w(&empty[stage], 0x3);
                        if (++stage == kFS) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    umma_commit_pair_w(&tfull[acc], 0x3);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------ epilogue (both CTAs)
        const int q = warp & 3;
        const int r = q * 32 + lane;
        const uint32_t leader_tempty0 = mapa_shared(&tempty[0], 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = pair; u < p.units; u += n_pairs) {
            const FUnit un = fwd_unit(p, u);
            if (un.m_pair * 256 >= n_eff) continue;
            const int64_t row = static_cast<int64_t>(un.m_pair) * 256 + rank * 128 + r;
            const bool row_ok = row < n_eff;
            bool skip = true;
            int64_t tcol = -1;
            if (row_ok) {
                const int64_t y = p.targets[row];
                skip = p.has_ignore && y == p.ignore_index;
                tcol = y - p.col_global0;
            }
            float m_run = -INFINITY, a_run = 0.f, zt = 0.f;
            bool found = false;
            for (int t = 0; t < un.nt; ++t) {
                const int n_tile = un.t0 + t;
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                       static_cast<uint32_t>(acc * kBN);
#pragma unroll 1
                for (int c = 0; c < kBN / 32; ++c) {
                    float v[32];
                    tmem_ld32(taddr + c * 32, v);
                    const int col0 = n_tile * kBN + c * 32;
                    if (col0 + 32 > p.v_cols) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j >= p.v_cols) v[j] = -INFINITY;
                    }
                    float cmax = v[0];
#pragma unroll
                    for (int j = 1; j < 32; ++j) cmax = fmaxf(cmax, v[j]);
                    if (cmax > m_run) {
                        a_run *= ex2((m_run - cmax) * kL2e);
                        m_run = cmax;
                    }
                    if (cmax != -INFINITY) {
                        float s0 = 0.f, s1 = 0.f;
#pragma unroll
                        for (int j = 0; j < 32; j += 2) {
                            s0 += ex2((v[j] - m_run) * kL2e);
                            s1 += ex2((v[j + 1] - m_run) * kL2e);
                        }
                        a_run += s0 + s1;
                    }
                    // target capture only inside this launch's valid columns
                    const int64_t tc = tcol - col0;
                    if (tc >= 0 && tc < 32 && col0 + tc < p.v_cols) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j == tc) zt = v[j];
                        found = true;
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(leader_tempty0 + acc * 8);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
            if (row_ok) {
                const size_t off = static_cast<size_t>(un.split) * p.n_rows + row;
                p.part_m[off] = skip ? -INFINITY : m_run;
                p.part_a[off] = skip ? 0.f : a_run;
                p.part_zt[off] = (skip || !found) ? 0.f : zt;
                p.part_found[off] = (skip || !found) ? 0 : 1;
            }
        }
    }

    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == 2) tmem_dealloc_pair<512>(tmem_base);
}

// p.m_blocks counts 256-row pairs here; grid = 2 x min(pairs on the device, units).
cudaError_t launch_fwd_pair(const TileParams& p, const TensorMaps& maps, int sms, cudaStream_t stream) {
    {
        cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fce_fwd_pair_kernel), kFwdPairSmem);
        if (e != cudaSuccess) return e;
    }
    int pairs = sms / 2;
    if (pairs > p.units) pairs = p.units;
    if (pairs < 1) pairs = 1;
    fce_fwd_pair_kernel<<<2 * pairs, kThreads, kFwdPairSmem, stream>>>(p, maps);
    return cudaGetLastError();
}

}  // namespace fce
