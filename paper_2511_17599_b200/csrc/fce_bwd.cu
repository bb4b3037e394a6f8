// Persistent fused backward (one launch per fce_backward call).
//
// The backward of the reference (fused_backward_recompute,
// proj/include/fusedce/fused_backward.hpp:118-140; per-(n, v) work in
// accumulate_grads_block 26-56) is three contractions over different index
// pairs: S = H.W^T (recompute, contract d), dH = G.W (contract v) and
// dW = G^T.H (contract n).  At D = 4096 neither dH[m,:] nor dW[v,:] fits TMEM,
// so each contraction stays output-stationary on the tensor cores and only
// G = gamma (softmax - onehot), bf16, moves between them through a ring of
// two group slots in HBM.
//
// Execution: CTA pairs (cluster of 2, tcgen05.mma.cta_group::2, M = 256): each
// CTA loads its 128 rows of A and its 128 columns of B per 64-deep K stage
// (32 KB, 6 stages), the even CTA issues the MMAs for both, and each CTA's
// epilogue drains its own 128 accumulator rows.  A unit is a 256 x 256 tile.
//
// Geometry: rows are cut into row chunks (nc_max rows), the vocabulary into
// bands (ldg columns); chunk c = (row chunk, band).  The bands of a row chunk
// form dH groups of kg consecutive bands: dH = G . W contracts a whole group
// (K = kg * band) before it is written, so the fp32 dH read-modify-write
// traffic (N x D x 4 B per write, the dominant HBM stream of the backward)
// drops kg-fold.  A group's G lives in ring slot (group & 1), band j of the
// group at columns [j * band, (j + 1) * band).
//
// Work units of one launch, dispatched in this order by an atomic counter
// (work stealing per pair); per group with chunks c0 .. c(nb-1):
//     G(c0)  G(c1) dW(c0)  G(c2) dW(c1) ...  G(c(nb-1))  dH(group)  dW(c(nb-1))
//   G(c):  256x256 S tiles of chunk c -> G tile into the group's ring slot
//   dW(c): 256 vocab rows x 256 d, K = row chunk, reading band c's G columns
//   dH(g): 256 rows x 256 d, K = the group's vocabulary
// (dW lags its G by one band so a dW unit rarely waits for G stragglers; with
// kg = 1 the order is G(c) dH(c) dW(c).)  Every chunk is counted at full
// (row_chunk x band) geometry so a unit index decodes in closed form; units
// that fall past N or V are empty (no loads, no MMA) but still signal.
// Dependencies (waited by the scheduler before it publishes a unit, released by
// the epilogue with a gpu-scope fence + atomic; every wait targets a unit
// dispatched earlier, so the schedule cannot deadlock):
//   G(c)       needs every dH / dW unit of group(c) - 2 complete (slot reuse)
//   dH(g, mb)  needs the G rows of mb in every chunk of g, and dH(g - 1) when g
//              is not the first group of its row chunk (fixed fp32 add order)
//   dW(c)      needs G(c) complete, and dW(c - bands) when c is not in the
//              first row chunk (store, then ordered adds)
#include <cmath>
#include <cstdio>

#include "fce_internal.h"
#include "sm100_ptx.cuh"

namespace fce {

using namespace ptx;

static constexpr float kL2e = 1.4426950408889634f;
constexpr int kUnitRing = 8;
constexpr int kPS = 6;                     // pipeline stages
constexpr int kPA = 128 * kBK * 2;         // this CTA's A rows per stage
constexpr int kPB = 128 * kBK * 2;         // this CTA's B columns per stage
constexpr int kPM = 256;                   // unit rows (pair)
constexpr int kEpiStage = 2 * 16384;       // epilogue staging: one 128-row x 128-byte slice per column group
// epilogue warps: 4 (one per TMEM lane quarter, 256 columns each) or 8 (two per
// quarter, 128 columns each); selected at launch (option "bwd_epi_warps")

enum UnitType : int { kUnitGrad = 0, kUnitDH = 1, kUnitDW = 2, kUnitStop = 3 };

struct BUnit {
    int type;     // UnitType
    int c;        // chunk (grad, dW); last chunk of the group (dH)
    int m_blk;    // 256-row block: chunk rows (grad, dH) or band vocab rows (dW)
    int n_tile;   // 256-wide tile: band vocab (grad) or d (dH, dW)
    int r0, nc;   // chunk rows [r0, r0 + nc)
    int vb, vc;   // vocab rows [vb, vb + vc): the band (grad, dW) or the group (dH)
    int slot;     // ring slot of the group
    int gcol;     // ring column of this band's G (grad, dW)
    int row_idx, gl, c0, nb;  // row chunk, group within it, its first chunk, bands
    bool empty;   // past N or V: no loads / MMA / stores, completion only
    bool zero_dw; // dW unit of the first row chunk with no live rows: stores zeros (no MMA)
};

// Closed-form decode of the dispatch order described at the top of the file.
// n_live: rows of the (compacted) problem that are real; the geometry is laid
// out for p.n rows and units past n_live are empty.
__device__ __forceinline__ BUnit decode_unit(const BwdParams& p, int u, int n_live) {
    BUnit r;
    r.zero_dw = false;
    if (u >= p.units) {
        r.type = kUnitStop;
        r.empty = true;
        return r;
    }
    r.row_idx = u / p.per_rc;
    const int lu = u - r.row_idx * p.per_rc;
    r.gl = min(lu / p.per_gf, p.gpr - 1);
    int l = lu - r.gl * p.per_gf;
    r.nb = min(p.kg, p.bands - r.gl * p.kg);
    r.c0 = r.row_idx * p.bands + r.gl * p.kg;
    r.slot = (r.row_idx * p.gpr + r.gl) & 1;
    const int blk = p.n_g + p.n_dw;
    int j, loc;
    if (l < p.n_g) {
        r.type = kUnitGrad;
        j = 0;
        loc = l;
    } else if ((l -= p.n_g) < (r.nb - 1) * blk) {
        j = 1 + l / blk;
        loc = l - (j - 1) * blk;
        if (loc < p.n_g) {
            r.type = kUnitGrad;
        } else {
            r.type = kUnitDW;
            loc -= p.n_g;
            j -= 1;
        }
    } else {
        l -= (r.nb - 1) * blk;
        j = r.nb - 1;
        if (l < p.n_dh) {
            r.type = kUnitDH;
            loc = l;
        } else {
            r.type = kUnitDW;
            loc = l - p.n_dh;
        }
    }
    r.c = r.c0 + j;
    r.r0 = r.row_idx * static_cast<int>(p.nc_max);
    r.nc = min(static_cast<int>(p.nc_max), n_live - r.r0);
    r.gcol = j * static_cast<int>(p.ldg);
    if (r.type == kUnitDH) {
        r.vb = r.gl * p.kg * static_cast<int>(p.ldg);
        r.vc = min(r.nb * static_cast<int>(p.ldg), p.v - r.vb);
        r.m_blk = loc / p.d_tiles;
        r.n_tile = loc - r.m_blk * p.d_tiles;
        r.empty = r.m_blk * kPM >= r.nc;
    } else {
        r.vb = (r.gl * p.kg + j) * static_cast<int>(p.ldg);
        r.vc = min(static_cast<int>(p.ldg), p.v - r.vb);
        if (r.type == kUnitGrad) {
            r.m_blk = loc / p.vt;
            r.n_tile = loc - r.m_blk * p.vt;
            r.empty = r.m_blk * kPM >= r.nc || r.n_tile * kBN >= r.vc;
        } else {
            r.n_tile = loc / p.vm;
            r.m_blk = loc - r.n_tile * p.vm;
            r.empty = r.m_blk * kPM >= r.vc;
        }
    }
    if (!((p.unit_mask >> r.type) & 1)) {
        r.empty = true;
    } else if (r.type == kUnitDW && !r.empty && r.nc <= 0) {
        // no live rows in this row chunk: nothing to add; the first chunk's
        // units still owe dW its (zero) value
        r.empty = true;
        r.zero_dw = r.row_idx == 0;
    }
    return r;
}

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* ptr) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ptr) : "memory");
    return v;
}

__device__ __forceinline__ void wait_at_least(const unsigned* ptr, unsigned target) {
    if (ld_acquire(ptr) >= target) return;
    while (ld_acquire(ptr) < target) __nanosleep(128);
}

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// counters: [0] scheduler; chunk c: [1+4c] G done, [2+4c] dH of the group ending
// at c done, [3+4c] dW done, [4+4c] dH + dW of the group starting at c done;
// then per (chunk, 256-row block) G done.  Both CTAs of a pair signal every
// unit, so every target is twice the unit count.
__device__ __forceinline__ unsigned* cnt(const BwdParams& p, int c, int k) {
    return p.counters + 1 + 4 * c + k;
}

__device__ __forceinline__ int unit_kblocks(const BwdParams& p, const BUnit& un) {
    if (un.type == kUnitGrad) return p.k_blocks_d;
    if (un.type == kUnitDH) return (un.vc + kBK - 1) / kBK;
    return (un.nc + kBK - 1) / kBK;
}

template <int kEpiWarps>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 32 * kEpiWarps, 1)
    fce_bwd_persistent_kernel(const __grid_constant__ BwdParams p, const __grid_constant__ BwdMaps maps) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kPS * kPA;
    uint8_t* sEpi = sB + kPS * kPB;  // 2 x 16 KB epilogue staging (TMA store / reduce-add)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sEpi + kEpiStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + kPS;
    uint64_t* tfull = bars + 2 * kPS;
    uint64_t* tempty = tfull + 2;
    uint64_t* ufull = tempty + 2;
    uint64_t* uempty = ufull + kUnitRing;
    int* unit_ring = reinterpret_cast<int*>(uempty + kUnitRing);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(unit_ring + kUnitRing);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const unsigned two = 2u;  // signals per unit (one per CTA of the pair)
    // Warp roles.  The SM sub-partition arbiter favours the highest warp id, so
    // the latency-critical MMA issuer and TMA producer take the top ids and the
    // (instruction-heavy) epilogue warps the bottom ones.
    constexpr int kWarpAlloc = kEpiWarps, kWarpSched = kEpiWarps + 1, kWarpTma = kEpiWarps + 2,
                  kWarpMma = kEpiWarps + 3;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kPS; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * kEpiWarps);  // epilogue warps of both CTAs (leader's copy)
        }
        for (int s = 0; s < kUnitRing; ++s) {
            mbar_init(&ufull[s], 1);
            // leader's copy: TMA producer + 4 epilogue warps of each CTA, + MMA thread
            mbar_init(&uempty[s], 3 + 2 * kEpiWarps);
        }
        fence_mbar_init();
    }
    if (warp == kWarpTma && lane == 0) {
        tma_prefetch_desc(&maps.h_k);
        tma_prefetch_desc(&maps.w_k);
        tma_prefetch_desc(&maps.g_k);
        tma_prefetch_desc(&maps.w_mn);
        tma_prefetch_desc(&maps.g_mn);
        tma_prefetch_desc(&maps.h_mn);
    }
    if (warp == kWarpAlloc) tmem_alloc_pair<512>(tmem_slot);
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t leader_uempty0 = mapa_shared(&uempty[0], 0);
    // compacted problems: the live row count is produced on the device
    const int n_live = p.n_valid ? static_cast<int>(min(static_cast<unsigned long long>(p.n), *p.n_valid)) : p.n;

    if (warp == kWarpSched) {
        // ------------------------------------------------ scheduler (even CTA)
        // Claims units (work stealing per pair), waits until their inputs are
        // complete, and only then publishes them to both CTAs' unit rings, so
        // dependency latency never sits on the TMA / MMA critical path.
        if (lane == 0 && rank == 0) {
            int us = 0;
            uint32_t uphase = 0;
            const uint32_t peer_ring0 = mapa_shared(&unit_ring[0], 1);
            const uint32_t peer_ufull0 = mapa_shared(&ufull[0], 1);
            const bool static_sched = (p.unit_mask >> 4) & 1;  // debug: round-robin schedule
            int u_static = blockIdx.x >> 1;
            for (;;) {
                int u;
                if (static_sched) {
                    u = u_static;
                    u_static += gridDim.x >> 1;
                } else {
                    u = static_cast<int>(atomicAdd(p.counters, 1u));
                }
                const BUnit un = decode_unit(p, u, n_live);
                if (un.type != kUnitStop && !un.empty) {
                    if (un.type == kUnitGrad) {
                        const int g = un.row_idx * p.gpr + un.gl;
                        if (g >= 2) {
                            // the slot's previous group: g - 2 (possibly in the previous row chunk)
                            const int g2 = g - 2, r2 = g2 / p.gpr, gl2 = g2 - r2 * p.gpr;
                            const int nb2 = min(p.kg, p.bands - gl2 * p.kg);
                            wait_at_least(cnt(p, r2 * p.bands + gl2 * p.kg, 3), two * (p.n_dh + nb2 * p.n_dw));
                        }
                    } else if (un.type == kUnitDH) {
                        for (int cc = un.c0; cc <= un.c; ++cc)
                            wait_at_least(p.counters + p.gm_base + cc * p.mb_max + un.m_blk, two * p.vt);
                        if (un.gl > 0) wait_at_least(cnt(p, un.c0 - 1, 1), two * p.n_dh);
                    } else {
                        wait_at_least(cnt(p, un.c, 0), two * p.n_g);
                        if (un.row_idx > 0) wait_at_least(cnt(p, un.c - p.bands, 2), two * p.n_dw);
                    }
                }
                mbar_wait_cluster(&uempty[us], uphase ^ 1);
                unit_ring[us] = u;
                st_shared_cluster_u32(peer_ring0 + 4 * us, static_cast<uint32_t>(u));
                mbar_arrive(&ufull[us]);
                mbar_arrive_cluster(peer_ufull0 + 8 * us);
                if (++us == kUnitRing) {
                    us = 0;
                    uphase ^= 1;
                }
                if (un.type == kUnitStop) break;
            }
        }
    } else if (warp == kWarpTma) {
        // ------------------------------------------------ TMA producer (both CTAs)
        // Whole warp, converged; one elected lane issues each TMA.
        {
            int stage = 0, us = 0;
            uint32_t phase = 0, uphase = 0;
            const uint64_t pol_norm = policy_evict_normal();
            const uint64_t pol_g = (p.l2_hints & 2) ? policy_evict_last() : pol_norm;
            const uint64_t pol_h = (p.l2_hints & 8) ? policy_evict_first() : pol_norm;
            const uint32_t leader_full0 = mapa_shared(&full[0], 0);
            const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
            for (;;) {
                mbar_wait_cluster(&ufull[us], uphase);
                const int u = unit_ring[us];
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(leader_uempty0 + 8 * us);
                __syncwarp();
                if (++us == kUnitRing) {
                    us = 0;
                    uphase ^= 1;
                }
                const BUnit un = decode_unit(p, u, n_live);
                if (un.type == kUnitStop) break;
                if (un.empty) continue;
                const CUtensorMap *ma, *mb;
                int a_mn, b_mn, a_row, b_row, a_k0, b_k0;
                uint64_t pa = pol_norm, pb = pol_norm;
                if (un.type == kUnitGrad) {
                    ma = &maps.h_k;
                    mb = &maps.w_k;
                    a_mn = b_mn = 0;
                    a_row = un.r0 + un.m_blk * kPM + rank * 128;
                    b_row = un.vb + un.n_tile * kBN + rank * 128;
                    a_k0 = b_k0 = 0;
                } else if (un.type == kUnitDH) {
                    ma = &maps.g_k;
                    mb = &maps.w_mn;
                    a_mn = 0;
                    b_mn = 1;
                    a_row = un.slot * static_cast<int>(p.nc_max) + un.m_blk * kPM + rank * 128;
                    b_row = un.n_tile * kBN + rank * 128;
                    a_k0 = 0;
                    b_k0 = un.vb;
                    pa = pol_g;
                } else {
                    ma = &maps.g_mn;
                    mb = &maps.h_mn;
                    a_mn = b_mn = 1;
                    a_row = un.gcol + un.m_blk * kPM + rank * 128;
                    b_row = un.n_tile * kBN + rank * 128;
                    a_k0 = un.slot * static_cast<int>(p.nc_max);
                    b_k0 = un.r0;
                    pa = pol_g;
                    pb = pol_h;
                }
                // the scheduler acquired this unit's inputs (gpu scope) before
                // publishing it; order that before this thread's async-proxy reads
                fence_proxy_async_global();
                const int kbs = unit_kblocks(p, un);
                for (int kb = 0; kb < kbs; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (rank == 0) mbar_arrive_expect_tx_w(&full[stage], 2 * (kPA + kPB));
                    const uint32_t fb = leader_full0 + stage * 8;
                    const uint32_t a_dst = sa0 + stage * kPA;
                    const uint32_t b_dst = sb0 + stage * kPB;
                    if (!a_mn) {
                        tma_load_2d_pair_w(a_dst, ma, fb, a_k0 + kb * kBK, a_row, pa);
                    } else {
                        tma_load_2d_pair_w(a_dst, ma, fb, a_row, a_k0 + kb * kBK, pa);
                        tma_load_2d_pair_w(a_dst + 8192, ma, fb, a_row + 64, a_k0 + kb * kBK, pa);
                    }
                    if (!b_mn) {
                        tma_load_2d_pair_w(b_dst, mb, fb, b_k0 + kb * kBK, b_row, pb);
                    } else {
                        tma_load_2d_pair_w(b_dst, mb, fb, b_row, b_k0 + kb * kBK, pb);
                        tma_load_2d_pair_w(b_dst + 8192, mb, fb, b_row + 64, b_k0 + kb * kBK, pb);
                    }
                    if (++stage == kPS) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == kWarpMma) {
        // ------------------------------------------------ MMA issuer (even CTA)
        // The whole warp runs the loop (converged, warp-uniform operands) and
        // one elected lane issues, so each MMA is a single UTCHMMA.2CTA; the
        // descriptors of every (stage, k) are a fixed offset from the unit's base.
        if (rank == 0) {
            int stage = 0, us = 0, acc = 0;
            uint32_t phase = 0, uphase = 0, acc_phase = 0;
            const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
            for (;;) {
                mbar_wait(&ufull[us], uphase);
                const int u = unit_ring[us];
                __syncwarp();
                if (lane == 0) mbar_arrive(&uempty[us]);
                __syncwarp();
                if (++us == kUnitRing) {
                    us = 0;
                    uphase ^= 1;
                }
                const BUnit un = decode_unit(p, u, n_live);
                if (un.type == kUnitStop) break;
                if (un.empty) continue;
                const uint32_t a_mn = un.type == kUnitDW ? 1u : 0u;
                const uint32_t b_mn = un.type == kUnitGrad ? 0u : 1u;
                const uint32_t idesc = make_idesc_bf16(kPM, kBN, a_mn, b_mn);
                // descriptor of stage 0, k 0 and the per-k step (in 16-byte units)
                const uint64_t ad0 = a_mn ? make_sdesc_sw128(sa0, 8192, 1024) : make_sdesc_sw128(sa0, 16, 1024);
                const uint64_t bd0 = b_mn ? make_sdesc_sw128(sb0, 8192, 1024) : make_sdesc_sw128(sb0, 16, 1024);
                const uint32_t astep = a_mn ? (2048u >> 4) : (32u >> 4);
                const uint32_t bstep = b_mn ? (2048u >> 4) : (32u >> 4);
                const int kbs = unit_kblocks(p, un);
                long long cyc0 = 0;
                if (p.trace && lane == 0) {
                    p.trace[8 * u + 0] = global_ns();
                    cyc0 = clock64();
                }
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                if (p.trace && lane == 0) p.trace[8 * u + 4] = global_ns();
                tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * kBN;
                long long wait_cyc = 0;
                for (int kb = 0; kb < kbs; ++kb) {
                    if (p.trace) {
                        const long long c0 = clock64();
                        mbar_wait(&full[stage], phase);
                        const long long c1 = clock64();
                        if (kb == 0) {
                            if (lane == 0) p.trace[8 * u + 5] = global_ns();
                        } else {
                            wait_cyc += c1 - c0;
                        }
                    } else {
                        mbar_wait(&full[stage], phase);
                    }
                    tc_fence_after();
                    const uint64_t ads = ad0 + static_cast<uint64_t>((stage * kPA) >> 4);
                    const uint64_t bds = bd0 + static_cast<uint64_t>((stage * kPB) >> 4);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                        umma_bf16_pair_w(d_tmem, ads + k * astep, bds + k * bstep, idesc, (kb | k) != 0 ? 1u : 0u);
                    umma_commit_pair_w(&empty[stage], 0x3);
                    if (++stage == kPS) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit_pair_w(&tfull[acc], 0x3);
                if (p.trace && lane == 0) {
                    p.trace[8 * u + 1] = global_ns();
                    p.trace[8 * u + 7] = clock64() - cyc0;
                }
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }
        }
    } else if (warp < kEpiWarps) {
        // ------------------------------------------------ epilogue (both CTAs)
        const int q = warp & 3;                 // TMEM lane quarter (hardware: warp id % 4)
        const int r = q * 32 + lane;            // accumulator row of this thread
        const int chalf = warp >> 2;            // which column slice (8 warps: halves)
        int us = 0, acc = 0;
        uint32_t uphase = 0, acc_phase = 0;
        const uint64_t pol_out = (p.l2_hints & 1) ? policy_evict_first() : policy_evict_normal();
        const uint64_t pol_gst = (p.l2_hints & 4) ? policy_evict_last() : policy_evict_normal();
        const uint32_t leader_tempty0 = mapa_shared(&tempty[0], 0);
        for (;;) {
            mbar_wait_cluster(&ufull[us], uphase);
            const int u = unit_ring[us];
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(leader_uempty0 + 8 * us);
            if (++us == kUnitRing) {
                us = 0;
                uphase ^= 1;
            }
            const BUnit un = decode_unit(p, u, n_live);
            if (un.type == kUnitStop) break;

            if (!un.empty) {
                mbar_wait(&tfull[acc], acc_phase);
                // trace slot 6: when the unit's last MMA completed (accumulator full)
                if (p.trace && rank == 0 && threadIdx.x == 0) p.trace[8 * u + 6] = global_ns();
                tc_fence_after();
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                       static_cast<uint32_t>(acc * kBN);
                const int lrow = un.m_blk * kPM + static_cast<int>(rank) * 128 + r;
                // tma_epi bit 0: G through SMEM + TMA store; bit 1: dH / dW through
                // SMEM + TMA store / reduce-add (otherwise per-thread vector stores)
                if (un.type == kUnitGrad ? (p.tma_epi & 1) : (p.tma_epi & 2)) {
                    // Each column group (4 warps, one TMEM lane quarter each) stages a
                    // 128-row x 128-byte slice in swizzled SMEM and one thread hands it
                    // to the TMA engine: full-line stores / reduce-adds instead of 32
                    // scattered 16-byte requests per warp instruction.
                    const int grp = warp >> 2;
                    const bool gl = (threadIdx.x & 127) == 0;  // group leader
                    const uint32_t sbuf = smem_u32(sEpi + grp * 16384);
                    const int ncols = kBN / (kEpiWarps / 4);
                    const int gcol0 = grp * ncols;
                    const uint32_t my_row = sbuf + static_cast<uint32_t>(r) * 128u;
                    const uint32_t sw = static_cast<uint32_t>(r & 7);
                    if (un.type == kUnitGrad) {
                        const bool row_ok = lrow < un.nc;
                        const int64_t grow = static_cast<int64_t>(un.r0) + lrow;
                        float gam = 0.f, lse_r = 0.f;
                        int64_t tcol = -1;
                        if (row_ok) {
                            const int64_t y = p.targets[grow];
                            const bool skip = p.has_ignore && y == p.ignore_index;
                            gam = skip ? 0.f : p.gamma[grow];
                            lse_r = skip ? 0.f : p.lse[grow];
                            tcol = y - (p.v_offset + un.vb);
                        }
#pragma unroll 1
                        for (int sl = 0; sl < ncols / 64; ++sl) {
                            const int c64 = gcol0 + sl * 64;
                            if (gl) bulk_wait_read0();
                            named_bar_sync(2 + grp, 128);
                            uint32_t packed[32];
#pragma unroll
                            for (int h2 = 0; h2 < 2; ++h2) {
                                float v[32];
                                tmem_ld32(taddr + c64 + h2 * 32, v);
                                const int col0 = un.n_tile * kBN + c64 + h2 * 32;
                                const int64_t tc = tcol - col0;
#pragma unroll
                                for (int j = 0; j < 32; j += 2) {
                                    float g0 = gam * (ex2((v[j] - lse_r) * kL2e) - (tc == j ? 1.f : 0.f));
                                    float g1 = gam * (ex2((v[j + 1] - lse_r) * kL2e) - (tc == j + 1 ? 1.f : 0.f));
                                    if (gam == 0.f || col0 + j >= un.vc) g0 = 0.f;
                                    if (gam == 0.f || col0 + j + 1 >= un.vc) g1 = 0.f;
                                    packed[h2 * 16 + (j >> 1)] = pack_bf16(g0, g1);
                                }
                            }
#pragma unroll
                            for (int ch = 0; ch < 8; ++ch)
                                st_shared_v4(my_row + ((static_cast<uint32_t>(ch) ^ sw) << 4), packed[4 * ch],
                                             packed[4 * ch + 1], packed[4 * ch + 2], packed[4 * ch + 3]);
                            fence_proxy_async_shared();
                            named_bar_sync(2 + grp, 128);
                            if (gl) {
                                tma_store_2d_hint(&maps.g_st, sbuf, un.gcol + un.n_tile * kBN + c64,
                                                  un.slot * static_cast<int>(p.nc_max) + un.m_blk * kPM +
                                                      static_cast<int>(rank) * 128,
                                                  pol_gst);
                                bulk_commit();
                            }
                        }
                    } else if (un.type == kUnitDW && p.dw_bf16) {
                        // bf16 dW (one row chunk: written exactly once): 64-column
                        // slices of RNE-rounded pairs, 128-byte rows through TMA
                        const int orow = un.vb + un.m_blk * kPM + static_cast<int>(rank) * 128;
                        const bool discard = ((p.unit_mask >> 5) & 1) || ((p.unit_mask >> 7) & 1);
#pragma unroll 1
                        for (int sl = 0; sl < ncols / 64; ++sl) {
                            const int c64 = gcol0 + sl * 64;
                            if (gl) bulk_wait_read0();
                            named_bar_sync(2 + grp, 128);
                            uint32_t packed[32];
#pragma unroll
                            for (int h2 = 0; h2 < 2; ++h2) {
                                float v[32];
                                tmem_ld32(taddr + c64 + h2 * 32, v);
#pragma unroll
                                for (int j = 0; j < 32; j += 2) packed[h2 * 16 + (j >> 1)] = pack_bf16(v[j], v[j + 1]);
                            }
#pragma unroll
                            for (int ch = 0; ch < 8; ++ch)
                                st_shared_v4(my_row + ((static_cast<uint32_t>(ch) ^ sw) << 4), packed[4 * ch],
                                             packed[4 * ch + 1], packed[4 * ch + 2], packed[4 * ch + 3]);
                            fence_proxy_async_shared();
                            named_bar_sync(2 + grp, 128);
                            if (gl && !discard) {
                                tma_store_2d_hint(&maps.dw_st, sbuf, un.n_tile * kBN + c64, orow, pol_out);
                                bulk_commit();
                            }
                        }
                    } else {
                        const bool is_dh = un.type == kUnitDH;
                        const bool accumulate = is_dh ? (un.gl > 0 || p.accumulate_dh) : (un.row_idx > 0);
                        const CUtensorMap* om = is_dh ? &maps.dh_st : &maps.dw_st;
                        const int orow = (is_dh ? un.r0 : un.vb) + un.m_blk * kPM + static_cast<int>(rank) * 128;
                        if (is_dh && p.dh_peers > 0) {
                            // reduce into the accumulator of the rank owning this 128-row block
                            const int blk = orow >> 7;
                            int q = 0;
                            while (q + 1 < p.dh_peers && blk >= p.peer_block0[q + 1]) ++q;
                            om = &maps.dh_peer[q];
                        }
                        // debug: bit 5 discards dH and dW writes, bit 6 only dH, bit 7 only dW
                        const bool discard = ((p.unit_mask >> 5) & 1) || ((p.unit_mask >> (is_dh ? 6 : 7)) & 1);
#pragma unroll 1
                        for (int sl = 0; sl < ncols / 32; ++sl) {
                            const int c32 = gcol0 + sl * 32;
                            if (gl) bulk_wait_read0();
                            named_bar_sync(2 + grp, 128);
                            float v[32];
                            tmem_ld32(taddr + c32, v);
                            const uint32_t* vu = reinterpret_cast<const uint32_t*>(v);
#pragma unroll
                            for (int ch = 0; ch < 8; ++ch)
                                st_shared_v4(my_row + ((static_cast<uint32_t>(ch) ^ sw) << 4), vu[4 * ch],
                                             vu[4 * ch + 1], vu[4 * ch + 2], vu[4 * ch + 3]);
                            fence_proxy_async_shared();
                            named_bar_sync(2 + grp, 128);
                            if (gl && !discard) {
                                if (accumulate)
                                    tma_reduce_add_2d_hint(om, sbuf, un.n_tile * kBN + c32, orow, pol_out);
                                else
                                    tma_store_2d_hint(om, sbuf, un.n_tile * kBN + c32, orow, pol_out);
                                bulk_commit();
                            }
                        }
                    }
                    // the unit's writes must be complete before its completion is published
                    if (gl) bulk_wait_all0();
                } else if (un.type == kUnitGrad) {
                    const bool row_ok = lrow < un.nc;
                    const int64_t grow = static_cast<int64_t>(un.r0) + lrow;
                    float gam = 0.f, lse_r = 0.f;
                    int64_t tcol = -1;
                    if (row_ok) {
                        const int64_t y = p.targets[grow];
                        const bool skip = p.has_ignore && y == p.ignore_index;
                        gam = skip ? 0.f : p.gamma[grow];
                        lse_r = skip ? 0.f : p.lse[grow];
                        tcol = y - (p.v_offset + un.vb);
                    }
                    __nv_bfloat16* grow_ptr =
                        p.g_ring + (static_cast<int64_t>(un.slot) * p.nc_max + lrow) * p.ldr + un.gcol;
#pragma unroll 1
                    for (int cc = 0; cc < kBN / 32 / (kEpiWarps / 4); ++cc) {
                        const int c = chalf * (kBN / 32 / (kEpiWarps / 4)) + cc;
                        float v[32];
                        tmem_ld32(taddr + c * 32, v);
                        const int col0 = un.n_tile * kBN + c * 32;
                        // rows past the live count inside the unit store zeros (gam = 0):
                        // dW units read them against zero H rows, so they must be finite
                        if (!((p.unit_mask >> 3) & 1)) {  // debug bit 3: skip G stores
                            const int64_t tc = tcol - col0;
                            uint32_t packed[16];
#pragma unroll
                            for (int j = 0; j < 32; j += 2) {
                                float g0 = gam * (ex2((v[j] - lse_r) * kL2e) - (tc == j ? 1.f : 0.f));
                                float g1 = gam * (ex2((v[j + 1] - lse_r) * kL2e) - (tc == j + 1 ? 1.f : 0.f));
                                if (gam == 0.f || col0 + j >= un.vc) g0 = 0.f;
                                if (gam == 0.f || col0 + j + 1 >= un.vc) g1 = 0.f;
                                packed[j >> 1] = pack_bf16(g0, g1);
                            }
                            __nv_bfloat16* dst = grow_ptr + col0;
                            st_v8_b32_hint(dst, packed, pol_gst);
                            st_v8_b32_hint(dst + 16, packed + 8, pol_gst);
                        }
                    }
                } else {
                    // dH rows = chunk rows into dH; dW rows = band vocab rows into dW
                    const bool is_dh = un.type == kUnitDH;
                    const int mrows = is_dh ? un.nc : un.vc;
                    const bool accumulate = is_dh ? (un.gl > 0 || p.accumulate_dh) : (un.row_idx > 0);
                    float* crow = is_dh ? p.dh + (static_cast<int64_t>(un.r0) + lrow) * p.lddh
                                        : p.dw + (static_cast<int64_t>(un.vb) + lrow) * p.lddw;
#pragma unroll 1
                    for (int cc = 0; cc < kBN / 32 / (kEpiWarps / 4); ++cc) {
                        const int c = chalf * (kBN / 32 / (kEpiWarps / 4)) + cc;
                        float v[32];
                        tmem_ld32(taddr + c * 32, v);
                        const int col0 = un.n_tile * kBN + c * 32;
                        if (lrow < mrows && !((p.unit_mask >> 5) & 1)) {  // debug bit 5: discard dH/dW
                            float* dst = crow + col0;
                            const bool vec = (col0 + 32 <= p.d) && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                            if (vec) {
                                if (accumulate) {
#pragma unroll
                                    for (int j = 0; j < 32; j += 4)
                                        red_add_v4_hint(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3], pol_out);
                                } else if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
#pragma unroll
                                    for (int j = 0; j < 32; j += 8) st_v8_f32_hint(dst + j, v + j, pol_out);
                                } else {
#pragma unroll
                                    for (int j = 0; j < 32; j += 4)
                                        st_v4_hint(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3], pol_out);
                                }
                            } else {
                                for (int j = 0; j < 32; ++j) {
                                    if (col0 + j < p.d) {
                                        if (accumulate)
                                            atomicAdd(dst + j, v[j]);
                                        else
                                            dst[j] = v[j];
                                    }
                                }
                            }
                        }
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(leader_tempty0 + 8 * acc);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
                // generic-proxy stores above are read later through TMA (async proxy)
                fence_proxy_async_global();
            }

            if (un.zero_dw) {
                // dW rows of a launch whose row chunks hold no live row: exact zeros
                const int lrow = un.m_blk * kPM + static_cast<int>(rank) * 128 + r;
                if (lrow < un.vc) {
                    const int c_per = kBN / (kEpiWarps / 4);
                    const int c0 = un.n_tile * kBN + chalf * c_per;
                    const int64_t vrow = static_cast<int64_t>(un.vb) + lrow;
                    for (int c = c0; c < c0 + c_per && c < p.d; ++c) {
                        if (p.dw_bf16)
                            reinterpret_cast<__nv_bfloat16*>(p.dw)[vrow * p.lddw + c] = __float2bfloat16(0.f);
                        else
                            p.dw[vrow * p.lddw + c] = 0.f;
                    }
                }
            }

            // publish completion of this CTA's half: all 128 epilogue threads'
            // stores, then one gpu-scope release
            named_bar_sync(1, 32 * kEpiWarps);
            if (threadIdx.x == 0) {
                __threadfence();
                if (p.trace && rank == 0) {
                    unsigned smid;
                    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                    p.trace[8 * u + 2] = global_ns();
                    p.trace[8 * u + 3] = smid;
                }
                if (un.type == kUnitGrad) {
                    atomicAdd(p.counters + p.gm_base + un.c * p.mb_max + un.m_blk, 1u);
                    atomicAdd(cnt(p, un.c, 0), 1u);
                } else if (un.type == kUnitDH) {
                    atomicAdd(cnt(p, un.c, 1), 1u);
                    atomicAdd(cnt(p, un.c0, 3), 1u);
                } else {
                    atomicAdd(cnt(p, un.c, 2), 1u);
                    atomicAdd(cnt(p, un.c0, 3), 1u);
                }
            }
        }
    }

    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    if (warp == kWarpAlloc) tmem_dealloc_pair<512>(tmem_base);
}

constexpr int kBwdSmem = kPS * (kPA + kPB) + kEpiStage + 1024 + 512;

cudaError_t launch_bwd_persistent(const BwdParams& p, const BwdMaps& maps, int grid,
                                  cudaStream_t stream) {
    const int wide = p.epi_warps == 4 ? 0 : 1;
    auto kern = wide ? fce_bwd_persistent_kernel<8> : fce_bwd_persistent_kernel<4>;
    {
        cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(kern), kBwdSmem);
        if (e != cudaSuccess) return e;
    }
    int pairs = grid / 2;
    if (pairs > p.units) pairs = p.units;
    if (pairs < 1) return cudaSuccess;
    kern<<<2 * pairs, 128 + 32 * (wide ? 8 : 4), kBwdSmem, stream>>>(p, maps);
    return cudaGetLastError();
}

}  // namespace fce
