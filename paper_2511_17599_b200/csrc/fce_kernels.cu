// sm_100a kernels of the fused linear-cross-entropy operator.
//
// One warp-specialised, persistent tcgen05 kernel template serves every
// contraction on the path; only its epilogue differs:
//
//   kEpiForward  S = H_m . W_v^T tile in TMEM -> online max / sum-exp over the
//                vocab tiles of a split + target-logit gather, written as one
//                (m, a, z_target, found) partial per row and split.  This is
//                Alg. 1 / accumulate_stats_block
//                (reference proj/include/fusedce/fused_forward.hpp:47-73) with
//                the dot products of detail::dot (detail/kernels.hpp:47-61)
//                replaced by UMMA tiles.  No N x V buffer exists.
//   kEpiGrad     recomputed S tile -> G = gamma * (exp(S - lse) - onehot) in
//                registers -> bf16 G band (Alg. 2, fused_backward.hpp:34-55).
//   kEpiGemm     plain C (+)= A . B^T with fp32 store or red.global.add; used
//                for dW_band = G_band^T . H and dH += G_band . W_band.
//
// Roles (256 threads, 1 CTA / SM): warp 0 (converged, one elect.sync lane
// per instruction) issues TMA into a 4-stage smem ring, warp 1 likewise issues
// tcgen05.mma (M=128, N=256, K=16) into one of two TMEM accumulators
// (2 x 256 fp32 columns), warp 2 owns the TMEM allocation, warps 4-7 drain
// TMEM with tcgen05.ld (thread = row).  Template flag MC: the forward on
// 2-CTA clusters with the W tile multicast to both CTAs (option fwd_mc).
// Compacted problems (ignored rows packed away) pass the device-resident live
// row count in TileParams::n_valid; the forward skips row blocks past it.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>
#include <cudaTypedefs.h>

#include "fce_internal.h"
#include "sm100_ptx.cuh"

namespace fce {

using namespace ptx;

static constexpr float kLog2e = 1.4426950408889634f;

struct Unit {
    int prob, m_blk, n_tile0, n_tiles, split;
};

__device__ __forceinline__ Unit get_unit(const TileParams& p, int u) {
    Unit r;
    r.prob = 0;
    r.split = 0;
    r.n_tiles = 1;
    if (p.mode == kEpiForward) {
        // L2 raster: groups of m_group row blocks; inside a group the split
        // index is slow and the row block fast, so the CTAs running at the
        // same time share one vocab range (W tiles hit in L2) and the group's
        // H rows stay L2 resident.
        const int per_group = p.m_group * p.splits;
        const int g = u / per_group;
        const int gsize = min(p.m_group, p.m_blocks - g * p.m_group);
        const int local = u - g * per_group;
        const int s = local / gsize;
        const int mi = local - s * gsize;
        r.m_blk = g * p.m_group + mi;
        r.split = s;
        const int t0 = static_cast<int>(static_cast<long long>(s) * p.v_tiles / p.splits);
        const int t1 = static_cast<int>(static_cast<long long>(s + 1) * p.v_tiles / p.splits);
        r.n_tile0 = t0;
        r.n_tiles = t1 - t0;
    } else if (p.mode == kEpiGrad) {
        r.m_blk = u / p.v_tiles;
        r.n_tile0 = u - r.m_blk * p.v_tiles;
    } else {
        const int pi = u < p.units0 ? 0 : 1;
        const int local = pi ? u - p.units0 : u;
        const GemmProblem& q = p.prob[pi];
        if (q.n_fastest) {
            r.m_blk = local / q.n_tiles;
            r.n_tile0 = local - r.m_blk * q.n_tiles;
        } else {
            r.n_tile0 = local / q.m_tiles;
            r.m_blk = local - r.n_tile0 * q.m_tiles;
        }
        r.prob = pi;
    }
    return r;
}

// MC (forward only): clusters of two CTAs on adjacent row blocks of the same
// vocab tiles; each CTA loads its own H rows and one 128-row half of the W tile
// and multicasts that half into both CTAs' stages, so every W byte leaves L2
// once per pair.  Stage slots are released by both CTAs' MMA commits.
template <int EPI, bool MC>
__global__ void __launch_bounds__(kThreads, 1)
    fce_tile_kernel(const __grid_constant__ TileParams p, const __grid_constant__ TensorMaps maps) {
    extern __shared__ uint8_t smem_raw[];
    const uint32_t raw_addr = smem_u32(smem_raw);
    uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
    uint8_t* sA = smem;
    uint8_t* sB = smem + kStages * kStageBytesA;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sB + kStages * kStageBytesB);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int rank = MC ? static_cast<int>(cluster_ctarank()) : 0;
    const int u_first = MC ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int u_step = MC ? static_cast<int>(gridDim.x >> 1) : static_cast<int>(gridDim.x);
    // compacted forward: rows past the device count are padding; every role
    // skips the units whose (first) row block lies past it
    const int n_eff = (EPI == kEpiForward && p.n_valid)
                          ? static_cast<int>(min(static_cast<unsigned long long>(p.n_rows), *p.n_valid))
                          : p.n_rows;
    auto dead = [&](const Unit& un) {
        return EPI == kEpiForward && (MC ? 2 * un.m_blk : un.m_blk) * kBM >= n_eff;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], MC ? 2 : 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&maps.a0);
        tma_prefetch_desc(&maps.b0);
        if (EPI == kEpiGemm) {
            tma_prefetch_desc(&maps.a1);
            tma_prefetch_desc(&maps.b1);
        }
    }
    if (warp == 2) {
        tmem_alloc<512>(tmem_slot);
    }
    tc_fence_before();
    if (MC)
        cluster_sync_all();  // the peer multicasts into this CTA's stages / barriers
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        // Whole warp, converged, warp-uniform operands; one elected lane issues
        // (a single UTMALDG per load instead of an ELECT / BRA.U.ANY loop).
        {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
            for (int u = u_first; u < p.units; u += u_step) {
                Unit un = get_unit(p, u);
                if (dead(un)) continue;
                if (MC) un.m_blk = 2 * un.m_blk + rank;
                const CUtensorMap* ma = un.prob ? &maps.a1 : &maps.a0;
                const CUtensorMap* mb = un.prob ? &maps.b1 : &maps.b0;
                int kbs = p.k_blocks, a_mn = 0, b_mn = 0;
                if (EPI == kEpiGemm) {
                    kbs = p.prob[un.prob].k_blocks;
                    a_mn = p.prob[un.prob].a_mn;
                    b_mn = p.prob[un.prob].b_mn;
                }
                for (int t = 0; t < un.n_tiles; ++t) {
                    const int n_tile = un.n_tile0 + t;
                    for (int kb = 0; kb < kbs; ++kb) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        mbar_arrive_expect_tx_w(&full[stage], kStageBytesA + kStageBytesB);
                        const uint32_t a_dst = sa0 + stage * kStageBytesA;
                        const uint32_t b_dst = sb0 + stage * kStageBytesB;
                        if (!a_mn) {
                            tma_load_2d_w(a_dst, ma, &full[stage], kb * kBK, un.m_blk * kBM, kEvictNormal);
                        } else {
#pragma unroll
                            for (int j = 0; j < kBM / 64; ++j)
                                tma_load_2d_w(a_dst + j * 8192, ma, &full[stage], un.m_blk * kBM + 64 * j, kb * kBK,
                                              kEvictNormal);
                        }
                        if (MC) {
                            tma_load_2d_mc_w(b_dst + rank * (kStageBytesB / 2), mb, &full[stage], kb * kBK,
                                             n_tile * kBN + rank * (kBN / 2), 0x3, kEvictNormal);
                        } else if (!b_mn) {
                            tma_load_2d_w(b_dst, mb, &full[stage], kb * kBK, n_tile * kBN, kEvictNormal);
                        } else {
#pragma unroll
                            for (int j = 0; j < kBN / 64; ++j)
                                tma_load_2d_w(b_dst + j * 8192, mb, &full[stage], n_tile * kBN + 64 * j, kb * kBK,
                                              kEvictNormal);
                        }
                        if (++stage == kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            const uint32_t sa0 = smem_u32(sA), sb0 = smem_u32(sB);
            for (int u = u_first; u < p.units; u += u_step) {
                const Unit un = get_unit(p, u);
                if (dead(un)) continue;
                int kbs = p.k_blocks;
                uint32_t a_mn = 0, b_mn = 0;
                if (EPI == kEpiGemm) {
                    kbs = p.prob[un.prob].k_blocks;
                    a_mn = p.prob[un.prob].a_mn;
                    b_mn = p.prob[un.prob].b_mn;
                }
                const uint32_t idesc = make_idesc_bf16(kBM, kBN, a_mn, b_mn);
                // K-major SW128: +32 B per K=16 step inside the 128-B atom.
                // MN-major SW128: +16 rows * 128 B = 2 KB per K=16 step; LBO = 8 KB
                // between 64-wide M/N column blocks.
                const uint64_t ad0 = a_mn ? make_sdesc_sw128(sa0, 8192, 1024) : make_sdesc_sw128(sa0, 16, 1024);
                const uint64_t bd0 = b_mn ? make_sdesc_sw128(sb0, 8192, 1024) : make_sdesc_sw128(sb0, 16, 1024);
                const uint32_t astep = a_mn ? (2048u >> 4) : (32u >> 4);
                const uint32_t bstep = b_mn ? (2048u >> 4) : (32u >> 4);
                for (int t = 0; t < un.n_tiles; ++t) {
                    mbar_wait(&tempty[acc], acc_phase ^ 1);
                    tc_fence_after();
                    const uint32_t d_tmem = tmem_base + acc * kBN;
                    for (int kb = 0; kb < kbs; ++kb) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                        const uint64_t ads = ad0 + static_cast<uint64_t>((stage * kStageBytesA) >> 4);
                        const uint64_t bds = bd0 + static_cast<uint64_t>((stage * kStageBytesB) >> 4);
#pragma unroll
                        for (int k = 0; k < kBK / 16; ++k)
                            umma_bf16_w(d_tmem, ads + k * astep, bds + k * bstep, idesc, (kb | k) != 0 ? 1u : 0u);
                        if (MC)
                            umma_commit_mc_w(&empty[stage], 0x3);
                        else
                            umma_commit_w(&empty[stage]);
                        if (++stage == kStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    umma_commit_w(&tfull[acc]);
                    acc ^= 1;
                    if (acc == 0) acc_phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------ epilogue
        const int q = warp & 3;
        const int r = q * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = u_first; u < p.units; u += u_step) {
            Unit un = get_unit(p, u);
            if (dead(un)) continue;
            if (MC) un.m_blk = 2 * un.m_blk + rank;
            const int64_t row = static_cast<int64_t>(un.m_blk) * kBM + r;

            // per-row state (forward / grad)
            bool row_ok = false, skip = true;
            int64_t tcol = -1;  // launch-local column of this row's target
            float m_run = -INFINITY, a_run = 0.f, zt = 0.f;
            bool found = false;
            float lse_r = 0.f, gam = 0.f;
            if (EPI != kEpiGemm) {
                row_ok = row < n_eff;
                if (row_ok) {
                    const int64_t y = p.targets[row];
                    skip = p.has_ignore && y == p.ignore_index;
                    tcol = y - p.col_global0;
                    if (EPI == kEpiGrad) {
                        gam = skip ? 0.f : p.gamma[row];
                        lse_r = skip ? 0.f : p.lse[row];
                    }
                }
            }

            for (int t = 0; t < un.n_tiles; ++t) {
                const int n_tile = un.n_tile0 + t;
                mbar_wait(&tfull[acc], acc_phase);
                tc_fence_after();
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) +
                                       static_cast<uint32_t>(acc * kBN);
#pragma unroll 1
                for (int c = 0; c < kBN / 32; ++c) {
                    float v[32];
                    tmem_ld32(taddr + c * 32, v);
                    const int col0 = n_tile * kBN + c * 32;
                    if (EPI == kEpiForward) {
                        if (col0 + 32 > p.v_cols) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (col0 + j >= p.v_cols) v[j] = -INFINITY;
                        }
                        float cmax = v[0];
#pragma unroll
                        for (int j = 1; j < 32; ++j) cmax = fmaxf(cmax, v[j]);
                        if (cmax > m_run) {
                            a_run *= ex2((m_run - cmax) * kLog2e);
                            m_run = cmax;
                        }
                        if (cmax != -INFINITY) {
                            float s0 = 0.f, s1 = 0.f;
#pragma unroll
                            for (int j = 0; j < 32; j += 2) {
                                s0 += ex2((v[j] - m_run) * kLog2e);
                                s1 += ex2((v[j + 1] - m_run) * kLog2e);
                            }
                            a_run += s0 + s1;
                        }
                        // target capture only inside this launch's valid columns: a
                        // shard's padded tail must not claim a neighbour's target
                        const int64_t tc = tcol - col0;
                        if (tc >= 0 && tc < 32 && col0 + tc < p.v_cols) {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (j == tc) zt = v[j];
                            found = true;
                        }
                    } else if (EPI == kEpiGrad) {
                        if (row_ok) {
                            const int64_t tc = tcol - col0;
                            uint32_t packed[16];
#pragma unroll
                            for (int j = 0; j < 32; j += 2) {
                                float g0 = gam * (ex2((v[j] - lse_r) * kLog2e) -
                                                  (tc == j ? 1.f : 0.f));
                                float g1 = gam * (ex2((v[j + 1] - lse_r) * kLog2e) -
                                                  (tc == j + 1 ? 1.f : 0.f));
                                if (gam == 0.f || col0 + j >= p.v_cols) g0 = 0.f;
                                if (gam == 0.f || col0 + j + 1 >= p.v_cols) g1 = 0.f;
                                packed[j >> 1] = pack_bf16(g0, g1);
                            }
                            __nv_bfloat16* dst = p.g_out + row * p.ldg + col0;
#pragma unroll
                            for (int j = 0; j < 4; ++j)
                                st_v4_b32(dst + 8 * j, packed[4 * j], packed[4 * j + 1],
                                          packed[4 * j + 2], packed[4 * j + 3]);
                        }
                    } else {
                        const GemmProblem& gq = p.prob[un.prob];
                        if (row < gq.m && gq.accumulate != 2) {  // 2: discard (benchmark only)
                            float* dst = gq.c + row * gq.ldc + col0;
                            const bool vec = (col0 + 32 <= gq.n) &&
                                             ((reinterpret_cast<uintptr_t>(dst) & 15) == 0);
                            if (vec) {
                                if (gq.accumulate) {
#pragma unroll
                                    for (int j = 0; j < 32; j += 4)
                                        red_add_v4(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
                                } else {
#pragma unroll
                                    for (int j = 0; j < 32; j += 4)
                                        st_v4(dst + j, v[j], v[j + 1], v[j + 2], v[j + 3]);
                                }
                            } else {
#pragma unroll
                                for (int j = 0; j < 32; ++j) {
                                    if (col0 + j < gq.n) {
                                        if (gq.accumulate)
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
                if (lane == 0) mbar_arrive(&tempty[acc]);
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1;
            }

            if (EPI == kEpiForward && row_ok) {
                const size_t off = static_cast<size_t>(un.split) * p.n_rows + row;
                p.part_m[off] = skip ? -INFINITY : m_run;
                p.part_a[off] = skip ? 0.f : a_run;
                p.part_zt[off] = (skip || !found) ? 0.f : zt;
                p.part_found[off] = (skip || !found) ? 0 : 1;
            }
        }
    }

    tc_fence_before();
    if (MC)
        cluster_sync_all();  // no CTA leaves while its peer may still signal it
    else
        __syncthreads();
    tc_fence_after();
    if (warp == 2) {
        tmem_dealloc<512>(tmem_base);
    }
}

// ============================================================== host helpers

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    // function-local static: initialised once, thread-safe
    static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
        return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }();
    return fn;
}

bool encode_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                   uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer, bool fp32) {
    auto fn = get_encode_fn();
    if (!fn) return false;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || (row_stride_bytes & 15)) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_stride_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(map, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

cudaError_t ensure_dyn_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({func, dev})) return cudaSuccess;
    e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({func, dev});
    return e;
}

int device_sm_count(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    return v;
}

template <int EPI>
static cudaError_t launch_one(const TileParams& p, const TensorMaps& maps, int grid,
                              cudaStream_t stream) {
    {
        cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fce_tile_kernel<EPI, false>), kSmemBytes);
        if (e != cudaSuccess) return e;
    }
    fce_tile_kernel<EPI, false><<<grid, kThreads, kSmemBytes, stream>>>(p, maps);
    return cudaGetLastError();
}

// Forward on 2-CTA clusters with W multicast (p.m_blocks counts row-block pairs).
cudaError_t launch_fwd_mc(const TileParams& p, const TensorMaps& maps, int sms, cudaStream_t stream) {
    if (p.units <= 0) return cudaSuccess;
    {
        cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void*>(fce_tile_kernel<kEpiForward, true>), kSmemBytes);
        if (e != cudaSuccess) return e;
    }
    int clusters = std::min(sms / 2, p.units);
    if (clusters < 1) clusters = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters, 1, 1);
    cfg.blockDim = dim3(kThreads, 1, 1);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fce_tile_kernel<kEpiForward, true>, p, maps);
}

cudaError_t launch_tile_kernel(const TileParams& p, const TensorMaps& maps, int grid,
                               cudaStream_t stream) {
    if (p.units <= 0) return cudaSuccess;
    if (grid > p.units) grid = p.units;
    switch (p.mode) {
        case kEpiForward: return launch_one<kEpiForward>(p, maps, grid, stream);
        case kEpiGrad: return launch_one<kEpiGrad>(p, maps, grid, stream);
        default: return launch_one<kEpiGemm>(p, maps, grid, stream);
    }
}

// ============================================================== small kernels

__global__ void k_prep_targets(const int64_t* __restrict__ targets, int64_t n, int has_ignore,
                               int64_t ignore_index, int64_t v_total, int* err,
                               unsigned long long* valid_count) {
    unsigned long long local = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t y = targets[i];
        if (has_ignore && y == ignore_index) continue;
        ++local;
        if (y < 0 || y >= v_total) atomicOr(&err[kErrTargetRange], 1);
    }
    // warp aggregate then one atomic per warp (integer: order-independent)
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(valid_count, local);
}

cudaError_t launch_prep_targets(const int64_t* targets, int64_t n, int has_ignore,
                                int64_t ignore_index, int64_t v_total, int* err_flags,
                                unsigned long long* valid_count, cudaStream_t stream) {
    int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 1184));
    if (blocks < 1) blocks = 1;
    k_prep_targets<<<blocks, 256, 0, stream>>>(targets, n, has_ignore, ignore_index, v_total,
                                               err_flags, valid_count);
    return cudaGetLastError();
}

// Ordered merge of `parts` partial stats per row, exactly the reference's
// merge_stats (softmax_stats.hpp:52-75) applied in ascending part order
// (fused_forward.hpp:112-123 for windows, parallel_sim.hpp:214-220 for
// ranks), then loss = (m - z_t) + log a (softmax_stats.hpp:45).
__global__ void k_merge_stats(int parts, int64_t n, int64_t stride, int64_t fstride, const float* __restrict__ pm,
                              const float* __restrict__ pa, const float* __restrict__ pzt,
                              const uint8_t* __restrict__ pf, const int64_t* __restrict__ targets,
                              int has_ignore, int64_t ignore_index, int emit_loss, float* m_out,
                              float* a_out, float* zt_out, uint8_t* f_out, float* lse_out,
                              float* loss_rows, double* block_sums, int* err,
                              const int* __restrict__ row_map) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    double my_loss = 0.0;
    if (i < n) {
        const bool ign = has_ignore && targets[i] == ignore_index;
        float M = -INFINITY, A = 0.f, Z = 0.f;
        bool F = false;
        // partials of compacted problems are indexed by the row's compact slot
        const int64_t src = row_map ? static_cast<int64_t>(row_map[i]) : i;
        if (!ign) {
            for (int s = 0; s < parts; ++s) {
                const int64_t o = s * stride + src;
                const float sm = pm[o], sa = pa[o];
                const bool sf = pf[s * fstride + src] != 0;
                if (F && sf) atomicOr(&err[kErrDuplicate], 1);
                const float nm = M > sm ? M : sm;
                float acc = 0.f;
                if (A != 0.f) acc += A * expf(M - nm);
                if (sa != 0.f) acc += sa * expf(sm - nm);
                M = nm;
                A = acc;
                if (!F && sf) {
                    Z = pzt[o];
                    F = true;
                }
            }
        }
        if (m_out) m_out[i] = M;
        if (a_out) a_out[i] = A;
        if (zt_out) zt_out[i] = Z;
        if (f_out) f_out[i] = F ? 1 : 0;
        if (emit_loss) {
            float loss = 0.f;
            if (!ign) {
                if (!F) atomicOr(&err[kErrNotFound], 1);
                loss = (M - Z) + logf(A);
            }
            if (loss_rows) loss_rows[i] = loss;
            if (lse_out) lse_out[i] = M + logf(A);
            my_loss = loss;
        }
    }
    if (emit_loss && block_sums) {
        __shared__ double red[256];
        red[threadIdx.x] = my_loss;
        __syncthreads();
        for (int o = 128; o > 0; o >>= 1) {
            if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
            __syncthreads();
        }
        if (threadIdx.x == 0) block_sums[blockIdx.x] = red[0];
    }
}

cudaError_t launch_merge_stats(int parts, int64_t n, int64_t part_stride, const float* pm,
                               const float* pa, const float* pzt, const uint8_t* pf,
                               const int64_t* targets, int has_ignore, int64_t ignore_index,
                               int emit_loss, float* m, float* a, float* zt, uint8_t* found,
                               float* lse, float* loss_rows, double* block_sums, int* err_flags,
                               cudaStream_t stream, int* blocks_out, const int* row_map,
                               int64_t found_stride) {
    const int blocks = static_cast<int>((n + 255) / 256);
    if (blocks_out) *blocks_out = blocks;
    k_merge_stats<<<blocks, 256, 0, stream>>>(parts, n, part_stride, found_stride >= 0 ? found_stride : part_stride,
                                              pm, pa, pzt, pf, targets,
                                              has_ignore, ignore_index, emit_loss, m, a, zt, found,
                                              lse, loss_rows, block_sums, err_flags, row_map);
    return cudaGetLastError();
}

// ------------------------------------------------- ignored-row compaction
// The reference never touches an ignored position: accumulate_stats_block and
// accumulate_grads_block skip rows whose tracking entry is kSkipPosition
// (fused_forward.hpp:57-59, fused_backward.hpp:37-39).  The device path gets
// the same saving by compacting the valid rows before the tile kernels:
// row_map[i] = slot of row i among the valid rows (ascending), -1 if ignored;
// rows[j] = original index of slot j.  One block scans N in 1024-row tiles.
__global__ void __launch_bounds__(1024) k_row_map(const int64_t* __restrict__ targets, int64_t n,
                                                  int64_t ignore_index, int* row_map, int* rows) {
    __shared__ int warp_sums[32];
    __shared__ int base_s;
    if (threadIdx.x == 0) base_s = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = 0; t0 < n; t0 += 1024) {
        const int64_t i = t0 + threadIdx.x;
        const int valid = (i < n && targets[i] != ignore_index) ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, valid);
        const int in_warp = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) warp_sums[wid] = __popc(bal);
        __syncthreads();
        if (wid == 0) {
            const int x = warp_sums[lane];
            int incl = x;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            warp_sums[lane] = incl - x;  // exclusive
        }
        __syncthreads();
        const int slot = base_s + warp_sums[wid] + in_warp;
        if (i < n) {
            row_map[i] = valid ? slot : -1;
            if (valid) rows[slot] = static_cast<int>(i);
        }
        __syncthreads();
        if (threadIdx.x == 1023) base_s = slot + valid;
        __syncthreads();
    }
}

cudaError_t launch_row_map(const int64_t* targets, int64_t n, int64_t ignore_index, int* row_map,
                           int* rows, cudaStream_t stream) {
    k_row_map<<<1, 1024, 0, stream>>>(targets, n, ignore_index, row_map, rows);
    return cudaGetLastError();
}

// dst[j, 0:cols) = src[rows[j], 0:cols) for 16-byte elements (cols16 per row)
// for the live slots j < *count; slots past it (the padding of the
// compacted problem, sized for N rows) are zero-filled
__global__ void k_gather_rows16(const uint4* __restrict__ src, int64_t ld_src16, uint4* __restrict__ dst,
                                int64_t ld_dst16, int64_t cols16, const int* __restrict__ rows,
                                int64_t n_slots, const unsigned long long* __restrict__ count) {
    const int64_t live = static_cast<int64_t>(*count);
    const int64_t total = n_slots * cols16;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = k / cols16, c = k - j * cols16;
        dst[j * ld_dst16 + c] = j < live ? src[static_cast<int64_t>(rows[j]) * ld_src16 + c] : make_uint4(0, 0, 0, 0);
    }
}

// per-slot row data: targets, and (backward) gamma / lse of the live rows;
// padding slots get target 0 and gamma = lse = 0 (they contribute nothing)
__global__ void k_gather_row_scalars(const int* __restrict__ rows, int64_t n_slots,
                                     const unsigned long long* __restrict__ count,
                                     const int64_t* __restrict__ t_in, int64_t* t_out,
                                     const float* __restrict__ g_in, float* g_out,
                                     const float* __restrict__ l_in, float* l_out) {
    const int64_t live = static_cast<int64_t>(*count);
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_slots;
         j += (int64_t)gridDim.x * blockDim.x) {
        const bool ok = j < live;
        const int64_t i = ok ? rows[j] : 0;
        if (t_out) t_out[j] = ok ? t_in[i] : 0;
        if (g_out) g_out[j] = ok ? g_in[i] : 0.f;
        if (l_out) l_out[j] = ok ? l_in[i] : 0.f;
    }
}

cudaError_t launch_gather_rows(const void* src, int64_t ld_src_bytes, void* dst, int64_t ld_dst_bytes,
                               int64_t row_bytes, const int* rows, int64_t n_slots,
                               const unsigned long long* count, const int64_t* t_in, int64_t* t_out,
                               const float* g_in, float* g_out, const float* l_in, float* l_out,
                               cudaStream_t stream) {
    if (n_slots <= 0) return cudaSuccess;
    if (src) {
        const int64_t cols16 = (row_bytes + 15) / 16;
        const int64_t total = n_slots * cols16;
        const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
        k_gather_rows16<<<blocks, 256, 0, stream>>>(static_cast<const uint4*>(src), ld_src_bytes / 16,
                                                    static_cast<uint4*>(dst), ld_dst_bytes / 16, cols16,
                                                    rows, n_slots, count);
    }
    const int blocks = static_cast<int>(std::min<int64_t>((n_slots + 255) / 256, 148 * 4));
    k_gather_row_scalars<<<blocks, 256, 0, stream>>>(rows, n_slots, count, t_in, t_out, g_in, g_out, l_in,
                                                     l_out);
    return cudaGetLastError();
}

// dH[i, :] = dH_c[row_map[i], :] (or += with accumulate); ignored rows are
// zeroed (left untouched with accumulate), as accumulate_grads_block leaves
// them (fused_backward.hpp:37-39 on zero-initialised gradients).
__global__ void k_scatter_rows_f32(const float* __restrict__ src, int64_t ld_src, float* dst,
                                   int64_t ld_dst, int64_t cols, const int* __restrict__ row_map,
                                   int64_t n, int accumulate) {
    const int64_t c4 = (cols + 3) / 4;
    const bool vec = (cols % 4 == 0) && (ld_src % 4 == 0) && (ld_dst % 4 == 0);
    const int64_t total = n * (vec ? c4 : cols);
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < total;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t per = vec ? c4 : cols;
        const int64_t i = k / per, c = k - i * per;
        const int j = row_map[i];
        if (j < 0 && accumulate) continue;
        if (vec) {
            float4 v = j >= 0 ? reinterpret_cast<const float4*>(src + j * ld_src)[c] : make_float4(0.f, 0.f, 0.f, 0.f);
            float4* d = reinterpret_cast<float4*>(dst + i * ld_dst) + c;
            if (accumulate) {
                const float4 o = *d;
                v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
            }
            *d = v;
        } else {
            const float v = j >= 0 ? src[j * ld_src + c] : 0.f;
            float* d = dst + i * ld_dst + c;
            *d = accumulate ? *d + v : v;
        }
    }
}

cudaError_t launch_scatter_rows_f32(const float* src, int64_t ld_src, float* dst, int64_t ld_dst,
                                    int64_t cols, const int* row_map, int64_t n, int accumulate,
                                    cudaStream_t stream) {
    const int64_t total = n * ((cols + 3) / 4);
    const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 148 * 16));
    k_scatter_rows_f32<<<std::max(blocks, 1), 256, 0, stream>>>(src, ld_src, dst, ld_dst, cols, row_map, n,
                                                                accumulate);
    return cudaGetLastError();
}

// Deterministic final reduction (fixed order), then reduce_losses semantics
// (reduction.hpp:37-54): mean over the valid count, 0 when nothing is valid.
__global__ void k_reduce_loss(const double* __restrict__ block_sums, int blocks,
                              const unsigned long long* valid_count, int reduction, float* out) {
    __shared__ double red[256];
    double s = 0.0;
    for (int i = threadIdx.x; i < blocks; i += 256) s += block_sums[i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double total = red[0];
        if (reduction == 0) {
            const unsigned long long c = *valid_count;
            total = c > 0 ? total / static_cast<double>(c) : 0.0;
        }
        *out = static_cast<float>(total);
    }
}

cudaError_t launch_reduce_loss(const double* block_sums, int blocks,
                               const unsigned long long* valid_count, int reduction,
                               float* loss_reduced, cudaStream_t stream) {
    k_reduce_loss<<<1, 256, 0, stream>>>(block_sums, blocks, valid_count, reduction, loss_reduced);
    return cudaGetLastError();
}

// gamma_n = effective upstream (reduction.hpp:110-126); lse_n = m + log a;
// require_stats (fused_backward.hpp:58-73): non-ignored rows need found && a > 0.
__global__ void k_gamma(int64_t n, const int64_t* __restrict__ targets, int has_ignore,
                        int64_t ignore_index, const float* __restrict__ m,
                        const float* __restrict__ a, const uint8_t* __restrict__ found,
                        int reduction, float upstream_scalar, const float* __restrict__ up_dev,
                        const float* __restrict__ up_rows, const unsigned long long* valid_count,
                        float* gamma, float* lse, int* err) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool ign = has_ignore && targets[i] == ignore_index;
    if (ign) {
        gamma[i] = 0.f;
        lse[i] = 0.f;
        return;
    }
    if (!(found[i] != 0) || !(a[i] > 0.f)) atomicOr(&err[kErrMissingStats], 1);
    float g;
    // scalar upstream: by value, or read on the device (graph-capturable autograd)
    const float up = up_dev ? *up_dev : upstream_scalar;
    if (reduction == 2) {
        g = up_rows[i];
    } else if (reduction == 0) {
        const unsigned long long c = *valid_count;
        g = c > 0 ? up / static_cast<float>(c) : 0.f;
    } else {
        g = up;
    }
    gamma[i] = g;
    lse[i] = m[i] + logf(a[i]);
}

cudaError_t launch_gamma(int64_t n, const int64_t* targets, int has_ignore, int64_t ignore_index,
                         const float* m, const float* a, const uint8_t* found, int reduction,
                         float upstream_scalar, const float* upstream_dev, const float* upstream_rows,
                         const unsigned long long* valid_count, float* gamma, float* lse,
                         int* err_flags, cudaStream_t stream) {
    const int blocks = static_cast<int>((n + 255) / 256);
    k_gamma<<<blocks, 256, 0, stream>>>(n, targets, has_ignore, ignore_index, m, a, found,
                                        reduction, upstream_scalar, upstream_dev, upstream_rows, valid_count,
                                        gamma, lse, err_flags);
    return cudaGetLastError();
}

__global__ void k_scale(float* x, int64_t count, const float* factor_dev, float factor) {
    const float f = factor_dev ? *factor_dev : factor;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
         i += (int64_t)gridDim.x * blockDim.x)
        x[i] *= f;
}

cudaError_t launch_scale(float* x, int64_t count, const float* factor_dev, float factor,
                         cudaStream_t stream) {
    int blocks = static_cast<int>(std::min<int64_t>((count + 255) / 256, 148 * 16));
    if (blocks < 1) blocks = 1;
    k_scale<<<blocks, 256, 0, stream>>>(x, count, factor_dev, factor);
    return cudaGetLastError();
}

// ------------------------------------------------- synthetic instance (device)
// Bit-identical to make_random_instance (reference instance.hpp:38-66):
// splitmix64 is counter based, so element i of a stream whose state starts at
// s0 is mix(s0 + (i + 1) * golden).
__device__ __forceinline__ uint64_t splitmix_at(uint64_t s0, uint64_t i) {
    uint64_t z = s0 + (i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ float round_bf16_dev(float x) {
    if (isnan(x)) return x;
    uint32_t bits = __float_as_uint(x);
    const uint32_t lsb = (bits >> 16) & 1u;
    bits += 0x7FFFu + lsb;
    bits &= 0xFFFF0000u;
    return __uint_as_float(bits);
}

__global__ void k_gen_matrix(__nv_bfloat16* out, int64_t rows, int64_t cols, int64_t ld,
                             uint64_t s0, double scale, float* out_f32) {
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t z = splitmix_at(s0, static_cast<uint64_t>(i));
        const double u = static_cast<double>(z >> 11) * 0x1.0p-53;
        const double x = __dmul_rn(__dsub_rn(__dmul_rn(2.0, u), 1.0), scale);
        const float xf = round_bf16_dev(__double2float_rn(x));
        const int64_t r = i / cols, c = i - r * cols;
        if (out) out[r * ld + c] = __float2bfloat16_rn(xf);
        if (out_f32) out_f32[r * ld + c] = xf;
    }
}

cudaError_t launch_gen_matrix(__nv_bfloat16* out, int64_t rows, int64_t cols, int64_t ld,
                              uint64_t seed_state, double scale, float* out_f32,
                              cudaStream_t stream) {
    k_gen_matrix<<<148 * 8, 256, 0, stream>>>(out, rows, cols, ld, seed_state, scale, out_f32);
    return cudaGetLastError();
}

__global__ void k_gen_targets(int64_t* out, int64_t n, int64_t v, uint64_t seed,
                              int64_t ignore_index, double ignore_fraction) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t t = static_cast<int64_t>(splitmix_at(seed ^ 0x5A5A5A5A5A5A5A5Aull, i) %
                                         static_cast<uint64_t>(v));
        if (ignore_fraction > 0.0) {
            const double u =
                static_cast<double>(splitmix_at(seed ^ 0x3C3C3C3C3C3C3C3Cull, i) >> 11) *
                0x1.0p-53;
            if (u < ignore_fraction) t = ignore_index;
        }
        out[i] = t;
    }
}

cudaError_t launch_gen_targets(int64_t* out, int64_t n, int64_t v, uint64_t seed,
                               int64_t ignore_index, double ignore_fraction, cudaStream_t stream) {
    int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 1184));
    if (blocks < 1) blocks = 1;
    k_gen_targets<<<blocks, 256, 0, stream>>>(out, n, v, seed, ignore_index, ignore_fraction);
    return cudaGetLastError();
}

// float (on the bf16 grid) -> bf16, flagging off-grid values (bf16.hpp:31-36).
__global__ void k_f32_to_bf16(const float* __restrict__ in, int64_t rows, int64_t cols,
                              int64_t ld_in, __nv_bfloat16* out, int64_t ld_out, int* err) {
    const int64_t total = rows * ld_out;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / ld_out, c = i - r * ld_out;
        float x = 0.f;
        if (c < cols) {
            x = in[r * ld_in + c];
            if (round_bf16_dev(x) != x && !isnan(x)) atomicOr(&err[kErrOffGrid], 1);
        }
        out[i] = __float2bfloat16_rn(x);
    }
}

// out[r, c] = bf16_rn(in[r, c]) for c < cols (padding columns untouched)
__global__ void k_round_to_bf16(const float* __restrict__ in, int64_t rows, int64_t cols, int64_t ld_in,
                                __nv_bfloat16* out, int64_t ld_out) {
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols, c = i - r * cols;
        out[r * ld_out + c] = __float2bfloat16_rn(in[r * ld_in + c]);
    }
}

cudaError_t launch_round_to_bf16(const float* in, int64_t rows, int64_t cols, int64_t ld_in,
                                 __nv_bfloat16* out, int64_t ld_out, cudaStream_t stream) {
    if (rows <= 0 || cols <= 0) return cudaSuccess;
    k_round_to_bf16<<<148 * 8, 256, 0, stream>>>(in, rows, cols, ld_in, out, ld_out);
    return cudaGetLastError();
}

cudaError_t launch_f32_to_bf16(const float* in, int64_t rows, int64_t cols, int64_t ld_in,
                               __nv_bfloat16* out, int64_t ld_out, int* err_flags,
                               cudaStream_t stream) {
    k_f32_to_bf16<<<148 * 8, 256, 0, stream>>>(in, rows, cols, ld_in, out, ld_out, err_flags);
    return cudaGetLastError();
}

}  // namespace fce
