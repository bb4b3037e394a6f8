// Internal (non-ABI) declarations shared by the C-ABI layer and the CUDA
// translation units.  Nothing here is exported from libfce.so.
#pragma once

#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <nvtx3/nvToolsExt.h>

#include "../../include/fce/fce.h"

namespace fce {

// NVTX range around a host entry point / launch group (header-only NVTX3:
// free when no profiler is attached; nsys / ncu --nvtx show the K1 / K2 /
// collective phases of a step).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Tile geometry of the tcgen05 kernel (one CTA per SM, 1-CTA UMMA).
constexpr int kBM = 128;      // rows per tile = TMEM lanes
constexpr int kBN = 256;      // columns per tile = UMMA N = TMEM columns per accumulator
constexpr int kBK = 64;       // K per pipeline stage = one 128-byte swizzle atom of bf16
constexpr int kStages = 4;    // TMA -> MMA smem ring depth
constexpr int kThreads = 256; // warp0 TMA, warp1 MMA, warp2 TMEM alloc, warp3 idle, warps4-7 epilogue
constexpr int kStageBytesA = kBM * kBK * 2;
constexpr int kStageBytesB = kBN * kBK * 2;
constexpr int kSmemBytes = kStages * (kStageBytesA + kStageBytesB) + 1024 /*align*/ + 256 /*barriers*/;

enum EpilogueMode : int { kEpiForward = 0, kEpiGrad = 1, kEpiGemm = 2 };

// Ranks whose dH accumulators one persistent backward can reduce into directly.
constexpr int kMaxDhPeers = 8;

// One GEMM problem C[M,N] (+)= A[M,K] * B[N,K]^T for the generic epilogue.
struct GemmProblem {
    int m, n, k_blocks;
    int m_tiles, n_tiles;
    int a_mn, b_mn;     // 1 = operand stored MN-major (M/N contiguous), 0 = K-major
    int n_fastest;      // tile order inside the problem
    int accumulate;     // 1 = red.global.add into C, 0 = plain store
    float* c;
    int64_t ldc;
};

struct TileParams {
    int mode;
    int units;               // total work units
    // forward / grad (A = H [N, D] K-major, B = W rows K-major)
    int n_rows;              // N (rows of the operand / partial arrays)
    const unsigned long long* n_valid;  // forward: device count of live rows (compacted problems); rows
                                        // past it are skipped on the device (NULL: all n_rows)
    int v_cols;              // valid columns of this launch (V_local for fwd, band width for grad)
    int m_blocks;            // ceil(N / kBM)
    int v_tiles;             // ceil(v_cols / kBN)
    int splits;              // forward split-V factor
    int m_group;             // m-blocks per L2 raster group
    int k_blocks;            // ceil(D / kBK)
    const int64_t* targets;  // [N] global target ids
    int64_t col_global0;     // global vocab id of launch column 0
    int has_ignore;
    int64_t ignore_index;
    float* part_m;           // [splits][N]
    float* part_a;
    float* part_zt;
    uint8_t* part_found;
    const float* lse;        // [N] (grad)
    const float* gamma;      // [N] (grad)
    __nv_bfloat16* g_out;    // grad: G band [N][ldg]
    int64_t ldg;
    // generic GEMM (two problems in one persistent launch)
    GemmProblem prob[2];
    int units0;
};

struct TensorMaps {
    CUtensorMap a0, b0, a1, b1;
};

// ----------------------------------------------------------- persistent backward
// Every (row chunk x vocab band) chunk is laid out at full geometry; see fce_bwd.cu.
struct BwdParams {
    int units;               // row chunks * per_rc
    int n_chunks, bands;     // chunks = row chunks x bands, chunk c = (c / bands, c % bands)
    int kg, gpr;             // bands per dH group, dH groups per row chunk
    int per_rc, per_gf;      // units per row chunk, per full group
    int n_g, n_dh, n_dw;     // grad / dH / dW units per chunk (padded geometry)
    int vt, vm;              // band / 256, band / 128
    int d_tiles, k_blocks_d, mb_max, gm_base;
    int n, v;                // rows, local vocab rows
    int has_ignore, accumulate_dh;
    int unit_mask;           // debug / profiling: bit0 grad, bit1 dH, bit2 dW units do work
    int epi_warps;           // 4 or 8 epilogue warps per CTA
    int tma_epi;             // 1: epilogue writes G / dH / dW through SMEM + TMA store / reduce-add
    int dw_bf16;             // 1: dW is bf16 (one row chunk, stored once from the accumulators)
    const unsigned long long* n_valid;  // device count of live rows (compacted problems; NULL: n)
    int l2_hints;            // bit0: evict_first on dH/dW writes, bit1: evict_last on G loads,
                             // bit2: evict_last on G stores, bit3: evict_first on H loads (dW)
    // dH reduced across ranks inside the kernel (vocab-parallel over peer
    // memory): every dH tile is TMA-reduce-added into the symmetric accumulator
    // of the rank owning its 128-row block; owners hold blocks
    // [peer_block0[q], peer_block0[q + 1]) (0 peers: local dH as usual)
    int dh_peers;
    int peer_block0[kMaxDhPeers + 1];
    int64_t nc_max, ldg, ldr, d, lddh, lddw, v_offset, ignore_index;  // ldg = band, ldr = kg * band
    unsigned* counters;      // [0] scheduler, 4 per chunk, then mb_max per chunk
    unsigned long long* trace;  // dev only: [units][8] = MMA start, MMA end, epilogue end, smid,
                                //   accumulator free, first stage ready, stage-wait cycles
    const int64_t* targets;
    const float* lse;
    const float* gamma;
    __nv_bfloat16* g_ring;   // [2 group slots][nc_max][ldr]: band j of a group at column j * ldg
    float* dh;
    float* dw;               // fp32 dW, or the bf16 dW (reinterpreted) when dw_bf16
};

struct BwdMaps {
    CUtensorMap h_k, w_k, g_k, w_mn, g_mn, h_mn;
    CUtensorMap g_st, dh_st, dw_st;  // epilogue TMA stores / reduce-adds (tma_epi)
    CUtensorMap dh_peer[kMaxDhPeers];  // owners' dH accumulators (dh_peers > 0)
};

cudaError_t launch_fwd_pair(const TileParams& p, const TensorMaps& maps, int sms, cudaStream_t stream);
cudaError_t launch_fwd_mc(const TileParams& p, const TensorMaps& maps, int sms, cudaStream_t stream);

cudaError_t launch_pair_gemm(const GemmProblem& q, const TensorMaps& maps, int sms,
                             cudaStream_t stream);

cudaError_t launch_bwd_persistent(const BwdParams& p, const BwdMaps& maps, int grid,
                                  cudaStream_t stream);

// fce_merge_partials with a separate stride (in bytes) for the found flags, so
// per-rank partials can travel as one packed block [m | a | z_t | found]
// (fce_api.cpp).
fce_status merge_partials(fce_handle h, int parts, int64_t n, int64_t part_stride, int64_t found_stride,
                          const float* m, const float* a, const float* z_target, const uint8_t* found,
                          const int64_t* targets, int32_t has_ignore, int64_t ignore_index, int reduction,
                          fce_stats merged, float* lse, float* loss_rows, float* loss_reduced);

// Overlapped vocab-parallel backward (fce_api.cpp): fce_backward with the rows
// cut into row chunks of `row_chunk`, the persistent kernel leaving
// `reserve_sms` SMs free for collectives, `counters_reset` recorded on the
// handle stream once the dependency counters are zeroed, and for every row
// chunk the device counter + value that mark its dH rows final.
struct DhChunkDone {
    const unsigned* counter;
    unsigned target;
    int64_t row0, rows;
};
struct LastBwdView {
    const unsigned* counters;
    int64_t row_chunk, n_rc, bands, n_dh;
};
fce_status backward_for_overlap(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                                float upstream_scalar, const float* upstream_rows, float* dhidden, int64_t lddh,
                                float* dweight, int64_t lddw, int64_t row_chunk, int reserve_sms,
                                cudaEvent_t counters_reset, std::vector<DhChunkDone>* done);
// fce_backward whose dH tiles are reduce-added (TMA, fp32) straight into the
// owning rank's dH accumulator: peer_dh[q] are the k ranks' [n, d]
// accumulators as mapped in this process (peer memory), rank q owning the
// 128-row blocks [block0[q], block0[q + 1]).  The accumulators must be zeroed
// (owned rows) before any rank's kernel starts; dW stays local (fce_api.cpp).
fce_status backward_dh_peers(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                             float upstream_scalar, const float* upstream_rows, float* const* peer_dh, int k,
                             const int* block0, float* dweight, int64_t lddw);
// Stream-ordered wait until *counter >= target (cuStreamWaitValue32, or a
// one-thread spin kernel where stream memory operations are unavailable).
cudaError_t stream_wait_geq(cudaStream_t s, const unsigned* counter, unsigned target);

// Stream a handle launches on (fce_api.cpp).
cudaStream_t handle_stream(fce_handle h);
int handle_device(fce_handle h);
// Options "vp_overlap_chunks" / "vp_reserve_sms" of the handle (fce_vp_backward).
int64_t handle_vp_overlap_chunks(fce_handle h);
int64_t handle_vp_reserve_sms(fce_handle h);
// Option "vp_fused_dh": fce_vp_backward reduces dH inside the kernel (peer memory).
int64_t handle_vp_fused_dh(fce_handle h);
// Option "validate" (multi-rank entry points also cross-check the ranks' shapes).
bool handle_validate(fce_handle h);
// Option "comm_trace_ptr" (dev): u64 slots for globaltimer stamps, 2 per chunk.
unsigned long long* handle_comm_trace(fce_handle h);
cudaError_t launch_stamp(cudaStream_t s, unsigned long long* slot);
// Thread-local message returned by fce_last_error (fce_api.cpp).
void set_last_error(const char* msg);

// Host helpers (fce_kernels.cu)
bool encode_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                   uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_outer,
                   bool fp32 = false);
cudaError_t launch_tile_kernel(const TileParams& p, const TensorMaps& maps, int grid,
                               cudaStream_t stream);
int device_sm_count(int device);
// One-time (per kernel and device, thread-safe) opt-in to `bytes` of dynamic
// shared memory; several host threads may drive handles on the same or on
// different devices (in-process communicator groups).
cudaError_t ensure_dyn_smem(const void* func, int bytes);

cudaError_t launch_prep_targets(const int64_t* targets, int64_t n, int has_ignore,
                                int64_t ignore_index, int64_t v_total, int* err_flags,
                                unsigned long long* valid_count, cudaStream_t stream);
cudaError_t launch_merge_stats(int parts, int64_t n, int64_t part_stride, const float* pm,
                               const float* pa, const float* pzt, const uint8_t* pf,
                               const int64_t* targets, int has_ignore, int64_t ignore_index,
                               int emit_loss, float* m, float* a, float* zt, uint8_t* found,
                               float* lse, float* loss_rows, double* block_sums, int* err_flags,
                               cudaStream_t stream, int* blocks_out, const int* row_map = nullptr,
                               int64_t found_stride = -1 /* -1: part_stride */);
cudaError_t launch_round_to_bf16(const float* in, int64_t rows, int64_t cols, int64_t ld_in,
                                 __nv_bfloat16* out, int64_t ld_out, cudaStream_t stream);
// ignored-row compaction (fce_kernels.cu)
cudaError_t launch_row_map(const int64_t* targets, int64_t n, int64_t ignore_index, int* row_map,
                           int* rows, cudaStream_t stream);
cudaError_t launch_gather_rows(const void* src, int64_t ld_src_bytes, void* dst, int64_t ld_dst_bytes,
                               int64_t row_bytes, const int* rows, int64_t n_slots,
                               const unsigned long long* count, const int64_t* t_in, int64_t* t_out,
                               const float* g_in, float* g_out, const float* l_in, float* l_out,
                               cudaStream_t stream);
cudaError_t launch_scatter_rows_f32(const float* src, int64_t ld_src, float* dst, int64_t ld_dst,
                                    int64_t cols, const int* row_map, int64_t n, int accumulate,
                                    cudaStream_t stream);
cudaError_t launch_reduce_loss(const double* block_sums, int blocks,
                               const unsigned long long* valid_count, int reduction,
                               float* loss_reduced, cudaStream_t stream);
cudaError_t launch_gamma(int64_t n, const int64_t* targets, int has_ignore, int64_t ignore_index,
                         const float* m, const float* a, const uint8_t* found, int reduction,
                         float upstream_scalar, const float* upstream_dev, const float* upstream_rows,
                         const unsigned long long* valid_count, float* gamma, float* lse,
                         int* err_flags, cudaStream_t stream);
cudaError_t launch_scale(float* x, int64_t count, const float* factor_dev, float factor,
                         cudaStream_t stream);
cudaError_t launch_gen_matrix(__nv_bfloat16* out, int64_t rows, int64_t cols, int64_t ld,
                              uint64_t seed_state, double scale, float* out_f32,
                              cudaStream_t stream);
cudaError_t launch_gen_targets(int64_t* out, int64_t n, int64_t v, uint64_t seed,
                               int64_t ignore_index, double ignore_fraction, cudaStream_t stream);
cudaError_t launch_f32_to_bf16(const float* in, int64_t rows, int64_t cols, int64_t ld_in,
                               __nv_bfloat16* out, int64_t ld_out, int* err_flags,
                               cudaStream_t stream);

// err_flags slots
enum ErrSlot : int {
    kErrTargetRange = 0,
    kErrDuplicate = 1,
    kErrNotFound = 2,
    kErrMissingStats = 3,
    kErrOffGrid = 4,
    kErrSlots = 8
};

}  // namespace fce
