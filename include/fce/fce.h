/*
 * fce.h — C-ABI of the B200-native fused linear-cross-entropy operator.
 *
 * The reference (arxiv/paper_2511_17599, proj/include/fusedce) is a
 * header-only C++20 template library with no FFI of its own; every entry
 * point below replaces one of its public L1 functions and is what a foreign
 * binding (ctypes / cgo / JNI) or the drop-in C++ headers in include/fusedce
 * bind to.  Plain pointers and sizes only: no C++ or torch types.
 *
 * Conventions
 *   - Every pointer argument of a compute entry point is a DEVICE pointer,
 *     caller-owned and stream-ordered on the handle's stream.
 *   - hidden / weight are bf16, row-major, leading dimension in elements,
 *     ld % 8 == 0 and 16-byte aligned base (TMA); d may be < ld (the tail is
 *     never read).  Outputs are fp32 (loss, stats, gradients).
 *   - No exception crosses the ABI: every function returns an fce_status and
 *     fce_last_error() holds a thread-local message for the last failure.
 *   - Validation happens before any output is written (reference:
 *     validate_problem, dense_matrix.hpp:182-211); the target check needs the
 *     targets, which are on the device, so it costs one stream sync per call.
 */
#ifndef FCE_FCE_H_
#define FCE_FCE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Codes 1..10 mirror fusedce::ErrorCode in declaration order
 * (reference proj/include/fusedce/errors.hpp:10-21), so a binding maps
 * status - 1 straight onto the reference enum. */
typedef enum fce_status {
    FCE_OK = 0,
    FCE_DIMENSION_MISMATCH = 1,
    FCE_TARGET_OUT_OF_RANGE = 2,
    FCE_UNDERFLOW_RELEASE = 3,
    FCE_DUPLICATE_TARGET = 4,
    FCE_MISSING_STATS = 5,
    FCE_INCONSISTENT_UPSTREAM = 6,
    FCE_UNSUPPORTED_REDUCTION = 7,
    FCE_INVALID_LAYOUT = 8,
    FCE_EMPTY_GRID = 9,
    FCE_EMPTY_INPUT = 10,
    FCE_CUDA_ERROR = 100,
    FCE_NCCL_ERROR = 101,
    FCE_INVALID_ARGUMENT = 102
} fce_status;

/* fusedce::ReductionMode order (reference reduction.hpp:12). */
typedef enum fce_reduction {
    FCE_REDUCTION_MEAN = 0,
    FCE_REDUCTION_SUM = 1,
    FCE_REDUCTION_NONE = 2
} fce_reduction;

typedef struct fce_handle_s* fce_handle;

/* One (rank-local) problem: H[n, d] . W[v, d]^T against global targets.
 * Replaces the (MatrixView hidden, MatrixView weights, TargetVector) triple of
 * the reference signatures (fused_forward.hpp:161-164) and, with v_offset,
 * a WeightShard (parallel_sim.hpp:72-76). */
typedef struct fce_problem {
    const void* hidden;      /* bf16 [n, ldh] */
    int64_t ldh;
    const void* weight;      /* bf16 [v, ldw]: this rank's vocabulary rows */
    int64_t ldw;
    int64_t n, d, v;
    int64_t v_offset;        /* global vocab id of weight row 0 (0 unless sharded) */
    int64_t v_total;         /* global vocabulary for target validation; 0 means v */
    const int64_t* targets;  /* int64 [n], global ids */
    int32_t has_ignore;      /* TargetVector::ignore_index() engaged */
    int64_t ignore_index;
} fce_problem;

/* Per-row stats cache, SoftmaxStats<float> split into arrays
 * (reference softmax_stats.hpp:14-46).  Any member may be NULL on output. */
typedef struct fce_stats {
    float* m;
    float* a;
    float* z_target;
    uint8_t* found;
} fce_stats;

/* ---------------------------------------------------------------- handle */
fce_status fce_create(fce_handle* out, int device, void* stream /* cudaStream_t, may be NULL */);
fce_status fce_destroy(fce_handle h);
/* Retarget the handle; the new stream is ordered after the work already queued
 * on the old one (the handle's workspaces are shared between them). */
fce_status fce_set_stream(fce_handle h, void* stream);
const char* fce_last_error(void);
const char* fce_status_string(fce_status s);
/* Tuning / behaviour knobs: "splits" (forward split-V factor, 0 = auto),
 * "band_cols" / "row_chunk" (backward G chunk, 0 = auto), "bwd_persistent"
 * (1 = one persistent backward launch, default; 0 = two launches per chunk), "validate"
 * (1 = sync and check targets / stats, default 1), "timing" (1 = per-kernel
 * event timing, see fce_kernel_stats; setting it resets the counters),
 * "skip_ignored" (1 = compact ignored rows away before the tile kernels,
 * default), "bwd_reserve_sms" (SMs the persistent backward leaves free),
 * "vp_overlap_chunks" (fce_vp_backward: 0 = one dH all-reduce after the
 * kernel, default; k >= 2 = rows in k chunks, each chunk's all-reduce
 * released by the kernel's completion counter and overlapped with the later
 * chunks) and "vp_reserve_sms" (SMs left to those collectives, default 8). */
fce_status fce_set_option(fce_handle h, const char* key, int64_t value);
/* Library-owned device workspace (the device analogue of MemoryLedger,
 * memory_ledger.hpp:18-62): bytes held now and the high-water mark. */
fce_status fce_workspace_bytes(fce_handle h, size_t* current, size_t* peak);
/* Number of kernels this handle launched since creation (for the bench). */
fce_status fce_launch_count(fce_handle h, int64_t* count);
/* With option "timing" = 1 every tile-kernel launch is bracketed by CUDA
 * events on the handle's stream.  kernel: 0 = forward (online-LSE epilogue),
 * 1 = gradient producer (recompute + softmax - onehot), 2 = dW / dH
 * contractions (per-band path), 3 = persistent fused backward (default).  Returns summed device time, launch count and algorithmic
 * flops (2 * M * N * K per contraction) since timing was (re)enabled. */
fce_status fce_kernel_stats(fce_handle h, int kernel, double* total_ms, int64_t* launches,
                            double* flops);

/* ---------------------------------------------------------------- forward
 * fused_forward (fused_forward.hpp:161-172); window > 0 gives
 * fused_forward_windowed (177-195) with window rounded to 256-column tiles.
 * Writes the stats cache, per-row lse = m + log a, per-row loss (0 on ignored
 * rows) and, for mean/sum, the reduced loss (one float). */
fce_status fce_forward(fce_handle h, const fce_problem* p, int reduction, int64_t window,
                       fce_stats stats, float* lse, float* loss_rows, float* loss_reduced);

/* tp_rank_partial (parallel_sim.hpp:165-181): stats of this rank's vocab
 * shard only (target captured only if it falls in the shard). */
fce_status fce_forward_partial(fce_handle h, const fce_problem* p, fce_stats partial);

/* Rank-ordered merge of `parts` partial stats laid out [parts][part_stride]
 * (parallel_sim.hpp:214-231, merge_stats softmax_stats.hpp:52-75), then
 * loss / lse / reduction as fce_forward.  Duplicate targets ->
 * FCE_DUPLICATE_TARGET; a valid row no part found -> FCE_TARGET_OUT_OF_RANGE. */
fce_status fce_merge_partials(fce_handle h, int parts, int64_t n, int64_t part_stride,
                              const float* m, const float* a, const float* z_target,
                              const uint8_t* found, const int64_t* targets, int32_t has_ignore,
                              int64_t ignore_index, int reduction, fce_stats merged, float* lse,
                              float* loss_rows, float* loss_reduced);

/* ---------------------------------------------------------------- backward
 * fused_backward_recompute (fused_backward.hpp:118-140) for this rank's
 * vocabulary rows: dH[n, lddh] (+)= G . W and dW[v, lddw] = G^T . H with
 * G = gamma (softmax - onehot) recomputed from `stats`.  reduction NONE takes
 * upstream_rows [n] (device), MEAN/SUM take upstream_scalar
 * (check_upstream, reduction.hpp:81-97).  accumulate_dhidden = 1 adds into
 * dH (vocab-parallel partial sums); dhidden or dweight may be NULL to skip. */
fce_status fce_backward(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                        float upstream_scalar, const float* upstream_rows, float* dhidden,
                        int64_t lddh, float* dweight, int64_t lddw, int accumulate_dhidden);

/* Element types of gradient outputs (fce_backward_ex). */
typedef enum fce_dtype {
    FCE_DTYPE_F32 = 0,
    FCE_DTYPE_BF16 = 1
} fce_dtype;

/* fce_backward with the gradient element types chosen per output: FCE_DTYPE_F32
 * (as fce_backward) or FCE_DTYPE_BF16 (round-to-nearest-even of the fp32 sums;
 * the framework-facing form, e.g. a bf16 lm_head's .grad).  bf16 dW is written
 * straight from the tensor-core accumulators when the backward runs in one row
 * chunk (no fp32 V x D buffer at all); bf16 dH is accumulated in an fp32
 * workspace across vocabulary bands and rounded once at the end.
 * accumulate_dhidden requires an fp32 dH. */
fce_status fce_backward_ex(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                           float upstream_scalar, const float* upstream_rows, void* dhidden,
                           int64_t lddh, int dh_dtype, void* dweight, int64_t lddw, int dw_dtype,
                           int accumulate_dhidden);

/* fce_backward_ex with the MEAN / SUM upstream scalar read from device memory
 * (one float, e.g. a framework's loss gradient tensor) instead of passed by
 * value: no host read of the gradient, so with option "validate" = 0 an
 * autograd backward is stream-ordered end to end and CUDA-graph capturable.
 * reduction NONE takes upstream_rows as fce_backward_ex. */
fce_status fce_backward_dev(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                            const float* upstream_scalar_dev, const float* upstream_rows, void* dhidden,
                            int64_t lddh, int dh_dtype, void* dweight, int64_t lddw, int dw_dtype,
                            int accumulate_dhidden);

/* The tile kernel's generic contraction (the dW / dH building block), exposed
 * for kernel-level tests and benchmarks: C[M, N] (+)= A . B^T in fp32 with bf16
 * operands; A is [M, K] (a_mn = 0, row stride lda) or stored as [K, M]
 * (a_mn = 1); B is [N, K] (b_mn = 0) or stored as [K, N] (b_mn = 1). */
fce_status fce_gemm_bf16(fce_handle h, const void* a, int64_t lda, int a_mn, const void* b,
                         int64_t ldb, int b_mn, int64_t m, int64_t n, int64_t k, float* c,
                         int64_t ldc, int accumulate);

/* scale_partial_grads (fused_backward.hpp:193-202): x[i] *= factor. */
fce_status fce_scale(fce_handle h, float* x, int64_t count, float factor);

/* ---------------------------------------------------------------- inputs
 * make_random_instance[_with_ignores] (instance.hpp:38-85), bit-identical,
 * including round_bf16 (bf16.hpp:14-23).  Any output may be NULL; the f32
 * copies use the same leading dimensions.  ignore_fraction <= 0: no ignores. */
fce_status fce_generate_instance(fce_handle h, int64_t n, int64_t d, int64_t v, uint64_t seed,
                                 void* hidden_bf16, int64_t ldh, void* weight_bf16, int64_t ldw,
                                 int64_t* targets, int64_t ignore_index, double ignore_fraction,
                                 float* hidden_f32, float* weight_f32);

/* fp32 rows on the bf16 grid -> bf16 [rows, ld_out] (zero-padded beyond
 * cols).  Off-grid values -> FCE_INVALID_LAYOUT (the GPU path is bf16-in). */
fce_status fce_f32_to_bf16(fce_handle h, const float* in, int64_t rows, int64_t cols,
                           int64_t ld_in, void* out, int64_t ld_out);

#ifdef __cplusplus
}
#endif

#endif /* FCE_FCE_H_ */
