/*
 * fce_oracle.h — CPU restatement of the reference fused-LCE algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline leg of bench.py may load this library, and only as the
 * checker; the product path (libfce.so) never links or calls it.
 *
 * Every function restates one reference function (cited file:line relative
 * to the reference's proj/include/fusedce/) in plain C11 with the same
 * evaluation order, for T = float.  Built with -ffp-contract=off, as is the
 * reference build in oracle/_ref, the two agree bit for bit (pinned by
 * tests/test_oracle.py against oracle/_ref and tests/golden/).
 */
#ifndef FCE_ORACLE_H_
#define FCE_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_MEAN = 0, ORC_SUM = 1, ORC_NONE = 2 };

/* status codes = fce_status (1 + fusedce::ErrorCode) */
enum {
    ORC_OK = 0,
    ORC_DIMENSION_MISMATCH = 1,
    ORC_TARGET_OUT_OF_RANGE = 2,
    ORC_DUPLICATE_TARGET = 4,
    ORC_MISSING_STATS = 5,
    ORC_INCONSISTENT_UPSTREAM = 6,
    ORC_UNSUPPORTED_REDUCTION = 7,
    ORC_INVALID_LAYOUT = 8,
    ORC_EMPTY_INPUT = 10
};

typedef struct orc_stats {
    float m, a, z_target;
    uint8_t found;
} orc_stats;

/* instance.hpp:15-20, 23-25 */
uint64_t orc_splitmix64(uint64_t* state);
double orc_splitmix_unit(uint64_t* state);
/* bf16.hpp:14-23, 31-36 */
float orc_round_bf16(float x);
int orc_is_bf16_value(float x);
/* instance.hpp:38-85; round = 1 applies DenseMatrix::round_to_bf16
 * (dense_matrix.hpp:86-92) to H and W.  ignore_fraction <= 0: no ignores. */
int orc_make_instance(size_t n, size_t d, size_t v, uint64_t seed, int64_t ignore_index,
                      double ignore_fraction, int round, float* hidden, float* weight,
                      int64_t* targets);

/* detail/kernels.hpp:11-61 */
float orc_dot(const float* a, const float* b, size_t n, size_t d_tile);

/* softmax_stats.hpp:23-45, 52-75 */
void orc_stats_update(orc_stats* s, float z);
float orc_stats_logsumexp(const orc_stats* s);
float orc_stats_loss(const orc_stats* s);
int orc_merge_stats(const orc_stats* s1, const orc_stats* s2, orc_stats* out);

/* exec.hpp:25-41 (ceil-first); out_lo/out_hi have `parts` entries */
int orc_partition_ranges(size_t total, size_t parts, size_t* out_lo, size_t* out_hi);

/* fused_forward.hpp:161-172 (window = 0) and 177-195 (window > 0), single
 * worker.  stats[n]; loss_rows[n] (0 on ignored rows); *loss_reduced for
 * mean/sum.  threads > 1 splits rows (bitwise identical: rows are
 * independent).  Returns a status code. */
int orc_fused_forward(const float* hidden, const float* weight, size_t n, size_t d, size_t v,
                      size_t v_offset, const int64_t* targets, int has_ignore, int64_t ignore_index,
                      int reduction, size_t window, int threads, orc_stats* stats,
                      float* loss_rows, float* loss_reduced);

/* tp_rank_partial (parallel_sim.hpp:165-181): stats of weight rows
 * [v_offset, v_offset + v_rows) with global targets, no validation. */
int orc_rank_partial(const float* hidden, const float* weight_shard, size_t n, size_t d,
                     size_t v_rows, size_t v_offset, const int64_t* targets, int has_ignore,
                     int64_t ignore_index, int threads, orc_stats* stats);

/* fused_backward.hpp:118-140 for weight rows [v_offset, v_offset + v) of a
 * v_total vocabulary (0: v) (single-worker accumulation order: dH rows over
 * ascending v, dW rows over ascending n).  upstream_rows used for NONE. */
int orc_fused_backward(const float* hidden, const float* weight, size_t n, size_t d, size_t v,
                       size_t v_offset, size_t v_total, const int64_t* targets, int has_ignore,
                       int64_t ignore_index, const orc_stats* stats, int reduction,
                       float upstream_scalar, const float* upstream_rows, int threads,
                       float* dhidden, float* dweight);

/* reduction.hpp:37-54 */
float orc_reduce_losses(const float* rows, size_t n, int reduction, size_t valid_count);

#ifdef __cplusplus
}
#endif

#endif
