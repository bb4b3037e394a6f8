/*
 * fce_vp.h — vocabulary-parallel (tensor-parallel over the vocab) C-ABI.
 *
 * Replaces the single-process rank simulation of the reference
 * (proj/include/fusedce/parallel_sim.hpp:158-290: tp_rank_partial,
 * tp_forward, tp_backward) with one process per GPU and NCCL over
 * NVLink / NVSwitch.  Each rank passes its own contiguous ceil-first W shard
 * (ShardLayout::tensor_parallel, parallel_sim.hpp:55-57, exec.hpp:25-41) in
 * an fce_problem with v_offset / v_total set; H and targets are replicated.
 */
#ifndef FCE_FCE_VP_H_
#define FCE_FCE_VP_H_

#include "fce.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fce_comm_s* fce_comm;

#define FCE_COMM_ID_BYTES 128

/* Rank 0 creates the id and ships it to the others (e.g. torch.distributed
 * broadcast); every rank then calls fce_comm_init. */
fce_status fce_comm_unique_id(uint8_t* out, size_t len);
fce_status fce_comm_init(fce_comm* out, int device, int nranks, int rank, const uint8_t* id,
                         size_t len);
fce_status fce_comm_destroy(fce_comm c);
const char* fce_vp_last_error(void);

/* tp_forward (parallel_sim.hpp:186-236): all-gather of the per-row
 * (m, a, z_target, found) partials + rank-ordered merge; every rank ends with
 * the same merged stats, lse and loss. */
fce_status fce_vp_forward(fce_handle h, fce_comm c, const fce_problem* p, int reduction,
                          fce_stats merged, float* lse, float* loss_rows, float* loss_reduced);

/* tp_backward (parallel_sim.hpp:246-290): local dW shard, all-reduced dH. */
fce_status fce_vp_backward(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged,
                           int reduction, float upstream_scalar, const float* upstream_rows,
                           float* dhidden, int64_t lddh, float* dweight_shard, int64_t lddw);

#ifdef __cplusplus
}
#endif

#endif /* FCE_FCE_VP_H_ */
