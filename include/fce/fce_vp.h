/*
 * fce_vp.h — multi-rank C-ABI: vocabulary-parallel (tensor-parallel over the
 * vocab), sequence-parallel gather / scatter and the data-parallel step.
 *
 * Replaces the single-process rank simulation of the reference
 * (proj/include/fusedce/parallel_sim.hpp:158-378: tp_rank_partial,
 * tp_forward, tp_backward, sp_to_tp_gather, dp_step) with real ranks.  Each
 * rank passes its own contiguous ceil-first W shard (ShardLayout::
 * tensor_parallel, parallel_sim.hpp:55-57, exec.hpp:25-41) in an fce_problem
 * with v_offset / v_total set; H and targets are replicated.
 *
 * A communicator (fce_comm) has one of three transports:
 *   NCCL  (fce_comm_init)        one process per GPU, NCCL over NVLink /
 *                                NVSwitch — the production layout;
 *   ipc   (fce_comm_init_ipc)    one process per rank on one node, the
 *                                library's own collectives over CUDA IPC peer
 *                                memory (no NCCL);
 *   local (fce_comm_init_local)  k ranks inside ONE process, each driven by
 *                                its own host thread, on any devices (several
 *                                may share one GPU); the same peer-memory
 *                                kernels.
 * Every collective entry point must be called by all ranks of the
 * communicator (for the local transport: concurrently, one thread per rank).
 * All device work is stream-ordered on the handle's stream.
 */
#ifndef FCE_FCE_VP_H_
#define FCE_FCE_VP_H_

#include "fce.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fce_comm_s* fce_comm;
typedef struct fce_comm_group_s* fce_comm_group;

#define FCE_COMM_ID_BYTES 128

enum { FCE_TRANSPORT_NCCL = 1, FCE_TRANSPORT_LOCAL = 2, FCE_TRANSPORT_IPC = 3 };

/* NCCL transport: rank 0 creates the id and ships it to the others (e.g. a
 * torch.distributed broadcast); every rank then calls fce_comm_init. */
fce_status fce_comm_unique_id(uint8_t* out, size_t len);
fce_status fce_comm_init(fce_comm* out, int device, int nranks, int rank, const uint8_t* id,
                         size_t len);
/* IPC transport: one process per rank on one node, collectives by the
 * library's own kernels over CUDA IPC peer memory (NVLink P2P; no NCCL).  Rank
 * 0 makes the id (a rendezvous name, FCE_COMM_ID_BYTES), the caller ships it to
 * the other processes, every rank calls fce_comm_init_ipc; ranks may share a
 * GPU. */
fce_status fce_comm_ipc_id(uint8_t* out, size_t len);
fce_status fce_comm_init_ipc(fce_comm* out, int device, int nranks, int rank, const uint8_t* id,
                             size_t len);
/* Local transport: one group object shared by the k ranks of this process. */
fce_status fce_comm_group_create(fce_comm_group* out, int nranks);
fce_status fce_comm_group_destroy(fce_comm_group g); /* the group lives on until its last comm is destroyed */
fce_status fce_comm_init_local(fce_comm* out, fce_comm_group g, int device, int rank);
fce_status fce_comm_destroy(fce_comm c);
fce_status fce_comm_query(fce_comm c, int* nranks, int* rank, int* transport);
const char* fce_vp_last_error(void);
/* Bytes of device scratch the communicator holds (gather / pack buffers). */
fce_status fce_comm_scratch_bytes(fce_comm c, size_t* bytes);

/* Raw collectives on the handle's stream (fp32 sums are added in rank order
 * on the local transport). */
fce_status fce_comm_all_gather(fce_handle h, fce_comm c, const void* send, void* recv, size_t bytes_per_rank);
fce_status fce_comm_all_reduce_f32(fce_handle h, fce_comm c, const float* send, float* recv, size_t count);
fce_status fce_comm_reduce_scatter_f32(fce_handle h, fce_comm c, const float* send, float* recv,
                                       size_t recv_count);

/* tp_forward (parallel_sim.hpp:186-236): this rank's partial stats over its
 * shard, one all-gather of the packed (m, a, z_target, found) block — 13 B per
 * row per rank — and a rank-ordered merge on every rank, so every rank ends
 * with the same merged stats, lse and loss. */
fce_status fce_vp_forward(fce_handle h, fce_comm c, const fce_problem* p, int reduction,
                          fce_stats merged, float* lse, float* loss_rows, float* loss_reduced);

/* tp_backward (parallel_sim.hpp:246-290): local dW shard, dH summed over
 * ranks (every rank ends with the full dH).  Any lddh >= d (a strided dH is
 * reduced through a packed buffer). */
fce_status fce_vp_backward(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged,
                           int reduction, float upstream_scalar, const float* upstream_rows,
                           float* dhidden, int64_t lddh, float* dweight_shard, int64_t lddw);

/* sp_to_tp_gather (parallel_sim.hpp:294-314): rank r holds position shard r
 * of H (bf16 [shard_rows, ld_shard]; shards are consecutive in rank order,
 * e.g. the ceil-first partition_ranges(n_total, nranks)); every rank receives
 * the full H (bf16 [n_total, ld_full]) in position order.  Shards may be ragged; the
 * ranks exchange their (rows, d) first (one host sync): rows that do not add
 * up to n_total -> FCE_DIMENSION_MISMATCH, disagreeing widths ->
 * FCE_INVALID_LAYOUT (sp_to_tp_gather's "hidden shards disagree on width"). */
fce_status fce_sp_gather(fce_handle h, fce_comm c, const void* shard, int64_t shard_rows, int64_t ld_shard,
                         int64_t d, int64_t n_total, void* full, int64_t ld_full);

/* The sequence-parallel -> vocab-parallel forward as one call: rank r passes
 * its position shard of H (bf16 [shard_rows, ld_shard]) and a problem whose
 * `hidden` / `ldh` name a caller-owned full-size buffer (bf16 [n, ldh]) that
 * receives the gathered H (the backward needs it); weight / v_offset / v_total
 * / targets as fce_vp_forward.  The other ranks' rows are all-gathered on the
 * communicator's stream while K1 runs over this rank's own rows, then K1 runs
 * over the rest and the stats merge as in fce_vp_forward. */
fce_status fce_sp_vp_forward(fce_handle h, fce_comm c, const fce_problem* p, const void* shard, int64_t shard_rows,
                             int64_t ld_shard, int reduction, fce_stats merged, float* lse, float* loss_rows,
                             float* loss_reduced);

/* The backward's inverse of fce_sp_gather: every rank holds a full-length dH
 * partial (fp32 [n_total, lddh], e.g. its vocab shard's contribution); rank r
 * receives the sum over ranks of rows of its position shard (a reduce-scatter
 * in place of fce_vp_backward's all-reduce when the caller is sequence
 * parallel). */
fce_status fce_sp_scatter(fce_handle h, fce_comm c, const float* dh_partial, int64_t n_total, int64_t lddh,
                          int64_t d, float* dh_shard, int64_t shard_rows, int64_t ld_shard);

/* tp_backward followed by the sequence-parallel reduce-scatter of dH, as one
 * call: rank r receives the summed dH rows of its position shard (fp32
 * [shard_rows, ld_shard]; shards consecutive in rank order) and its local dW
 * shard.  With a peer-memory transport (local, ipc) and no ignore_index the
 * reduction happens inside the backward kernel: every dH tile is
 * TMA-reduce-added into the accumulator of the rank owning its rows while the
 * kernel runs (no separate reduce-scatter pass; sums across ranks in arrival
 * order).  Otherwise: local dH, then fce_sp_scatter. */
fce_status fce_sp_vp_backward(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged, int reduction,
                              float upstream_scalar, const float* upstream_rows, float* dh_shard, int64_t shard_rows,
                              int64_t ld_shard, float* dweight_shard, int64_t lddw);

/* dp_step (parallel_sim.hpp:334-378): every rank runs the fused forward and
 * backward on its micro-batch (p), then loss and dW are averaged over the
 * ranks (all-reduce / nranks); dH stays rank-local (may be NULL).  Micro-
 * batches must have equal sizes (FCE_INVALID_LAYOUT), and reduction must be
 * mean or sum (FCE_UNSUPPORTED_REDUCTION).  loss: one device float. */
fce_status fce_dp_step(fce_handle h, fce_comm c, const fce_problem* p, int reduction, float* loss,
                       float* dhidden, int64_t lddh, float* dweight, int64_t lddw);

#ifdef __cplusplus
}
#endif

#endif /* FCE_FCE_VP_H_ */
