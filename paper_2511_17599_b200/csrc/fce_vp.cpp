// Multi-rank entry points (include/fce/fce_vp.h) over the communicator
// interface of fce_comm.h (NCCL or the in-process local transport).
//
// Replaces the in-process simulation of the reference
// (proj/include/fusedce/parallel_sim.hpp:158-378) with real ranks:
//   fce_vp_forward  : fce_forward_partial on the local W shard (v_offset set),
//                     one all-gather of the packed per-row (m, a, z_t, found)
//                     block (13 B per row per rank) and a rank-ordered merge on
//                     every rank (tp_forward, parallel_sim.hpp:186-236).
//   fce_vp_backward : fce_backward on the shard with the merged stats; dW stays
//                     local (parallel_sim.hpp:240-244), dH partials summed with
//                     one all-reduce (parallel_sim.hpp:276-288).
//   fce_sp_gather / fce_sp_scatter : the sequence-parallel <-> vocab-parallel
//                     switch (sp_to_tp_gather, parallel_sim.hpp:294-314) as an
//                     all-gather of H shards and a reduce-scatter of dH.
//   fce_dp_step     : dp_step (parallel_sim.hpp:334-378): local fused step,
//                     all-reduce of loss and dW, scaled by 1 / nranks.
#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <vector>

#include "../../include/fce/fce.h"
#include "../../include/fce/fce_vp.h"
#include "fce_comm.h"
#include "fce_internal.h"

struct fce_comm_s {
    fce::Comm* impl = nullptr;
    void* buf = nullptr;       // grow-only scratch (pack / gather buffers)
    size_t buf_size = 0;
    int64_t* xchg = nullptr;   // small exchange area: [8] send + [8 * nranks] recv
    int64_t* xchg_host = nullptr;
    // overlapped backward: the collectives' stream and its two fences
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t reset_ev = nullptr, done_ev = nullptr;
};

struct fce_comm_group_s {
    fce::LocalGroup* g = nullptr;
};

namespace {

fce_status vp_fail(fce_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    fce::set_last_error(buf);
    return s;
}

#define VP_CUDA(call)                                                                             \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return vp_fail(FCE_CUDA_ERROR, "%s failed: %s", #call, cudaGetErrorString(e_));       \
    } while (0)

size_t round_up(size_t a, size_t b) { return (a + b - 1) / b * b; }

// Grow-only scratch of the communicator.  Peers of the local transport read
// this rank's buffers only inside a collective, which ends with this stream
// waiting for their reads, so a stream sync makes the old buffer free.
fce_status scratch(fce_comm c, size_t bytes, cudaStream_t s, char** out) {
    if (bytes > c->buf_size) {
        if (c->buf) {
            VP_CUDA(cudaStreamSynchronize(s));
            cudaFree(c->buf);
            c->buf = nullptr;
            c->buf_size = 0;
        }
        VP_CUDA(cudaMalloc(&c->buf, bytes));
        c->buf_size = bytes;
    }
    *out = static_cast<char*>(c->buf);
    return FCE_OK;
}

constexpr int kXchg = 8;  // int64 values per rank in exchange()

fce_status finish_comm_init(fce_comm c) {
    const size_t bytes = sizeof(int64_t) * kXchg * (1 + static_cast<size_t>(c->impl->nranks));
    VP_CUDA(cudaMalloc(&c->xchg, bytes));
    VP_CUDA(cudaMallocHost(&c->xchg_host, bytes));
    return FCE_OK;
}

// All-gather of up to kXchg int64 per rank through the device (host sync):
// out[r * 4 + i] = rank r's vals[i] for i < 4, and (8-value calls)
// out[4 * k + r * 4 + i - 4] for i >= 4 — callers index with xval().
fce_status exchange(fce_comm c, cudaStream_t s, const int64_t* vals, int cnt, std::vector<int64_t>* out) {
    const int k = c->impl->nranks;
    int64_t* host = c->xchg_host;
    for (int i = 0; i < kXchg; ++i) host[i] = i < cnt ? vals[i] : 0;
    VP_CUDA(cudaMemcpyAsync(c->xchg, host, kXchg * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    fce_status st = c->impl->all_gather(c->xchg, c->xchg + kXchg, kXchg * sizeof(int64_t), s);
    if (st) return st;
    VP_CUDA(cudaMemcpyAsync(host + kXchg, c->xchg + kXchg, kXchg * sizeof(int64_t) * k, cudaMemcpyDeviceToHost, s));
    VP_CUDA(cudaStreamSynchronize(s));
    // keep the 4-per-rank layout the callers index (r * 4 + i), then the upper halves
    out->assign(static_cast<size_t>(kXchg) * k, 0);
    for (int q = 0; q < k; ++q)
        for (int i = 0; i < kXchg; ++i)
            (*out)[i < 4 ? q * 4 + i : 4 * k + q * 4 + (i - 4)] = host[kXchg + q * kXchg + i];
    return FCE_OK;
}

int64_t xval(const std::vector<int64_t>& all, int k, int q, int i) {
    return i < 4 ? all[q * 4 + i] : all[4 * k + q * 4 + (i - 4)];
}

fce_status check_args(fce_handle h, fce_comm c) {
    if (!h || !c || !c->impl) return vp_fail(FCE_INVALID_ARGUMENT, "null handle or communicator");
    return FCE_OK;
}

// With validation on, the ranks agree on (N, d, V_total, ignore sentinel)
// before any size-dependent collective: a mismatch is an error on every rank
// instead of a hang in the collective.
// (the backward modes — in-kernel peer reduction, overlapped chunks — decide
// which collectives run, so they must agree too).
fce_status check_same_problem(fce_handle h, fce_comm c, const fce_problem* p) {
    if (!fce::handle_validate(h) || c->impl->nranks == 1) return FCE_OK;
    std::vector<int64_t> all;
    const int64_t vt = p->v_total ? p->v_total : p->v;
    const int64_t mine[6] = {p->n, p->d, vt, p->has_ignore ? p->ignore_index : INT64_MIN,
                             fce::handle_vp_fused_dh(h), fce::handle_vp_overlap_chunks(h)};
    fce_status s = exchange(c, fce::handle_stream(h), mine, 6, &all);
    if (s) return s;
    const int k = c->impl->nranks;
    for (int q = 0; q < k; ++q)
        for (int i = 0; i < 6; ++i)
            if (xval(all, k, q, i) != mine[i])
                return vp_fail(i < 4 ? FCE_DIMENSION_MISMATCH : FCE_INVALID_ARGUMENT,
                               "ranks disagree on the problem / mode (N, d, V_total, ignore, vp_fused_dh, "
                               "vp_overlap_chunks): rank %d has %lld where this rank has %lld (field %d)",
                               q, (long long)xval(all, k, q, i), (long long)mine[i], i);
    return FCE_OK;
}

// dst[rows, ld_dst] (+ tight copy) of a row-major block of `row_bytes` per row.
fce_status copy_rows(void* dst, size_t ld_dst_bytes, const void* src, size_t ld_src_bytes, size_t row_bytes,
                     size_t rows, cudaStream_t s) {
    if (!rows || !row_bytes) return FCE_OK;
    VP_CUDA(cudaMemcpy2DAsync(dst, ld_dst_bytes, src, ld_src_bytes, row_bytes, rows, cudaMemcpyDeviceToDevice, s));
    return FCE_OK;
}

// tp_backward with the dH all-reduce overlapped with the kernel
// (parallel_sim.hpp:276-288 reduces dH after every rank's shard is done; here
// the rows are cut into `chunks` row chunks and chunk c's all-reduce runs on the
// communicator's stream while the persistent kernel computes chunk c + 1).
// The comm stream starts after the kernel's dependency counters are reset,
// then waits on the device counter that marks each chunk's dH rows final; the
// kernel leaves vp_reserve_sms SMs free so the collective's kernels run beside
// it.  The handle stream resumes after the last collective.
// The communicator's own (high-priority) stream for collectives that overlap
// the handle stream's kernels, with its two fences.
fce_status ensure_comm_stream(fce_handle h, fce_comm c) {
    VP_CUDA(cudaSetDevice(fce::handle_device(h)));
    if (!c->comm_stream) {
        int lo = 0, hi = 0;
        VP_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        VP_CUDA(cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi));
        VP_CUDA(cudaEventCreateWithFlags(&c->reset_ev, cudaEventDisableTiming));
        VP_CUDA(cudaEventCreateWithFlags(&c->done_ev, cudaEventDisableTiming));
    }
    return FCE_OK;
}

fce_status vp_backward_overlapped(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged, int reduction,
                                  float upstream_scalar, const float* upstream_rows, float* dhidden,
                                  float* dweight_shard, int64_t lddw, int64_t chunks) {
    cudaStream_t stream = fce::handle_stream(h);
    fce_status es = ensure_comm_stream(h, c);
    if (es) return es;
    // the comm stream follows everything already queued (inputs of the reduce)
    VP_CUDA(cudaEventRecord(c->done_ev, stream));
    VP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->done_ev, 0));
    std::vector<fce::DhChunkDone> done;
    const int64_t row_chunk = (p->n + chunks - 1) / chunks;
    fce_status s = fce::backward_for_overlap(h, p, merged, reduction, upstream_scalar, upstream_rows, dhidden, p->d,
                                             dweight_shard, lddw, row_chunk,
                                             static_cast<int>(fce::handle_vp_reserve_sms(h)), c->reset_ev, &done);
    if (s) return s;
    VP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->reset_ev, 0));
    unsigned long long* trace = fce::handle_comm_trace(h);
    for (size_t i = 0; i < done.size(); ++i) {
        const fce::DhChunkDone& d = done[i];
        VP_CUDA(fce::stream_wait_geq(c->comm_stream, d.counter, d.target));
        if (trace) VP_CUDA(fce::launch_stamp(c->comm_stream, trace + 2 * i));
        float* rows = dhidden + d.row0 * p->d;
        if ((s = c->impl->all_reduce_sum(rows, rows, static_cast<size_t>(d.rows) * p->d, c->comm_stream))) return s;
        if (trace) VP_CUDA(fce::launch_stamp(c->comm_stream, trace + 2 * i + 1));
    }
    VP_CUDA(cudaEventRecord(c->done_ev, c->comm_stream));
    VP_CUDA(cudaStreamWaitEvent(stream, c->done_ev, 0));
    return FCE_OK;
}

// dH reduced inside the backward over peer memory (local / ipc transports):
// every rank's dH tiles are TMA-reduce-added straight into the symmetric
// accumulator of the rank owning their 128-row block, while the kernel runs —
// the dH reduce-scatter costs no separate pass.  owner q holds the blocks
// [block0[q], block0[q + 1]).  Then each rank copies out the rows it needs:
// every owner's rows (tp_backward semantics: the full dH) or the rows of its own
// position shard [sp_lo, sp_hi) (sequence-parallel semantics).
fce_status vp_backward_fused(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged, int reduction,
                             float upstream_scalar, const float* upstream_rows, const int* block0, float* out,
                             int64_t ld_out, int64_t out_row0, int64_t out_rows, float* dweight_shard,
                             int64_t lddw) {
    const int k = c->impl->nranks, r = c->impl->rank;
    cudaStream_t stream = fce::handle_stream(h);
    const int64_t n = p->n, d = p->d;
    void* sym[fce::kMaxDhPeers];
    fce_status s = c->impl->sym_buffers(sizeof(float) * static_cast<size_t>(n) * d, stream, sym);
    if (s) return s;
    auto own_lo = [&](int q) { return std::min<int64_t>(n, int64_t(block0[q]) * 128); };
    // zero the rows this rank owns, then no rank's kernel starts before every
    // owner has zeroed
    if (own_lo(r + 1) > own_lo(r))
        VP_CUDA(cudaMemsetAsync(static_cast<float*>(sym[r]) + own_lo(r) * d, 0,
                                sizeof(float) * (own_lo(r + 1) - own_lo(r)) * d, stream));
    if ((s = c->impl->fence(stream))) return s;
    float* peers[fce::kMaxDhPeers];
    for (int q = 0; q < k; ++q) peers[q] = static_cast<float*>(sym[q]);
    if ((s = fce::backward_dh_peers(h, p, merged, reduction, upstream_scalar, upstream_rows, peers, k, block0,
                                    dweight_shard, lddw)))
        return s;
    // every rank's reduce-adds have landed
    if ((s = c->impl->fence(stream))) return s;
    for (int q = 0; q < k; ++q) {
        const int64_t lo = std::max(own_lo(q), out_row0), hi = std::min(own_lo(q + 1), out_row0 + out_rows);
        if (hi <= lo) continue;
        VP_CUDA(cudaMemcpy2DAsync(out + (lo - out_row0) * ld_out, sizeof(float) * ld_out, peers[q] + lo * d,
                                  sizeof(float) * d, sizeof(float) * d, hi - lo, cudaMemcpyDefault, stream));
    }
    // peers are done reading this rank's accumulator before it is reused
    return c->impl->fence(stream);
}

bool fused_dh_possible(fce_comm c, const fce_problem* p) {
    return c->impl->has_peer_memory() && c->impl->nranks <= fce::kMaxDhPeers && !p->has_ignore &&
           (p->d * 4) % 16 == 0;
}

}  // namespace

extern "C" {

const char* fce_vp_last_error(void) { return fce_last_error(); }

fce_status fce_comm_unique_id(uint8_t* out, size_t len) { return fce::nccl_unique_id(out, len); }

fce_status fce_comm_init(fce_comm* out, int device, int nranks, int rank, const uint8_t* id, size_t len) {
    if (!out) return vp_fail(FCE_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return vp_fail(FCE_INVALID_LAYOUT, "bad rank layout");
    fce::Comm* impl = nullptr;
    fce_status s = fce::make_nccl_comm(&impl, device, nranks, rank, id, len);
    if (s) return s;
    fce_comm c = new fce_comm_s();
    c->impl = impl;
    if ((s = finish_comm_init(c))) {
        fce_comm_destroy(c);
        return s;
    }
    *out = c;
    return FCE_OK;
}

fce_status fce_comm_ipc_id(uint8_t* out, size_t len) { return fce::ipc_unique_id(out, len); }

fce_status fce_comm_init_ipc(fce_comm* out, int device, int nranks, int rank, const uint8_t* id, size_t len) {
    if (!out) return vp_fail(FCE_INVALID_ARGUMENT, "null output");
    *out = nullptr;
    fce::Comm* impl = nullptr;
    fce_status s = fce::make_ipc_comm(&impl, device, nranks, rank, id, len);
    if (s) return s;
    fce_comm c = new fce_comm_s();
    c->impl = impl;
    if ((s = finish_comm_init(c))) {
        fce_comm_destroy(c);
        return s;
    }
    *out = c;
    return FCE_OK;
}

fce_status fce_comm_group_create(fce_comm_group* out, int nranks) {
    if (!out) return vp_fail(FCE_INVALID_ARGUMENT, "null output");
    fce::LocalGroup* g = nullptr;
    fce_status s = fce::make_local_group(&g, nranks);
    if (s) return s;
    *out = new fce_comm_group_s{g};
    return FCE_OK;
}

fce_status fce_comm_group_destroy(fce_comm_group g) {
    if (!g) return FCE_OK;
    fce::release_local_group(g->g);
    delete g;
    return FCE_OK;
}

fce_status fce_comm_init_local(fce_comm* out, fce_comm_group g, int device, int rank) {
    if (!out || !g) return vp_fail(FCE_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    fce::Comm* impl = nullptr;
    fce_status s = fce::make_local_comm(&impl, g->g, device, rank);
    if (s) return s;
    fce_comm c = new fce_comm_s();
    c->impl = impl;
    if ((s = finish_comm_init(c))) {
        fce_comm_destroy(c);
        return s;
    }
    *out = c;
    return FCE_OK;
}

fce_status fce_comm_destroy(fce_comm c) {
    if (!c) return FCE_OK;
    if (c->impl) cudaSetDevice(c->impl->device);
    if (c->buf) cudaFree(c->buf);
    if (c->xchg) cudaFree(c->xchg);
    if (c->xchg_host) cudaFreeHost(c->xchg_host);
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->reset_ev) cudaEventDestroy(c->reset_ev);
    if (c->done_ev) cudaEventDestroy(c->done_ev);
    delete c->impl;
    delete c;
    return FCE_OK;
}

fce_status fce_comm_query(fce_comm c, int* nranks, int* rank, int* transport) {
    if (!c || !c->impl) return vp_fail(FCE_INVALID_ARGUMENT, "null communicator");
    if (nranks) *nranks = c->impl->nranks;
    if (rank) *rank = c->impl->rank;
    if (transport) *transport = c->impl->transport();
    return FCE_OK;
}

fce_status fce_comm_scratch_bytes(fce_comm c, size_t* bytes) {
    if (!c || !bytes) return vp_fail(FCE_INVALID_ARGUMENT, "null argument");
    *bytes = c->buf_size;
    return FCE_OK;
}

fce_status fce_comm_all_gather(fce_handle h, fce_comm c, const void* send, void* recv, size_t bytes_per_rank) {
    fce_status s = check_args(h, c);
    if (s) return s;
    return c->impl->all_gather(send, recv, bytes_per_rank, fce::handle_stream(h));
}

fce_status fce_comm_all_reduce_f32(fce_handle h, fce_comm c, const float* send, float* recv, size_t count) {
    fce_status s = check_args(h, c);
    if (s) return s;
    return c->impl->all_reduce_sum(send, recv, count, fce::handle_stream(h));
}

fce_status fce_comm_reduce_scatter_f32(fce_handle h, fce_comm c, const float* send, float* recv,
                                       size_t recv_count) {
    fce_status s = check_args(h, c);
    if (s) return s;
    return c->impl->reduce_scatter_sum(send, recv, recv_count, fce::handle_stream(h));
}

fce_status fce_vp_forward(fce_handle h, fce_comm c, const fce_problem* p, int reduction, fce_stats merged,
                          float* lse, float* loss_rows, float* loss_reduced) {
    fce::NvtxRange nvtx_("fce_vp_forward");
    fce_status s = check_args(h, c);
    if (s) return s;
    if (!p) return vp_fail(FCE_INVALID_ARGUMENT, "null problem");
    if (p->n <= 0) return vp_fail(FCE_EMPTY_INPUT, "tp forward requires N > 0 and d > 0");
    if ((s = check_same_problem(h, c, p))) return s;
    const int k = c->impl->nranks;
    const int64_t n = p->n;
    cudaStream_t stream = fce::handle_stream(h);
    // per rank: [m (n f32) | a (n f32) | z_t (n f32) | found (n u8)], 256-byte aligned
    const size_t rank_bytes = round_up(13 * static_cast<size_t>(n), 256);
    char* buf = nullptr;
    if ((s = scratch(c, rank_bytes * (1 + static_cast<size_t>(k)), stream, &buf))) return s;
    float* lm = reinterpret_cast<float*>(buf);
    fce_stats part{lm, lm + n, lm + 2 * n, reinterpret_cast<uint8_t*>(buf + 12 * n)};
    if ((s = fce_forward_partial(h, p, part))) return s;
    char* g = buf + rank_bytes;
    if ((s = c->impl->all_gather(buf, g, rank_bytes, stream))) return s;
    const float* gm = reinterpret_cast<const float*>(g);
    return fce::merge_partials(h, k, n, static_cast<int64_t>(rank_bytes / 4), static_cast<int64_t>(rank_bytes), gm,
                               gm + n, gm + 2 * n, reinterpret_cast<const uint8_t*>(g + 12 * n), p->targets,
                               p->has_ignore, p->ignore_index, reduction, merged, lse, loss_rows, loss_reduced);
}

fce_status fce_vp_backward(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged, int reduction,
                           float upstream_scalar, const float* upstream_rows, float* dhidden, int64_t lddh,
                           float* dweight_shard, int64_t lddw) {
    fce::NvtxRange nvtx_("fce_vp_backward");
    fce_status s = check_args(h, c);
    if (s) return s;
    if (!p) return vp_fail(FCE_INVALID_ARGUMENT, "null problem");
    if (!dhidden)
        return fce_backward(h, p, merged, reduction, upstream_scalar, upstream_rows, nullptr, 0, dweight_shard,
                            lddw, 0);
    if ((s = check_same_problem(h, c, p))) return s;
    if (lddh < p->d) return vp_fail(FCE_DIMENSION_MISMATCH, "lddh < d");
    cudaStream_t stream = fce::handle_stream(h);
    if (fce::handle_vp_fused_dh(h) && fused_dh_possible(c, p)) {
        // owners: ceil-first partition of the 128-row blocks over the ranks
        const int k = c->impl->nranks;
        const int64_t nb = (p->n + 127) / 128;
        int block0[fce::kMaxDhPeers + 1];
        for (int q = 0; q <= k; ++q) block0[q] = static_cast<int>((nb / k) * q + std::min<int64_t>(q, nb % k));
        return vp_backward_fused(h, c, p, merged, reduction, upstream_scalar, upstream_rows, block0, dhidden, lddh,
                                 0, p->n, dweight_shard, lddw);
    }
    const int64_t chunks = fce::handle_vp_overlap_chunks(h);
    if (chunks > 1 && lddh == p->d && !p->has_ignore && p->n >= 256 * chunks)
        return vp_backward_overlapped(h, c, p, merged, reduction, upstream_scalar, upstream_rows, dhidden,
                                      dweight_shard, lddw, chunks);
    // a strided dH is reduced through a packed [n, d] buffer (one collective)
    float* dst = dhidden;
    if (lddh != p->d) {
        char* buf = nullptr;
        if ((s = scratch(c, sizeof(float) * static_cast<size_t>(p->n) * p->d, stream, &buf))) return s;
        dst = reinterpret_cast<float*>(buf);
    }
    if ((s = fce_backward(h, p, merged, reduction, upstream_scalar, upstream_rows, dst, p->d, dweight_shard, lddw,
                          0)))
        return s;
    if ((s = c->impl->all_reduce_sum(dst, dst, static_cast<size_t>(p->n) * p->d, stream))) return s;
    if (dst != dhidden)
        return copy_rows(dhidden, sizeof(float) * lddh, dst, sizeof(float) * p->d, sizeof(float) * p->d, p->n,
                         stream);
    return FCE_OK;
}

fce_status fce_sp_gather(fce_handle h, fce_comm c, const void* shard, int64_t shard_rows, int64_t ld_shard,
                         int64_t d, int64_t n_total, void* full, int64_t ld_full) {
    fce::NvtxRange nvtx_("fce_sp_gather");
    fce_status s = check_args(h, c);
    if (s) return s;
    if (d <= 0 || n_total <= 0) return vp_fail(FCE_EMPTY_INPUT, "sp gather requires d > 0 and N > 0");
    if (shard_rows < 0 || (shard_rows > 0 && (!shard || ld_shard < d)) || !full || ld_full < d)
        return vp_fail(FCE_INVALID_ARGUMENT, "bad shard / output buffers");
    const int k = c->impl->nranks;
    cudaStream_t stream = fce::handle_stream(h);
    std::vector<int64_t> all;
    const int64_t mine[2] = {shard_rows, d};
    if ((s = exchange(c, stream, mine, 2, &all))) return s;
    int64_t total = 0, rows_max = 0;
    for (int q = 0; q < k; ++q) {
        if (all[4 * q + 1] != d) return vp_fail(FCE_INVALID_LAYOUT, "hidden shards disagree on width");
        total += all[4 * q];
        rows_max = std::max(rows_max, all[4 * q]);
    }
    if (total != n_total)
        return vp_fail(FCE_DIMENSION_MISMATCH, "shard rows add up to %lld, not N = %lld", (long long)total,
                       (long long)n_total);
    const size_t row_b = sizeof(uint16_t) * d;
    const size_t blk = round_up(row_b * rows_max, 256);
    char* buf = nullptr;
    if ((s = scratch(c, blk * (1 + static_cast<size_t>(k)), stream, &buf))) return s;
    if ((s = copy_rows(buf, row_b, shard, sizeof(uint16_t) * ld_shard, row_b, shard_rows, stream))) return s;
    if ((s = c->impl->all_gather(buf, buf + blk, blk, stream))) return s;
    int64_t at = 0;
    for (int q = 0; q < k; ++q) {
        if ((s = copy_rows(static_cast<char*>(full) + sizeof(uint16_t) * ld_full * at, sizeof(uint16_t) * ld_full,
                           buf + blk * (1 + q), row_b, row_b, all[4 * q], stream)))
            return s;
        at += all[4 * q];
    }
    return FCE_OK;
}

fce_status fce_sp_vp_forward(fce_handle h, fce_comm c, const fce_problem* p, const void* shard, int64_t shard_rows,
                             int64_t ld_shard, int reduction, fce_stats merged, float* lse, float* loss_rows,
                             float* loss_reduced) {
    fce::NvtxRange nvtx_("fce_sp_vp_forward");
    fce_status s = check_args(h, c);
    if (s) return s;
    if (!p || !p->hidden) return vp_fail(FCE_INVALID_ARGUMENT, "null problem or gather buffer");
    if (p->n <= 0 || p->d <= 0) return vp_fail(FCE_EMPTY_INPUT, "tp forward requires N > 0 and d > 0");
    if (shard_rows < 0 || (shard_rows > 0 && (!shard || ld_shard < p->d)))
        return vp_fail(FCE_INVALID_ARGUMENT, "bad hidden shard");
    const int k = c->impl->nranks, r = c->impl->rank;
    const int64_t n = p->n, d = p->d;
    cudaStream_t stream = fce::handle_stream(h);
    if ((s = ensure_comm_stream(h, c))) return s;
    // the ranks' position shards
    std::vector<int64_t> all;
    const int64_t mine[2] = {shard_rows, d};
    if ((s = exchange(c, stream, mine, 2, &all))) return s;
    std::vector<int64_t> start(k + 1, 0);
    int64_t rows_max = 0;
    for (int q = 0; q < k; ++q) {
        if (all[4 * q + 1] != d) return vp_fail(FCE_INVALID_LAYOUT, "hidden shards disagree on width");
        start[q + 1] = start[q] + all[4 * q];
        rows_max = std::max(rows_max, all[4 * q]);
    }
    if (start[k] != n)
        return vp_fail(FCE_DIMENSION_MISMATCH, "shard rows add up to %lld, not N = %lld", (long long)start[k],
                       (long long)n);
    const int64_t lo = start[r], hi = start[r + 1];
    // scratch: [packed partials: rank block + k-rank gather] [shard staging + k-rank gather of H shards]
    const size_t rank_bytes = round_up(13 * static_cast<size_t>(n), 256);
    const size_t row_b = sizeof(uint16_t) * d;
    const size_t blk = round_up(row_b * rows_max, 256);
    char* buf = nullptr;
    if ((s = scratch(c, rank_bytes * (1 + static_cast<size_t>(k)) + blk * (1 + static_cast<size_t>(k)), stream,
                     &buf)))
        return s;
    char* hbuf = buf + rank_bytes * (1 + static_cast<size_t>(k));
    char* full = static_cast<char*>(const_cast<void*>(p->hidden));
    const size_t ldf_b = sizeof(uint16_t) * p->ldh;
    // 1. this rank's rows into the full H (handle stream), then the other ranks'
    //    rows arrive on the communicator's stream while K1 runs on these
    if ((s = copy_rows(full + lo * ldf_b, ldf_b, shard, sizeof(uint16_t) * ld_shard, row_b, shard_rows, stream)))
        return s;
    VP_CUDA(cudaEventRecord(c->done_ev, stream));
    VP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->done_ev, 0));
    if ((s = copy_rows(hbuf, row_b, shard, sizeof(uint16_t) * ld_shard, row_b, shard_rows, c->comm_stream))) return s;
    if ((s = c->impl->all_gather(hbuf, hbuf + blk, blk, c->comm_stream))) return s;
    for (int q = 0; q < k; ++q) {
        if (q == r) continue;
        if ((s = copy_rows(full + start[q] * ldf_b, ldf_b, hbuf + blk * (1 + q), row_b, row_b, all[4 * q],
                           c->comm_stream)))
            return s;
    }
    VP_CUDA(cudaEventRecord(c->reset_ev, c->comm_stream));
    // 2. K1 over this rank's rows, then (after the gather) over the others
    float* lm = reinterpret_cast<float*>(buf);
    uint8_t* lf = reinterpret_cast<uint8_t*>(buf + 12 * n);
    auto partial = [&](int64_t r0, int64_t r1) -> fce_status {
        if (r1 <= r0) return FCE_OK;
        fce_problem q = *p;
        q.hidden = full + r0 * ldf_b;
        q.n = r1 - r0;
        q.targets = p->targets + r0;
        fce_stats part{lm + r0, lm + n + r0, lm + 2 * n + r0, lf + r0};
        return fce_forward_partial(h, &q, part);
    };
    if ((s = partial(lo, hi))) return s;
    VP_CUDA(cudaStreamWaitEvent(stream, c->reset_ev, 0));
    if ((s = partial(0, lo)) || (s = partial(hi, n))) return s;
    // 3. the packed partials of every rank, merged in rank order (as fce_vp_forward)
    char* g = buf + rank_bytes;
    if ((s = c->impl->all_gather(buf, g, rank_bytes, stream))) return s;
    const float* gm = reinterpret_cast<const float*>(g);
    return fce::merge_partials(h, k, n, static_cast<int64_t>(rank_bytes / 4), static_cast<int64_t>(rank_bytes), gm,
                               gm + n, gm + 2 * n, reinterpret_cast<const uint8_t*>(g + 12 * n), p->targets,
                               p->has_ignore, p->ignore_index, reduction, merged, lse, loss_rows, loss_reduced);
}

fce_status fce_sp_scatter(fce_handle h, fce_comm c, const float* dh_partial, int64_t n_total, int64_t lddh,
                          int64_t d, float* dh_shard, int64_t shard_rows, int64_t ld_shard) {
    fce::NvtxRange nvtx_("fce_sp_scatter");
    fce_status s = check_args(h, c);
    if (s) return s;
    if (d <= 0 || n_total <= 0) return vp_fail(FCE_EMPTY_INPUT, "sp scatter requires d > 0 and N > 0");
    if (!dh_partial || lddh < d || shard_rows < 0 || (shard_rows > 0 && (!dh_shard || ld_shard < d)))
        return vp_fail(FCE_INVALID_ARGUMENT, "bad dH / shard buffers");
    const int k = c->impl->nranks, r = c->impl->rank;
    cudaStream_t stream = fce::handle_stream(h);
    std::vector<int64_t> all;
    const int64_t mine[2] = {shard_rows, d};
    if ((s = exchange(c, stream, mine, 2, &all))) return s;
    int64_t total = 0, rows_max = 0;
    for (int q = 0; q < k; ++q) {
        if (all[4 * q + 1] != d) return vp_fail(FCE_INVALID_LAYOUT, "dH shards disagree on width");
        total += all[4 * q];
        rows_max = std::max(rows_max, all[4 * q]);
    }
    if (total != n_total)
        return vp_fail(FCE_DIMENSION_MISMATCH, "shard rows add up to %lld, not N = %lld", (long long)total,
                       (long long)n_total);
    // send: [k][rows_max][d] with block q = rows of rank q's shard (zero padded)
    const size_t row_b = sizeof(float) * d;
    const size_t blk_elems = round_up(static_cast<size_t>(rows_max) * d, 64);
    char* buf = nullptr;
    if ((s = scratch(c, sizeof(float) * blk_elems * (1 + static_cast<size_t>(k)), stream, &buf))) return s;
    float* send = reinterpret_cast<float*>(buf);
    float* recv = send + blk_elems * k;
    VP_CUDA(cudaMemsetAsync(send, 0, sizeof(float) * blk_elems * k, stream));
    int64_t at = 0;
    for (int q = 0; q < k; ++q) {
        if ((s = copy_rows(send + blk_elems * q, row_b, dh_partial + at * lddh, sizeof(float) * lddh, row_b,
                           all[4 * q], stream)))
            return s;
        at += all[4 * q];
    }
    if ((s = c->impl->reduce_scatter_sum(send, recv, blk_elems, stream))) return s;
    return copy_rows(dh_shard, sizeof(float) * ld_shard, recv, row_b, row_b, all[4 * r], stream);
}

fce_status fce_sp_vp_backward(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged, int reduction,
                              float upstream_scalar, const float* upstream_rows, float* dh_shard, int64_t shard_rows,
                              int64_t ld_shard, float* dweight_shard, int64_t lddw) {
    fce::NvtxRange nvtx_("fce_sp_vp_backward");
    fce_status s = check_args(h, c);
    if (s) return s;
    if (!p) return vp_fail(FCE_INVALID_ARGUMENT, "null problem");
    if (shard_rows < 0 || (shard_rows > 0 && (!dh_shard || ld_shard < p->d)))
        return vp_fail(FCE_INVALID_ARGUMENT, "bad dH shard buffer");
    const int k = c->impl->nranks, r = c->impl->rank;
    cudaStream_t stream = fce::handle_stream(h);
    // the ranks' position shards (consecutive in rank order)
    std::vector<int64_t> all;
    const int64_t mine[1] = {shard_rows};
    if ((s = exchange(c, stream, mine, 1, &all))) return s;
    int64_t total = 0, lo = 0;
    std::vector<int64_t> starts(k + 1, 0);
    for (int q = 0; q < k; ++q) {
        starts[q] = total;
        if (q == r) lo = total;
        total += all[4 * q];
    }
    starts[k] = total;
    if (total != p->n)
        return vp_fail(FCE_DIMENSION_MISMATCH, "shard rows add up to %lld, not N = %lld", (long long)total,
                       (long long)p->n);
    if (fused_dh_possible(c, p)) {
        // block b belongs to the rank whose shard holds its first row
        int block0[fce::kMaxDhPeers + 1];
        const int64_t nb = (p->n + 127) / 128;
        for (int q = 0; q < k; ++q) block0[q] = static_cast<int>(std::min<int64_t>(nb, (starts[q] + 127) / 128));
        block0[k] = static_cast<int>(nb);
        for (int q = k - 1; q >= 0; --q) block0[q] = std::min(block0[q], block0[q + 1]);
        return vp_backward_fused(h, c, p, merged, reduction, upstream_scalar, upstream_rows, block0, dh_shard,
                                 ld_shard, lo, shard_rows, dweight_shard, lddw);
    }
    // NCCL (or ignore_index): local dH of this shard's vocabulary, then a reduce-scatter
    char* buf = nullptr;
    const size_t dh_b = sizeof(float) * static_cast<size_t>(p->n) * p->d;
    VP_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&buf), dh_b, stream));
    s = fce_backward(h, p, merged, reduction, upstream_scalar, upstream_rows, reinterpret_cast<float*>(buf), p->d,
                     dweight_shard, lddw, 0);
    if (!s) s = fce_sp_scatter(h, c, reinterpret_cast<float*>(buf), p->n, p->d, p->d, dh_shard, shard_rows, ld_shard);
    cudaFreeAsync(buf, stream);
    return s;
}

fce_status fce_dp_step(fce_handle h, fce_comm c, const fce_problem* p, int reduction, float* loss, float* dhidden,
                       int64_t lddh, float* dweight, int64_t lddw) {
    fce::NvtxRange nvtx_("fce_dp_step");
    fce_status s = check_args(h, c);
    if (s) return s;
    if (!p || !loss || !dweight) return vp_fail(FCE_INVALID_ARGUMENT, "null problem, loss or dW");
    if (reduction == FCE_REDUCTION_NONE)
        return vp_fail(FCE_UNSUPPORTED_REDUCTION, "data-parallel loss sync requires a scalar reduction");
    if (reduction != FCE_REDUCTION_MEAN && reduction != FCE_REDUCTION_SUM)
        return vp_fail(FCE_UNSUPPORTED_REDUCTION, "unknown reduction %d", reduction);
    if (lddw < p->d) return vp_fail(FCE_DIMENSION_MISMATCH, "lddw < d");
    const int k = c->impl->nranks;
    cudaStream_t stream = fce::handle_stream(h);
    std::vector<int64_t> all;
    const int64_t mine[3] = {p->n, p->d, p->v};
    if ((s = exchange(c, stream, mine, 3, &all))) return s;
    for (int q = 0; q < k; ++q) {
        if (all[4 * q] != p->n) return vp_fail(FCE_INVALID_LAYOUT, "replica micro-batches must have equal sizes");
        if (all[4 * q + 1] != p->d || all[4 * q + 2] != p->v)
            return vp_fail(FCE_DIMENSION_MISMATCH, "replicas disagree on the weight shape");
    }
    const size_t n = static_cast<size_t>(std::max<int64_t>(p->n, 1));
    // scratch: stats (13 B / row) + lse + per-row loss, then (strided dW) a packed dW
    const size_t rows_off = round_up(17 * n, 16);
    const size_t st_b = round_up(rows_off + 4 * n, 256);
    const size_t dw_b = lddw != p->d ? sizeof(float) * static_cast<size_t>(p->v) * p->d : 0;
    char* buf = nullptr;
    if ((s = scratch(c, st_b + dw_b, stream, &buf))) return s;
    float* fm = reinterpret_cast<float*>(buf);
    fce_stats st{fm, fm + n, fm + 2 * n, reinterpret_cast<uint8_t*>(fm + 4 * n)};
    float* lse = fm + 3 * n;
    float* rows = reinterpret_cast<float*>(buf + rows_off);
    if ((s = fce_forward(h, p, reduction, 0, st, lse, rows, loss))) return s;
    float* dw = dw_b ? reinterpret_cast<float*>(buf + st_b) : dweight;
    if ((s = fce_backward(h, p, st, reduction, 1.0f, nullptr, dhidden, lddh, dw, p->d, 0))) return s;
    // loss and dW: mean over replicas (sum in rank order, then x 1 / nranks)
    const size_t dw_count = static_cast<size_t>(p->v) * p->d;
    if ((s = c->impl->all_reduce_sum(loss, loss, 1, stream))) return s;
    if ((s = c->impl->all_reduce_sum(dw, dw, dw_count, stream))) return s;
    const float inv = 1.0f / static_cast<float>(k);
    if ((s = fce_scale(h, loss, 1, inv))) return s;
    if ((s = fce_scale(h, dw, static_cast<int64_t>(dw_count), inv))) return s;
    if (dw != dweight)
        return copy_rows(dweight, sizeof(float) * lddw, dw, sizeof(float) * p->d, sizeof(float) * p->d, p->v, stream);
    return FCE_OK;
}

}  // extern "C"
