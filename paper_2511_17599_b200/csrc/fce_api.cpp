// C-ABI implementation (include/fce/fce.h): argument validation with the
// reference's error taxonomy, the per-handle device workspace + ledger, and
// the launch plans of the forward / backward passes.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fce/fce.h"
#include "fce_internal.h"

using namespace fce;

namespace {

thread_local std::string g_last_error;

fce_status fail(fce_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return s;
}

#define FCE_CUDA(call)                                                                          \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            return fail(FCE_CUDA_ERROR, "%s failed: %s", #call, cudaGetErrorString(e_));        \
    } while (0)

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

}  // namespace

struct fce_handle_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sms = 148;
    // scratch workspace (grow-only) + the persistent small block
    void* ws = nullptr;
    size_t ws_size = 0;
    size_t ws_peak = 0;
    size_t ws_in_use = 0;
    int* err = nullptr;                     // kErrSlots ints
    unsigned long long* count = nullptr;    // valid-target count
    int* host_err = nullptr;                // pinned mirror
    int64_t splits = 0, band_cols = 0, row_chunk = 0, validate = 1, bwd_persistent = 1;
    int64_t l2_hints = 1;
    int64_t gemm_pair = 1;
    int64_t fwd_m_group = 0;  // forward raster: row blocks per L2 group (0 = default)
    int64_t fwd_pair = 0;     // forward on CTA pairs (fce_fwd_pair.cu); measured slower under the power cap
    int64_t fwd_mc = 0;       // forward on 2-CTA clusters with W multicast
    int64_t bwd_unit_mask = 7;
    int64_t trace_ptr = 0;
    int64_t bwd_epi_warps = 4;  // measured: -1.5 to -2.4% backward, -0.8 to -1.6% step vs 8 (profiles/r02_epi_warps_ab.log)
    int64_t bwd_tma_epi = 3;
    int64_t dh_group = 1;     // bands per dH group in the persistent backward
    int64_t skip_ignored = 1; // compact away ignored rows before the tile kernels
    int64_t bwd_reserve_sms = 0;  // SMs the persistent backward leaves free (overlapped collectives)
    int64_t vp_overlap_chunks = 0;  // fce_vp_backward: row chunks whose dH all-reduce overlaps the kernel (0: off)
    int64_t vp_reserve_sms = 8;     // ... and the SMs the kernel leaves to the collectives
    int64_t comm_trace_ptr = 0;     // dev only: globaltimer stamps of the overlapped collectives
    int64_t vp_fused_dh = 0;        // fce_vp_backward: reduce dH inside the kernel over peer memory
    // last persistent backward launch: where each row chunk's dH completion is counted
    struct LastBwd {
        bool valid = false;
        const unsigned* counters = nullptr;
        int64_t row_chunk = 0, n_rc = 0, bands = 0, n_dh = 0;
    } last_bwd;
    cudaEvent_t ctr_reset_ev = nullptr;  // when set: recorded right after the counter reset
    // when k > 0: the next persistent backward reduces dH into these owners' accumulators
    struct DhPeers {
        int k = 0;
        float* ptr[kMaxDhPeers] = {};
        int block0[kMaxDhPeers + 1] = {};
    } dh_peers;
    // compaction buffers (grow-only, separate from ws so both can be live)
    void* cws = nullptr;
    size_t cws_size = 0;
    int64_t launches = 0;
    size_t bwd_scratch[2] = {0, 0};  // workspace offsets of the G ring and the dependency counters
    // optional per-kernel CUDA-event timing of the tile kernels (bench roofline)
    int64_t timing = 0;
    struct Pending {
        int mode;
        cudaEvent_t start, stop;
        double flops;                 // total, or per live row when `live` is set
        unsigned long long* live;     // pinned snapshot of the device live-row count (compacted problems)
    };
    std::vector<Pending> pending;
    std::vector<cudaEvent_t> event_pool;
    cudaEvent_t switch_ev = nullptr;           // orders a new stream after the old one (fce_set_stream)
    unsigned long long* live_host = nullptr;  // pinned slots for the live-row snapshots
    int live_used = 0;
    static constexpr int kLiveSlots = 1024;
    double k_ms[4] = {0, 0, 0, 0};
    double k_flops[4] = {0, 0, 0, 0};
    int64_t k_launches[4] = {0, 0, 0, 0};
};

namespace fce {
cudaStream_t handle_stream(fce_handle h) { return h ? h->stream : nullptr; }
int64_t handle_vp_overlap_chunks(fce_handle h) { return h ? h->vp_overlap_chunks : 0; }
int64_t handle_vp_reserve_sms(fce_handle h) { return h ? h->vp_reserve_sms : 0; }
int handle_device(fce_handle h) { return h ? h->device : 0; }
int64_t handle_vp_fused_dh(fce_handle h) { return h ? h->vp_fused_dh : 0; }
bool handle_validate(fce_handle h) { return h && h->validate != 0; }
unsigned long long* handle_comm_trace(fce_handle h) {
    return h ? reinterpret_cast<unsigned long long*>(h->comm_trace_ptr) : nullptr;
}
void set_last_error(const char* msg) { g_last_error = msg; }
}  // namespace fce

namespace {

struct Scratch {
    fce_handle h;
    void** buf;
    size_t* size;
    size_t off = 0;
    explicit Scratch(fce_handle hh) : h(hh), buf(&hh->ws), size(&hh->ws_size) {}
    Scratch(fce_handle hh, void** b, size_t* sz) : h(hh), buf(b), size(sz) {}
    // Carves 256-byte aligned pieces out of the handle workspace; call
    // commit() once the layout is known so the workspace grows in one go.
    size_t take(size_t bytes) {
        size_t o = (off + 255) & ~size_t(255);
        off = o + bytes;
        return o;
    }
    fce_status commit() {
        if (off > *size) {
            if (*buf) {
                cudaStreamSynchronize(h->stream);
                cudaFree(*buf);
                *buf = nullptr;
                *size = 0;
            }
            cudaError_t e = cudaMalloc(buf, off);
            if (e != cudaSuccess)
                return fail(FCE_CUDA_ERROR, "workspace allocation of %zu bytes failed: %s", off,
                            cudaGetErrorString(e));
            *size = off;
        }
        if (buf == &h->ws) h->ws_in_use = off;
        h->ws_peak = std::max(h->ws_peak, h->ws_size + h->cws_size + 64 + 3 * sizeof(int) * kErrSlots);
        return FCE_OK;
    }
    template <typename T>
    T* ptr(size_t o) const {
        return reinterpret_cast<T*>(static_cast<char*>(*buf) + o);
    }
};

fce_status check_handle(fce_handle h) {
    if (!h) return fail(FCE_INVALID_ARGUMENT, "null handle");
    cudaError_t e = cudaSetDevice(h->device);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "cudaSetDevice: %s", cudaGetErrorString(e));
    return FCE_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// validate_problem (dense_matrix.hpp:182-211) for what the host can see, plus
// the TMA layout contract of the device path.
fce_status check_problem(const fce_problem* p) {
    if (!p) return fail(FCE_INVALID_ARGUMENT, "null problem");
    if (p->n <= 0 || p->d <= 0 || p->v <= 0)
        return fail(FCE_EMPTY_INPUT, "problem requires N > 0, d > 0, V > 0 (got N=%lld, d=%lld, V=%lld)",
                    (long long)p->n, (long long)p->d, (long long)p->v);
    if (!p->hidden || !p->weight || !p->targets)
        return fail(FCE_INVALID_ARGUMENT, "null hidden / weight / targets pointer");
    if (p->ldh < p->d || p->ldw < p->d)
        return fail(FCE_DIMENSION_MISMATCH, "leading dimension smaller than d (ldh=%lld ldw=%lld d=%lld)",
                    (long long)p->ldh, (long long)p->ldw, (long long)p->d);
    if (p->ldh % 8 || p->ldw % 8 || !aligned16(p->hidden) || !aligned16(p->weight))
        return fail(FCE_INVALID_LAYOUT,
                    "bf16 operands need ld %% 8 == 0 and 16-byte aligned bases (TMA); ldh=%lld ldw=%lld",
                    (long long)p->ldh, (long long)p->ldw);
    if (p->v_offset < 0 || (p->v_total && p->v_offset + p->v > p->v_total))
        return fail(FCE_INVALID_LAYOUT, "vocab shard [%lld, %lld) outside [0, %lld)",
                    (long long)p->v_offset, (long long)(p->v_offset + p->v), (long long)p->v_total);
    if (p->n > INT32_MAX / 2 || p->v > INT32_MAX / 2 || p->d > (1 << 20))
        return fail(FCE_INVALID_LAYOUT, "problem too large for 32-bit tile indices");
    return FCE_OK;
}

fce_status read_errors(fce_handle h, bool sync) {
    if (!sync) return FCE_OK;
    FCE_CUDA(cudaMemcpyAsync(h->host_err, h->err, sizeof(int) * kErrSlots, cudaMemcpyDeviceToHost,
                             h->stream));
    FCE_CUDA(cudaStreamSynchronize(h->stream));
    if (h->host_err[kErrTargetRange])
        return fail(FCE_TARGET_OUT_OF_RANGE, "a non-ignored target lies outside [0, V)");
    if (h->host_err[kErrDuplicate])
        return fail(FCE_DUPLICATE_TARGET, "both stats claim the target logit");
    if (h->host_err[kErrNotFound])
        return fail(FCE_TARGET_OUT_OF_RANGE, "target of a position not covered by any shard");
    if (h->host_err[kErrMissingStats])
        return fail(FCE_MISSING_STATS, "a non-ignored position has no usable forward stats");
    if (h->host_err[kErrOffGrid])
        return fail(FCE_INVALID_LAYOUT, "input value is not on the bf16 grid");
    return FCE_OK;
}

fce_status reset_flags(fce_handle h) {
    FCE_CUDA(cudaMemsetAsync(h->err, 0, sizeof(int) * kErrSlots + 64, h->stream));
    return FCE_OK;
}

// Ignored-row compaction (the reference skips ignored positions outright,
// fused_forward.hpp:57-59, fused_backward.hpp:37-39): when the targets carry
// ignored rows, the valid rows are packed to the front of an N-row problem
// (row map by a one-block scan, gather of H rows and targets, zero padding)
// and the tile kernels skip everything past the live count, which they read
// from device memory.  No host sync: the count never leaves the GPU, so the
// path stays stream-ordered (and CUDA-graph capturable with validation off).
struct Compact {
    bool on = false;
    int* map = nullptr;        // [N] slot or -1
    int* rows = nullptr;       // [N] original row of each live slot
    int64_t* targets = nullptr;
    void* hidden = nullptr;    // [N, ldh] bf16, live rows first, zero padding
    int64_t ldh = 0;
    float* gamma = nullptr;    // backward: per-slot effective upstream / lse
    float* lse = nullptr;
    float* dh = nullptr;       // backward: [N, lddh] fp32
    int64_t lddh = 0;
};

fce_status plan_compaction(fce_handle h, const fce_problem* p, bool backward, bool want_dh, Compact* c,
                           fce_problem* pc) {
    *pc = *p;
    if (!p->has_ignore || !h->skip_ignored) return FCE_OK;
    const int64_t n = p->n;
    c->on = true;
    c->ldh = round_up(p->d, 8);
    c->lddh = round_up(p->d, 4);
    Scratch cs(h, &h->cws, &h->cws_size);
    const size_t o_map = cs.take(sizeof(int) * n);
    const size_t o_rows = cs.take(sizeof(int) * n);
    const size_t o_t = cs.take(sizeof(int64_t) * n);
    const size_t o_h = cs.take(sizeof(__nv_bfloat16) * n * c->ldh);
    size_t o_g = 0, o_l = 0, o_dh = 0;
    if (backward) {
        o_g = cs.take(sizeof(float) * n);
        o_l = cs.take(sizeof(float) * n);
        if (want_dh) o_dh = cs.take(sizeof(float) * n * c->lddh);
    }
    fce_status s = cs.commit();
    if (s) return s;
    c->map = cs.ptr<int>(o_map);
    c->rows = cs.ptr<int>(o_rows);
    c->targets = cs.ptr<int64_t>(o_t);
    c->hidden = cs.ptr<void>(o_h);
    if (backward) {
        c->gamma = cs.ptr<float>(o_g);
        c->lse = cs.ptr<float>(o_l);
        if (want_dh) c->dh = cs.ptr<float>(o_dh);
    }
    cudaError_t e = launch_row_map(p->targets, n, p->ignore_index, c->map, c->rows, h->stream);
    if (e == cudaSuccess)
        e = launch_gather_rows(p->hidden, p->ldh * 2, c->hidden, c->ldh * 2, p->d * 2, c->rows, n, h->count,
                               p->targets, c->targets, nullptr, nullptr, nullptr, nullptr, h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "compaction kernels: %s", cudaGetErrorString(e));
    h->launches += 3;
    pc->hidden = c->hidden;
    pc->ldh = c->ldh;
    pc->targets = c->targets;
    pc->has_ignore = 0;
    return FCE_OK;
}

// Forward split-V factor: units = m_blocks * splits spread over the SMs of a
// persistent grid; pick the factor with the best tile balance.
int choose_splits(int64_t m_blocks, int64_t v_tiles, int sms, int64_t requested) {
    if (requested > 0) return static_cast<int>(std::min<int64_t>(requested, v_tiles));
    int best = 1;
    double best_eff = -1.0;
    const int64_t max_s = std::min<int64_t>(v_tiles, 256);
    for (int64_t s = 1; s <= max_s; ++s) {
        const int64_t units = m_blocks * s;
        const int64_t per_cta = ceil_div(units, sms);
        const int64_t tiles_per_unit = ceil_div(v_tiles, s);
        const double eff = static_cast<double>(m_blocks * v_tiles) /
                           static_cast<double>(sms * per_cta * tiles_per_unit);
        // prefer fewer splits when efficiency is within noise (less merge work)
        if (eff > best_eff + 0.005) {
            best_eff = eff;
            best = static_cast<int>(s);
        }
    }
    return best;
}

cudaEvent_t pool_event(fce_handle h) {
    if (!h->event_pool.empty()) {
        cudaEvent_t e = h->event_pool.back();
        h->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void drain_timing(fce_handle h) {
    for (auto& q : h->pending) {
        cudaEventSynchronize(q.stop);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, q.start, q.stop);
        h->k_ms[q.mode] += ms;
        // compacted problems: algorithmic flops of the rows that were live
        h->k_flops[q.mode] += q.live ? q.flops * static_cast<double>(*q.live) : q.flops;
        h->k_launches[q.mode] += 1;
        h->event_pool.push_back(q.start);
        h->event_pool.push_back(q.stop);
    }
    h->pending.clear();
    h->live_used = 0;
}

// With timing on: events around the launch on the handle's stream and the
// algorithmic flop count.  For a compacted problem (n_valid set) the count is
// `flops_per_row` times the live-row count, which only the device knows: a
// pinned snapshot of it is queued right after the launch and read when the
// timing is drained.
struct TimedRegion {
    fce_handle h;
    cudaEvent_t e0 = nullptr;
    TimedRegion(fce_handle hh) : h(hh) {
        if (h->timing) {
            e0 = pool_event(h);
            cudaEventRecord(e0, h->stream);
        }
    }
    void done(int mode, double flops_total, double flops_per_row, const unsigned long long* n_valid) {
        if (!h->timing) return;
        cudaEvent_t e1 = pool_event(h);
        cudaEventRecord(e1, h->stream);
        unsigned long long* live = nullptr;
        if (n_valid) {
            if (!h->live_host && cudaMallocHost(&h->live_host, sizeof(unsigned long long) * h->kLiveSlots) != cudaSuccess)
                h->live_host = nullptr;
            if (h->live_host && h->live_used == h->kLiveSlots) drain_timing(h);
            if (h->live_host) {
                live = h->live_host + h->live_used++;
                cudaMemcpyAsync(live, n_valid, sizeof(unsigned long long), cudaMemcpyDeviceToHost, h->stream);
            }
        }
        h->pending.push_back({mode, e0, e1, live ? flops_per_row : flops_total, live});
    }
};

// Launches one tile kernel (timed when timing is on).
cudaError_t timed_launch(fce_handle h, const TileParams& p, const TensorMaps& maps, double flops,
                         int fwd_variant = 0, double flops_per_row = 0, const unsigned long long* n_valid = nullptr) {
    TimedRegion tr(h);
    cudaError_t e = fwd_variant == 1   ? launch_fwd_pair(p, maps, h->sms, h->stream)
                    : fwd_variant == 2 ? launch_fwd_mc(p, maps, h->sms, h->stream)
                                       : launch_tile_kernel(p, maps, h->sms, h->stream);
    tr.done(p.mode, flops, flops_per_row, n_valid);
    h->launches += 1;
    return e;
}

// Forward geometry: row blocks of 256 (CTA pairs) or 128 rows, and the
// split-V factor over the persistent grid (pairs count as one slot each).
struct FwdGeom {
    bool pair;
    bool mc;  // 2-CTA clusters with W multicast (cta_group::1 MMAs)
    int64_t m_blocks, v_tiles;
    int splits;
};

FwdGeom forward_geometry(fce_handle h, const fce_problem* p, int64_t window) {
    FwdGeom g;
    g.pair = h->fwd_pair != 0;
    g.mc = !g.pair && h->fwd_mc != 0;
    g.m_blocks = ceil_div(p->n, (g.pair || g.mc) ? 256 : kBM);
    g.v_tiles = ceil_div(p->v, kBN);
    g.splits = choose_splits(g.m_blocks, g.v_tiles, (g.pair || g.mc) ? h->sms / 2 : h->sms, h->splits);
    if (window > 0) g.splits = static_cast<int>(std::min<int64_t>(g.v_tiles, ceil_div(p->v, window)));
    return g;
}

fce_status run_forward_tiles(fce_handle h, const fce_problem* p, const FwdGeom& g, float* pm, float* pa,
                             float* pzt, uint8_t* pf, const unsigned long long* n_valid = nullptr) {
    fce::NvtxRange nvtx_("K1 forward tiles (tcgen05, online LSE)");
    TileParams tp;
    std::memset(&tp, 0, sizeof(tp));
    TensorMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    // pair: each CTA stages its 128 rows of H and its 128-row half of the W tile
    const uint32_t b_box = (g.pair || g.mc) ? 128 : kBN;
    if (!encode_map_2d(&maps.a0, p->hidden, p->d, p->n, p->ldh * 2, kBK, kBM) ||
        !encode_map_2d(&maps.b0, p->weight, p->d, p->v, p->ldw * 2, kBK, b_box))
        return fail(FCE_CUDA_ERROR, "cuTensorMapEncodeTiled failed for H / W");
    tp.mode = kEpiForward;
    tp.n_rows = static_cast<int>(p->n);
    tp.n_valid = n_valid;
    tp.v_cols = static_cast<int>(p->v);
    tp.m_blocks = static_cast<int>(g.m_blocks);
    tp.v_tiles = static_cast<int>(g.v_tiles);
    tp.splits = g.splits;
    tp.m_group = static_cast<int>(
        std::min<int64_t>(tp.m_blocks, h->fwd_m_group ? h->fwd_m_group : (g.pair ? 8 : g.mc ? 16 : 32)));
    tp.k_blocks = static_cast<int>(ceil_div(p->d, kBK));
    tp.units = tp.m_blocks * tp.splits;
    tp.targets = p->targets;
    tp.col_global0 = p->v_offset;
    tp.has_ignore = p->has_ignore;
    tp.ignore_index = p->ignore_index;
    tp.part_m = pm;
    tp.part_a = pa;
    tp.part_zt = pzt;
    tp.part_found = pf;
    cudaError_t e = timed_launch(h, tp, maps, 2.0 * p->n * p->d * p->v, g.pair ? 1 : g.mc ? 2 : 0,
                                 2.0 * p->d * p->v, n_valid);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "forward tile kernel: %s", cudaGetErrorString(e));
    return FCE_OK;
}

// Persistent backward: one launch of fce_bwd_persistent_kernel over every
// (row chunk x vocab band) chunk; see fce_bwd.cu for the schedule.
fce_status run_backward_persistent(fce_handle h, const fce_problem* p, const float* gamma,
                                   const float* lse, int64_t row_chunk, int64_t band, int kg,
                                   float* dhidden, int64_t lddh, float* dweight, int64_t lddw,
                                   int accumulate_dhidden, bool dw_bf16 = false,
                                   const unsigned long long* n_valid = nullptr) {
    fce::NvtxRange nvtx_("K2 persistent backward (S -> G -> dH, dW)");
    char* ws = static_cast<char*>(h->ws);
    __nv_bfloat16* g_ring = reinterpret_cast<__nv_bfloat16*>(ws + h->bwd_scratch[0]);
    unsigned* d_ctr = reinterpret_cast<unsigned*>(ws + h->bwd_scratch[1]);

    const int64_t n_rc = ceil_div(p->n, row_chunk), n_bd = ceil_div(p->v, band);
    const int64_t n_chunks = n_rc * n_bd;
    const int mb_max = static_cast<int>(row_chunk / 256);  // 256-row pair units
    const int d_tiles = static_cast<int>(ceil_div(p->d, kBN));
    BwdParams bp;
    std::memset(&bp, 0, sizeof(bp));
    bp.n_chunks = static_cast<int>(n_chunks);
    bp.bands = static_cast<int>(n_bd);
    bp.vt = static_cast<int>(band / kBN);
    bp.vm = static_cast<int>(band / 256);
    bp.n_g = mb_max * bp.vt;
    bp.n_dh = dhidden ? mb_max * d_tiles : 0;
    bp.n_dw = dweight ? bp.vm * d_tiles : 0;
    bp.kg = kg;
    bp.gpr = static_cast<int>(ceil_div(n_bd, kg));
    bp.per_gf = kg * (bp.n_g + bp.n_dw) + bp.n_dh;
    const int64_t per_rc = n_bd * (bp.n_g + bp.n_dw) + bp.gpr * bp.n_dh;
    const int64_t units = n_rc * per_rc;
    if (units >= INT32_MAX) return fail(FCE_INVALID_LAYOUT, "too many backward work units");
    bp.units = static_cast<int>(units);
    bp.per_rc = static_cast<int>(per_rc);
    bp.d_tiles = d_tiles;
    bp.k_blocks_d = static_cast<int>(ceil_div(p->d, kBK));
    bp.mb_max = mb_max;
    bp.gm_base = static_cast<int>(1 + 4 * n_chunks);
    bp.n = static_cast<int>(p->n);
    bp.v = static_cast<int>(p->v);
    bp.has_ignore = p->has_ignore;
    bp.accumulate_dh = accumulate_dhidden;
    bp.l2_hints = static_cast<int>(h->l2_hints);
    bp.unit_mask = static_cast<int>(h->bwd_unit_mask);
    bp.epi_warps = static_cast<int>(h->bwd_epi_warps);
    bp.dw_bf16 = dw_bf16 ? 1 : 0;
    bp.n_valid = n_valid;
    bp.trace = reinterpret_cast<unsigned long long*>(h->trace_ptr);
    bp.nc_max = row_chunk;
    bp.ldg = band;
    bp.ldr = band * kg;
    bp.d = p->d;
    bp.lddh = lddh;
    bp.lddw = lddw;
    bp.v_offset = p->v_offset;
    bp.ignore_index = p->ignore_index;
    bp.counters = d_ctr;
    bp.dh_peers = dhidden ? h->dh_peers.k : 0;
    for (int q = 0; q <= kMaxDhPeers; ++q) bp.peer_block0[q] = h->dh_peers.block0[q];
    bp.targets = p->targets;
    bp.lse = lse;
    bp.gamma = gamma;
    bp.g_ring = g_ring;
    bp.dh = dhidden;
    bp.dw = dweight;

    FCE_CUDA(cudaMemsetAsync(d_ctr, 0, sizeof(unsigned) * (1 + 4 * n_chunks + n_chunks * mb_max), h->stream));
    if (h->ctr_reset_ev) FCE_CUDA(cudaEventRecord(h->ctr_reset_ev, h->stream));
    h->last_bwd.valid = dhidden != nullptr;
    h->last_bwd.counters = d_ctr;
    h->last_bwd.row_chunk = row_chunk;
    h->last_bwd.n_rc = n_rc;
    h->last_bwd.bands = n_bd;
    h->last_bwd.n_dh = bp.n_dh;
    // ring rows past a short last row chunk (up to its 256-row unit edge) are
    // read by dW units and multiplied by zero-filled H rows: keep them finite
    const int64_t nc_last = p->n - (n_rc - 1) * row_chunk;
    const int64_t tail = std::min(round_up(nc_last, 256), row_chunk) - nc_last;
    if (tail > 0)
        for (int s2 = 0; s2 < 2; ++s2)
            FCE_CUDA(cudaMemsetAsync(g_ring + (s2 * row_chunk + nc_last) * bp.ldr, 0,
                                     sizeof(__nv_bfloat16) * tail * bp.ldr, h->stream));

    BwdMaps maps;
    std::memset(&maps, 0, sizeof(maps));
    const uint64_t ring_rows = static_cast<uint64_t>(2 * row_chunk);
    // pair units: every CTA loads 128 rows of K-major operands per stage
    if (!encode_map_2d(&maps.h_k, p->hidden, p->d, p->n, p->ldh * 2, kBK, 128) ||
        !encode_map_2d(&maps.w_k, p->weight, p->d, p->v, p->ldw * 2, kBK, 128) ||
        !encode_map_2d(&maps.g_k, g_ring, bp.ldr, ring_rows, bp.ldr * 2, kBK, 128) ||
        !encode_map_2d(&maps.w_mn, p->weight, p->d, p->v, p->ldw * 2, 64, 64) ||
        !encode_map_2d(&maps.g_mn, g_ring, bp.ldr, ring_rows, bp.ldr * 2, 64, 64) ||
        !encode_map_2d(&maps.h_mn, p->hidden, p->d, p->n, p->ldh * 2, 64, 64))
        return fail(FCE_CUDA_ERROR, "cuTensorMapEncodeTiled failed (persistent backward)");

    // epilogue through SMEM + TMA store / reduce-add when the outputs allow
    // TMA (16-byte aligned rows); otherwise per-thread vector stores
    bp.tma_epi = 0;
    if (h->bwd_tma_epi) {
        bool ok = encode_map_2d(&maps.g_st, g_ring, bp.ldr, ring_rows, bp.ldr * 2, 64, 128);
        if (ok && dhidden) ok = encode_map_2d(&maps.dh_st, dhidden, p->d, p->n, lddh * 4, 32, 128, true);
        if (ok && dweight)
            ok = dw_bf16 ? encode_map_2d(&maps.dw_st, dweight, p->d, p->v, lddw * 2, 64, 128)
                         : encode_map_2d(&maps.dw_st, dweight, p->d, p->v, lddw * 4, 32, 128, true);
        bp.tma_epi = ok ? static_cast<int>(h->bwd_tma_epi & 3) : 0;
    }
    if (dw_bf16 && !(bp.tma_epi & 2))
        return fail(FCE_CUDA_ERROR, "bf16 dW needs the TMA epilogue (16-byte aligned rows)");
    if (bp.dh_peers > 0) {
        // every dH tile is reduce-added into its owner rank's accumulator
        bool ok = (bp.tma_epi & 2) != 0;
        for (int q = 0; ok && q < bp.dh_peers; ++q)
            ok = encode_map_2d(&maps.dh_peer[q], h->dh_peers.ptr[q], p->d, p->n, lddh * 4, 32, 128, true);
        if (!ok) return fail(FCE_CUDA_ERROR, "peer dH reduction needs the TMA epilogue and aligned accumulators");
        bp.accumulate_dh = 1;
    }
    TimedRegion tr(h);
    const int grid = static_cast<int>(std::max<int64_t>(2, h->sms - h->bwd_reserve_sms));
    cudaError_t e = launch_bwd_persistent(bp, maps, grid, h->stream);
    const double per_row = 2.0 * p->d * p->v * (1 + (dhidden ? 1 : 0) + (dweight ? 1 : 0));
    tr.done(3, per_row * p->n, per_row, n_valid);
    h->launches += 1;
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "persistent backward kernel: %s", cudaGetErrorString(e));
    return FCE_OK;
}

}  // namespace

extern "C" {

const char* fce_last_error(void) { return g_last_error.c_str(); }

const char* fce_status_string(fce_status s) {
    switch (s) {
        case FCE_OK: return "ok";
        case FCE_DIMENSION_MISMATCH: return "DimensionMismatch";
        case FCE_TARGET_OUT_OF_RANGE: return "TargetOutOfRange";
        case FCE_UNDERFLOW_RELEASE: return "UnderflowRelease";
        case FCE_DUPLICATE_TARGET: return "DuplicateTarget";
        case FCE_MISSING_STATS: return "MissingStats";
        case FCE_INCONSISTENT_UPSTREAM: return "InconsistentUpstream";
        case FCE_UNSUPPORTED_REDUCTION: return "UnsupportedReduction";
        case FCE_INVALID_LAYOUT: return "InvalidLayout";
        case FCE_EMPTY_GRID: return "EmptyGrid";
        case FCE_EMPTY_INPUT: return "EmptyInput";
        case FCE_CUDA_ERROR: return "CudaError";
        case FCE_NCCL_ERROR: return "NcclError";
        case FCE_INVALID_ARGUMENT: return "InvalidArgument";
    }
    return "unknown";
}

fce_status fce_create(fce_handle* out, int device, void* stream) {
    if (!out) return fail(FCE_INVALID_ARGUMENT, "null output handle");
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(FCE_CUDA_ERROR, "no CUDA device available (%s); the fused LCE operator has no CPU path",
                    cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(FCE_INVALID_ARGUMENT, "device %d out of range", device);
    FCE_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    FCE_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(FCE_CUDA_ERROR, "device %d is sm_%d%d; this library is built for sm_100a only",
                    device, prop.major, prop.minor);
    fce_handle h = new fce_handle_s();
    h->device = device;
    h->stream = static_cast<cudaStream_t>(stream);
    h->sms = prop.multiProcessorCount;
    e = cudaMalloc(&h->err, sizeof(int) * kErrSlots + 64);
    if (e != cudaSuccess) {
        delete h;
        return fail(FCE_CUDA_ERROR, "cudaMalloc: %s", cudaGetErrorString(e));
    }
    h->count = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(h->err) +
                                                     sizeof(int) * kErrSlots);
    e = cudaMallocHost(&h->host_err, sizeof(int) * kErrSlots + 64);
    if (e != cudaSuccess) {
        cudaFree(h->err);
        delete h;
        return fail(FCE_CUDA_ERROR, "cudaMallocHost: %s", cudaGetErrorString(e));
    }
    *out = h;
    return FCE_OK;
}

fce_status fce_destroy(fce_handle h) {
    if (!h) return FCE_OK;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->stream);
    drain_timing(h);
    for (cudaEvent_t e : h->event_pool) cudaEventDestroy(e);
    if (h->live_host) cudaFreeHost(h->live_host);
    if (h->switch_ev) cudaEventDestroy(h->switch_ev);
    if (h->ws) cudaFree(h->ws);
    if (h->cws) cudaFree(h->cws);
    if (h->err) cudaFree(h->err);
    if (h->host_err) cudaFreeHost(h->host_err);
    delete h;
    return FCE_OK;
}

fce_status fce_set_stream(fce_handle h, void* stream) {
    if (!h) return fail(FCE_INVALID_ARGUMENT, "null handle");
    cudaStream_t ns = static_cast<cudaStream_t>(stream);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (ns != h->stream) FCE_CUDA(cudaStreamIsCapturing(ns, &cap));
    if (ns != h->stream && cap == cudaStreamCaptureStatusNone) {
        // Work already queued on the old stream may still read or write the
        // handle's workspaces and flag block: the new stream starts after it.
        // (A stream under graph capture cannot wait on outside work; ordering
        // a graph's launches is the caller's, as for any captured work.)
        FCE_CUDA(cudaSetDevice(h->device));
        if (!h->switch_ev) FCE_CUDA(cudaEventCreateWithFlags(&h->switch_ev, cudaEventDisableTiming));
        FCE_CUDA(cudaEventRecord(h->switch_ev, h->stream));
        FCE_CUDA(cudaStreamWaitEvent(ns, h->switch_ev, 0));
    }
    h->stream = ns;
    return FCE_OK;
}

fce_status fce_set_option(fce_handle h, const char* key, int64_t value) {
    if (!h || !key) return fail(FCE_INVALID_ARGUMENT, "null handle or key");
    if (value < 0) return fail(FCE_INVALID_ARGUMENT, "option %s must be >= 0", key);
    if (!std::strcmp(key, "splits")) {
        h->splits = value;
    } else if (!std::strcmp(key, "band_cols")) {
        if (value % kBN) return fail(FCE_INVALID_LAYOUT, "band_cols must be a multiple of %d", kBN);
        h->band_cols = value;
    } else if (!std::strcmp(key, "row_chunk")) {
        if (value % kBM) return fail(FCE_INVALID_LAYOUT, "row_chunk must be a multiple of %d", kBM);
        h->row_chunk = value;
    } else if (!std::strcmp(key, "validate")) {
        h->validate = value ? 1 : 0;
    } else if (!std::strcmp(key, "bwd_tma_epi")) {
        // 0: per-thread stores, 1: G via TMA, 2: dH / dW via TMA, 3: both
        h->bwd_tma_epi = value > 3 ? 3 : value;
    } else if (!std::strcmp(key, "bwd_epi_warps")) {
        if (value != 4 && value != 8) return fail(FCE_INVALID_ARGUMENT, "bwd_epi_warps must be 4 or 8");
        h->bwd_epi_warps = value;
    } else if (!std::strcmp(key, "trace_ptr")) {
        h->trace_ptr = value;
    } else if (!std::strcmp(key, "bwd_unit_mask")) {
        h->bwd_unit_mask = value & 255;
    } else if (!std::strcmp(key, "dh_group")) {
        if (value < 1 || value > 64) return fail(FCE_INVALID_ARGUMENT, "dh_group must be in [1, 64]");
        h->dh_group = value;
    } else if (!std::strcmp(key, "bwd_reserve_sms")) {
        if (value > h->sms - 2) return fail(FCE_INVALID_ARGUMENT, "bwd_reserve_sms must leave at least one CTA pair");
        h->bwd_reserve_sms = value;
    } else if (!std::strcmp(key, "vp_overlap_chunks")) {
        if (value == 1 || value > 64) return fail(FCE_INVALID_ARGUMENT, "vp_overlap_chunks must be 0 or in [2, 64]");
        h->vp_overlap_chunks = value;
    } else if (!std::strcmp(key, "vp_fused_dh")) {
        h->vp_fused_dh = value ? 1 : 0;
    } else if (!std::strcmp(key, "comm_trace_ptr")) {
        h->comm_trace_ptr = value;
    } else if (!std::strcmp(key, "vp_reserve_sms")) {
        if (value > h->sms - 2) return fail(FCE_INVALID_ARGUMENT, "vp_reserve_sms must leave at least one CTA pair");
        h->vp_reserve_sms = value;
    } else if (!std::strcmp(key, "skip_ignored")) {
        h->skip_ignored = value ? 1 : 0;
    } else if (!std::strcmp(key, "fwd_m_group")) {
        h->fwd_m_group = value;
    } else if (!std::strcmp(key, "fwd_mc")) {
        h->fwd_mc = value ? 1 : 0;
    } else if (!std::strcmp(key, "fwd_pair")) {
        h->fwd_pair = value ? 1 : 0;
    } else if (!std::strcmp(key, "gemm_pair")) {
        h->gemm_pair = value ? 1 : 0;
    } else if (!std::strcmp(key, "l2_hints")) {
        h->l2_hints = value;
    } else if (!std::strcmp(key, "bwd_persistent")) {
        h->bwd_persistent = value ? 1 : 0;
    } else if (!std::strcmp(key, "timing")) {
        drain_timing(h);
        for (int i = 0; i < 4; ++i) h->k_ms[i] = h->k_flops[i] = 0, h->k_launches[i] = 0;
        h->timing = value ? 1 : 0;
    } else {
        return fail(FCE_INVALID_ARGUMENT, "unknown option '%s'", key);
    }
    return FCE_OK;
}

fce_status fce_workspace_bytes(fce_handle h, size_t* current, size_t* peak) {
    if (!h) return fail(FCE_INVALID_ARGUMENT, "null handle");
    if (current) *current = h->ws_size + sizeof(int) * kErrSlots + 64;
    if (peak) *peak = h->ws_peak;
    return FCE_OK;
}

fce_status fce_kernel_stats(fce_handle h, int kernel, double* total_ms, int64_t* launches,
                            double* flops) {
    if (!h) return fail(FCE_INVALID_ARGUMENT, "null handle");
    if (kernel < 0 || kernel > 3) return fail(FCE_INVALID_ARGUMENT, "kernel id must be 0..3");
    drain_timing(h);
    if (total_ms) *total_ms = h->k_ms[kernel];
    if (launches) *launches = h->k_launches[kernel];
    if (flops) *flops = h->k_flops[kernel];
    return FCE_OK;
}

fce_status fce_launch_count(fce_handle h, int64_t* count) {
    if (!h || !count) return fail(FCE_INVALID_ARGUMENT, "null argument");
    *count = h->launches;
    return FCE_OK;
}

fce_status fce_forward(fce_handle h, const fce_problem* p, int reduction, int64_t window,
                       fce_stats stats, float* lse, float* loss_rows, float* loss_reduced) {
    fce::NvtxRange nvtx_("fce_forward");
    fce_status s = check_handle(h);
    if (s) return s;
    if ((s = check_problem(p))) return s;
    if (reduction < 0 || reduction > 2) return fail(FCE_UNSUPPORTED_REDUCTION, "unknown reduction %d", reduction);
    if (window < 0) return fail(FCE_INVALID_LAYOUT, "window size must be at least 1");
    const int64_t v_total = p->v_total ? p->v_total : p->v;
    if ((s = reset_flags(h))) return s;
    cudaError_t e = launch_prep_targets(p->targets, p->n, p->has_ignore, p->ignore_index, v_total,
                                        h->err, h->count, h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "prep kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    if ((s = read_errors(h, h->validate != 0))) return s;
    Compact cp;
    fce_problem pc;
    if ((s = plan_compaction(h, p, false, false, &cp, &pc))) return s;
    const int64_t nc = std::max<int64_t>(pc.n, 1);  // partial rows (>= 1 keeps pointers valid)

    const FwdGeom geom = forward_geometry(h, &pc, window);
    const int splits = std::max(geom.splits, 1);

    Scratch sc(h);
    const size_t o_m = sc.take(sizeof(float) * splits * nc);
    const size_t o_a = sc.take(sizeof(float) * splits * nc);
    const size_t o_z = sc.take(sizeof(float) * splits * nc);
    const size_t o_f = sc.take(splits * nc);
    const size_t o_b = sc.take(sizeof(double) * (ceil_div(p->n, 256) + 1));
    if ((s = sc.commit())) return s;

    if ((s = run_forward_tiles(h, &pc, geom, sc.ptr<float>(o_m), sc.ptr<float>(o_a), sc.ptr<float>(o_z),
                               sc.ptr<uint8_t>(o_f), cp.on ? h->count : nullptr)))
        return s;
    int blocks = 0;
    e = launch_merge_stats(splits, p->n, nc, sc.ptr<float>(o_m), sc.ptr<float>(o_a),
                           sc.ptr<float>(o_z), sc.ptr<uint8_t>(o_f), p->targets, p->has_ignore,
                           p->ignore_index, 1, stats.m, stats.a, stats.z_target, stats.found, lse,
                           loss_rows, sc.ptr<double>(o_b), h->err, h->stream, &blocks,
                           cp.on ? cp.map : nullptr);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "merge kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    if (reduction != FCE_REDUCTION_NONE && loss_reduced) {
        e = launch_reduce_loss(sc.ptr<double>(o_b), blocks, h->count, reduction, loss_reduced, h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "reduce kernel: %s", cudaGetErrorString(e));
        h->launches += 1;
    }
    return FCE_OK;
}

fce_status fce_forward_partial(fce_handle h, const fce_problem* p, fce_stats partial) {
    fce::NvtxRange nvtx_("fce_forward_partial");
    fce_status s = check_handle(h);
    if (s) return s;
    if ((s = check_problem(p))) return s;
    const int64_t v_total = p->v_total ? p->v_total : p->v;
    if ((s = reset_flags(h))) return s;
    cudaError_t e = launch_prep_targets(p->targets, p->n, p->has_ignore, p->ignore_index, v_total,
                                        h->err, h->count, h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "prep kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    if ((s = read_errors(h, h->validate != 0))) return s;
    Compact cp;
    fce_problem pc;
    if ((s = plan_compaction(h, p, false, false, &cp, &pc))) return s;
    const int64_t nc = std::max<int64_t>(pc.n, 1);
    const FwdGeom geom = forward_geometry(h, &pc, 0);
    const int splits = std::max(geom.splits, 1);
    Scratch sc(h);
    const size_t o_m = sc.take(sizeof(float) * splits * nc);
    const size_t o_a = sc.take(sizeof(float) * splits * nc);
    const size_t o_z = sc.take(sizeof(float) * splits * nc);
    const size_t o_f = sc.take(splits * nc);
    if ((s = sc.commit())) return s;
    if ((s = run_forward_tiles(h, &pc, geom, sc.ptr<float>(o_m), sc.ptr<float>(o_a), sc.ptr<float>(o_z),
                               sc.ptr<uint8_t>(o_f), cp.on ? h->count : nullptr)))
        return s;
    e = launch_merge_stats(splits, p->n, nc, sc.ptr<float>(o_m), sc.ptr<float>(o_a),
                           sc.ptr<float>(o_z), sc.ptr<uint8_t>(o_f), p->targets, p->has_ignore,
                           p->ignore_index, 0, partial.m, partial.a, partial.z_target, partial.found,
                           nullptr, nullptr, nullptr, h->err, h->stream, nullptr,
                           cp.on ? cp.map : nullptr);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "merge kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    return FCE_OK;
}

fce_status fce_merge_partials(fce_handle h, int parts, int64_t n, int64_t part_stride,
                              const float* m, const float* a, const float* z_target,
                              const uint8_t* found, const int64_t* targets, int32_t has_ignore,
                              int64_t ignore_index, int reduction, fce_stats merged, float* lse,
                              float* loss_rows, float* loss_reduced) {
    return fce::merge_partials(h, parts, n, part_stride, part_stride, m, a, z_target, found, targets, has_ignore,
                               ignore_index, reduction, merged, lse, loss_rows, loss_reduced);
}

}  // extern "C"

namespace fce {

fce_status merge_partials(fce_handle h, int parts, int64_t n, int64_t part_stride, int64_t found_stride,
                          const float* m, const float* a, const float* z_target, const uint8_t* found,
                          const int64_t* targets, int32_t has_ignore, int64_t ignore_index, int reduction,
                          fce_stats merged, float* lse, float* loss_rows, float* loss_reduced) {
    fce::NvtxRange nvtx_("fce_merge_partials");
    fce_status s = check_handle(h);
    if (s) return s;
    if (parts <= 0) return fail(FCE_INVALID_LAYOUT, "no partials to merge");
    if (n <= 0) return fail(FCE_EMPTY_INPUT, "merge requires N > 0");
    if (part_stride < n || found_stride < n) return fail(FCE_DIMENSION_MISMATCH, "part stride smaller than N");
    if (!m || !a || !z_target || !found || !targets) return fail(FCE_INVALID_ARGUMENT, "null partial");
    if (reduction < 0 || reduction > 2) return fail(FCE_UNSUPPORTED_REDUCTION, "unknown reduction %d", reduction);
    if ((s = reset_flags(h))) return s;
    // count of valid rows (targets already validated by the rank partials)
    cudaError_t e = launch_prep_targets(targets, n, has_ignore, ignore_index, INT64_MAX, h->err,
                                        h->count, h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "prep kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    Scratch sc(h);
    const size_t o_b = sc.take(sizeof(double) * (ceil_div(n, 256) + 1));
    if ((s = sc.commit())) return s;
    int blocks = 0;
    e = launch_merge_stats(parts, n, part_stride, m, a, z_target, found, targets, has_ignore,
                           ignore_index, 1, merged.m, merged.a, merged.z_target, merged.found, lse,
                           loss_rows, sc.ptr<double>(o_b), h->err, h->stream, &blocks, nullptr, found_stride);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "merge kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    if (reduction != FCE_REDUCTION_NONE && loss_reduced) {
        e = launch_reduce_loss(sc.ptr<double>(o_b), blocks, h->count, reduction, loss_reduced, h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "reduce kernel: %s", cudaGetErrorString(e));
        h->launches += 1;
    }
    return read_errors(h, h->validate != 0);
}

}  // namespace fce

extern "C" {

static fce_status run_backward_tiles(fce_handle h, const fce_problem* p, const float* gamma,
                                     const float* lse, int64_t row_chunk, int64_t band, __nv_bfloat16* G,
                                     float* dhidden, int64_t lddh, float* dweight, int64_t lddw,
                                     int accumulate_dhidden);

fce_status fce_backward(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                        float upstream_scalar, const float* upstream_rows, float* dhidden,
                        int64_t lddh, float* dweight, int64_t lddw, int accumulate_dhidden) {
    return fce_backward_ex(h, p, stats, reduction, upstream_scalar, upstream_rows, dhidden, lddh, FCE_DTYPE_F32,
                           dweight, lddw, FCE_DTYPE_F32, accumulate_dhidden);
}

static fce_status backward_impl(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                                float upstream_scalar, const float* upstream_dev, const float* upstream_rows,
                                void* dhidden_out, int64_t lddh, int dh_dtype, void* dweight_out, int64_t lddw,
                                int dw_dtype, int accumulate_dhidden);

fce_status fce_backward_ex(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                           float upstream_scalar, const float* upstream_rows, void* dhidden_out,
                           int64_t lddh, int dh_dtype, void* dweight_out, int64_t lddw, int dw_dtype,
                           int accumulate_dhidden) {
    return backward_impl(h, p, stats, reduction, upstream_scalar, nullptr, upstream_rows, dhidden_out, lddh,
                         dh_dtype, dweight_out, lddw, dw_dtype, accumulate_dhidden);
}

fce_status fce_backward_dev(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                            const float* upstream_scalar_dev, const float* upstream_rows, void* dhidden,
                            int64_t lddh, int dh_dtype, void* dweight, int64_t lddw, int dw_dtype,
                            int accumulate_dhidden) {
    if (reduction != FCE_REDUCTION_NONE && !upstream_scalar_dev)
        return fail(FCE_INCONSISTENT_UPSTREAM, "scalar reductions require the device upstream scalar");
    return backward_impl(h, p, stats, reduction, 0.f, upstream_scalar_dev, upstream_rows, dhidden, lddh, dh_dtype,
                         dweight, lddw, dw_dtype, accumulate_dhidden);
}

static fce_status backward_impl(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                                float upstream_scalar, const float* upstream_dev, const float* upstream_rows,
                                void* dhidden_out, int64_t lddh, int dh_dtype, void* dweight_out, int64_t lddw,
                                int dw_dtype, int accumulate_dhidden) {
    fce::NvtxRange nvtx_("fce_backward");
    fce_status s = check_handle(h);
    if (s) return s;
    if ((s = check_problem(p))) return s;
    if ((dh_dtype != FCE_DTYPE_F32 && dh_dtype != FCE_DTYPE_BF16) ||
        (dw_dtype != FCE_DTYPE_F32 && dw_dtype != FCE_DTYPE_BF16))
        return fail(FCE_INVALID_ARGUMENT, "gradient dtype must be FCE_DTYPE_F32 or FCE_DTYPE_BF16");
    if (dh_dtype == FCE_DTYPE_BF16 && accumulate_dhidden)
        return fail(FCE_INVALID_ARGUMENT, "accumulate_dhidden requires an fp32 dH");
    const bool dh_bf16 = dhidden_out && dh_dtype == FCE_DTYPE_BF16;
    const bool dw_bf16 = dweight_out && dw_dtype == FCE_DTYPE_BF16;
    // fp32 views; bf16 outputs are redirected below
    float* dhidden = dh_bf16 ? nullptr : static_cast<float*>(dhidden_out);
    float* dweight = dw_bf16 ? nullptr : static_cast<float*>(dweight_out);
    if (reduction < 0 || reduction > 2) return fail(FCE_UNSUPPORTED_REDUCTION, "unknown reduction %d", reduction);
    if (reduction == FCE_REDUCTION_NONE && !upstream_rows)
        return fail(FCE_INCONSISTENT_UPSTREAM, "reduction none requires a per-position upstream gradient");
    if (reduction != FCE_REDUCTION_NONE && upstream_rows)
        return fail(FCE_INCONSISTENT_UPSTREAM, "scalar reductions require a scalar upstream gradient");
    if (!stats.m || !stats.a || !stats.found)
        return fail(FCE_MISSING_STATS, "stats cache (m, a, found) is required");
    if (dhidden_out && lddh < p->d) return fail(FCE_DIMENSION_MISMATCH, "lddh < d");
    if (dweight_out && lddw < p->d) return fail(FCE_DIMENSION_MISMATCH, "lddw < d");
    const int64_t v_total = p->v_total ? p->v_total : p->v;

    if ((s = reset_flags(h))) return s;
    cudaError_t e = launch_prep_targets(p->targets, p->n, p->has_ignore, p->ignore_index, v_total,
                                        h->err, h->count, h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "prep kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    // ignored rows compacted away (their gradient rows are exactly zero)
    Compact cp;
    fce_problem pcv;
    if ((s = plan_compaction(h, p, true, dhidden_out != nullptr, &cp, &pcv))) return s;
    const fce_problem* pk = &pcv;  // the problem the tile kernels see
    const int64_t n_k = std::max<int64_t>(pk->n, 1);

    // chunking of G = N_c x V_c bf16
    // defaults measured best on B200 at the Llama-3-8B shape
    int64_t row_chunk = h->row_chunk;
    if (!row_chunk && h->bwd_persistent) {
        // As few row chunks as the G ring cap (1 GiB at kg = 1) allows, of equal
        // size: every extra row chunk is another fp32 read-modify-write pass
        // over dW (measured: Gemma-2-2B shape 213 -> 178 ms going from 4 chunks
        // of 16384 to 1-2 chunks; profiles/r01_energy.md).
        const int64_t band_guess = h->band_cols ? h->band_cols : 3072;
        const int64_t cap = std::max<int64_t>(256, ((int64_t(1) << 30) / (2 * 2 * band_guess)) / 256 * 256);
        row_chunk = ceil_div(n_k, ceil_div(n_k, cap));
    } else if (!row_chunk) {
        row_chunk = 16384;
    }
    row_chunk = std::min(row_chunk, round_up(n_k, h->bwd_persistent ? 256 : kBM));
    if (h->bwd_persistent) row_chunk = round_up(row_chunk, 256);
    int64_t band = h->band_cols;
    if (!band) {
        if (h->bwd_persistent) {
            // Base band by width (interleaved A/B on B200, profiles/r02_band_ab.log):
            // D <= 3072 (Gemma-2-2B) 4096; long row chunks at D >= 6144
            // (Llama-3-70B) 3072; otherwise (Llama-3-8B, Qwen2.5-7B) 3584.
            // Shorter row chunks take wider bands (fewer dH passes, more units
            // per phase): 3072 * sqrt(16384 / rows) to a multiple of 1024,
            // measured best at 1024 / 4096 / 8192 rows: 12288 / 6144 / 6144
            // (profiles/r01_band_small.log).
            const int64_t base = p->d <= 3072 ? 4096 : (row_chunk >= 32768 && p->d >= 6144) ? 3072 : 3584;
            const double w = 3072.0 * std::sqrt(16384.0 / static_cast<double>(row_chunk));
            band = std::max<int64_t>(base, static_cast<int64_t>(std::llround(w / 1024.0)) * 1024);
        } else {
            // ~32 MB of G per chunk so it stays L2 resident between producer and consumers
            band = std::max<int64_t>(kBN, ((int64_t(16) << 20) / row_chunk) / kBN * kBN);
        }
    }
    band = std::min(band, round_up(p->v, kBN));
    // bands per dH group (persistent backward): dH is written once per group
    const int64_t n_bd_all = ceil_div(p->v, band);
    const int kg = h->bwd_persistent ? static_cast<int>(std::min<int64_t>(h->dh_group, n_bd_all)) : 1;

    Scratch sc(h);
    const size_t o_g = sc.take(sizeof(float) * p->n);
    const size_t o_l = sc.take(sizeof(float) * p->n);
    const size_t o_G = sc.take(sizeof(__nv_bfloat16) * row_chunk * band * (h->bwd_persistent ? 2 * kg : 1));
    const int64_t n_rc = ceil_div(n_k, row_chunk), n_bd = ceil_div(p->v, band);
    const int64_t n_chunks = n_rc * n_bd;
    const int64_t mb_max = ceil_div(row_chunk, 128);
    const size_t o_ctr = sc.take(sizeof(unsigned) * (1 + 4 * n_chunks + n_chunks * mb_max));
    // bf16 outputs: dH is summed in fp32 over the bands (workspace, rounded at the
    // end); dW goes out as bf16 straight from the accumulators when it is written
    // once (persistent backward, one row chunk, TMA epilogue), else via fp32
    const int64_t ld32 = round_up(p->d, 4);
    const bool dw_direct = dw_bf16 && h->bwd_persistent && n_rc == 1 && (h->bwd_tma_epi & 2) && lddw % 8 == 0 &&
                           aligned16(dweight_out);
    const size_t o_dhf = dh_bf16 ? sc.take(sizeof(float) * p->n * ld32) : 0;
    const size_t o_dwf = (dw_bf16 && !dw_direct) ? sc.take(sizeof(float) * p->v * ld32) : 0;
    if ((s = sc.commit())) return s;
    h->bwd_scratch[0] = o_G;
    h->bwd_scratch[1] = o_ctr;
    float* gamma = sc.ptr<float>(o_g);
    float* lse = sc.ptr<float>(o_l);
    __nv_bfloat16* G = sc.ptr<__nv_bfloat16>(o_G);
    const int64_t lddh_out = lddh;  // caller's dH leading dimension (bf16 output)
    if (dh_bf16) {
        dhidden = sc.ptr<float>(o_dhf);
        lddh = ld32;
    }
    float* dw_store = dweight;  // what the kernels write (fp32, or bf16 reinterpreted)
    int64_t lddw_k = lddw;
    if (dw_bf16 && dw_direct) {
        dw_store = static_cast<float*>(dweight_out);
    } else if (dw_bf16) {
        dw_store = sc.ptr<float>(o_dwf);
        lddw_k = ld32;
    }

    e = launch_gamma(p->n, p->targets, p->has_ignore, p->ignore_index, stats.m, stats.a, stats.found,
                     reduction, upstream_scalar, upstream_dev, upstream_rows, h->count, gamma, lse, h->err,
                     h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "gamma kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    if ((s = read_errors(h, h->validate != 0))) return s;
    if (!dhidden && !dw_store) return FCE_OK;

    float* dh_k = dhidden;
    int64_t lddh_k = lddh;
    int acc_k = accumulate_dhidden;
    if (cp.on) {
        e = launch_gather_rows(nullptr, 0, nullptr, 0, 0, cp.rows, p->n, h->count, nullptr, nullptr, gamma,
                               cp.gamma, lse, cp.lse, h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "compaction gather: %s", cudaGetErrorString(e));
        h->launches += 1;
        gamma = cp.gamma;
        lse = cp.lse;
        dh_k = cp.dh;
        lddh_k = cp.lddh;
        acc_k = 0;
    }
    {
        if (h->bwd_persistent) {
            s = run_backward_persistent(h, pk, gamma, lse, row_chunk, band, kg, dh_k, lddh_k, dw_store,
                                        lddw_k, acc_k, dw_direct, cp.on ? h->count : nullptr);
        } else {
            s = run_backward_tiles(h, pk, gamma, lse, row_chunk, band, G, dh_k, lddh_k, dw_store, lddw_k,
                                   acc_k);
        }
        if (s) return s;
    }
    if (cp.on && dhidden) {
        e = launch_scatter_rows_f32(cp.dh, cp.lddh, dhidden, lddh, p->d, cp.map, p->n, accumulate_dhidden,
                                    h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "scatter kernel: %s", cudaGetErrorString(e));
        h->launches += 1;
    }
    if (dh_bf16) {
        e = launch_round_to_bf16(dhidden, p->n, p->d, lddh, static_cast<__nv_bfloat16*>(dhidden_out), lddh_out,
                                 h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "bf16 rounding: %s", cudaGetErrorString(e));
        h->launches += 1;
    }
    if (dw_bf16 && !dw_direct) {
        e = launch_round_to_bf16(dw_store, p->v, p->d, lddw_k, static_cast<__nv_bfloat16*>(dweight_out), lddw,
                                 h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "bf16 rounding: %s", cudaGetErrorString(e));
        h->launches += 1;
    }
    return FCE_OK;
}

// Non-persistent backward (option bwd_persistent = 0): per (row chunk, band)
// a G tile launch and one dW / dH GEMM launch.
static fce_status run_backward_tiles(fce_handle h, const fce_problem* p, const float* gamma,
                                     const float* lse, int64_t row_chunk, int64_t band, __nv_bfloat16* G,
                                     float* dhidden, int64_t lddh, float* dweight, int64_t lddw,
                                     int accumulate_dhidden) {
    cudaError_t e;
    const int k_blocks_d = static_cast<int>(ceil_div(p->d, kBK));
    for (int64_t r0 = 0; r0 < p->n; r0 += row_chunk) {
        const int64_t nc = std::min(row_chunk, p->n - r0);
        const void* h_chunk = static_cast<const __nv_bfloat16*>(p->hidden) + r0 * p->ldh;
        for (int64_t vb = 0; vb < p->v; vb += band) {
            const int64_t vc = std::min(band, p->v - vb);
            const void* w_band = static_cast<const __nv_bfloat16*>(p->weight) + vb * p->ldw;

            // K2a: recompute S tiles, G = gamma (softmax - onehot) -> bf16 chunk
            TileParams tp;
            std::memset(&tp, 0, sizeof(tp));
            TensorMaps maps;
            std::memset(&maps, 0, sizeof(maps));
            if (!encode_map_2d(&maps.a0, h_chunk, p->d, nc, p->ldh * 2, kBK, kBM) ||
                !encode_map_2d(&maps.b0, w_band, p->d, vc, p->ldw * 2, kBK, kBN))
                return fail(FCE_CUDA_ERROR, "cuTensorMapEncodeTiled failed (grad)");
            tp.mode = kEpiGrad;
            tp.n_rows = static_cast<int>(nc);
            tp.v_cols = static_cast<int>(vc);
            tp.m_blocks = static_cast<int>(ceil_div(nc, kBM));
            tp.v_tiles = static_cast<int>(ceil_div(vc, kBN));
            tp.k_blocks = k_blocks_d;
            tp.units = tp.m_blocks * tp.v_tiles;
            tp.targets = p->targets + r0;
            tp.col_global0 = p->v_offset + vb;
            tp.has_ignore = p->has_ignore;
            tp.ignore_index = p->ignore_index;
            tp.lse = lse + r0;
            tp.gamma = gamma + r0;
            tp.g_out = G;
            tp.ldg = band;
            e = timed_launch(h, tp, maps, 2.0 * nc * p->d * vc);
            if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "grad tile kernel: %s", cudaGetErrorString(e));

            // K2b + K2c in one persistent launch:
            //   prob 0: dW[vb:vb+vc] (+)= G^T . H[r0:r0+nc]   (A, B MN-major)
            //   prob 1: dH[r0:r0+nc] (+)= G . W[vb:vb+vc]      (A K-major, B MN-major)
            TileParams gp;
            std::memset(&gp, 0, sizeof(gp));
            TensorMaps gm;
            std::memset(&gm, 0, sizeof(gm));
            int np = 0;
            if (dweight) {
                GemmProblem& q = gp.prob[np];
                if (!encode_map_2d(np ? &gm.a1 : &gm.a0, G, band, nc, band * 2, 64, 64) ||
                    !encode_map_2d(np ? &gm.b1 : &gm.b0, h_chunk, p->d, nc, p->ldh * 2, 64, 64))
                    return fail(FCE_CUDA_ERROR, "cuTensorMapEncodeTiled failed (dW)");
                q.m = static_cast<int>(vc);
                q.n = static_cast<int>(p->d);
                q.k_blocks = static_cast<int>(ceil_div(nc, kBK));
                q.m_tiles = static_cast<int>(ceil_div(vc, kBM));
                q.n_tiles = static_cast<int>(ceil_div(p->d, kBN));
                q.a_mn = 1;
                q.b_mn = 1;
                q.n_fastest = 0;
                q.accumulate = r0 > 0 ? 1 : 0;
                q.c = dweight + vb * lddw;
                q.ldc = lddw;
                ++np;
            }
            if (dhidden) {
                GemmProblem& q = gp.prob[np];
                if (!encode_map_2d(np ? &gm.a1 : &gm.a0, G, band, nc, band * 2, kBK, kBM) ||
                    !encode_map_2d(np ? &gm.b1 : &gm.b0, w_band, p->d, vc, p->ldw * 2, 64, 64))
                    return fail(FCE_CUDA_ERROR, "cuTensorMapEncodeTiled failed (dH)");
                q.m = static_cast<int>(nc);
                q.n = static_cast<int>(p->d);
                q.k_blocks = static_cast<int>(ceil_div(vc, kBK));
                q.m_tiles = static_cast<int>(ceil_div(nc, kBM));
                q.n_tiles = static_cast<int>(ceil_div(p->d, kBN));
                q.a_mn = 0;
                q.b_mn = 1;
                q.n_fastest = 1;
                q.accumulate = (vb > 0 || accumulate_dhidden) ? 1 : 0;
                q.c = dhidden + r0 * lddh;
                q.ldc = lddh;
                ++np;
            }
            gp.mode = kEpiGemm;
            gp.units0 = gp.prob[0].m_tiles * gp.prob[0].n_tiles;
            gp.units = gp.units0 + (np > 1 ? gp.prob[1].m_tiles * gp.prob[1].n_tiles : 0);
            e = timed_launch(h, gp, gm, 2.0 * nc * p->d * vc * np);
            if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "gemm tile kernel: %s", cudaGetErrorString(e));
        }
    }
    return FCE_OK;
}

fce_status fce_gemm_bf16(fce_handle h, const void* a, int64_t lda, int a_mn, const void* b,
                         int64_t ldb, int b_mn, int64_t m, int64_t n, int64_t k, float* c,
                         int64_t ldc, int accumulate) {
    fce_status s = check_handle(h);
    if (s) return s;
    if (m <= 0 || n <= 0 || k <= 0) return fail(FCE_EMPTY_INPUT, "gemm requires M, N, K > 0");
    if (!a || !b || !c) return fail(FCE_INVALID_ARGUMENT, "null operand");
    if (lda % 8 || ldb % 8 || !aligned16(a) || !aligned16(b))
        return fail(FCE_INVALID_LAYOUT, "bf16 operands need ld %% 8 == 0 and 16-byte aligned bases");
    if (m > INT32_MAX / 2 || n > INT32_MAX / 2 || k > INT32_MAX / 2)
        return fail(FCE_INVALID_LAYOUT, "gemm too large");
    TileParams gp;
    std::memset(&gp, 0, sizeof(gp));
    TensorMaps gm;
    std::memset(&gm, 0, sizeof(gm));
    // A: [M, K] K-major (lda >= K) or stored [K, M] MN-major (lda >= M)
    const bool ok_a = a_mn ? encode_map_2d(&gm.a0, a, m, k, lda * 2, 64, 64)
                           : encode_map_2d(&gm.a0, a, k, m, lda * 2, kBK, kBM);
    const bool ok_b = b_mn ? encode_map_2d(&gm.b0, b, n, k, ldb * 2, 64, 64)
                           : encode_map_2d(&gm.b0, b, k, n, ldb * 2, kBK, h->gemm_pair ? 128 : kBN);
    if (!ok_a || !ok_b) return fail(FCE_CUDA_ERROR, "cuTensorMapEncodeTiled failed (gemm)");
    GemmProblem& q = gp.prob[0];
    q.m = static_cast<int>(m);
    q.n = static_cast<int>(n);
    q.k_blocks = static_cast<int>(ceil_div(k, kBK));
    q.m_tiles = static_cast<int>(ceil_div(m, kBM));
    q.n_tiles = static_cast<int>(ceil_div(n, kBN));
    q.a_mn = a_mn ? 1 : 0;
    q.b_mn = b_mn ? 1 : 0;
    q.n_fastest = 0;
    q.accumulate = accumulate == 2 ? 2 : (accumulate ? 1 : 0);
    q.c = c;
    q.ldc = ldc;
    gp.mode = kEpiGemm;
    gp.units0 = q.m_tiles * q.n_tiles;
    gp.units = gp.units0;
    cudaError_t e;
    if (h->gemm_pair) {
        e = launch_pair_gemm(q, gm, h->sms, h->stream);
        h->launches += 1;
    } else {
        e = timed_launch(h, gp, gm, 2.0 * m * n * k);
    }
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "gemm tile kernel: %s", cudaGetErrorString(e));
    return FCE_OK;
}

fce_status fce_scale(fce_handle h, float* x, int64_t count, float factor) {
    fce_status s = check_handle(h);
    if (s) return s;
    if (count <= 0) return FCE_OK;
    if (!x) return fail(FCE_INVALID_ARGUMENT, "null buffer");
    cudaError_t e = launch_scale(x, count, nullptr, factor, h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "scale kernel: %s", cudaGetErrorString(e));
    h->launches += 1;
    return FCE_OK;
}

fce_status fce_generate_instance(fce_handle h, int64_t n, int64_t d, int64_t v, uint64_t seed,
                                 void* hidden_bf16, int64_t ldh, void* weight_bf16, int64_t ldw,
                                 int64_t* targets, int64_t ignore_index, double ignore_fraction,
                                 float* hidden_f32, float* weight_f32) {
    fce_status s = check_handle(h);
    if (s) return s;
    if (n <= 0 || d <= 0 || v <= 0) return fail(FCE_EMPTY_INPUT, "instance requires N > 0, d > 0, V > 0");
    if (ldh < d || ldw < d) return fail(FCE_DIMENSION_MISMATCH, "leading dimension < d");
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    cudaError_t e;
    if (hidden_bf16 || hidden_f32) {
        if (hidden_bf16) FCE_CUDA(cudaMemsetAsync(hidden_bf16, 0, sizeof(__nv_bfloat16) * n * ldh, h->stream));
        e = launch_gen_matrix(static_cast<__nv_bfloat16*>(hidden_bf16), n, d, ldh, seed, scale,
                              hidden_f32, h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "gen kernel: %s", cudaGetErrorString(e));
    }
    if (weight_bf16 || weight_f32) {
        if (weight_bf16) FCE_CUDA(cudaMemsetAsync(weight_bf16, 0, sizeof(__nv_bfloat16) * v * ldw, h->stream));
        e = launch_gen_matrix(static_cast<__nv_bfloat16*>(weight_bf16), v, d, ldw,
                              seed ^ 0xA5A5A5A5A5A5A5A5ull, scale, weight_f32, h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "gen kernel: %s", cudaGetErrorString(e));
    }
    if (targets) {
        e = launch_gen_targets(targets, n, v, seed, ignore_index, ignore_fraction, h->stream);
        if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "gen kernel: %s", cudaGetErrorString(e));
    }
    return FCE_OK;
}

fce_status fce_f32_to_bf16(fce_handle h, const float* in, int64_t rows, int64_t cols,
                           int64_t ld_in, void* out, int64_t ld_out) {
    fce_status s = check_handle(h);
    if (s) return s;
    if (rows <= 0 || cols <= 0) return FCE_OK;
    if (!in || !out) return fail(FCE_INVALID_ARGUMENT, "null buffer");
    if (ld_out < cols || ld_in < cols) return fail(FCE_DIMENSION_MISMATCH, "leading dimension < cols");
    if ((s = reset_flags(h))) return s;
    cudaError_t e = launch_f32_to_bf16(in, rows, cols, ld_in, static_cast<__nv_bfloat16*>(out),
                                       ld_out, h->err, h->stream);
    if (e != cudaSuccess) return fail(FCE_CUDA_ERROR, "convert kernel: %s", cudaGetErrorString(e));
    return read_errors(h, true);
}

}  // extern "C"

namespace fce {

fce_status backward_for_overlap(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                                float upstream_scalar, const float* upstream_rows, float* dhidden, int64_t lddh,
                                float* dweight, int64_t lddw, int64_t row_chunk, int reserve_sms,
                                cudaEvent_t counters_reset, std::vector<DhChunkDone>* done) {
    fce_status s = check_handle(h);
    if (s) return s;
    if (!h->bwd_persistent || p->has_ignore || !dhidden)
        return fail(FCE_INVALID_ARGUMENT, "overlapped backward needs the persistent kernel, dH and no ignore_index");
    const int64_t saved_rc = h->row_chunk, saved_res = h->bwd_reserve_sms;
    h->row_chunk = round_up(row_chunk, 256);
    h->bwd_reserve_sms = std::min<int64_t>(reserve_sms, h->sms - 2);
    h->ctr_reset_ev = counters_reset;
    h->last_bwd.valid = false;
    s = backward_impl(h, p, stats, reduction, upstream_scalar, nullptr, upstream_rows, dhidden, lddh, FCE_DTYPE_F32,
                      dweight, lddw, FCE_DTYPE_F32, 0);
    h->row_chunk = saved_rc;
    h->bwd_reserve_sms = saved_res;
    h->ctr_reset_ev = nullptr;
    if (s) return s;
    if (!h->last_bwd.valid) return fail(FCE_INVALID_ARGUMENT, "no persistent backward was launched");
    const LastBwdView lb{h->last_bwd.counters, h->last_bwd.row_chunk, h->last_bwd.n_rc, h->last_bwd.bands,
                         h->last_bwd.n_dh};
    done->clear();
    for (int64_t rc = 0; rc < lb.n_rc; ++rc) {
        // dH of a row chunk is final when the dH units of its last vocabulary
        // band are: dH groups of one row chunk complete in band order (each
        // waits for the previous one), every unit signals from both CTAs
        const int64_t c_last = rc * lb.bands + lb.bands - 1;
        DhChunkDone d;
        d.counter = lb.counters + 1 + 4 * c_last + 1;
        d.target = static_cast<unsigned>(2 * lb.n_dh);
        d.row0 = rc * lb.row_chunk;
        d.rows = std::min(lb.row_chunk, p->n - d.row0);
        done->push_back(d);
    }
    return FCE_OK;
}

fce_status backward_dh_peers(fce_handle h, const fce_problem* p, fce_stats stats, int reduction,
                             float upstream_scalar, const float* upstream_rows, float* const* peer_dh, int k,
                             const int* block0, float* dweight, int64_t lddw) {
    fce_status s = check_handle(h);
    if (s) return s;
    if (k < 1 || k > kMaxDhPeers) return fail(FCE_INVALID_LAYOUT, "peer dH reduction supports 1..%d ranks", kMaxDhPeers);
    if (!h->bwd_persistent || p->has_ignore)
        return fail(FCE_INVALID_ARGUMENT, "peer dH reduction needs the persistent backward and no ignore_index");
    h->dh_peers.k = k;
    for (int q = 0; q < k; ++q) h->dh_peers.ptr[q] = peer_dh[q];
    for (int q = 0; q <= k; ++q) h->dh_peers.block0[q] = block0[q];
    s = backward_impl(h, p, stats, reduction, upstream_scalar, nullptr, upstream_rows, peer_dh[0], p->d, FCE_DTYPE_F32,
                      dweight, lddw, FCE_DTYPE_F32, 1);
    h->dh_peers.k = 0;
    return s;
}

}  // namespace fce
