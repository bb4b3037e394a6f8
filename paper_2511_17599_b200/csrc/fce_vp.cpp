// Vocabulary-parallel split over k GPUs (one process per GPU).
//
// Replaces the in-process simulation of tp_forward / tp_backward
// (reference proj/include/fusedce/parallel_sim.hpp:186-290) with real ranks:
//   forward : fce_forward_partial on the local W shard (v_offset set), then
//             ncclAllGather of the per-row (m, a, z_t, found) partials
//             (16 B per row per rank) and a rank-ordered merge on every rank,
//             so loss / lse / stats are identical everywhere.
//   backward: fce_backward on the shard with the merged stats; dW stays local
//             (parallel_sim.hpp:240-244), dH partials are summed with
//             ncclAllReduce (parallel_sim.hpp:276-288).
// NCCL is resolved with dlopen at first use, so a process that already
// loaded torch's libnccl.so.2 shares that copy and the library carries no
// link-time NCCL dependency.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/fce/fce.h"
#include "../../include/fce/fce_vp.h"
#include "fce_internal.h"

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                               ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!lib) {
            api.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
#define FCE_SYM(field, name)                                                 \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(lib, name));    \
    if (!api.field) {                                                        \
        api.why = std::string("missing NCCL symbol ") + name;                \
        return;                                                              \
    }
        FCE_SYM(get_unique_id, "ncclGetUniqueId");
        FCE_SYM(comm_init_rank, "ncclCommInitRank");
        FCE_SYM(comm_destroy, "ncclCommDestroy");
        FCE_SYM(all_gather, "ncclAllGather");
        FCE_SYM(all_reduce, "ncclAllReduce");
        FCE_SYM(group_start, "ncclGroupStart");
        FCE_SYM(group_end, "ncclGroupEnd");
        FCE_SYM(error_string, "ncclGetErrorString");
#undef FCE_SYM
        api.ok = true;
    });
    return api;
}

fce_status vp_fail(fce_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    fce::set_last_error(buf);
    return s;
}

}  // namespace

struct fce_comm_s {
    ncclComm_t comm = nullptr;
    int nranks = 1;
    int rank = 0;
    // gather buffers, grown on demand
    void* buf = nullptr;
    size_t buf_size = 0;
};

extern "C" {

const char* fce_vp_last_error(void) { return fce_last_error(); }

fce_status fce_comm_unique_id(uint8_t* out, size_t len) {
    if (!out || len < sizeof(ncclUniqueId)) return vp_fail(FCE_INVALID_ARGUMENT, "id buffer too small");
    NcclApi& api = nccl();
    if (!api.ok) return vp_fail(FCE_NCCL_ERROR, "%s", api.why.c_str());
    ncclUniqueId id;
    ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return vp_fail(FCE_NCCL_ERROR, "ncclGetUniqueId: %s", api.error_string(r));
    std::memcpy(out, &id, sizeof(id));
    return FCE_OK;
}

fce_status fce_comm_init(fce_comm* out, int device, int nranks, int rank, const uint8_t* id,
                         size_t len) {
    if (!out || !id || len < sizeof(ncclUniqueId)) return vp_fail(FCE_INVALID_ARGUMENT, "bad arguments");
    if (nranks < 1 || rank < 0 || rank >= nranks) return vp_fail(FCE_INVALID_LAYOUT, "bad rank layout");
    NcclApi& api = nccl();
    if (!api.ok) return vp_fail(FCE_NCCL_ERROR, "%s", api.why.c_str());
    if (cudaSetDevice(device) != cudaSuccess) return vp_fail(FCE_CUDA_ERROR, "cudaSetDevice failed");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    fce_comm c = new fce_comm_s();
    ncclResult_t r = api.comm_init_rank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return vp_fail(FCE_NCCL_ERROR, "ncclCommInitRank: %s", api.error_string(r));
    }
    c->nranks = nranks;
    c->rank = rank;
    *out = c;
    return FCE_OK;
}

fce_status fce_comm_destroy(fce_comm c) {
    if (!c) return FCE_OK;
    if (c->comm && nccl().ok) nccl().comm_destroy(c->comm);
    if (c->buf) cudaFree(c->buf);
    delete c;
    return FCE_OK;
}

fce_status fce_vp_forward(fce_handle h, fce_comm c, const fce_problem* p, int reduction,
                          fce_stats merged, float* lse, float* loss_rows, float* loss_reduced) {
    if (!h || !c || !p) return vp_fail(FCE_INVALID_ARGUMENT, "null argument");
    const int64_t n = p->n;
    const size_t per_rank = (3 * sizeof(float) + 1) * static_cast<size_t>(n);
    const size_t need = 2 * per_rank * static_cast<size_t>(c->nranks) + 1024;
    if (need > c->buf_size) {
        if (c->buf) cudaFree(c->buf);
        c->buf = nullptr;
        if (cudaMalloc(&c->buf, need) != cudaSuccess) return vp_fail(FCE_CUDA_ERROR, "gather buffer");
        c->buf_size = need;
    }
    char* base = static_cast<char*>(c->buf);
    // local partial: [m | a | zt] floats then found bytes
    float* lm = reinterpret_cast<float*>(base);
    float* la = lm + n;
    float* lz = la + n;
    uint8_t* lf = reinterpret_cast<uint8_t*>(lz + n);
    char* gbase = base + ((per_rank + 255) & ~size_t(255));
    float* gm = reinterpret_cast<float*>(gbase);
    float* ga = gm + n * c->nranks;
    float* gz = ga + n * c->nranks;
    uint8_t* gf = reinterpret_cast<uint8_t*>(gz + n * c->nranks);

    fce_stats part{lm, la, lz, lf};
    fce_status s = fce_forward_partial(h, p, part);
    if (s) return s;
    // collectives run on the handle's stream, ordered after the partial kernels
    cudaStream_t stream = fce::handle_stream(h);
    NcclApi& api = nccl();
    api.group_start();
    api.all_gather(lm, gm, n, ncclFloat32, c->comm, stream);
    api.all_gather(la, ga, n, ncclFloat32, c->comm, stream);
    api.all_gather(lz, gz, n, ncclFloat32, c->comm, stream);
    api.all_gather(lf, gf, n, ncclUint8, c->comm, stream);
    ncclResult_t r = api.group_end();
    if (r != ncclSuccess) return vp_fail(FCE_NCCL_ERROR, "all-gather of stats: %s", api.error_string(r));
    return fce_merge_partials(h, c->nranks, n, n, gm, ga, gz, gf, p->targets, p->has_ignore,
                              p->ignore_index, reduction, merged, lse, loss_rows, loss_reduced);
}

fce_status fce_vp_backward(fce_handle h, fce_comm c, const fce_problem* p, fce_stats merged,
                           int reduction, float upstream_scalar, const float* upstream_rows,
                           float* dhidden, int64_t lddh, float* dweight_shard, int64_t lddw) {
    if (!h || !c || !p) return vp_fail(FCE_INVALID_ARGUMENT, "null argument");
    fce_status s = fce_backward(h, p, merged, reduction, upstream_scalar, upstream_rows, dhidden,
                                lddh, dweight_shard, lddw, 0);
    if (s) return s;
    if (!dhidden || c->nranks == 1) return FCE_OK;
    cudaStream_t stream = fce::handle_stream(h);
    NcclApi& api = nccl();
    ncclResult_t r;
    if (lddh == p->d) {
        r = api.all_reduce(dhidden, dhidden, static_cast<size_t>(p->n * p->d), ncclFloat32, ncclSum,
                           c->comm, stream);
    } else {
        api.group_start();
        for (int64_t i = 0; i < p->n; ++i)
            api.all_reduce(dhidden + i * lddh, dhidden + i * lddh, static_cast<size_t>(p->d),
                           ncclFloat32, ncclSum, c->comm, stream);
        r = api.group_end();
    }
    if (r != ncclSuccess) return vp_fail(FCE_NCCL_ERROR, "all-reduce of dH: %s", api.error_string(r));
    return FCE_OK;
}

}  // extern "C"
