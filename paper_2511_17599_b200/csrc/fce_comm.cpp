// Communicator transports behind fce_comm (see fce_comm.h).
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <random>
#include <thread>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "fce_comm.h"
#include "fce_internal.h"

namespace fce {

namespace {

fce_status comm_fail(fce_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    set_last_error(buf);
    return s;
}

#define FCE_COMM_CUDA(call)                                                                       \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return comm_fail(FCE_CUDA_ERROR, "%s failed: %s", #call, cudaGetErrorString(e_));     \
    } while (0)

// ------------------------------------------------------------------ NCCL
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*reduce_scatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                   cudaStream_t) = nullptr;
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
#define FCE_SYM(field, name)                                              \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(lib, name)); \
    if (!api.field) {                                                     \
        api.why = std::string("missing NCCL symbol ") + name;             \
        return;                                                           \
    }
        FCE_SYM(get_unique_id, "ncclGetUniqueId");
        FCE_SYM(comm_init_rank, "ncclCommInitRank");
        FCE_SYM(comm_destroy, "ncclCommDestroy");
        FCE_SYM(all_gather, "ncclAllGather");
        FCE_SYM(all_reduce, "ncclAllReduce");
        FCE_SYM(reduce_scatter, "ncclReduceScatter");
        FCE_SYM(error_string, "ncclGetErrorString");
#undef FCE_SYM
        api.ok = true;
    });
    return api;
}

class NcclComm final : public Comm {
public:
    ncclComm_t comm = nullptr;
    ~NcclComm() override {
        if (comm && nccl().ok) nccl().comm_destroy(comm);
    }
    int transport() const override { return kTransportNccl; }
    fce_status check(ncclResult_t r, const char* what) {
        if (r == ncclSuccess) return FCE_OK;
        return comm_fail(FCE_NCCL_ERROR, "%s: %s", what, nccl().error_string(r));
    }
    fce_status all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        NvtxRange nvtx_("nccl all_gather");
        return check(nccl().all_gather(send, recv, bytes, ncclUint8, comm, s), "ncclAllGather");
    }
    fce_status all_reduce_sum(const float* send, float* recv, size_t count, cudaStream_t s) override {
        NvtxRange nvtx_("nccl all_reduce");
        return check(nccl().all_reduce(send, recv, count, ncclFloat32, ncclSum, comm, s), "ncclAllReduce");
    }
    fce_status reduce_scatter_sum(const float* send, float* recv, size_t recv_count, cudaStream_t s) override {
        NvtxRange nvtx_("nccl reduce_scatter");
        return check(nccl().reduce_scatter(send, recv, recv_count, ncclFloat32, ncclSum, comm, s),
                     "ncclReduceScatter");
    }
};

}  // namespace

fce_status Comm::sym_buffers(size_t, cudaStream_t, void**) {
    return comm_fail(FCE_INVALID_ARGUMENT, "this transport has no peer memory (use the local or ipc transport)");
}
fce_status Comm::fence(cudaStream_t) {
    return comm_fail(FCE_INVALID_ARGUMENT, "this transport has no stream fence");
}

fce_status nccl_unique_id(uint8_t* out, size_t len) {
    if (!out || len < sizeof(ncclUniqueId)) return comm_fail(FCE_INVALID_ARGUMENT, "id buffer too small");
    NcclApi& api = nccl();
    if (!api.ok) return comm_fail(FCE_NCCL_ERROR, "%s", api.why.c_str());
    ncclUniqueId id;
    ncclResult_t r = api.get_unique_id(&id);
    if (r != ncclSuccess) return comm_fail(FCE_NCCL_ERROR, "ncclGetUniqueId: %s", api.error_string(r));
    std::memcpy(out, &id, sizeof(id));
    return FCE_OK;
}

fce_status make_nccl_comm(Comm** out, int device, int nranks, int rank, const uint8_t* id, size_t len) {
    if (!id || len < sizeof(ncclUniqueId)) return comm_fail(FCE_INVALID_ARGUMENT, "bad NCCL id");
    NcclApi& api = nccl();
    if (!api.ok) return comm_fail(FCE_NCCL_ERROR, "%s", api.why.c_str());
    FCE_COMM_CUDA(cudaSetDevice(device));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    NcclComm* c = new NcclComm();
    ncclResult_t r = api.comm_init_rank(&c->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
        c->comm = nullptr;
        delete c;
        return comm_fail(FCE_NCCL_ERROR, "ncclCommInitRank: %s", api.error_string(r));
    }
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    *out = c;
    return FCE_OK;
}

// ------------------------------------------------------------------ local
// Rendezvous state shared by the k ranks of one in-process group.  Each
// collective is a sequence of phases; in a phase every rank records an event
// on its stream after the work the phase depends on, meets the others at a
// host barrier, then makes its stream wait for every peer's event.  Device
// work is never blocked on the host beyond the barrier itself.
struct LocalGroup {
    int nranks = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    bool aborted = false;
    int refs = 1;
    std::vector<int> device;       // per rank, -1 until joined
    std::vector<const void*> send; // published buffers of the current collective
    std::vector<void*> recv;
    std::vector<cudaEvent_t> ev;   // [phase][rank] published events
    std::vector<void*> sym;        // per rank: symmetric peer-memory region
    double timeout_s = 600.0;
};

namespace {

constexpr int kPhases = 3;

class LocalComm final : public Comm {
public:
    LocalGroup* g = nullptr;
    cudaEvent_t ev[kPhases] = {nullptr, nullptr, nullptr};
    bool peers_ready = false;
    void* sym = nullptr;
    size_t sym_bytes = 0;

    ~LocalComm() override {
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (sym) cudaFree(sym);
        release_local_group(g);
    }
    bool has_peer_memory() const override { return true; }

    fce_status fence(cudaStream_t s) override { return sync_phase(0, s); }

    fce_status sym_buffers(size_t bytes, cudaStream_t s, void** ptrs) override {
        if (bytes > sym_bytes) {
            if (sym) {
                // the last use ended with a fence: peers no longer read it
                FCE_COMM_CUDA(cudaStreamSynchronize(s));
                FCE_COMM_CUDA(cudaFree(sym));
                sym = nullptr;
            }
            FCE_COMM_CUDA(cudaMalloc(&sym, bytes));
            sym_bytes = bytes;
        }
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->sym[rank] = sym;
        }
        fce_status st = sync_phase(0, s);
        if (st) return st;
        if ((st = enable_peers())) return st;
        std::lock_guard<std::mutex> lk(g->mu);
        for (int q = 0; q < nranks; ++q) ptrs[q] = g->sym[q];
        return FCE_OK;
    }
    int transport() const override { return kTransportLocal; }

    fce_status barrier() {
        std::unique_lock<std::mutex> lk(g->mu);
        if (g->aborted) return comm_fail(FCE_NCCL_ERROR, "local communicator group was aborted by a peer");
        const uint64_t my = g->gen;
        if (++g->arrived == g->nranks) {
            g->arrived = 0;
            ++g->gen;
            g->cv.notify_all();
            return FCE_OK;
        }
        const bool ok = g->cv.wait_for(lk, std::chrono::duration<double>(g->timeout_s),
                                       [&] { return g->gen != my || g->aborted; });
        if (g->gen != my) return FCE_OK;
        g->aborted = true;
        g->cv.notify_all();
        return comm_fail(FCE_NCCL_ERROR, ok ? "local communicator group aborted"
                                            : "local collective timed out waiting for peer ranks "
                                              "(every rank must call it, each from its own thread)");
    }

    // Record this rank's event for `phase`, meet the peers, wait for theirs.
    fce_status sync_phase(int phase, cudaStream_t s) {
        FCE_COMM_CUDA(cudaEventRecord(ev[phase], s));
        {
            std::lock_guard<std::mutex> lk(g->mu);
            g->ev[phase * nranks + rank] = ev[phase];
        }
        fce_status st = barrier();
        if (st) return st;
        for (int q = 0; q < nranks; ++q)
            if (q != rank) FCE_COMM_CUDA(cudaStreamWaitEvent(s, g->ev[phase * nranks + q], 0));
        return FCE_OK;
    }

    void publish(const void* send, void* recv) {
        std::lock_guard<std::mutex> lk(g->mu);
        g->send[rank] = send;
        g->recv[rank] = recv;
    }

    // Kernels of this rank read peers' buffers: peer access to every other device.
    fce_status enable_peers() {
        if (peers_ready) return FCE_OK;
        for (int q = 0; q < nranks; ++q) {
            const int pd = g->device[q];
            if (pd == device || pd < 0) continue;
            int can = 0;
            FCE_COMM_CUDA(cudaDeviceCanAccessPeer(&can, device, pd));
            if (!can) return comm_fail(FCE_NCCL_ERROR, "device %d cannot access peer device %d", device, pd);
            cudaError_t e = cudaDeviceEnablePeerAccess(pd, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) {
                cudaGetLastError();
            } else if (e != cudaSuccess) {
                return comm_fail(FCE_CUDA_ERROR, "cudaDeviceEnablePeerAccess(%d): %s", pd, cudaGetErrorString(e));
            }
        }
        peers_ready = true;
        return FCE_OK;
    }

    fce_status all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        NvtxRange nvtx_("local all_gather");
        publish(send, recv);
        fce_status st = sync_phase(0, s);
        if (st) return st;
        for (int q = 0; q < nranks; ++q) {
            char* dst = static_cast<char*>(recv) + static_cast<size_t>(q) * bytes;
            if (dst != g->send[q] && bytes)
                FCE_COMM_CUDA(cudaMemcpyAsync(dst, g->send[q], bytes, cudaMemcpyDefault, s));
        }
        // peers may overwrite their send buffers only after everyone copied them
        return sync_phase(1, s);
    }

    fce_status all_reduce_sum(const float* send, float* recv, size_t count, cudaStream_t s) override {
        NvtxRange nvtx_("local all_reduce");
        publish(send, recv);
        fce_status st = sync_phase(0, s);
        if (st) return st;
        if ((st = enable_peers())) return st;
        // reduce-scatter: rank r sums slice r of every rank's input into its own
        // output (in place is safe: no peer reads slice r of this rank's buffer)
        const size_t per = ((count + nranks - 1) / nranks + 3) / 4 * 4;
        auto lo = [&](int q) { return std::min(count, static_cast<size_t>(q) * per); };
        PeerPtrs src;
        for (int q = 0; q < nranks; ++q) src.p[q] = static_cast<const float*>(g->send[q]) + lo(rank);
        FCE_COMM_CUDA(launch_sum_peers(src, nranks, recv + lo(rank), lo(rank + 1) - lo(rank), s));
        if ((st = sync_phase(1, s))) return st;
        // all-gather of the reduced slices straight from the peers' outputs
        for (int q = 0; q < nranks; ++q) {
            if (q == rank || lo(q + 1) == lo(q)) continue;
            FCE_COMM_CUDA(cudaMemcpyAsync(recv + lo(q), static_cast<float*>(g->recv[q]) + lo(q),
                                          (lo(q + 1) - lo(q)) * sizeof(float), cudaMemcpyDefault, s));
        }
        return sync_phase(2, s);
    }

    fce_status reduce_scatter_sum(const float* send, float* recv, size_t recv_count, cudaStream_t s) override {
        NvtxRange nvtx_("local reduce_scatter");
        publish(send, recv);
        fce_status st = sync_phase(0, s);
        if (st) return st;
        if ((st = enable_peers())) return st;
        PeerPtrs src;
        for (int q = 0; q < nranks; ++q)
            src.p[q] = static_cast<const float*>(g->send[q]) + static_cast<size_t>(rank) * recv_count;
        FCE_COMM_CUDA(launch_sum_peers(src, nranks, recv, recv_count, s));
        return sync_phase(1, s);
    }
};


// ------------------------------------------------------------------ ipc
// One process per rank on one node, collectives by the library's own kernels
// over CUDA IPC peer memory (NVLink P2P between GPUs; plain HBM when ranks
// share a GPU) — no NCCL.  Rendezvous through a POSIX shared-memory segment
// named by the id: every rank publishes the IPC handles of its registered
// staging buffer and of its phase events there, and the host barrier of a
// phase is a generation counter in the segment.  Each collective stages its
// input in the rank's registered buffer, so peers read it directly:
//   all_gather      copy-in, phase, copy every peer's block out, phase
//   all_reduce      copy-in, phase, sum slice r of every peer's input into
//                   this rank's second region (rank order), phase, copy every
//                   peer's reduced slice out, phase
//   reduce_scatter  copy-in, phase, sum block r of every peer's input, phase
struct IpcRankSlot {
    int device;
    int pid;
    uint64_t buf_version;  // bumps whenever the rank re-registers its buffer
    uint64_t buf_bytes;
    cudaIpcMemHandle_t buf;
    cudaIpcEventHandle_t ev[kPhases];
    uint64_t sym_version;  // symmetric peer-memory region (fused dH reduction)
    uint64_t sym_bytes;
    cudaIpcMemHandle_t sym;
};

struct IpcShared {
    uint32_t magic;
    int nranks;
    std::atomic<int> joined;
    std::atomic<int> arrived;
    std::atomic<uint64_t> gen;
    std::atomic<int> aborted;
    IpcRankSlot slot[kMaxLocalRanks];
};
static_assert(std::atomic<int>::is_always_lock_free && std::atomic<uint64_t>::is_always_lock_free,
              "cross-process atomics must be lock free");
constexpr uint32_t kIpcMagic = 0xFCE1BC01u;

class IpcComm final : public Comm {
public:
    IpcShared* sh = nullptr;
    std::string name;
    cudaEvent_t ev[kPhases] = {nullptr, nullptr, nullptr};
    cudaEvent_t peer_ev[kMaxLocalRanks][kPhases] = {};
    char* buf = nullptr;  // registered staging buffer
    size_t buf_bytes = 0;
    uint64_t buf_version = 0;
    char* peer_buf[kMaxLocalRanks] = {};
    uint64_t peer_version[kMaxLocalRanks] = {};
    char* sym = nullptr;
    size_t sym_bytes = 0;
    uint64_t sym_version = 0;
    char* peer_sym[kMaxLocalRanks] = {};
    uint64_t peer_sym_version[kMaxLocalRanks] = {};
    double timeout_s = 600.0;

    ~IpcComm() override {
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) continue;
            if (peer_buf[q]) cudaIpcCloseMemHandle(peer_buf[q]);
            if (peer_sym[q]) cudaIpcCloseMemHandle(peer_sym[q]);
            for (int ph = 0; ph < kPhases; ++ph)
                if (peer_ev[q][ph]) cudaEventDestroy(peer_ev[q][ph]);
        }
        if (buf) cudaFree(buf);
        if (sym) cudaFree(sym);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (sh) munmap(sh, sizeof(IpcShared));
    }
    int transport() const override { return kTransportIpc; }
    bool has_peer_memory() const override { return true; }

    fce_status fence(cudaStream_t s) override { return sync_phase(0, s); }

    fce_status sym_buffers(size_t bytes, cudaStream_t s, void** ptrs) override {
        IpcRankSlot& me = sh->slot[rank];
        if (bytes > sym_bytes) {
            if (sym) {
                FCE_COMM_CUDA(cudaStreamSynchronize(s));
                FCE_COMM_CUDA(cudaFree(sym));
                sym = nullptr;
            }
            FCE_COMM_CUDA(cudaMalloc(&sym, bytes));
            sym_bytes = bytes;
            FCE_COMM_CUDA(cudaIpcGetMemHandle(&me.sym, sym));
            me.sym_bytes = bytes;
            me.sym_version = ++sym_version;
        }
        fce_status st = sync_phase(0, s);
        if (st) return st;
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) {
                ptrs[q] = sym;
                continue;
            }
            const IpcRankSlot& p = sh->slot[q];
            if (p.sym_version != peer_sym_version[q] || !peer_sym[q]) {
                if (peer_sym[q]) FCE_COMM_CUDA(cudaIpcCloseMemHandle(peer_sym[q]));
                void* ptr = nullptr;
                FCE_COMM_CUDA(cudaIpcOpenMemHandle(&ptr, p.sym, cudaIpcMemLazyEnablePeerAccess));
                peer_sym[q] = static_cast<char*>(ptr);
                peer_sym_version[q] = p.sym_version;
            }
            ptrs[q] = peer_sym[q];
        }
        return FCE_OK;
    }

    fce_status barrier() {
        const uint64_t my = sh->gen.load();
        if (sh->arrived.fetch_add(1) + 1 == nranks) {
            sh->arrived.store(0);
            sh->gen.fetch_add(1);
            return FCE_OK;
        }
        const auto t0 = std::chrono::steady_clock::now();
        int spins = 0;
        while (sh->gen.load() == my) {
            if (sh->aborted.load()) return comm_fail(FCE_NCCL_ERROR, "ipc communicator aborted by a peer rank");
            if (++spins > 64) {
                std::this_thread::sleep_for(std::chrono::microseconds(20));
                if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
                    sh->aborted.store(1);
                    return comm_fail(FCE_NCCL_ERROR, "ipc collective timed out waiting for peer ranks");
                }
            }
        }
        return FCE_OK;
    }

    fce_status sync_phase(int phase, cudaStream_t s) {
        FCE_COMM_CUDA(cudaEventRecord(ev[phase], s));
        fce_status st = barrier();
        if (st) return st;
        for (int q = 0; q < nranks; ++q)
            if (q != rank) FCE_COMM_CUDA(cudaStreamWaitEvent(s, peer_ev[q][phase], 0));
        return FCE_OK;
    }

    // Grow the registered buffer (peers re-open it at their next collective).
    fce_status ensure(size_t bytes, cudaStream_t s) {
        if (bytes <= buf_bytes) return FCE_OK;
        if (buf) {
            // this stream already waited for every peer's reads of the old buffer
            FCE_COMM_CUDA(cudaStreamSynchronize(s));
            FCE_COMM_CUDA(cudaFree(buf));
            buf = nullptr;
        }
        const size_t sz = std::max<size_t>(bytes, size_t(64) << 20);
        FCE_COMM_CUDA(cudaMalloc(&buf, sz));
        buf_bytes = sz;
        IpcRankSlot& me = sh->slot[rank];
        FCE_COMM_CUDA(cudaIpcGetMemHandle(&me.buf, buf));
        me.buf_bytes = sz;
        me.buf_version = ++buf_version;
        return FCE_OK;
    }

    // After the first barrier of a collective: (re-)open peers' buffers that changed.
    fce_status refresh_peers() {
        for (int q = 0; q < nranks; ++q) {
            if (q == rank) {
                peer_buf[q] = buf;
                continue;
            }
            const IpcRankSlot& p = sh->slot[q];
            if (p.buf_version == peer_version[q] && peer_buf[q]) continue;
            if (peer_buf[q]) FCE_COMM_CUDA(cudaIpcCloseMemHandle(peer_buf[q]));
            void* ptr = nullptr;
            FCE_COMM_CUDA(cudaIpcOpenMemHandle(&ptr, p.buf, cudaIpcMemLazyEnablePeerAccess));
            peer_buf[q] = static_cast<char*>(ptr);
            peer_version[q] = p.buf_version;
        }
        return FCE_OK;
    }

    fce_status all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
        NvtxRange nvtx_("ipc all_gather");
        fce_status st = ensure(bytes, s);
        if (st) return st;
        if (bytes) FCE_COMM_CUDA(cudaMemcpyAsync(buf, send, bytes, cudaMemcpyDeviceToDevice, s));
        if ((st = sync_phase(0, s)) || (st = refresh_peers())) return st;
        for (int q = 0; q < nranks; ++q)
            if (bytes)
                FCE_COMM_CUDA(cudaMemcpyAsync(static_cast<char*>(recv) + static_cast<size_t>(q) * bytes, peer_buf[q],
                                              bytes, cudaMemcpyDefault, s));
        return sync_phase(1, s);
    }

    fce_status all_reduce_sum(const float* send, float* recv, size_t count, cudaStream_t s) override {
        NvtxRange nvtx_("ipc all_reduce");
        const size_t region = (count * sizeof(float) + 255) / 256 * 256;
        fce_status st = ensure(2 * region, s);
        if (st) return st;
        if (count) FCE_COMM_CUDA(cudaMemcpyAsync(buf, send, count * sizeof(float), cudaMemcpyDeviceToDevice, s));
        if ((st = sync_phase(0, s)) || (st = refresh_peers())) return st;
        const size_t per = ((count + nranks - 1) / nranks + 3) / 4 * 4;
        auto lo = [&](int q) { return std::min(count, static_cast<size_t>(q) * per); };
        PeerPtrs src;
        for (int q = 0; q < nranks; ++q) src.p[q] = reinterpret_cast<const float*>(peer_buf[q]) + lo(rank);
        FCE_COMM_CUDA(launch_sum_peers(src, nranks, reinterpret_cast<float*>(buf + region) + lo(rank),
                                       lo(rank + 1) - lo(rank), s));
        if ((st = sync_phase(1, s))) return st;
        for (int q = 0; q < nranks; ++q) {
            if (lo(q + 1) == lo(q)) continue;
            FCE_COMM_CUDA(cudaMemcpyAsync(recv + lo(q), reinterpret_cast<const float*>(peer_buf[q] + region) + lo(q),
                                          (lo(q + 1) - lo(q)) * sizeof(float), cudaMemcpyDefault, s));
        }
        return sync_phase(2, s);
    }

    fce_status reduce_scatter_sum(const float* send, float* recv, size_t recv_count, cudaStream_t s) override {
        NvtxRange nvtx_("ipc reduce_scatter");
        const size_t bytes = recv_count * sizeof(float) * nranks;
        fce_status st = ensure(bytes, s);
        if (st) return st;
        if (bytes) FCE_COMM_CUDA(cudaMemcpyAsync(buf, send, bytes, cudaMemcpyDeviceToDevice, s));
        if ((st = sync_phase(0, s)) || (st = refresh_peers())) return st;
        PeerPtrs src;
        for (int q = 0; q < nranks; ++q)
            src.p[q] = reinterpret_cast<const float*>(peer_buf[q]) + static_cast<size_t>(rank) * recv_count;
        FCE_COMM_CUDA(launch_sum_peers(src, nranks, recv, recv_count, s));
        return sync_phase(1, s);
    }
};

}  // namespace

fce_status ipc_unique_id(uint8_t* out, size_t len) {
    if (!out || len < 64) return comm_fail(FCE_INVALID_ARGUMENT, "id buffer too small");
    std::random_device rd;
    char name[64];
    snprintf(name, sizeof(name), "/fce_ipc_%d_%08x%08x", static_cast<int>(getpid()), rd(), rd());
    std::memset(out, 0, len);
    std::memcpy(out, name, std::strlen(name) + 1);
    return FCE_OK;
}

fce_status make_ipc_comm(Comm** out, int device, int nranks, int rank, const uint8_t* id, size_t len) {
    if (!out || !id || len < 64) return comm_fail(FCE_INVALID_ARGUMENT, "bad ipc id");
    if (nranks < 1 || nranks > kMaxLocalRanks || rank < 0 || rank >= nranks)
        return comm_fail(FCE_INVALID_LAYOUT, "ipc group size must be in [1, %d]", kMaxLocalRanks);
    char name[64];
    std::memcpy(name, id, 63);
    name[63] = 0;
    if (name[0] != '/') return comm_fail(FCE_INVALID_ARGUMENT, "not an ipc id (use fce_comm_ipc_id)");
    FCE_COMM_CUDA(cudaSetDevice(device));
    double timeout_s = 600.0;
    if (const char* t = std::getenv("FCE_LOCAL_TIMEOUT_S")) timeout_s = std::atof(t) > 0 ? std::atof(t) : 600.0;
    // rank 0 creates and sizes the segment; the others wait for it to appear
    int fd = -1;
    const auto t0 = std::chrono::steady_clock::now();
    if (rank == 0) {
        fd = shm_open(name, O_CREAT | O_RDWR, 0600);
        if (fd < 0 || ftruncate(fd, sizeof(IpcShared)) != 0) {
            if (fd >= 0) close(fd);
            return comm_fail(FCE_NCCL_ERROR, "shm_open/ftruncate %s failed", name);
        }
    } else {
        for (;;) {
            fd = shm_open(name, O_RDWR, 0600);
            if (fd >= 0) {
                struct stat stt;
                if (fstat(fd, &stt) == 0 && static_cast<size_t>(stt.st_size) >= sizeof(IpcShared)) break;
                close(fd);
                fd = -1;
            }
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s)
                return comm_fail(FCE_NCCL_ERROR, "ipc rendezvous %s not created by rank 0", name);
            std::this_thread::sleep_for(std::chrono::milliseconds(2));
        }
    }
    void* mem = mmap(nullptr, sizeof(IpcShared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (mem == MAP_FAILED) return comm_fail(FCE_NCCL_ERROR, "mmap of %s failed", name);
    IpcShared* sh = static_cast<IpcShared*>(mem);
    if (rank == 0) {
        sh->nranks = nranks;
        sh->joined.store(0);
        sh->arrived.store(0);
        sh->gen.store(0);
        sh->aborted.store(0);
        std::atomic_thread_fence(std::memory_order_seq_cst);
        reinterpret_cast<std::atomic<uint32_t>*>(&sh->magic)->store(kIpcMagic);
    } else {
        while (reinterpret_cast<std::atomic<uint32_t>*>(&sh->magic)->load() != kIpcMagic) {
            if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
                munmap(mem, sizeof(IpcShared));
                return comm_fail(FCE_NCCL_ERROR, "ipc rendezvous %s never initialised", name);
            }
            std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
        if (sh->nranks != nranks) {
            munmap(mem, sizeof(IpcShared));
            return comm_fail(FCE_INVALID_LAYOUT, "ipc group has %d ranks, this rank expects %d", sh->nranks, nranks);
        }
    }
    IpcComm* c = new IpcComm();
    c->sh = sh;
    c->name = name;
    c->nranks = nranks;
    c->rank = rank;
    c->device = device;
    c->timeout_s = timeout_s;
    IpcRankSlot& me = sh->slot[rank];
    me.device = device;
    me.pid = static_cast<int>(getpid());
    for (int ph = 0; ph < kPhases; ++ph) {
        cudaError_t e = cudaEventCreateWithFlags(&c->ev[ph], cudaEventInterprocess | cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaIpcGetEventHandle(&me.ev[ph], c->ev[ph]);
        if (e != cudaSuccess) {
            delete c;
            return comm_fail(FCE_CUDA_ERROR, "ipc event: %s", cudaGetErrorString(e));
        }
    }
    fce_status st = c->ensure(1, nullptr);
    if (st) {
        delete c;
        return st;
    }
    // join: everyone's handles are published before anyone opens a peer's
    sh->joined.fetch_add(1);
    while (sh->joined.load() < nranks) {
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s) {
            delete c;
            return comm_fail(FCE_NCCL_ERROR, "ipc rendezvous: only %d of %d ranks joined", sh->joined.load(), nranks);
        }
        std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
    for (int q = 0; q < nranks; ++q) {
        if (q == rank) continue;
        for (int ph = 0; ph < kPhases; ++ph) {
            cudaError_t e = cudaIpcOpenEventHandle(&c->peer_ev[q][ph], sh->slot[q].ev[ph]);
            if (e != cudaSuccess) {
                delete c;
                return comm_fail(FCE_CUDA_ERROR, "cudaIpcOpenEventHandle (rank %d): %s", q, cudaGetErrorString(e));
            }
        }
    }
    if ((st = c->refresh_peers())) {
        delete c;
        return st;
    }
    // every rank has opened the segment: the name can go (the mappings stay)
    if ((st = c->barrier())) {
        delete c;
        return st;
    }
    if (rank == 0) shm_unlink(name);
    *out = c;
    return FCE_OK;
}

fce_status make_local_group(LocalGroup** out, int nranks) {
    if (!out) return comm_fail(FCE_INVALID_ARGUMENT, "null output");
    if (nranks < 1 || nranks > kMaxLocalRanks)
        return comm_fail(FCE_INVALID_LAYOUT, "local group size must be in [1, %d]", kMaxLocalRanks);
    LocalGroup* g = new LocalGroup();
    g->nranks = nranks;
    g->device.assign(nranks, -1);
    g->send.assign(nranks, nullptr);
    g->recv.assign(nranks, nullptr);
    g->ev.assign(kPhases * nranks, nullptr);
    g->sym.assign(nranks, nullptr);
    if (const char* t = std::getenv("FCE_LOCAL_TIMEOUT_S")) g->timeout_s = std::atof(t) > 0 ? std::atof(t) : 600.0;
    *out = g;
    return FCE_OK;
}

void release_local_group(LocalGroup* g) {
    if (!g) return;
    bool last;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        last = --g->refs == 0;
    }
    if (last) delete g;
}

fce_status make_local_comm(Comm** out, LocalGroup* g, int device, int rank) {
    if (!out || !g) return comm_fail(FCE_INVALID_ARGUMENT, "null argument");
    if (rank < 0 || rank >= g->nranks) return comm_fail(FCE_INVALID_LAYOUT, "rank %d outside [0, %d)", rank, g->nranks);
    FCE_COMM_CUDA(cudaSetDevice(device));
    LocalComm* c = new LocalComm();
    for (auto& e : c->ev) {
        cudaError_t err = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        if (err != cudaSuccess) {
            delete c;  // g not yet referenced: c->g is null
            return comm_fail(FCE_CUDA_ERROR, "cudaEventCreate: %s", cudaGetErrorString(err));
        }
    }
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (g->device[rank] >= 0) {
            delete c;
            return comm_fail(FCE_INVALID_LAYOUT, "rank %d of the local group is already taken", rank);
        }
        g->device[rank] = device;
        ++g->refs;
    }
    c->g = g;
    c->nranks = g->nranks;
    c->rank = rank;
    c->device = device;
    *out = c;
    return FCE_OK;
}

}  // namespace fce
