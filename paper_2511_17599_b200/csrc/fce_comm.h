// Internal communicator interface behind the fce_comm handle of fce_vp.h.
//
// The vocabulary-parallel, sequence-parallel and data-parallel entry points
// (fce_vp.cpp) need three collectives, all stream-ordered on the caller's
// handle stream (inputs are read after the work already queued there, outputs
// are visible to the work queued after):
//   all_gather          every rank's `bytes` land in recv[rank * bytes]
//   all_reduce_sum      fp32 element-wise sum over ranks (in place allowed)
//   reduce_scatter_sum  rank r receives the sum of every rank's block r
// Two transports implement them:
//   NCCL   one process per GPU (the production layout): NCCL over NVLink /
//          NVSwitch, resolved with dlopen so a torch process shares its copy.
//   local  k ranks inside ONE process, each driven by its own host thread, on
//          any devices (several may share one GPU).  Collectives are the
//          library's own kernels reading the peers' buffers directly
//          (reduce-scatter then all-gather, sums in rank order) — the
//          peer-memory data path NVLink P2P gives a single-process multi-GPU
//          job, and the way the k-rank code runs on a one-GPU box.
//   ipc    one process per rank on one node, the same kernels over CUDA IPC
//          mappings of each rank's registered staging buffer (no NCCL).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/fce/fce.h"

namespace fce {

enum Transport : int { kTransportNccl = 1, kTransportLocal = 2, kTransportIpc = 3 };

class Comm {
public:
    virtual ~Comm() = default;
    virtual int transport() const = 0;
    virtual fce_status all_gather(const void* send, void* recv, size_t bytes, cudaStream_t s) = 0;
    virtual fce_status all_reduce_sum(const float* send, float* recv, size_t count, cudaStream_t s) = 0;
    virtual fce_status reduce_scatter_sum(const float* send, float* recv, size_t recv_count,
                                          cudaStream_t s) = 0;
    // Peer-memory transports only (local, ipc).  Collective: every rank's
    // symmetric region of >= bytes, as pointers usable by this rank's kernels
    // (its own first at ptrs[rank]); the regions persist between calls.
    virtual bool has_peer_memory() const { return false; }
    virtual fce_status sym_buffers(size_t bytes, cudaStream_t s, void** ptrs);
    // Collective stream fence: work queued on every rank's stream before it
    // completes before work queued after it on any rank's stream.
    virtual fce_status fence(cudaStream_t s);
    int nranks = 1;
    int rank = 0;
    int device = 0;
};

// Transports (fce_comm.cpp).  Errors are reported through set_last_error.
fce_status make_nccl_comm(Comm** out, int device, int nranks, int rank, const uint8_t* id, size_t len);
fce_status nccl_unique_id(uint8_t* out, size_t len);

// IPC transport: one process per rank on one node, the library's own
// collectives over CUDA IPC peer memory; rendezvous through a POSIX
// shared-memory segment named by the id (fce_comm.cpp).
fce_status ipc_unique_id(uint8_t* out, size_t len);
fce_status make_ipc_comm(Comm** out, int device, int nranks, int rank, const uint8_t* id, size_t len);

struct LocalGroup;
fce_status make_local_group(LocalGroup** out, int nranks);
fce_status make_local_comm(Comm** out, LocalGroup* g, int device, int rank);
void release_local_group(LocalGroup* g);

// Peer-sum kernel of the local transport (fce_comm.cu): dst[i] = sum over
// ranks p (ascending) of src[p][i], i < count.
constexpr int kMaxLocalRanks = 64;
struct PeerPtrs {
    const float* p[kMaxLocalRanks];
};
cudaError_t launch_sum_peers(const PeerPtrs& src, int k, float* dst, size_t count, cudaStream_t s);

}  // namespace fce
