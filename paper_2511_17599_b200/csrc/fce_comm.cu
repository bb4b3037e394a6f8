// Peer-sum kernel of the in-process ("local") communicator transport.
//
// dst[i] = src[0][i] + src[1][i] + ... + src[k-1][i], added in rank order —
// the order of the reference's dH sum over ranks (tp_backward,
// proj/include/fusedce/parallel_sim.hpp:276-288) — so a k-rank all-reduce
// over this transport is deterministic.  The sources are the ranks' own
// buffers (same device, or a peer device with P2P access over NVLink); the
// kernel is pure HBM streaming: (k + 1) x 4 B per element, 16-byte vector
// loads when every pointer allows it.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

#include "fce_comm.h"
#include "fce_internal.h"

namespace fce {

__global__ void __launch_bounds__(256) k_sum_peers_v4(PeerPtrs src, int k, float* __restrict__ dst,
                                                      size_t count4) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count4; i += stride) {
        float4 acc = reinterpret_cast<const float4*>(src.p[0])[i];
        for (int r = 1; r < k; ++r) {
            const float4 x = reinterpret_cast<const float4*>(src.p[r])[i];
            acc.x += x.x;
            acc.y += x.y;
            acc.z += x.z;
            acc.w += x.w;
        }
        reinterpret_cast<float4*>(dst)[i] = acc;
    }
}

__global__ void __launch_bounds__(256) k_sum_peers(PeerPtrs src, int k, float* __restrict__ dst, size_t begin,
                                                   size_t count) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    for (size_t i = begin + blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count; i += stride) {
        float acc = src.p[0][i];
        for (int r = 1; r < k; ++r) acc += src.p[r][i];
        dst[i] = acc;
    }
}

cudaError_t launch_sum_peers(const PeerPtrs& src, int k, float* dst, size_t count, cudaStream_t s) {
    if (count == 0) return cudaSuccess;
    bool vec = (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
    for (int r = 0; r < k; ++r) vec = vec && (reinterpret_cast<uintptr_t>(src.p[r]) & 15) == 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    size_t done = 0;
    if (vec && count >= 4) {
        const size_t c4 = count / 4;
        const size_t want = (c4 + 255) / 256;
        const int blocks = static_cast<int>(want < static_cast<size_t>(4 * sms) ? want : 4 * sms);
        k_sum_peers_v4<<<blocks, 256, 0, s>>>(src, k, dst, c4);
        done = c4 * 4;
    }
    if (done < count) {
        const size_t rest = count - done;
        const size_t want = (rest + 255) / 256;
        const int blocks = static_cast<int>(want < static_cast<size_t>(4 * sms) ? want : 4 * sms);
        k_sum_peers<<<blocks, 256, 0, s>>>(src, k, dst, done, count);
    }
    return cudaGetLastError();
}

// ------------------------------------------------ stream wait on a device counter
// The overlapped vocab-parallel backward releases the collective of a row chunk
// from the comm stream as soon as the persistent kernel's dependency counter
// says the chunk's dH rows are final.  cuStreamWaitValue32 holds the stream in
// the front end (no SM is occupied); where stream memory operations are not
// available a one-thread kernel spins on the counter instead.
__global__ void k_wait_geq(const unsigned* counter, unsigned target) {
    unsigned v;
    for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
        if (v >= target) break;
        __nanosleep(1000);
    }
}

cudaError_t stream_wait_geq(cudaStream_t s, const unsigned* counter, unsigned target) {
    // function-local static: resolved once (the driver entry point; no -lcuda)
    static const PFN_cuStreamWaitValue32_v8000 fn = [] {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuStreamWaitValue32_v8000>(ptr);
        return static_cast<PFN_cuStreamWaitValue32_v8000>(nullptr);
    }();
    if (fn) {
        CUresult r = fn(s, reinterpret_cast<CUdeviceptr>(counter), target, CU_STREAM_WAIT_VALUE_GEQ);
        if (r == CUDA_SUCCESS) return cudaSuccess;  // else (memory ops unsupported): spin kernel
    }
    k_wait_geq<<<1, 1, 0, s>>>(counter, target);
    return cudaGetLastError();
}

// globaltimer stamp when the stream reaches this point (device traces)
__global__ void k_stamp(unsigned long long* slot) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *slot = t;
}

cudaError_t launch_stamp(cudaStream_t s, unsigned long long* slot) {
    k_stamp<<<1, 1, 0, s>>>(slot);
    return cudaGetLastError();
}

}  // namespace fce
