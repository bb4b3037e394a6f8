// Peer-sum kernel of the in-process ("local") communicator transport.
//
// dst[i] = src[0][i] + src[1][i] + ... + src[k-1][i], added in rank order —
// the order of the reference's dH sum over ranks (tp_backward,
// proj/include/fusedce/parallel_sim.hpp:276-288) — so a k-rank all-reduce
// over this transport is deterministic.  The sources are the ranks' own
// buffers (same device, or a peer device with P2P access over NVLink); the
// kernel is pure HBM streaming: (k + 1) x 4 B per element, 16-byte vector
// loads when every pointer allows it.
#include <cstdint>

#include "fce_comm.h"

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

}  // namespace fce
