// Host <-> device plumbing of the drop-in API: one fce handle per device and
// thread, RAII device buffers, and the float (bf16 grid) -> bf16 upload that
// the sm_100a path consumes.  There is no CPU fallback: without a B200 the
// first call throws DeviceError.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <type_traits>
#include <vector>

#include "fce/fce.h"
#include "fusedce/bf16.hpp"
#include "fusedce/dense_matrix.hpp"
#include "fusedce/errors.hpp"

namespace fusedce::detail {

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

class DeviceBuffer {
  public:
    DeviceBuffer() = default;
    explicit DeviceBuffer(std::size_t bytes) : bytes_(bytes) {
        if (bytes) cuda_check(cudaMalloc(&p_, bytes), "cudaMalloc");
    }
    DeviceBuffer(const DeviceBuffer&) = delete;
    DeviceBuffer& operator=(const DeviceBuffer&) = delete;
    DeviceBuffer(DeviceBuffer&& o) noexcept : p_(o.p_), bytes_(o.bytes_) { o.p_ = nullptr; }
    DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
        if (this != &o) {
            if (p_) cudaFree(p_);
            p_ = o.p_;
            bytes_ = o.bytes_;
            o.p_ = nullptr;
        }
        return *this;
    }
    ~DeviceBuffer() {
        if (p_) cudaFree(p_);
    }
    template <typename U = void>
    U* get() const noexcept {
        return static_cast<U*>(p_);
    }
    std::size_t bytes() const noexcept { return bytes_; }
    void upload(const void* src, std::size_t n) { cuda_check(cudaMemcpy(p_, src, n, cudaMemcpyHostToDevice), "H2D"); }
    void download(void* dst, std::size_t n) const {
        cuda_check(cudaMemcpy(dst, p_, n, cudaMemcpyDeviceToHost), "D2H");
    }

  private:
    void* p_ = nullptr;
    std::size_t bytes_ = 0;
};

class HandleCache {
  public:
    ~HandleCache() {
        for (auto& [dev, h] : handles_) fce_destroy(h);
    }
    fce_handle get(int device) {
        auto it = handles_.find(device);
        if (it != handles_.end()) return it->second;
        fce_handle h = nullptr;
        throw_status(fce_create(&h, device, nullptr), "fce_create");
        handles_[device] = h;
        return h;
    }

  private:
    std::map<int, fce_handle> handles_;
};

inline fce_handle handle_for(int device) {
    thread_local HandleCache cache;
    return cache.get(device);
}

template <typename T>
void require_float() {
    if constexpr (!std::is_same_v<T, float>)
        throw InvalidLayout("the sm_100a path computes bf16-in / fp32-accumulate: use T = float on the bf16 grid");
}

inline std::int64_t padded_ld(std::size_t cols) { return static_cast<std::int64_t>((cols + 7) / 8 * 8); }

// float rows on the bf16 grid -> device bf16 [rows, ld] (exact conversion).
// The rows go up as fp32 in chunks of <= 64 MB and are checked and converted
// on the device (fce_f32_to_bf16: off-grid values -> InvalidLayout), so the
// host never walks the V x D weights element by element.
inline DeviceBuffer upload_bf16(const float* src, std::size_t rows, std::size_t cols, std::int64_t ld,
                                const char* name) {
    int dev = 0;
    cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
    fce_handle h = handle_for(dev);
    DeviceBuffer buf(rows * static_cast<std::size_t>(ld) * sizeof(std::uint16_t));
    if (!rows || !cols) return buf;
    const std::size_t chunk = std::max<std::size_t>(1, (std::size_t(16) << 20) / cols);
    DeviceBuffer f32(std::min(chunk, rows) * cols * sizeof(float));
    cuda_check(cudaMemset(buf.get(), 0, buf.bytes()), "cudaMemset");
    for (std::size_t r0 = 0; r0 < rows; r0 += chunk) {
        const std::size_t nr = std::min(chunk, rows - r0);
        f32.upload(src + r0 * cols, nr * cols * sizeof(float));
        const fce_status s = fce_f32_to_bf16(h, f32.get<float>(), static_cast<std::int64_t>(nr),
                                             static_cast<std::int64_t>(cols), static_cast<std::int64_t>(cols),
                                             buf.get<std::uint16_t>() + r0 * static_cast<std::size_t>(ld), ld);
        if (s == FCE_INVALID_LAYOUT)
            throw InvalidLayout(std::string(name) + " has a value in rows [" + std::to_string(r0) + ", " +
                                std::to_string(r0 + nr) + ") that is not on the bf16 grid (round_to_bf16 first)");
        throw_status(s, "upload");
    }
    return buf;
}

inline DeviceBuffer upload_targets(const TargetVector& t) {
    DeviceBuffer buf(t.size() * sizeof(std::int64_t));
    buf.upload(t.values().data(), buf.bytes());
    return buf;
}

}  // namespace fusedce::detail
