// bf16 grid helpers (reference bf16.hpp:14-36): round-to-nearest-even onto the
// top 16 bits of the float encoding.  The device path consumes bf16, so a
// float input is accepted only if it already lies on this grid.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>

namespace fusedce {

inline float round_bf16(float x) noexcept {
    if (std::isnan(x)) return x;
    std::uint32_t bits;
    std::memcpy(&bits, &x, 4);
    bits += 0x7FFFu + ((bits >> 16) & 1u);
    bits &= 0xFFFF0000u;
    float y;
    std::memcpy(&y, &bits, 4);
    return y;
}

inline double round_bf16(double x) noexcept { return static_cast<double>(round_bf16(static_cast<float>(x))); }

inline bool is_bf16_value(float x) noexcept { return std::isnan(x) || round_bf16(x) == x; }

// raw bf16 bits of a float that is on the grid (exact)
inline std::uint16_t bf16_bits(float x) noexcept {
    std::uint32_t bits;
    std::memcpy(&bits, &x, 4);
    return static_cast<std::uint16_t>(bits >> 16);
}

}  // namespace fusedce
