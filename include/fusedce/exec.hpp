// Execution policy and the ceil-first partition of the reference
// (exec.hpp:17-41).  `workers` / `vocab_tile` / `d_tile` drive CPU threads in
// the reference; on the device they are accepted and ignored (the tile
// schedule is the library's), except that `device` selects the GPU.
#pragma once

#include <cstddef>
#include <utility>
#include <vector>

#include "fusedce/errors.hpp"

namespace fusedce {

struct ExecPolicy {
    std::size_t workers = 1;
    std::size_t vocab_tile = 64;
    std::size_t d_tile = 64;
    int device = 0;
};

inline std::vector<std::pair<std::size_t, std::size_t>> partition_ranges(std::size_t total, std::size_t parts) {
    if (parts == 0) throw InvalidLayout("cannot partition into 0 parts");
    std::vector<std::pair<std::size_t, std::size_t>> out(parts);
    std::size_t lo = 0;
    for (std::size_t p = 0; p < parts; ++p) {
        const std::size_t len = total / parts + (p < total % parts ? 1 : 0);
        out[p] = {lo, lo + len};
        lo += len;
    }
    return out;
}

}  // namespace fusedce
