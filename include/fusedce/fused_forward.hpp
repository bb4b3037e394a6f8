// Drop-in fused forward (reference fused_forward.hpp:21-195): same types and
// signatures, computed by the sm_100a kernels behind fce_forward.  Inputs are
// host MatrixViews (copied to the GPU per call); outputs are host values.
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <vector>

#include "fusedce/dense_matrix.hpp"
#include "fusedce/detail/device.hpp"
#include "fusedce/exec.hpp"
#include "fusedce/memory_ledger.hpp"
#include "fusedce/reduction.hpp"
#include "fusedce/softmax_stats.hpp"

namespace fusedce {

template <typename T>
struct FusedOutput {
    LossValue<T> loss;
    std::vector<SoftmaxStats<T>> stats;
};

struct WindowConfig {
    std::size_t window_size = 0;
    std::size_t worker_count = 1;
};

namespace detail {

struct DeviceProblem {
    DeviceBuffer hidden, weight, targets;
    fce_problem p{};
};

template <typename T>
DeviceProblem upload_problem(const MatrixView<T>& hidden, const MatrixView<T>& weights, const TargetVector& targets,
                             std::size_t v_offset = 0, std::size_t v_total = 0) {
    require_float<T>();
    DeviceProblem dp;
    const std::int64_t ld = padded_ld(hidden.cols);
    if constexpr (std::is_same_v<T, float>) {
        dp.hidden = upload_bf16(hidden.data, hidden.rows, hidden.cols, ld, "hidden");
        dp.weight = upload_bf16(weights.data, weights.rows, weights.cols, ld, "weights");
    }
    dp.targets = upload_targets(targets);
    dp.p.hidden = dp.hidden.get();
    dp.p.ldh = ld;
    dp.p.weight = dp.weight.get();
    dp.p.ldw = ld;
    dp.p.n = static_cast<std::int64_t>(hidden.rows);
    dp.p.d = static_cast<std::int64_t>(hidden.cols);
    dp.p.v = static_cast<std::int64_t>(weights.rows);
    dp.p.v_offset = static_cast<std::int64_t>(v_offset);
    dp.p.v_total = static_cast<std::int64_t>(v_total);
    dp.p.targets = dp.targets.get<std::int64_t>();
    dp.p.has_ignore = targets.ignore_index().has_value() ? 1 : 0;
    dp.p.ignore_index = targets.ignore_index().value_or(0);
    return dp;
}

inline std::size_t staged_bytes(const DeviceProblem& dp) {
    return dp.hidden.bytes() + dp.weight.bytes() + dp.targets.bytes();
}

template <typename T>
std::vector<SoftmaxStats<T>> download_stats(const DeviceBuffer& m, const DeviceBuffer& a, const DeviceBuffer& z,
                                            const DeviceBuffer& f, std::size_t n) {
    std::vector<float> hm(n), ha(n), hz(n);
    std::vector<std::uint8_t> hf(n);
    m.download(hm.data(), n * 4);
    a.download(ha.data(), n * 4);
    z.download(hz.data(), n * 4);
    f.download(hf.data(), n);
    std::vector<SoftmaxStats<T>> out(n);
    for (std::size_t i = 0; i < n; ++i) out[i] = SoftmaxStats<T>{hm[i], ha[i], hz[i], hf[i] != 0};
    return out;
}

template <typename T>
FusedOutput<T> forward_device(const MatrixView<T>& hidden, const MatrixView<T>& weights, const TargetVector& targets,
                              ReductionMode reduction, std::size_t window, MemoryLedger& ledger,
                              const ExecPolicy& policy) {
    const ProblemDims dims = validate_problem(hidden, weights, targets);
    DeviceProblem dp = upload_problem(hidden, weights, targets);
    const std::size_t n = dims.n;
    DeviceBuffer m(n * 4), a(n * 4), z(n * 4), f(n), rows(n * 4), red(4);
    // the reference's accounting of forward_core (fused_forward.hpp:103-105):
    // merged + window stats and the per-row losses, independent of V.  The
    // device copies of the inputs are staging, not auxiliary memory (the
    // library's own workspace is reported by fce_workspace_bytes).
    ScopedCharge charge(ledger, 2 * n * sizeof(SoftmaxStats<T>) + n * sizeof(T));
    fce_handle h = handle_for(policy.device);
    fce_stats st{m.get<float>(), a.get<float>(), z.get<float>(), f.get<std::uint8_t>()};
    throw_status(fce_forward(h, &dp.p, to_fce(reduction), static_cast<std::int64_t>(window), st, nullptr,
                             rows.get<float>(), red.get<float>()),
                 "fused_forward");
    FusedOutput<T> out;
    out.stats = download_stats<T>(m, a, z, f, n);
    if (reduction == ReductionMode::None) {
        std::vector<float> hr(n);
        rows.download(hr.data(), n * 4);
        out.loss.per_position = std::vector<T>(hr.begin(), hr.end());
    } else {
        float r = 0.f;
        red.download(&r, 4);
        out.loss.reduced = static_cast<T>(r);
    }
    return out;
}

}  // namespace detail

// fused_forward (reference fused_forward.hpp:161-172)
template <typename T>
FusedOutput<T> fused_forward(const MatrixView<T>& hidden, const MatrixView<T>& weights, const TargetVector& targets,
                             ReductionMode reduction, MemoryLedger& ledger, const ExecPolicy& policy = {}) {
    return detail::forward_device(hidden, weights, targets, reduction, 0, ledger, policy);
}

// fused_forward_windowed (reference fused_forward.hpp:177-195); the window
// becomes the split-V factor of the tile schedule (rounded to 256 columns).
template <typename T>
FusedOutput<T> fused_forward_windowed(const MatrixView<T>& hidden, const MatrixView<T>& weights,
                                      const TargetVector& targets, ReductionMode reduction, const WindowConfig& cfg,
                                      MemoryLedger& ledger, const ExecPolicy& policy = {}) {
    if (cfg.window_size == 0) throw InvalidLayout("window size must be at least 1");
    if (cfg.worker_count == 0) throw InvalidLayout("worker count must be at least 1");
    validate_problem(hidden, weights, targets);
    return detail::forward_device(hidden, weights, targets, reduction, std::min(cfg.window_size, weights.rows), ledger,
                                  policy);
}

// stream_stats (reference fused_forward.hpp:137-154): one row over the
// vocabulary range [lo, hi); the empty range is the identity.
template <typename T>
SoftmaxStats<T> stream_stats(std::span<const T> h, const MatrixView<T>& weights, std::optional<std::int64_t> target,
                             std::size_t lo, std::size_t hi, const ExecPolicy& policy = {}) {
    if (h.size() != weights.cols)
        throw DimensionMismatch("hidden length " + std::to_string(h.size()) + " != weight cols " +
                                std::to_string(weights.cols));
    if (lo > hi || hi > weights.rows)
        throw DimensionMismatch("vocab range [" + std::to_string(lo) + ", " + std::to_string(hi) +
                                ") not contained in [0, " + std::to_string(weights.rows) + ")");
    if (lo == hi) return SoftmaxStats<T>{};
    // target outside [lo, hi) (or none): a sentinel the kernel never matches —
    // the reference never validates it, the result just has found = false
    const std::int64_t y = target.value_or(-1);
    const bool in_range = y >= static_cast<std::int64_t>(lo) && y < static_cast<std::int64_t>(hi);
    TargetVector tv(std::vector<std::int64_t>{in_range ? y : static_cast<std::int64_t>(hi)});
    MatrixView<T> row(h.data(), 1, h.size());
    detail::DeviceProblem dp = detail::upload_problem(row, weights.rows_slice(lo, hi), tv, lo, 0);
    dp.p.v_total = static_cast<std::int64_t>(std::max<std::size_t>(hi + 1, weights.rows + 1));
    detail::DeviceBuffer m(4), a(4), z(4), f(1);
    fce_stats st{m.get<float>(), a.get<float>(), z.get<float>(), f.get<std::uint8_t>()};
    throw_status(fce_forward_partial(detail::handle_for(policy.device), &dp.p, st), "stream_stats");
    return detail::download_stats<T>(m, a, z, f, 1)[0];
}

}  // namespace fusedce
