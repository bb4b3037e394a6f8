// Drop-in fused backward (reference fused_backward.hpp:118-202): recompute
// logits from H and W with the cached stats and return dH, dW, computed by the
// persistent sm_100a backward behind fce_backward.
#pragma once

#include <span>
#include <vector>

#include "fusedce/fused_forward.hpp"

namespace fusedce {

namespace detail {

template <typename T>
void require_stats(const TargetVector& targets, std::span<const SoftmaxStats<T>> stats) {
    if (stats.size() != targets.size())
        throw MissingStats("stats cache has " + std::to_string(stats.size()) + " entries for " +
                           std::to_string(targets.size()) + " positions");
}

template <typename T>
Gradients<T> backward_device(const MatrixView<T>& hidden, const MatrixView<T>& weights, const TargetVector& targets,
                             std::span<const SoftmaxStats<T>> stats, ReductionMode reduction, T up_scalar,
                             const std::vector<T>* up_rows, MemoryLedger& ledger, const ExecPolicy& policy) {
    const ProblemDims dims = validate_problem(hidden, weights, targets);
    require_stats(targets, stats);
    DeviceProblem dp = upload_problem(hidden, weights, targets);
    const std::size_t n = dims.n, d = dims.d, v = dims.v;
    std::vector<float> hm(n), ha(n), hz(n);
    std::vector<std::uint8_t> hf(n);
    for (std::size_t i = 0; i < n; ++i) {
        hm[i] = static_cast<float>(stats[i].m);
        ha[i] = static_cast<float>(stats[i].a);
        hz[i] = static_cast<float>(stats[i].z_target);
        hf[i] = stats[i].target_found ? 1 : 0;
    }
    DeviceBuffer m(n * 4), a(n * 4), z(n * 4), f(n), up(up_rows ? n * 4 : 0), dh(n * d * 4), dw(v * d * 4);
    m.upload(hm.data(), n * 4);
    a.upload(ha.data(), n * 4);
    z.upload(hz.data(), n * 4);
    f.upload(hf.data(), n);
    if (up_rows) {
        std::vector<float> u(up_rows->begin(), up_rows->end());
        up.upload(u.data(), n * 4);
    }
    // the reference's accounting (fused_backward.hpp:128, 135): gamma and the
    // two gradient buffers; the device path has no private dW partials
    ScopedCharge charge(ledger, n * sizeof(T) + (n + v) * d * sizeof(T));
    fce_stats st{m.get<float>(), a.get<float>(), z.get<float>(), f.get<std::uint8_t>()};
    throw_status(fce_backward(handle_for(policy.device), &dp.p, st, to_fce(reduction), static_cast<float>(up_scalar),
                              up_rows ? up.get<float>() : nullptr, dh.get<float>(), static_cast<std::int64_t>(d),
                              dw.get<float>(), static_cast<std::int64_t>(d), 0),
                 "fused_backward_recompute");
    Gradients<T> g{DenseMatrix<T>(n, d), DenseMatrix<T>(v, d)};
    if constexpr (std::is_same_v<T, float>) {
        dh.download(g.hidden.data(), dh.bytes());
        dw.download(g.weights.data(), dw.bytes());
    }
    return g;
}

}  // namespace detail

// fused_backward_recompute (reference fused_backward.hpp:118-140)
template <typename T>
Gradients<T> fused_backward_recompute(const MatrixView<T>& hidden, const MatrixView<T>& weights,
                                      const TargetVector& targets, std::span<const SoftmaxStats<T>> stats,
                                      const UpstreamGradient<T>& upstream, ReductionMode reduction,
                                      MemoryLedger& ledger, const ExecPolicy& policy = {}) {
    check_upstream(upstream, reduction, targets.size());
    using Kind = typename UpstreamGradient<T>::Kind;
    return detail::backward_device(hidden, weights, targets, stats, reduction, upstream.scalar,
                                   upstream.kind == Kind::PerPosition ? &upstream.vector : nullptr, ledger, policy);
}

template <typename T>
struct PartialGradients {
    DenseMatrix<T> hidden;
    DenseMatrix<T> weights;
};

template <typename T>
struct PartialGradOutput {
    LossValue<T> loss;
    std::vector<SoftmaxStats<T>> stats;
    PartialGradients<T> partials;
};

// Alg. 3 (reference fused_backward.hpp:162-188): forward + unscaled partials.
template <typename T>
PartialGradOutput<T> fused_forward_with_partial_grads(const MatrixView<T>& hidden, const MatrixView<T>& weights,
                                                      const TargetVector& targets, ReductionMode reduction,
                                                      MemoryLedger& ledger, const ExecPolicy& policy = {}) {
    if (reduction == ReductionMode::None)
        throw UnsupportedReduction("partial-gradient accumulation requires a scalar-upstream reduction (mean or sum)");
    PartialGradOutput<T> out;
    FusedOutput<T> fwd = fused_forward(hidden, weights, targets, reduction, ledger, policy);
    out.loss = std::move(fwd.loss);
    out.stats = std::move(fwd.stats);
    Gradients<T> g = detail::backward_device(hidden, weights, targets, std::span<const SoftmaxStats<T>>(out.stats),
                                             ReductionMode::Sum, T{1}, static_cast<const std::vector<T>*>(nullptr),
                                             ledger, policy);
    out.partials.hidden = std::move(g.hidden);
    out.partials.weights = std::move(g.weights);
    return out;
}

// Alg. 4 (reference fused_backward.hpp:193-202)
template <typename T>
Gradients<T> scale_partial_grads(PartialGradients<T> partials, T gamma_eff) {
    for (T& x : partials.hidden.storage()) x *= gamma_eff;
    for (T& x : partials.weights.storage()) x *= gamma_eff;
    return Gradients<T>{std::move(partials.hidden), std::move(partials.weights)};
}

}  // namespace fusedce
