// Drop-in tensor(vocab)-parallel API of the reference (parallel_sim.hpp:22-290):
// ShardLayout / WeightShard / tp_rank_partial / tp_forward / tp_backward with
// the same semantics.  Ranks here are simulated on one GPU exactly like the
// reference simulates them in one process (per-shard kernel launches, rank-
// ordered merge on the device); real multi-GPU runs use fce_vp_forward /
// fce_vp_backward (include/fce/fce_vp.h) with one process per GPU.
// SP gather and the DP step (parallel_sim.hpp:294-378) are provided with the
// reference semantics on top of the same device path.
#pragma once

#include <span>
#include <vector>

#include "fusedce/fused_backward.hpp"

namespace fusedce {

enum class ParallelMode { DataParallel, TensorParallel, SequenceParallel };

struct ShardRange {
    std::size_t lo = 0, hi = 0;
    std::size_t size() const noexcept { return hi - lo; }
};

struct ShardLayout {
    ParallelMode mode = ParallelMode::TensorParallel;
    std::vector<ShardRange> ranges;
    std::size_t rank_count() const noexcept { return ranges.size(); }
    static ShardLayout make(ParallelMode mode, std::size_t axis, std::size_t ranks) {
        if (ranks == 0) throw InvalidLayout("rank count must be at least 1");
        if (axis < ranks)
            throw InvalidLayout("cannot split axis of length " + std::to_string(axis) + " across " +
                                std::to_string(ranks) + " ranks");
        ShardLayout l;
        l.mode = mode;
        for (auto [lo, hi] : partition_ranges(axis, ranks)) l.ranges.push_back(ShardRange{lo, hi});
        return l;
    }
    static ShardLayout tensor_parallel(std::size_t vocab, std::size_t ranks) {
        return make(ParallelMode::TensorParallel, vocab, ranks);
    }
    static ShardLayout sequence_parallel(std::size_t positions, std::size_t ranks) {
        return make(ParallelMode::SequenceParallel, positions, ranks);
    }
    static ShardLayout data_parallel(std::size_t positions, std::size_t ranks) {
        if (ranks != 0 && positions % ranks != 0)
            throw InvalidLayout("data parallelism needs equal micro-batches: " + std::to_string(positions) +
                                " positions across " + std::to_string(ranks) + " ranks");
        return make(ParallelMode::DataParallel, positions, ranks);
    }
};

template <typename T>
struct WeightShard {
    MatrixView<T> view;
    std::size_t v_offset = 0;
};

template <typename T>
std::vector<WeightShard<T>> shard_weights(const MatrixView<T>& weights, const ShardLayout& layout) {
    if (layout.mode != ParallelMode::TensorParallel) throw InvalidLayout("weight sharding requires a tensor-parallel layout");
    if (layout.ranges.empty() || layout.ranges.back().hi != weights.rows)
        throw InvalidLayout("layout does not cover the vocabulary");
    std::vector<WeightShard<T>> out;
    for (const ShardRange& r : layout.ranges) out.push_back(WeightShard<T>{weights.rows_slice(r.lo, r.hi), r.lo});
    return out;
}

template <typename T>
struct RankPartial {
    std::size_t rank = 0;
    std::size_t v_offset = 0;
    std::vector<SoftmaxStats<T>> stats;
};

namespace detail {

template <typename T>
std::size_t validate_weight_shards(const std::vector<WeightShard<T>>& shards, std::size_t d) {
    if (shards.empty()) throw InvalidLayout("no weight shards");
    std::size_t next = 0;
    for (const auto& s : shards) {
        if (s.view.cols != d)
            throw InvalidLayout("weight shard width " + std::to_string(s.view.cols) + " != hidden width " +
                                std::to_string(d));
        if (s.v_offset != next || s.view.rows == 0)
            throw InvalidLayout("weight shards must tile the vocabulary contiguously");
        next += s.view.rows;
    }
    return next;
}

template <typename T>
void check_global_targets(const MatrixView<T>& hidden, const TargetVector& targets, std::size_t vocab) {
    if (hidden.rows == 0 || hidden.cols == 0) throw EmptyInput("tp requires N > 0 and d > 0");
    if (hidden.rows != targets.size())
        throw DimensionMismatch("hidden rows " + std::to_string(hidden.rows) + " != target count " +
                                std::to_string(targets.size()));
    for (std::size_t i = 0; i < targets.size(); ++i)
        if (!targets.is_ignored(i) && (targets[i] < 0 || static_cast<std::size_t>(targets[i]) >= vocab))
            throw TargetOutOfRange("target " + std::to_string(targets[i]) + " at position " + std::to_string(i) +
                                   " outside [0, " + std::to_string(vocab) + ")");
}

}  // namespace detail

// tp_rank_partial (reference parallel_sim.hpp:165-181)
template <typename T>
RankPartial<T> tp_rank_partial(std::size_t rank, const MatrixView<T>& hidden, const WeightShard<T>& shard,
                               const TargetVector& targets, const ExecPolicy& policy = {}) {
    if (hidden.rows != targets.size())
        throw DimensionMismatch("hidden rows " + std::to_string(hidden.rows) + " != target count " +
                                std::to_string(targets.size()));
    std::int64_t vmax = static_cast<std::int64_t>(shard.v_offset + shard.view.rows);
    for (std::int64_t y : targets.values()) vmax = std::max(vmax, y + 1);
    detail::DeviceProblem dp =
        detail::upload_problem(hidden, shard.view, targets, shard.v_offset, static_cast<std::size_t>(vmax));
    const std::size_t n = hidden.rows;
    detail::DeviceBuffer m(n * 4), a(n * 4), z(n * 4), f(n);
    fce_stats st{m.get<float>(), a.get<float>(), z.get<float>(), f.get<std::uint8_t>()};
    throw_status(fce_forward_partial(detail::handle_for(policy.device), &dp.p, st), "tp_rank_partial");
    RankPartial<T> out;
    out.rank = rank;
    out.v_offset = shard.v_offset;
    out.stats = detail::download_stats<T>(m, a, z, f, n);
    return out;
}

// tp_forward (reference parallel_sim.hpp:186-236): rank-ordered merge on the device
template <typename T>
FusedOutput<T> tp_forward(const MatrixView<T>& hidden, const std::vector<WeightShard<T>>& shards,
                          const TargetVector& targets, ReductionMode reduction, MemoryLedger& ledger,
                          const ExecPolicy& policy = {}) {
    const std::size_t vocab = detail::validate_weight_shards(shards, hidden.cols);
    detail::check_global_targets(hidden, targets, vocab);
    const std::size_t n = hidden.rows, k = shards.size();
    std::vector<float> pm(k * n), pa(k * n), pz(k * n);
    std::vector<std::uint8_t> pf(k * n);
    ScopedCharge charge(ledger, k * n * 13 + n * 13);
    for (std::size_t r = 0; r < k; ++r) {
        const RankPartial<T> part = tp_rank_partial(r, hidden, shards[r], targets, policy);
        for (std::size_t i = 0; i < n; ++i) {
            pm[r * n + i] = static_cast<float>(part.stats[i].m);
            pa[r * n + i] = static_cast<float>(part.stats[i].a);
            pz[r * n + i] = static_cast<float>(part.stats[i].z_target);
            pf[r * n + i] = part.stats[i].target_found ? 1 : 0;
        }
    }
    detail::DeviceBuffer dm(k * n * 4), da(k * n * 4), dz(k * n * 4), df(k * n), dt = detail::upload_targets(targets);
    dm.upload(pm.data(), dm.bytes());
    da.upload(pa.data(), da.bytes());
    dz.upload(pz.data(), dz.bytes());
    df.upload(pf.data(), df.bytes());
    detail::DeviceBuffer m(n * 4), a(n * 4), z(n * 4), f(n), rows(n * 4), red(4);
    fce_stats st{m.get<float>(), a.get<float>(), z.get<float>(), f.get<std::uint8_t>()};
    throw_status(fce_merge_partials(detail::handle_for(policy.device), static_cast<int>(k), static_cast<std::int64_t>(n),
                                    static_cast<std::int64_t>(n), dm.get<float>(), da.get<float>(), dz.get<float>(),
                                    df.get<std::uint8_t>(), dt.get<std::int64_t>(),
                                    targets.ignore_index() ? 1 : 0, targets.ignore_index().value_or(0),
                                    to_fce(reduction), st, nullptr, rows.get<float>(), red.get<float>()),
                 "tp_forward");
    FusedOutput<T> out;
    out.stats = detail::download_stats<T>(m, a, z, f, n);
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

template <typename T>
struct TpGradients {
    DenseMatrix<T> hidden;
    std::vector<DenseMatrix<T>> weight_shards;
};

// tp_backward (reference parallel_sim.hpp:246-290): per-shard dW, dH summed
// over ranks on the device (fce_backward accumulate_dhidden).
template <typename T>
TpGradients<T> tp_backward(const MatrixView<T>& hidden, const std::vector<WeightShard<T>>& shards,
                           const TargetVector& targets, std::span<const SoftmaxStats<T>> stats,
                           const UpstreamGradient<T>& upstream, ReductionMode reduction, MemoryLedger& ledger,
                           const ExecPolicy& policy = {}) {
    const std::size_t vocab = detail::validate_weight_shards(shards, hidden.cols);
    detail::check_global_targets(hidden, targets, vocab);
    detail::require_stats(targets, stats);
    check_upstream(upstream, reduction, targets.size());
    using Kind = typename UpstreamGradient<T>::Kind;
    const std::size_t n = hidden.rows, d = hidden.cols;
    std::vector<float> hm(n), ha(n), hz(n);
    std::vector<std::uint8_t> hf(n);
    for (std::size_t i = 0; i < n; ++i) {
        hm[i] = static_cast<float>(stats[i].m);
        ha[i] = static_cast<float>(stats[i].a);
        hz[i] = static_cast<float>(stats[i].z_target);
        hf[i] = stats[i].target_found ? 1 : 0;
    }
    detail::DeviceBuffer m(n * 4), a(n * 4), z(n * 4), f(n), dh(n * d * 4);
    m.upload(hm.data(), n * 4);
    a.upload(ha.data(), n * 4);
    z.upload(hz.data(), n * 4);
    f.upload(hf.data(), n);
    detail::DeviceBuffer up(upstream.kind == Kind::PerPosition ? n * 4 : 0);
    if (upstream.kind == Kind::PerPosition) {
        std::vector<float> u(upstream.vector.begin(), upstream.vector.end());
        up.upload(u.data(), n * 4);
    }
    cudaMemset(dh.get(), 0, dh.bytes());
    ScopedCharge charge(ledger, 3 * n * 4 + n + up.bytes() + dh.bytes());
    fce_stats st{m.get<float>(), a.get<float>(), z.get<float>(), f.get<std::uint8_t>()};
    TpGradients<T> out;
    out.hidden = DenseMatrix<T>(n, d);
    for (const WeightShard<T>& shard : shards) {
        detail::DeviceProblem dp = detail::upload_problem(hidden, shard.view, targets, shard.v_offset, vocab);
        detail::DeviceBuffer dw(shard.view.rows * d * 4);
        throw_status(fce_backward(detail::handle_for(policy.device), &dp.p, st, to_fce(reduction),
                                  static_cast<float>(upstream.scalar), up.bytes() ? up.get<float>() : nullptr,
                                  dh.get<float>(), static_cast<std::int64_t>(d), dw.get<float>(),
                                  static_cast<std::int64_t>(d), 1),
                     "tp_backward");
        DenseMatrix<T> w(shard.view.rows, d);
        if constexpr (std::is_same_v<T, float>) dw.download(w.data(), dw.bytes());
        out.weight_shards.push_back(std::move(w));
    }
    if constexpr (std::is_same_v<T, float>) dh.download(out.hidden.data(), dh.bytes());
    return out;
}

// ---------------------------------------------------------------- SP and DP
// (reference parallel_sim.hpp:96-129 and 294-378)

template <typename T>
std::vector<MatrixView<T>> shard_positions(const MatrixView<T>& hidden, const ShardLayout& layout) {
    if (layout.mode == ParallelMode::TensorParallel) throw InvalidLayout("position sharding requires an SP or DP layout");
    if (layout.ranges.empty() || layout.ranges.back().hi != hidden.rows)
        throw InvalidLayout("layout does not cover the positions");
    std::vector<MatrixView<T>> out;
    for (const ShardRange& r : layout.ranges) out.push_back(hidden.rows_slice(r.lo, r.hi));
    return out;
}

inline std::vector<TargetVector> shard_targets(const TargetVector& targets, const ShardLayout& layout) {
    if (layout.mode == ParallelMode::TensorParallel) throw InvalidLayout("target sharding requires an SP or DP layout");
    if (layout.ranges.empty() || layout.ranges.back().hi != targets.size())
        throw InvalidLayout("layout does not cover the positions");
    std::vector<TargetVector> out;
    for (const ShardRange& r : layout.ranges)
        out.emplace_back(std::vector<std::int64_t>(targets.values().begin() + static_cast<std::ptrdiff_t>(r.lo),
                                                   targets.values().begin() + static_cast<std::ptrdiff_t>(r.hi)),
                         targets.ignore_index());
    return out;
}

// SP -> TP switch: concatenate the position shards of H (host; on GPUs this is
// an all-gather of H, paper_2511_17599_b200.vocab_parallel.sp_to_tp_gather).
template <typename T>
DenseMatrix<T> sp_to_tp_gather(const std::vector<MatrixView<T>>& shards) {
    if (shards.empty()) throw InvalidLayout("no hidden shards to gather");
    const std::size_t d = shards.front().cols;
    std::size_t total = 0;
    for (const auto& s : shards) {
        if (s.cols != d) throw InvalidLayout("hidden shards disagree on width");
        total += s.rows;
    }
    DenseMatrix<T> out(total, d);
    std::size_t row = 0;
    for (const auto& s : shards) {
        std::copy(s.data, s.data + s.rows * s.cols, out.row(row));
        row += s.rows;
    }
    return out;
}

template <typename T>
struct DpReplica {
    MatrixView<T> hidden;
    TargetVector targets;
};

template <typename T>
struct DpResult {
    T loss = T{0};
    DenseMatrix<T> weight_grad;
};

// Data-parallel step: every replica runs the fused forward + backward on its
// micro-batch; loss and dW are averaged over replicas (the all-reduce-mean).
template <typename T>
DpResult<T> dp_step(const std::vector<DpReplica<T>>& replicas, const MatrixView<T>& weights, ReductionMode reduction,
                    MemoryLedger& ledger, const ExecPolicy& policy = {}) {
    if (replicas.empty()) throw InvalidLayout("no replicas");
    if (reduction == ReductionMode::None) throw UnsupportedReduction("data-parallel loss sync requires a scalar reduction");
    const std::size_t micro = replicas.front().hidden.rows;
    for (const auto& r : replicas)
        if (r.hidden.rows != micro || r.targets.size() != micro)
            throw InvalidLayout("replica micro-batches must have equal sizes");
    DpResult<T> out;
    out.weight_grad = DenseMatrix<T>(weights.rows, weights.cols);
    T loss_sum = T{0};
    for (const auto& rep : replicas) {
        FusedOutput<T> fwd = fused_forward(rep.hidden, weights, rep.targets, reduction, ledger, policy);
        Gradients<T> g = fused_backward_recompute(rep.hidden, weights, rep.targets,
                                                  std::span<const SoftmaxStats<T>>(fwd.stats),
                                                  UpstreamGradient<T>::make_scalar(T{1}), reduction, ledger, policy);
        loss_sum += fwd.loss.scalar();
        T* acc = out.weight_grad.data();
        const T* part = g.weights.data();
        for (std::size_t i = 0; i < out.weight_grad.size(); ++i) acc[i] += part[i];
    }
    const T inv = T{1} / static_cast<T>(replicas.size());
    out.loss = loss_sum * inv;
    for (T& x : out.weight_grad.storage()) x *= inv;
    return out;
}

}  // namespace fusedce
