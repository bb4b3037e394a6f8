// extern "C" shim over the UNMODIFIED reference headers (compiled in place
// from /root/reference/proj/include with -Dfusedce=fusedce_ref; see
// oracle/Makefile target `ref`).  TEST INFRASTRUCTURE ONLY: used by tests/ to
// pin the C restatement and golden fixtures, and by bench.py's reference /
// cpu_baseline arm.  No reference source is copied into this repository.
#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <vector>

#include "fusedce/errors.hpp"
#include "fusedce/fused_backward.hpp"
#include "fusedce/fused_forward.hpp"
#include "fusedce/instance.hpp"
#include "fusedce/parallel_sim.hpp"
#include "fusedce/reference.hpp"

using namespace fusedce;

namespace {

template <typename Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return 0;
    } catch (const Error& e) {
        return static_cast<int>(e.code()) + 1;
    } catch (...) {
        return 100;
    }
}

ReductionMode red(int r) {
    return r == 0 ? ReductionMode::Mean : (r == 1 ? ReductionMode::Sum : ReductionMode::None);
}

TargetVector tv(const int64_t* y, size_t n, int has_ignore, int64_t ignore_index) {
    std::vector<int64_t> t(y, y + n);
    return has_ignore ? TargetVector(std::move(t), ignore_index) : TargetVector(std::move(t));
}

void put_stats(const std::vector<SoftmaxStats<float>>& s, float* m, float* a, float* zt,
               uint8_t* f) {
    for (size_t i = 0; i < s.size(); ++i) {
        if (m) m[i] = s[i].m;
        if (a) a[i] = s[i].a;
        if (zt) zt[i] = s[i].z_target;
        if (f) f[i] = s[i].target_found ? 1 : 0;
    }
}

std::vector<SoftmaxStats<float>> get_stats(size_t n, const float* m, const float* a,
                                           const float* zt, const uint8_t* f) {
    std::vector<SoftmaxStats<float>> s(n);
    for (size_t i = 0; i < n; ++i) {
        s[i].m = m[i];
        s[i].a = a[i];
        s[i].z_target = zt ? zt[i] : 0.f;
        s[i].target_found = f[i] != 0;
    }
    return s;
}

void put_loss(const LossValue<float>& l, float* rows, float* reduced) {
    if (l.per_position && rows) std::memcpy(rows, l.per_position->data(), l.per_position->size() * 4);
    if (l.reduced && reduced) *reduced = *l.reduced;
}

UpstreamGradient<float> upstream(int reduction, float s, const float* rows, size_t n) {
    if (reduction == 2 && rows) return UpstreamGradient<float>::make_per_position(std::vector<float>(rows, rows + n));
    if (reduction != 2 && rows) return UpstreamGradient<float>::make_per_position(std::vector<float>(rows, rows + n));
    return UpstreamGradient<float>::make_scalar(s);
}

}  // namespace

extern "C" {

int ref_make_instance(size_t n, size_t d, size_t v, uint64_t seed, int64_t ignore_index,
                      double ignore_fraction, int round, float* H, float* W, int64_t* Y) {
    return guarded([&] {
        Instance<float> inst = ignore_fraction > 0.0
                                   ? make_random_instance_with_ignores<float>(n, d, v, seed, ignore_index, ignore_fraction)
                                   : make_random_instance<float>(n, d, v, seed);
        if (round) {
            inst.hidden.round_to_bf16();
            inst.weights.round_to_bf16();
        }
        if (H) std::memcpy(H, inst.hidden.data(), inst.hidden.bytes());
        if (W) std::memcpy(W, inst.weights.data(), inst.weights.bytes());
        if (Y) std::memcpy(Y, inst.targets.values().data(), n * sizeof(int64_t));
    });
}

int ref_fused_forward(const float* H, const float* W, size_t n, size_t d, size_t v, const int64_t* Y,
                      int has_ignore, int64_t ignore_index, int reduction, size_t window,
                      size_t workers, float* m, float* a, float* zt, uint8_t* found,
                      float* loss_rows, float* loss_reduced, size_t* ledger_peak) {
    return guarded([&] {
        MemoryLedger ledger;
        ExecPolicy pol;
        pol.workers = workers ? workers : 1;
        MatrixView<float> hv(H, n, d), wv(W, v, d);
        FusedOutput<float> out =
            window ? fused_forward_windowed(hv, wv, tv(Y, n, has_ignore, ignore_index), red(reduction),
                                            WindowConfig{window, pol.workers}, ledger, pol)
                   : fused_forward(hv, wv, tv(Y, n, has_ignore, ignore_index), red(reduction), ledger, pol);
        put_stats(out.stats, m, a, zt, found);
        put_loss(out.loss, loss_rows, loss_reduced);
        if (ledger_peak) *ledger_peak = ledger.peak_bytes();
    });
}

int ref_fused_backward(const float* H, const float* W, size_t n, size_t d, size_t v, const int64_t* Y,
                       int has_ignore, int64_t ignore_index, const float* m, const float* a,
                       const float* zt, const uint8_t* found, int reduction, float up_scalar,
                       const float* up_rows, size_t workers, float* dH, float* dW) {
    return guarded([&] {
        MemoryLedger ledger;
        ExecPolicy pol;
        pol.workers = workers ? workers : 1;
        const auto stats = get_stats(n, m, a, zt, found);
        Gradients<float> g = fused_backward_recompute(
            MatrixView<float>(H, n, d), MatrixView<float>(W, v, d), tv(Y, n, has_ignore, ignore_index),
            std::span<const SoftmaxStats<float>>(stats), upstream(reduction, up_scalar, up_rows, n),
            red(reduction), ledger, pol);
        if (dH) std::memcpy(dH, g.hidden.data(), g.hidden.bytes());
        if (dW) std::memcpy(dW, g.weights.data(), g.weights.bytes());
    });
}

int ref_partial_grads(const float* H, const float* W, size_t n, size_t d, size_t v, const int64_t* Y,
                      int has_ignore, int64_t ignore_index, int reduction, float gamma_eff,
                      float* loss_reduced, float* dH, float* dW) {
    return guarded([&] {
        MemoryLedger ledger;
        PartialGradOutput<float> out = fused_forward_with_partial_grads(
            MatrixView<float>(H, n, d), MatrixView<float>(W, v, d), tv(Y, n, has_ignore, ignore_index),
            red(reduction), ledger);
        if (loss_reduced) *loss_reduced = out.loss.scalar();
        Gradients<float> g = scale_partial_grads(std::move(out.partials), gamma_eff);
        if (dH) std::memcpy(dH, g.hidden.data(), g.hidden.bytes());
        if (dW) std::memcpy(dW, g.weights.data(), g.weights.bytes());
    });
}

int ref_tp_forward(const float* H, const float* W, size_t n, size_t d, size_t v, const int64_t* Y,
                   int has_ignore, int64_t ignore_index, size_t ranks, int reduction, float* m,
                   float* a, float* zt, uint8_t* found, float* loss_rows, float* loss_reduced) {
    return guarded([&] {
        MemoryLedger ledger;
        MatrixView<float> wv(W, v, d);
        const auto shards = shard_weights(wv, ShardLayout::tensor_parallel(v, ranks));
        FusedOutput<float> out = tp_forward(MatrixView<float>(H, n, d), shards,
                                            tv(Y, n, has_ignore, ignore_index), red(reduction), ledger);
        put_stats(out.stats, m, a, zt, found);
        put_loss(out.loss, loss_rows, loss_reduced);
    });
}

int ref_tp_rank_partial(const float* H, const float* W_shard, size_t n, size_t d, size_t v_rows,
                        size_t v_offset, const int64_t* Y, int has_ignore, int64_t ignore_index,
                        float* m, float* a, float* zt, uint8_t* found) {
    return guarded([&] {
        WeightShard<float> sh{MatrixView<float>(W_shard, v_rows, d), v_offset};
        RankPartial<float> p = tp_rank_partial(0, MatrixView<float>(H, n, d), sh, tv(Y, n, has_ignore, ignore_index));
        put_stats(p.stats, m, a, zt, found);
    });
}

int ref_tp_backward(const float* H, const float* W, size_t n, size_t d, size_t v, const int64_t* Y,
                    int has_ignore, int64_t ignore_index, size_t ranks, const float* m, const float* a,
                    const float* zt, const uint8_t* found, int reduction, float up_scalar,
                    const float* up_rows, float* dH, float* dW) {
    return guarded([&] {
        MemoryLedger ledger;
        MatrixView<float> wv(W, v, d);
        const auto shards = shard_weights(wv, ShardLayout::tensor_parallel(v, ranks));
        const auto stats = get_stats(n, m, a, zt, found);
        TpGradients<float> g = tp_backward(MatrixView<float>(H, n, d), shards, tv(Y, n, has_ignore, ignore_index),
                                           std::span<const SoftmaxStats<float>>(stats),
                                           upstream(reduction, up_scalar, up_rows, n), red(reduction), ledger);
        if (dH) std::memcpy(dH, g.hidden.data(), g.hidden.bytes());
        if (dW) {
            size_t row = 0;
            for (const auto& s : g.weight_shards) {
                std::memcpy(dW + row * d, s.data(), s.bytes());
                row += s.rows();
            }
        }
    });
}

int ref_two_stage(const float* H, const float* W, size_t n, size_t d, size_t v, const int64_t* Y,
                  int has_ignore, int64_t ignore_index, int reduction, float up_scalar,
                  const float* up_rows, float* loss_rows, float* loss_reduced, float* dH, float* dW) {
    return guarded([&] {
        MemoryLedger ledger;
        MatrixView<float> hv(H, n, d), wv(W, v, d);
        const auto t = tv(Y, n, has_ignore, ignore_index);
        DenseMatrix<float> z = project_logits(hv, wv, ledger);
        put_loss(ce_loss_from_logits(MatrixView<float>(z), t, red(reduction)), loss_rows, loss_reduced);
        if (dH || dW) {
            Gradients<float> g = reference_backward(hv, wv, t, upstream(reduction, up_scalar, up_rows, n),
                                                    red(reduction), ledger);
            if (dH) std::memcpy(dH, g.hidden.data(), g.hidden.bytes());
            if (dW) std::memcpy(dW, g.weights.data(), g.weights.bytes());
        }
    });
}

int ref_stats_example(double* out) {
    // softmax_stats.hpp recurrence on logits (0, 1, 2), target 2
    // (the reference's worked example, tests/test_core_types.cpp:281-302)
    return guarded([&] {
        SoftmaxStats<double> s;
        s.update(0.0);
        s.update(1.0);
        s.update(2.0);
        s.update_target(2.0);
        out[0] = s.a;
        out[1] = s.logsumexp();
        out[2] = s.loss();
        SoftmaxStats<double> s1, s2;
        s1.m = 1.0; s1.a = 2.0; s2.m = 3.0; s2.a = 1.0;
        out[3] = merge_stats(s1, s2).a;
    });
}

}  // extern "C"
