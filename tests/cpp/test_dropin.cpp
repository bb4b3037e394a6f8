// C++ parity tests of the drop-in API (include/fusedce) against the CPU
// oracle (oracle/liboracle.so, test infrastructure), re-expressing the
// reference's own unit tests (proj/tests/*.cpp) for the device path.
// Built by `make tests/cpp/test_dropin`; run by tests/test_dropin_cpp.py on a B200.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "../../oracle/fce_oracle.h"
#include "fusedce/fused_backward.hpp"
#include "fusedce/fused_forward.hpp"
#include "fusedce/instance.hpp"
#include "fusedce/parallel_sim.hpp"

using namespace fusedce;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                 \
    do {                                                                            \
        ++g_checks;                                                                 \
        if (!(cond)) {                                                              \
            ++g_fail;                                                               \
            std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);   \
        }                                                                           \
    } while (0)

template <typename E, typename F>
static bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static double relmax(const float* got, const float* ref, std::size_t n) {
    double num = 0, den = 0;
    for (std::size_t i = 0; i < n; ++i) {
        num = std::max(num, std::fabs(double(got[i]) - double(ref[i])));
        den = std::max(den, std::fabs(double(ref[i])));
    }
    return den > 0 ? num / den : num;
}

static Instance<float> instance(std::size_t n, std::size_t d, std::size_t v, std::uint64_t seed, double frac) {
    Instance<float> inst = frac > 0 ? make_random_instance_with_ignores<float>(n, d, v, seed, -100, frac)
                                    : make_random_instance<float>(n, d, v, seed);
    inst.hidden.round_to_bf16();
    inst.weights.round_to_bf16();
    return inst;
}

static void test_worked_example() {
    // test_core_types.cpp:281-302
    SoftmaxStats<double> s;
    s.update(0.0);
    s.update(1.0);
    s.update(2.0);
    s.update_target(2.0);
    CHECK(std::fabs(s.a - 1.503214724408055) < 1e-14);
    CHECK(std::fabs(s.loss() - 0.4076059644443806) < 1e-13);
    SoftmaxStats<double> x, y;
    x.m = 1.0, x.a = 2.0, y.m = 3.0, y.a = 1.0;
    CHECK(std::fabs(merge_stats(x, y).a - 1.2706705664732254) < 1e-15);
}

static void test_forward_backward_vs_oracle(std::size_t n, std::size_t d, std::size_t v, std::uint64_t seed,
                                            double frac, ReductionMode red) {
    Instance<float> inst = instance(n, d, v, seed, frac);
    MemoryLedger ledger;
    FusedOutput<float> out = fused_forward(MatrixView<float>(inst.hidden), MatrixView<float>(inst.weights),
                                           inst.targets, red, ledger);
    CHECK(ledger.current_bytes() == 0);
    std::vector<orc_stats> st(n);
    std::vector<float> rows(n);
    float lred = 0;
    const int ign = inst.targets.ignore_index().has_value();
    const int orc_red = red == ReductionMode::Mean ? ORC_MEAN : (red == ReductionMode::Sum ? ORC_SUM : ORC_NONE);
    CHECK(orc_fused_forward(inst.hidden.data(), inst.weights.data(), n, d, v, 0, inst.targets.values().data(), ign,
                            -100, orc_red, 0, 1, st.data(), rows.data(), &lred) == 0);
    for (std::size_t i = 0; i < n; ++i) {
        CHECK(out.stats[i].target_found == (st[i].found != 0));
        if (st[i].found) CHECK(std::fabs(out.stats[i].logsumexp() - (st[i].m + std::log(st[i].a))) < 1e-3);
    }
    if (red != ReductionMode::None)
        CHECK(std::fabs(out.loss.scalar() - lred) <= 1e-3 * std::max(1.0f, std::fabs(lred)));
    else
        for (std::size_t i = 0; i < n; ++i) CHECK(std::fabs(out.loss.vector()[i] - rows[i]) < 1e-3 * std::max(1.f, rows[i]));

    std::vector<float> up(n, 0.75f);
    UpstreamGradient<float> ug = red == ReductionMode::None ? UpstreamGradient<float>::make_per_position(up)
                                                            : UpstreamGradient<float>::make_scalar(1.0f);
    Gradients<float> g = fused_backward_recompute(MatrixView<float>(inst.hidden), MatrixView<float>(inst.weights),
                                                  inst.targets, std::span<const SoftmaxStats<float>>(out.stats), ug,
                                                  red, ledger);
    CHECK(ledger.current_bytes() == 0);
    std::vector<float> dh(n * d), dw(v * d);
    CHECK(orc_fused_backward(inst.hidden.data(), inst.weights.data(), n, d, v, 0, 0, inst.targets.values().data(), ign,
                             -100, st.data(), orc_red, 1.0f, red == ReductionMode::None ? up.data() : nullptr, 1,
                             dh.data(), dw.data()) == 0);
    const double eh = relmax(g.hidden.data(), dh.data(), dh.size());
    const double ew = relmax(g.weights.data(), dw.data(), dw.size());
    std::printf("  n=%zu d=%zu v=%zu %s: dH err %.2e dW err %.2e\n", n, d, v, reduction_name(red).c_str(), eh, ew);
    CHECK(eh < 1e-2);
    CHECK(ew < 1e-2);
}

static void test_two_class_hand_example() {
    // test_reference.cpp:180-195
    DenseMatrix<float> h(1, 1, {1.0f});
    DenseMatrix<float> w(2, 1, {0.0f, 1.0f});
    TargetVector y({1});
    MemoryLedger ledger;
    auto out = fused_forward(MatrixView<float>(h), MatrixView<float>(w), y, ReductionMode::Sum, ledger);
    auto g = fused_backward_recompute(MatrixView<float>(h), MatrixView<float>(w), y,
                                      std::span<const SoftmaxStats<float>>(out.stats),
                                      UpstreamGradient<float>::make_scalar(1.0f), ReductionMode::Sum, ledger);
    const double sig = 0.2689414213699951;
    CHECK(std::fabs(g.weights.at(0, 0) - sig) < 1e-2 * sig);
    CHECK(std::fabs(g.weights.at(1, 0) + sig) < 1e-2 * sig);
    CHECK(std::fabs(g.hidden.at(0, 0) + sig) < 1e-2 * sig);
    CHECK(std::fabs(out.loss.scalar() - 0.3132616875182228) < 1e-5);
}

static void test_errors() {
    Instance<float> inst = instance(8, 16, 10, 1, 0.0);
    MemoryLedger ledger;
    MatrixView<float> hv(inst.hidden), wv(inst.weights);
    TargetVector bad({0, 1, 2, 3, 4, 5, 6, 10});
    CHECK(throws_as<TargetOutOfRange>([&] { fused_forward(hv, wv, bad, ReductionMode::Mean, ledger); }));
    CHECK(throws_as<DimensionMismatch>([&] { fused_forward(hv, wv.rows_slice(0, 10), TargetVector({0}), ReductionMode::Mean, ledger); }));
    DenseMatrix<float> off(8, 16);
    off.at(0, 0) = 0.1f;  // not on the bf16 grid
    CHECK(throws_as<InvalidLayout>([&] { fused_forward(MatrixView<float>(off), wv, inst.targets, ReductionMode::Mean, ledger); }));
    auto out = fused_forward(hv, wv, inst.targets, ReductionMode::Mean, ledger);
    CHECK(throws_as<InconsistentUpstream>([&] {
        fused_backward_recompute(hv, wv, inst.targets, std::span<const SoftmaxStats<float>>(out.stats),
                                 UpstreamGradient<float>::make_scalar(1.f), ReductionMode::None, ledger);
    }));
    std::vector<SoftmaxStats<float>> short_stats(out.stats.begin(), out.stats.begin() + 3);
    CHECK(throws_as<MissingStats>([&] {
        fused_backward_recompute(hv, wv, inst.targets, std::span<const SoftmaxStats<float>>(short_stats),
                                 UpstreamGradient<float>::make_scalar(1.f), ReductionMode::Mean, ledger);
    }));
    std::vector<SoftmaxStats<float>> lost = out.stats;
    lost[2].target_found = false;
    CHECK(throws_as<MissingStats>([&] {
        fused_backward_recompute(hv, wv, inst.targets, std::span<const SoftmaxStats<float>>(lost),
                                 UpstreamGradient<float>::make_scalar(1.f), ReductionMode::Mean, ledger);
    }));
    CHECK(throws_as<UnsupportedReduction>([&] { fused_forward_with_partial_grads(hv, wv, inst.targets, ReductionMode::None, ledger); }));
    CHECK(throws_as<InvalidLayout>([&] {
        fused_forward_windowed(hv, wv, inst.targets, ReductionMode::Mean, WindowConfig{0, 1}, ledger);
    }));
    DenseMatrix<double> hd(2, 2), wd(2, 2);
    CHECK(throws_as<InvalidLayout>([&] {
        fused_forward(MatrixView<double>(hd), MatrixView<double>(wd), TargetVector({0, 1}), ReductionMode::Mean, ledger);
    }));
    CHECK(ledger.current_bytes() == 0);
}

static void test_tp_matches_single() {
    Instance<float> inst = instance(40, 24, 301, 5, 0.25);
    MemoryLedger ledger;
    MatrixView<float> hv(inst.hidden), wv(inst.weights);
    auto single = fused_forward(hv, wv, inst.targets, ReductionMode::Mean, ledger);
    for (std::size_t ranks : {1u, 2u, 3u, 4u}) {
        auto shards = shard_weights(wv, ShardLayout::tensor_parallel(301, ranks));
        auto tp = tp_forward(hv, shards, inst.targets, ReductionMode::Mean, ledger);
        CHECK(std::fabs(tp.loss.scalar() - single.loss.scalar()) < 1e-5);
        for (std::size_t i = 0; i < 40; ++i) CHECK(tp.stats[i].target_found == single.stats[i].target_found);
        auto g1 = fused_backward_recompute(hv, wv, inst.targets, std::span<const SoftmaxStats<float>>(single.stats),
                                           UpstreamGradient<float>::make_scalar(1.f), ReductionMode::Mean, ledger);
        auto g2 = tp_backward(hv, shards, inst.targets, std::span<const SoftmaxStats<float>>(tp.stats),
                              UpstreamGradient<float>::make_scalar(1.f), ReductionMode::Mean, ledger);
        CHECK(relmax(g2.hidden.data(), g1.hidden.data(), g1.hidden.size()) < 1e-5);
        std::size_t row = 0;
        for (const auto& s : g2.weight_shards) {
            CHECK(relmax(s.data(), g1.weights.row(row), s.size()) < 1e-2);
            row += s.rows();
        }
    }
    CHECK(ledger.current_bytes() == 0);
    // stream_stats over a sub-range equals the rank partial of that range
    auto part = tp_rank_partial(0, hv, WeightShard<float>{wv.rows_slice(100, 200), 100}, inst.targets);
    auto s = stream_stats(inst.hidden.row_span(3), wv, std::optional<std::int64_t>(inst.targets[3]), 100, 200);
    CHECK(std::fabs(s.a - part.stats[3].a) < 1e-5 * std::max(1.f, part.stats[3].a));
    CHECK(s.target_found == part.stats[3].target_found);
}

static void test_sp_dp() {
    // SP round trip (test_parallel_sim.cpp:240-252) and DP equivalence (271-298)
    Instance<float> inst = instance(48, 16, 200, 9, 0.0);
    MemoryLedger ledger;
    MatrixView<float> hv(inst.hidden), wv(inst.weights);
    auto sp = shard_positions(hv, ShardLayout::sequence_parallel(48, 3));
    DenseMatrix<float> back = sp_to_tp_gather(sp);
    CHECK(back.storage() == inst.hidden.storage());
    auto layout = ShardLayout::data_parallel(48, 4);
    auto hs = shard_positions(hv, layout);
    auto ts = shard_targets(inst.targets, layout);
    std::vector<DpReplica<float>> reps;
    for (std::size_t r = 0; r < 4; ++r) reps.push_back(DpReplica<float>{hs[r], ts[r]});
    DpResult<float> dp = dp_step(reps, wv, ReductionMode::Mean, ledger);
    // equal micro-batches with mean reduction: DP mean == global mean
    auto full = fused_forward(hv, wv, inst.targets, ReductionMode::Mean, ledger);
    CHECK(std::fabs(dp.loss - full.loss.scalar()) < 1e-5);
    auto g = fused_backward_recompute(hv, wv, inst.targets, std::span<const SoftmaxStats<float>>(full.stats),
                                      UpstreamGradient<float>::make_scalar(1.f), ReductionMode::Mean, ledger);
    CHECK(relmax(dp.weight_grad.data(), g.weights.data(), g.weights.size()) < 1e-2);
    CHECK(throws_as<InvalidLayout>([&] { ShardLayout::data_parallel(10, 4); }));
    CHECK(throws_as<UnsupportedReduction>([&] { dp_step(reps, wv, ReductionMode::None, ledger); }));
    CHECK(ledger.current_bytes() == 0);
}

static void test_forward_memory_is_v_independent() {
    // test_fused_forward.cpp:217-232: the forward's auxiliary memory is
    // 2 N sizeof(SoftmaxStats) + N sizeof(T), whatever V is
    const std::size_t n = 16, d = 8;
    const std::size_t expect = 2 * n * sizeof(SoftmaxStats<float>) + n * sizeof(float);
    for (std::size_t v : {64, 512, 2048}) {
        Instance<float> inst = instance(n, d, v, 13, 0.0);
        MemoryLedger ledger;
        (void)fused_forward(MatrixView<float>(inst.hidden), MatrixView<float>(inst.weights), inst.targets,
                            ReductionMode::Mean, ledger);
        CHECK(ledger.peak_bytes() == expect);
        CHECK(ledger.current_bytes() == 0);
    }
}

int main() {
    std::printf("drop-in C++ API tests\n");
    test_worked_example();
    test_forward_backward_vs_oracle(256, 512, 32000, 42, 0.0, ReductionMode::Mean);
    test_forward_backward_vs_oracle(130, 40, 1000, 7, 0.25, ReductionMode::Sum);
    test_forward_backward_vs_oracle(33, 17, 257, 3, 0.3, ReductionMode::None);
    test_two_class_hand_example();
    test_errors();
    test_tp_matches_single();
    test_sp_dp();
    test_forward_memory_is_v_independent();
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
