// End-to-end timing of the drop-in C++ API (include/fusedce) with HOST buffers:
// what a caller of the reference's fused_forward / fused_backward_recompute
// gets when it switches the include path.  Every call uploads H, W (fp32 on the
// bf16 grid; checked and converted on the device) and the targets, runs the
// sm_100a kernels and returns owning host results (stats, loss, dH, dW), like
// the reference's bench run_iteration (proj/src/bench.cpp:89-124, 145-154).
//
//   tests/cpp/bench_dropin [N D V reps]      (default: the Llama-3-8B head)
// Prints one JSON line.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fusedce/fused_backward.hpp"
#include "fusedce/fused_forward.hpp"
#include "fusedce/instance.hpp"

using namespace fusedce;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    const std::size_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 16384;
    const std::size_t d = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 4096;
    const std::size_t v = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 128256;
    const int reps = argc > 4 ? std::atoi(argv[4]) : 3;
    auto t0 = clk::now();
    Instance<float> inst = make_random_instance<float>(n, d, v, 42);
    inst.hidden.round_to_bf16();
    inst.weights.round_to_bf16();
    const double gen_s = std::chrono::duration<double>(clk::now() - t0).count();
    MatrixView<float> hv(inst.hidden), wv(inst.weights);
    MemoryLedger ledger;
    double fwd_s = 0, bwd_s = 0, loss = 0, checksum = 0;
    for (int r = 0; r <= reps; ++r) {  // r = 0 warms up (handle, workspace)
        auto a = clk::now();
        FusedOutput<float> out = fused_forward(hv, wv, inst.targets, ReductionMode::Mean, ledger);
        auto b = clk::now();
        Gradients<float> g = fused_backward_recompute(hv, wv, inst.targets, std::span<const SoftmaxStats<float>>(out.stats),
                                                      UpstreamGradient<float>::make_scalar(1.0f), ReductionMode::Mean,
                                                      ledger);
        auto c = clk::now();
        if (r > 0) {
            fwd_s += std::chrono::duration<double>(b - a).count();
            bwd_s += std::chrono::duration<double>(c - b).count();
        }
        loss = out.loss.scalar();
        checksum = g.hidden.data()[0] + g.weights.data()[g.weights.size() - 1];
    }
    fwd_s /= reps;
    bwd_s /= reps;
    const double h2d = static_cast<double>(n * d + v * d) * 4 * 2 + n * 8;  // fwd + bwd uploads (fp32)
    const double d2h = static_cast<double>(n * 13 + (n + v) * d * 4);       // stats + dH + dW
    std::printf("{\"path\": \"fusedce::fused_forward + fused_backward_recompute (drop-in C++ API, host buffers)\", "
                "\"N\": %zu, \"D\": %zu, \"V\": %zu, \"reps\": %d, \"forward_s\": %.4f, \"backward_s\": %.4f, "
                "\"value\": %.1f, \"unit\": \"tokens/s\", \"h2d_bytes_per_step\": %.0f, \"d2h_bytes_per_step\": %.0f, "
                "\"loss\": %.6f, \"checksum\": %.6g, \"host_instance_s\": %.2f}\n",
                n, d, v, reps, fwd_s, bwd_s, n / (fwd_s + bwd_s), h2d, d2h, loss, checksum, gen_s);
    return 0;
}
