"""`fusedce`-style command line for the device path (reference CLI:
proj/tools/fusedce_main.cpp, flags in proj/README.md), with `--device cuda`
semantics: every fused method runs through libfce.so on a B200.

    python -m paper_2511_17599_b200.cli bench --bt 1024,4096 --vocab 8192,32768 --hidden 256
    python -m paper_2511_17599_b200.cli verify

`bench` sweeps the (B*T, V) grid per method and emits the reference's CSV
schema (bench.cpp:200-211): bt,vocab,hidden,method,precision,latency_s,
latency_min_s,latency_max_s,aux_peak_bytes,loss (`--extended` appends
tokens_per_s,tflops,pct_peak,peak_hbm_bytes,gpus) — `canonical` is the
two-stage PyTorch path (bf16 cuBLAS lm_head GEMM + fp32 cross-entropy,
materialises N x V logits; the paper's Table 2 baseline).
`verify` checks the fused device path against that two-stage path in fp32 on
random instances (loss equivalence, gradients, window sweep, shard invariance,
large-offset stability, k-rank vocab-parallel over the in-process transport
against the one-rank path) and prints one line per suite.  Exit codes follow the
reference CLI: 0 pass, 1 tolerance failure, 2 usage / library error.
"""
from __future__ import annotations

import argparse
import math
import os
import statistics
import sys
import tempfile
import time

import paper_2511_17599_b200 as fce


def _csv_list(s):
    return [int(x) for x in s.split(",") if x]


def _deliver(text: str, output):
    """Atomic write (reference deliver(), fusedce_main.cpp:71-90)."""
    if not output:
        sys.stdout.write(text)
        return
    d = os.path.dirname(os.path.abspath(output)) or "."
    fd, tmp = tempfile.mkstemp(dir=d, prefix=".fusedce.")
    with os.fdopen(fd, "w") as f:
        f.write(text)
    os.replace(tmp, output)


def _two_stage(H, W, Y, reduction, ign, grads=False, bf16=False):
    """The canonical path: lm_head GEMM (materialises N x V logits) + cross-entropy.
    fp32 GEMM for verify (a float reference); bench uses the bf16 cuBLAS GEMM with an
    fp32 cross-entropy, the paper's Table 2 "canonical"."""
    import torch
    dt = torch.bfloat16 if bf16 else torch.float32
    Hf = H.to(dt).detach().requires_grad_(grads)
    Wf = W.to(dt).detach().requires_grad_(grads)
    z = (Hf @ Wf.t()).float()
    loss = torch.nn.functional.cross_entropy(z, Y, reduction=reduction,
                                             ignore_index=-100 if ign is None else ign)
    if not grads:
        return loss.detach(), None, None
    (loss.sum() if reduction == "none" else loss).backward()
    return loss.detach(), Hf.grad, Wf.grad


def _peak_tflops() -> float:
    """Measured dense bf16 peak of this pool's B200s (MEASURED_PEAKS.json), else the spec."""
    import json
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return 2250.0


def cmd_bench(a) -> int:
    import torch
    h = fce.default_handle(0)
    rows = []
    for bt in a.bt:
        for v in a.vocab:
            H, W, Y = fce.generate_instance(bt, a.hidden, v, a.seed)
            for method in a.methods:
                def run():
                    if method == "canonical":
                        with torch.no_grad() if a.forward_only else torch.enable_grad():
                            loss, _, _ = _two_stage(H, W, Y, a.reduction, None, grads=not a.forward_only,
                                                    bf16=True)
                        return loss
                    if method == "fused_partial_grad":
                        out, parts = fce.fused_forward_with_partial_grads(H, W, Y, a.reduction)
                        if a.reduction == "mean":
                            fce.scale_partial_grads(parts, 1.0 / bt)
                        return out.loss
                    window = a.window if method == "fused_windowed" else 0
                    out = fce.fused_forward(H, W, Y, a.reduction, window=window)
                    if not a.forward_only:
                        fce.fused_backward_recompute(H, W, Y, out.stats, a.reduction, 1.0 if a.reduction != "none"
                                                     else torch.ones(bt, device="cuda"))
                    return out.loss
                for _ in range(a.warmup):
                    run()
                torch.cuda.synchronize()
                base = torch.cuda.memory_allocated()
                torch.cuda.reset_peak_memory_stats()
                ws0 = h.workspace_bytes()[0]
                times = []
                for _ in range(a.repeats):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    loss = run()
                    torch.cuda.synchronize()
                    times.append(time.perf_counter() - t0)
                aux = max(0, torch.cuda.max_memory_allocated() - base)
                if method != "canonical":
                    aux = max(aux, h.workspace_bytes()[0] - ws0) + h.workspace_bytes()[1]
                lv = float(loss.sum().item() if loss.dim() else loss.item())
                peak_hbm = torch.cuda.max_memory_allocated() + (h.workspace_bytes()[1] if method != "canonical" else 0)
                rows.append((bt, v, a.hidden, method, "bf16", statistics.median(times), min(times), max(times),
                             int(aux), lv, int(peak_hbm)))
    if a.format == "csv":
        text = "bt,vocab,hidden,method,precision,latency_s,latency_min_s,latency_max_s,aux_peak_bytes,loss"
        text += ",tokens_per_s,tflops,pct_peak,peak_hbm_bytes,gpus\n" if a.extended else "\n"
        peak = _peak_tflops()
        for r in rows:
            text += f"{r[0]},{r[1]},{r[2]},{r[3]},{r[4]},{r[5]:.9f},{r[6]:.9f},{r[7]:.9f},{r[8]},{r[9]:.8f}"
            if a.extended:
                # algorithmic flops: 2NDV forward; the fused fwd+bwd recomputes the logits (8NDV),
                # the canonical fwd+bwd does not (6NDV)
                mult = 2 if a.forward_only else (6 if r[3] == "canonical" else 8)
                tf = mult * r[0] * r[2] * r[1] / r[5] / 1e12
                text += f",{r[0] / r[5]:.1f},{tf:.2f},{tf / peak:.4f},{r[10]},1"
            text += "\n"
    else:
        text = "| B*T | V | method | latency ms | aux MB | loss |\n|---|---|---|---|---|---|\n"
        text += "".join(f"| {r[0]} | {r[1]} | {r[3]} | {r[5] * 1e3:.3f} | {r[8] / 2**20:.1f} | {r[9]:.6f} |\n"
                        for r in rows)
    _deliver(text, a.output)
    return 0


def cmd_verify(a) -> int:
    import numpy as np
    import torch
    g = np.random.default_rng(a.seed)
    results = []

    def suite(name, tol, fn):
        worst = 0.0
        for i in range(fn.count):
            worst = max(worst, fn(i))
        results.append((name, worst <= tol, worst, tol))

    def rel(x, y):
        return float((x.float() - y.float()).abs().max() / y.float().abs().max().clamp_min(1e-30))

    def loss_eq(i):
        n, d, v = int(g.integers(1, 200)), int(g.integers(1, 96)), int(g.integers(2, 700))
        frac = 0.25 if i % 2 else 0.0
        H, W, Y = fce.generate_instance(n, d, v, a.seed + i, -100, frac)
        ign = -100 if frac else None
        red = ("mean", "sum", "none")[i % 3]
        got = fce.fused_forward(H, W, Y, red, ign).loss
        ref, _, _ = _two_stage(H, W, Y, red, ign)
        return rel(got, ref) if ref.dim() else abs(got.item() - ref.item()) / max(1.0, abs(ref.item()))
    loss_eq.count = a.loss_instances

    def grads(i):
        n, d, v = int(g.integers(1, 160)), int(g.integers(1, 80)), int(g.integers(2, 600))
        H, W, Y = fce.generate_instance(n, d, v, 1000 + a.seed + i)
        out = fce.fused_forward(H, W, Y, "sum")
        dh, dw = fce.fused_backward_recompute(H, W, Y, out.stats, "sum")
        _, rh, rw = _two_stage(H, W, Y, "sum", None, grads=True)
        return max(rel(dh, rh), rel(dw, rw))
    grads.count = a.grad_instances

    def window(i):
        H, W, Y = fce.generate_instance(32, 32, 257, a.seed)
        base = fce.fused_forward(H, W, Y, "mean").loss.item()
        w = (1, 3, 16, 128, 256, 257)[i]
        return abs(fce.fused_forward_windowed(H, W, Y, w).loss.item() - base) / abs(base)
    window.count = 6

    def shards(i):
        H, W, Y = fce.generate_instance(48, 40, 301, a.seed + 7, -100, 0.25)
        base = fce.fused_forward(H, W, Y, "mean", -100).loss.item()
        k = a.ranks + i
        parts = [fce.tp_rank_partial(H, W[lo:hi], lo, 301, Y, -100) for lo, hi in fce.shard_ranges(301, k)]
        return abs(fce.merge_rank_partials(parts, Y, "mean", -100).loss.item() - base) / abs(base)
    shards.count = 3

    def stability(i):
        # +10240 shared offset through an extra column (verify.cpp:422-492, bf16 variant)
        n, dq, v = 4, 8, 12
        gen = np.random.default_rng(a.seed + i)
        H = (gen.integers(0, 9, (n, dq + 1)) - 4) / 4.0
        H[:, dq] = 1.0
        W = (gen.integers(0, 9, (v, dq + 1)) - 4) / 4.0
        Wb, Ws = W.copy(), W.copy()
        Wb[:, dq] = 0.0
        Ws[:, dq] = 10240.0
        Y = torch.from_numpy(gen.integers(0, v, n)).cuda()
        t = lambda x: torch.from_numpy(x.astype(np.float32)).cuda()  # noqa: E731
        got = fce.fused_forward(t(H), t(Ws), Y, "none").loss
        ref, _, _ = _two_stage(t(H), t(Wb), Y, "none", None)
        return float("inf") if not torch.isfinite(got).all() else rel(got, ref)
    stability.count = 3

    def vocab_parallel(i):
        # tp_forward / tp_backward over k real ranks (in-process local transport:
        # k threads, each with its own stream / handle / communicator) against
        # the one-rank path (verify.cpp shard-invariance suite, parallel_sim.hpp)
        from paper_2511_17599_b200 import vocab_parallel as vp
        k = 2 + i
        n, d, v = 96, 72, 777
        H, W, Y = fce.generate_instance(n, d, v, a.seed + 31 + i, -100, 0.2)
        one = fce.fused_forward(H, W, Y, "mean", -100)
        dh1, dw1 = fce.fused_backward_recompute(H, W, Y, one.stats, "mean", 1.0, -100)
        ranges = fce.shard_ranges(v, k)

        def rank_fn(r, comm, hh):
            lo, hi = ranges[r]
            out = vp.native_forward(comm, H, W[lo:hi], Y, lo, v, "mean", -100, handle=hh)
            dh, dw = vp.native_backward(comm, H, W[lo:hi], Y, lo, v, out.stats, "mean", 1.0, -100, handle=hh)
            return out.loss, dh, dw

        res = vp.run_ranks(k, rank_fn)
        err = abs(res[0][0].item() - one.loss.item()) / abs(one.loss.item())
        err = max(err, rel(res[0][1], dh1), rel(torch.cat([x[2] for x in res]), dw1))
        return err
    vocab_parallel.count = 3

    try:
        suite("loss_equivalence", 1e-3, loss_eq)
        suite("gradient_recompute", 1e-2, grads)
        suite("window_sweep", 1e-5, window)
        suite("shard_invariance", 1e-5, shards)
        suite("stability", 1e-4, stability)
        suite("vocab_parallel_ranks", 1e-3, vocab_parallel)
    except fce.FusedCEError as e:
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 2
    text = "".join(f"{name:20s} {'PASS' if ok else 'FAIL'}  max_err={err:.3e}  tol={tol:.0e}\n"
                   for name, ok, err, tol in results)
    ok = all(r[1] for r in results)
    text += f"overall: {'PASS' if ok else 'FAIL'}\n"
    _deliver(text, a.output)
    return 0 if ok else 1


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="fusedce", description=__doc__.split("\n\n")[0])
    ap.add_argument("--device", default="cuda", choices=["cuda"], help="device path (the B200 kernels)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--bt", type=_csv_list, default=[1024, 4096])
    b.add_argument("--vocab", type=_csv_list, default=[8192, 32768])
    b.add_argument("--hidden", type=int, default=256)
    b.add_argument("--methods", type=lambda s: s.split(","), default=["canonical", "fused"])
    b.add_argument("--reduction", default="mean", choices=["mean", "sum", "none"])
    b.add_argument("--window", type=int, default=0)
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--warmup", type=int, default=2)
    b.add_argument("--forward-only", action="store_true")
    b.add_argument("--format", default="csv", choices=["csv", "markdown"])
    b.add_argument("--extended", action="store_true",
                   help="append tokens_per_s,tflops,pct_peak,peak_hbm_bytes,gpus to the reference CSV schema")
    b.add_argument("--seed", type=int, default=42)
    b.add_argument("--output")
    v = sub.add_parser("verify")
    v.add_argument("--seed", type=int, default=42)
    v.add_argument("--loss-instances", type=int, default=40)
    v.add_argument("--grad-instances", type=int, default=12)
    v.add_argument("--ranks", type=int, default=2)
    v.add_argument("--output")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code not in (0, None) else 0
    known = {"canonical", "fused", "fused_windowed", "fused_partial_grad"}
    if a.cmd == "bench" and not set(a.methods) <= known:
        print(f"unknown method in {a.methods}", file=sys.stderr)
        return 2
    try:
        return cmd_bench(a) if a.cmd == "bench" else cmd_verify(a)
    except (fce.FusedCEError, ImportError) as e:
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
