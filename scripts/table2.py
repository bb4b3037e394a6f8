"""Reproduce the paper's Table 2 (canonical two-stage vs fused) on
B200: forward latency and peak memory for d = 4096, bf16, over the B*T x V grid.

canonical = torch bf16 lm_head GEMM (cuBLAS) + fp32 cross-entropy (materialises
N x V logits); proposed = this repository's fused forward (libfce.so).  Also
reports fwd+bwd for both.  Writes a markdown table to stdout.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402

D = 4096
BT = [int(x) for x in os.environ.get("BT", "1024,4096,8192,16384,32768").split(",")]
VS = [int(x) for x in os.environ.get("VS", "32768,65536,131072,262144").split(",")]
PAPER_MS = {(16384, 131072): (26.67, 13.20), (32768, 262144): (96.52, 53.61), (1024, 32768): (0.73, 0.69),
            (4096, 131072): (6.78, 2.86), (8192, 65536): (6.08, 2.90)}


def timeit(f, it=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


def peak_of(f):
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    f()
    torch.cuda.synchronize()
    return (torch.cuda.max_memory_allocated() - base) / 2**20


h = fce.default_handle(0)
h.set_option("validate", 0)
print("| B·T | V | canonical fwd ms | fused fwd ms | speed-up | canonical fwd MB (extra) | fused fwd MB (extra) | "
      "canonical fwd+bwd ms | fused fwd+bwd ms | paper GB200 canonical / fused fwd ms |")
print("|---|---|---|---|---|---|---|---|---|---|")
for bt in BT:
    for v in VS:
        H, W, Y = fce.generate_instance(bt, D, v, 42, handle=h)
        H, W = H.contiguous(), W.contiguous()

        def canon_fwd():
            return torch.nn.functional.cross_entropy((H @ W.t()).float(), Y)

        def fused_fwd():
            return fce.fused_forward(H, W, Y, "mean", handle=h).loss

        Hg = H.detach().clone().requires_grad_(True)
        Wg = W.detach().clone().requires_grad_(True)

        def canon_step():
            loss = torch.nn.functional.cross_entropy((Hg @ Wg.t()).float(), Y)
            loss.backward()
            Hg.grad = None
            Wg.grad = None

        def fused_step():
            out = fce.fused_forward(H, W, Y, "mean", handle=h)
            fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h)

        try:
            tc = timeit(canon_fwd)
            mc = peak_of(canon_fwd)
            tcs = timeit(canon_step, 3)
        except torch.OutOfMemoryError:
            tc = mc = tcs = float("nan")
        torch.cuda.empty_cache()
        tf = timeit(fused_fwd)
        mf = peak_of(fused_fwd)
        tfs = timeit(fused_step, 3)
        pc, pf = PAPER_MS.get((bt, v), (None, None))
        paper = f"{pc} / {pf}" if pc else "—"
        print(f"| {bt} | {v} | {tc:.2f} | {tf:.2f} | {tc / tf:.2f}x | {mc:.0f} | {mf:.0f} | {tcs:.2f} | {tfs:.2f} | {paper} |",
              flush=True)
        del H, W, Y, Hg, Wg
        torch.cuda.empty_cache()
