"""Backward time with fp32 vs bf16 gradient outputs at the Llama-3-8B shape (dev tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
n, d, v = 16384, 4096, 128256
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.Handle(0)
h.set_option("validate", 0)
out = fce.fused_forward(H, W, Y, "mean", handle=h)
res = {}
for blk in range(4):
    for gdt in ((torch.float32, torch.bfloat16) if blk % 2 == 0 else (torch.bfloat16, torch.float32)):
        fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, grad_dtype=gdt)
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            g = fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, grad_dtype=gdt)
            del g
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(gdt, []).append((e0.elapsed_time(e1) / 5, (torch.cuda.max_memory_allocated() - base) / 1e9))
for gdt, r in res.items():
    r.sort()
    print(f"{gdt}: bwd {r[len(r) // 2][0]:.2f} ms (min {r[0][0]:.2f}), peak extra alloc {r[0][1]:.2f} GB, "
          f"workspace {h.workspace_bytes()[1] / 1e9:.2f} GB")
