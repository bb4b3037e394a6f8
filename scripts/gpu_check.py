"""Quick numerics check of the CUDA path against a torch fp32 reference (dev tool)."""
import sys, time, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import paper_2511_17599_b200 as fce

def ref(Hf, Wf, Y, ign=None, reduction="mean"):
    H = Hf.clone().requires_grad_(True); W = Wf.clone().requires_grad_(True)
    z = H @ W.t()
    lse = torch.logsumexp(z, 1)
    valid = torch.ones_like(Y, dtype=torch.bool) if ign is None else (Y != ign)
    yy = torch.where(valid, Y, torch.zeros_like(Y))
    rows = torch.where(valid, lse - z.gather(1, yy[:, None])[:, 0], torch.zeros_like(lse))
    loss = rows.sum() / max(int(valid.sum()), 1) if reduction == "mean" else rows.sum()
    loss.backward()
    return loss.detach(), lse.detach(), rows.detach(), H.grad, W.grad

def relmax(a, b):
    return ((a.float() - b.float()).abs().max() / b.float().abs().max().clamp_min(1e-30)).item()

for (n, d, v, ign, frac, seed) in [(256, 512, 32000, None, 0.0, 42), (300, 136, 1000, -100, 0.25, 7), (1000, 4096, 5000, None, 0.0, 3), (129, 64, 257, -100, 0.3, 9)]:
    t0 = time.time()
    H, W, Y, Hf, Wf = fce.generate_instance(n, d, v, seed, -100, frac, want_f32=True)
    torch.cuda.synchronize()
    out = fce.fused_forward(H, W, Y, "mean", ign)
    torch.cuda.synchronize()
    rl, rlse, rrows, rdh, rdw = ref(Hf, Wf, Y, ign)
    valid = torch.ones_like(Y, dtype=torch.bool) if ign is None else (Y != ign)
    print(f"[{n}x{d}x{v} ign={ign}] loss gpu={out.loss.item():.7f} ref={rl.item():.7f} rel={abs(out.loss.item()-rl.item())/abs(rl.item()):.2e} "
          f"lse rel={relmax(out.lse[valid], rlse[valid]):.2e} rows rel={relmax(out.loss_rows, rrows):.2e} found={int(out.stats.found.sum())}/{int(valid.sum())}", flush=True)
    dh, dw = fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, ign)
    torch.cuda.synchronize()
    print(f"    dH relmax={relmax(dh, rdh):.2e} dW relmax={relmax(dw, rdw):.2e}  ({time.time()-t0:.1f}s)", flush=True)
