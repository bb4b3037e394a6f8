"""Quick device-time probe of forward / backward at a named shape (dev tool)."""
import sys, os, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
n, d, v = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 4096, 128256)))
opts = dict(a.split("=") for a in sys.argv[4:])
frac = float(opts.pop("ignore_fraction", 0.0))
H, W, Y = fce.generate_instance(n, d, v, 42, -100, frac)
ign = -100 if frac > 0 else None
h = fce.default_handle(0)
for k, val in opts.items():
    h.set_option(k, int(val))
h.set_option("validate", 0)
def fwd():
    return fce.fused_forward(H, W, Y, "mean", ign, handle=h)
out = fwd()
def bwd():
    return fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, ign, handle=h)
for f in (fwd, bwd): f()
torch.cuda.synchronize()
def t(f, it=3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(it): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
tf = t(fwd); tb = t(bwd)
fl = 2.0 * n * d * v
print(f"N={n} D={d} V={v} fwd {tf:.2f} ms ({fl/tf/1e9:.0f} TF/s)  bwd {tb:.2f} ms ({3*fl/tb/1e9:.0f} TF/s)  total {tf+tb:.2f} ms ({4*fl/(tf+tb)/1e9:.0f} TF/s, {n/(tf+tb)*1e3:.0f} tok/s) loss={out.loss.item():.6f}", flush=True)
