"""Per-unit timeline of the persistent backward (dev tool)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
n, d, v = 16384, 4096, 128256
opts = dict(kv.split("=") for kv in sys.argv[1:])
rc, bc = int(opts.get("row_chunk", 16384)), int(opts.get("band_cols", 3072))
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.default_handle(0)
for k, val in opts.items(): h.set_option(k, int(val))
out = fce.fused_forward(H, W, Y, "mean", handle=h)
NR, NB = -(-n // rc), -(-v // bc)
mb, vt, vm, dt = rc // 256, bc // 256, bc // 256, d // 256
ng, nh, nw = mb * vt, mb * dt, vm * dt
per = ng + nh + nw
units = NR * NB * per
tr = torch.zeros(units * 8, dtype=torch.int64, device="cuda")
h.set_option("trace_ptr", tr.data_ptr())
dh = torch.empty(n, d, device="cuda")
for _ in range(2):
    tr.zero_()
    fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
torch.cuda.synchronize()
t = tr.view(units, 8).cpu().numpy().astype(np.int64)
h.set_option("trace_ptr", 0)
ok = (t[:, 0] > 0) & (t[:, 1] > 0) & (t[:, 2] > 0)
t = t[ok]
l = (np.arange(units)[ok]) % per
typ = np.where(l < ng, 0, np.where(l < ng + nh, 1, 2))
kb = np.where(typ == 0, d // 64, np.where(typ == 1, bc // 64, rc // 64))
span_ns = (t[:, 1] - t[:, 0]).astype(float)
clk = float(np.median(t[:, 7] / np.maximum(span_ns, 1))) * 1e3  # SM cycles per us, measured
print(f"measured SM clock during the backward: {clk:.0f} MHz")
for k, name in enumerate(["grad", "dH", "dW"]):
    s = typ == k
    span = (t[s, 1] - t[s, 0]) / 1e3
    acc_wait = (t[s, 4] - t[s, 0]) / 1e3
    first = (t[s, 5] - t[s, 4]) / 1e3
    epi = (t[s, 2] - t[s, 1]) / 1e3
    print(f"{name:4s}: n={s.sum():6d} span {span.mean():6.1f} us = acc-free wait {acc_wait.mean():5.1f} + first-stage {first.mean():5.1f} "
          f"+ rest {span.mean()-acc_wait.mean()-first.mean():6.1f} (of which stage waits ~{steady.mean():5.1f});"
          f" ideal {kb[s].mean()*512/clk:5.1f}; issue-end->epi-end {epi.mean():5.1f}")
t0 = t[:, 0].min()
print(f"backward span {(t[:, 2].max() - t0) / 1e6:.2f} ms")
