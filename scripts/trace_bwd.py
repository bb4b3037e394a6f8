"""Per-unit timeline of the persistent backward (dev tool)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
n, d, v = 16384, 4096, 128256
opts = dict(kv.split("=") for kv in sys.argv[1:])
rc, bc = int(opts.get("row_chunk", 16384)), int(opts.get("band_cols", 2048))
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.default_handle(0)
for k, val in opts.items(): h.set_option(k, int(val))
out = fce.fused_forward(H, W, Y, "mean", handle=h)
NR, NB = -(-n // rc), -(-v // bc)
mb, vt, vm, dt = rc // 256, bc // 256, bc // 256, d // 256
ng, nh, nw = mb * vt, mb * dt, vm * dt
per = ng + nh + nw
units = NR * NB * per
tr = torch.zeros(units * 4, dtype=torch.int64, device="cuda")
h.set_option("trace_ptr", tr.data_ptr())
dh = torch.empty(n, d, device="cuda")
for _ in range(2):
    fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
torch.cuda.synchronize()
t = tr.view(units, 4).cpu().numpy().astype(np.int64)
h.set_option("trace_ptr", 0)
l = np.arange(units) % per
typ = np.where(l < ng, 0, np.where(l < ng + nh, 1, 2))
t0 = t[:, 0].min()
dur_mma = (t[:, 1] - t[:, 0]) / 1e3
dur_all = (t[:, 2] - t[:, 0]) / 1e3
kb = np.where(typ == 0, d // 64, np.where(typ == 1, bc // 64, rc // 64))
for k, name in enumerate(["grad", "dH", "dW"]):
    s = typ == k
    print(f"{name}: units {s.sum()}  mma-issue span mean {dur_mma[s].mean():.1f} us  start->epi-end mean {dur_all[s].mean():.1f} us  "
          f"ideal {kb[s].mean()*512/1.5e3:.1f} us  kblocks {kb[s].mean():.0f}")
total = (t[:, 2].max() - t0) / 1e6
print(f"backward span {total:.2f} ms")
# per-SM busy fraction: sum of MMA spans / total
sm = t[:, 3]
busy = np.bincount(sm.astype(int), weights=(t[:, 1] - t[:, 0]).astype(float)) / 1e6
busy = busy[busy > 0]
print(f"pairs {len(busy)}  MMA-issue busy per pair: mean {busy.mean():.2f} ms, min {busy.min():.2f}, max {busy.max():.2f}")
# gaps: for each SM, time between consecutive units' MMA start
order = np.lexsort((t[:, 0], sm))
ts, sms = t[order, 0], sm[order]
gaps = np.diff(ts)[np.diff(sms) == 0] / 1e3
print(f"start-to-start per pair: mean {gaps.mean():.1f} us median {np.median(gaps):.1f}")
