"""Tensor-pipe gaps between consecutive units of the persistent backward (dev
tool).  Trace slots per unit: [0] MMA issue start, [5] first operand stage
ready, [6] accumulator full (last MMA of the unit completed), [3] SM of the
pair's even CTA.  Per pair, the pipe idles before unit i for
max(0, first_stage_ready(i) - acc_full(i-1)); inside a unit it runs from
max(first_stage_ready(i), acc_full(i-1)) to acc_full(i)."""
import os, sys, torch, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
n, d, v = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 4096, 128256)))
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.default_handle(0)
out = fce.fused_forward(H, W, Y, "mean", handle=h)
units = 4_000_000
tr = torch.zeros(units * 8, dtype=torch.int64, device="cuda")
h.set_option("trace_ptr", tr.data_ptr())
dh = torch.empty(n, d, device="cuda")
for _ in range(2):
    tr.zero_()
    fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
torch.cuda.synchronize()
h.set_option("trace_ptr", 0)
t = tr.view(units, 8).cpu().numpy().astype(np.int64)
ok = (t[:, 0] > 0) & (t[:, 5] > 0) & (t[:, 6] > 0)
uid = np.arange(units)[ok]
t = t[ok]
# unit type (kg = 1 layout: per chunk G, dH, dW units) and k-blocks
rc, bc = int(os.environ.get("ROW_CHUNK", min(n, 16384))), int(os.environ.get("BAND", 3072))
mb, vt, dt = rc // 256, bc // 256, d // 256
per = mb * vt + mb * dt + vt * dt
loc = uid % per
typ = np.where(loc < mb * vt, 0, np.where(loc < mb * vt + mb * dt, 1, 2))
kbs = np.where(typ == 0, d // 64, np.where(typ == 1, bc // 64, rc // 64))
clk_ghz = float(np.median(t[:, 7] / np.maximum(t[:, 1] - t[:, 0], 1)))
start, end = t[:, 0].min(), t[:, 6].max()
span = (end - start) / 1e3
gaps, busy, first_gap = [], [], []
busy_t = {0: [], 1: [], 2: []}
ideal_t = {0: [], 1: [], 2: []}
for sm in np.unique(t[:, 3]):
    sel = t[:, 3] == sm
    u, ty, kb = t[sel], typ[sel], kbs[sel]
    order = np.argsort(u[:, 5])
    u, ty, kb = u[order], ty[order], kb[order]
    prev_full = None
    for row, tt, k in zip(u, ty, kb):
        fs, full = row[5], row[6]
        if prev_full is None:
            first_gap.append((fs - start) / 1e3)
            b = (full - fs) / 1e3
        else:
            g = max(0, fs - prev_full)
            gaps.append(g / 1e3)
            b = (full - max(fs, prev_full)) / 1e3
        busy.append(b)
        busy_t[int(tt)].append(b)
        ideal_t[int(tt)].append(k * 512 / (clk_ghz * 1e3))
        prev_full = full
pairs = len(np.unique(t[:, 3]))
print(f"pairs {pairs}, units {len(t)}, kernel span {span:.0f} us")
print(f"tensor-pipe time inside units: {sum(busy) / pairs:.0f} us per pair ({100 * sum(busy) / pairs / span:.1f}% of span)")
print(f"gaps between units: {sum(gaps) / pairs:.0f} us per pair ({100 * sum(gaps) / pairs / span:.1f}%), "
      f"mean {np.mean(gaps):.2f} us, p90 {np.percentile(gaps, 90):.2f} us, units with a gap > 0.2 us: "
      f"{100 * np.mean(np.array(gaps) > 0.2):.1f}%")
print(f"start-up (first unit's first stage): {np.mean(first_gap):.1f} us; "
      f"tail (last acc-full to kernel end): {np.mean([(end - t[t[:, 3] == sm][:, 6].max()) / 1e3 for sm in np.unique(t[:, 3])]):.1f} us")
print(f"measured SM clock {clk_ghz:.3f} GHz")
for k, name in enumerate(["G", "dH", "dW"]):
    b, i = np.array(busy_t[k]), np.array(ideal_t[k])
    if len(b):
        print(f"{name:2s}: {len(b):6d} units, busy {b.mean():6.1f} us vs ideal {i.mean():6.1f} us "
              f"-> {100 * i.sum() / b.sum():5.1f}% of tensor peak inside the unit")
