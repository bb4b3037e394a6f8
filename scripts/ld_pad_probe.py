"""Does a power-of-two row pitch hurt the L2?  The forward (and optionally the
backward) on H / W with ld = D and with ld = D + pad, one measured launch each
after a warm-up, for an ncu DRAM capture:

  ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
      -k regex:fce_ --csv python scripts/ld_pad_probe.py --shape 16384,8192,128256 --pads 0,64
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="16384,8192,128256")
ap.add_argument("--pads", default="0,64")
ap.add_argument("--bwd", action="store_true")
a = ap.parse_args()
n, d, v = (int(x) for x in a.shape.split(","))
H0, W0, Y = fce.generate_instance(n, d, v, 42)
h = fce.Handle(0)
h.set_option("validate", 0)
for pad in (int(x) for x in a.pads.split(",")):
    H = torch.empty(n, d + pad, dtype=torch.bfloat16, device="cuda")[:, :d]
    W = torch.empty(v, d + pad, dtype=torch.bfloat16, device="cuda")[:, :d]
    H.copy_(H0)
    W.copy_(W0)
    for _ in range(2):
        out = fce.fused_forward(H, W, Y, "mean", handle=h)
    if a.bwd:
        for _ in range(2):
            fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h)
    torch.cuda.synchronize()
    print(f"pad {pad}: loss {out.loss.item():.6f}", flush=True)
    del H, W
