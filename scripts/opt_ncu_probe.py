"""One warm-up + one measured launch of the forward or the backward per handle
option set, for an ncu capture (DRAM bytes, L2 hit, time) per set:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:fce_bwd_persistent --csv python scripts/opt_ncu_probe.py --what bwd "" "bwd_unit_mask=1"
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("sets", nargs="+")
ap.add_argument("--what", default="bwd", choices=["fwd", "bwd"])
ap.add_argument("--shape", default="16384,4096,128256")
a = ap.parse_args()
n, d, v = (int(x) for x in a.shape.split(","))
H, W, Y = fce.generate_instance(n, d, v, 42)
dh = torch.empty(n, d, device="cuda")
for s in a.sets:
    h = fce.Handle(0)
    h.set_option("validate", 0)
    out = fce.fused_forward(H, W, Y, "mean", handle=h)
    for kv in filter(None, s.split(",")):
        k, x = kv.split("=")
        h.set_option(k, int(x))
    for _ in range(2):
        if a.what == "fwd":
            fce.fused_forward(H, W, Y, "mean", handle=h)
        else:
            fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
    torch.cuda.synchronize()
    print(f"[{s or 'default'}] done", flush=True)
    h.close()
