"""Forward variants, one measured launch each after a warm-up launch, for an
ncu capture of DRAM bytes / L2 hit rate per option set:

  ncu --metrics dram__bytes_read.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum \
      -k regex:fce_tile_kernel --csv python scripts/fwd_variant_probe.py --shape 131072,8192,128256 \
      "" "fwd_m_group=16,splits=10"
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("sets", nargs="+")
ap.add_argument("--shape", default="131072,8192,128256")
a = ap.parse_args()
n, d, v = (int(x) for x in a.shape.split(","))
H, W, Y = fce.generate_instance(n, d, v, 42)
for s in a.sets:
    h = fce.Handle(0)
    h.set_option("validate", 0)
    for kv in filter(None, s.split(",")):
        k, x = kv.split("=")
        h.set_option(k, int(x))
    for _ in range(2):
        out = fce.fused_forward(H, W, Y, "mean", handle=h)
    torch.cuda.synchronize()
    print(f"[{s or 'default'}] loss {out.loss.item():.6f}", flush=True)
    h.close()
