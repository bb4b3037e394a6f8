"""One warm-up step, then one fwd+bwd step inside cudaProfilerStart/Stop (for
ncu --profile-from-start off).

    python scripts/profile_step.py [--config llama3-8b] [option=value ...]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2511_17599_b200 as fce  # noqa: E402
from bench import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="llama3-8b", choices=sorted(CONFIGS))
ap.add_argument("opts", nargs="*")
a = ap.parse_args()
n, d, v, frac = CONFIGS[a.config]
ign = -100 if frac > 0 else None
H, W, Y = fce.generate_instance(n, d, v, 42, -100, frac)
h = fce.default_handle(0)
for kv in a.opts:
    k, val = kv.split("=")
    h.set_option(k, int(val))
dh = torch.empty(n, d, device="cuda")


def step():
    out = fce.fused_forward(H, W, Y, "mean", ign, handle=h)
    fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, ign, handle=h, dhidden=dh)
    return out


step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
