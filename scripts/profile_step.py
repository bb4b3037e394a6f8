"""One warm-up step, then one step inside cudaProfilerStart/Stop (for ncu --profile-from-start off)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402

n, d, v = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (16384, 4096, 128256)))
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.default_handle(0)
for kv in sys.argv[4:]:
    k, val = kv.split("=")
    h.set_option(k, int(val))
dh = torch.empty(n, d, device="cuda")
dw = torch.empty(v, d, device="cuda")


def step():
    out = fce.fused_forward(H, W, Y, "mean", handle=h)
    fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
    return out


step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
step()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
