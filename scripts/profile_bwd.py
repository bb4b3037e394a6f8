"""Forward once, then the backward inside cudaProfilerStart/Stop (ncu --profile-from-start off)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
n, d, v = 16384, 4096, 128256
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.default_handle(0)
for kv in sys.argv[1:]:
    k, val = kv.split("=")
    h.set_option(k, int(val))
out = fce.fused_forward(H, W, Y, "mean", handle=h)
dh = torch.empty(n, d, device="cuda")
fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
