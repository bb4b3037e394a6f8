"""A/B of a handle option over whole fwd+bwd steps, interleaved blocks (dev tool).
    python scripts/pair_probe.py fwd_pair 0 1 [blocks] [steps]"""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
key = sys.argv[1]
vals = [int(x) for x in sys.argv[2:4]]
blocks = int(sys.argv[4]) if len(sys.argv) > 4 else 4
steps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
n, d, v = 16384, 4096, 128256
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.default_handle(0)
h.set_option("validate", 0)
def step():
    out = fce.fused_forward(H, W, Y, "mean", handle=h)
    fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h)
for _ in range(3): step()
res = {x: [] for x in vals}
for b in range(blocks):
    for x in (vals if b % 2 == 0 else vals[::-1]):
        h.set_option(key, x)
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(steps): step()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        res[x].append(ms)
        print(f"{key}={x} block {b}: {ms:.2f} ms/step", flush=True)
for x in vals:
    r = sorted(res[x])
    print(f"{key}={x}: median {r[len(r)//2]:.2f} min {r[0]:.2f}  ({16384/r[len(r)//2]*1e3:.0f} tok/s)")
