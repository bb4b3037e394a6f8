"""Steady-state clock / power of the forward and backward kernels per handle
option (dev tool): each variant loops ~2 s while nvidia-smi samples SM clock
and board power.   python scripts/power_probe.py fwd_pair 0 1"""
import os, subprocess, statistics, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce
key = sys.argv[1]
vals = [int(x) for x in sys.argv[2:]]
n, d, v = 16384, 4096, 128256
H, W, Y = fce.generate_instance(n, d, v, 42)
h = fce.default_handle(0)
h.set_option("validate", 0)
out = fce.fused_forward(H, W, Y, "mean", handle=h)

def sample(fn, seconds=2.0):
    f = open("/tmp/clk.csv", "w")
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                          "-lms", "50"], stdout=f)
    time.sleep(0.2)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    k = 0
    e0.record()
    t0 = time.time()
    while time.time() - t0 < seconds:
        fn(); k += 1
        if k % 4 == 0: torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    p.terminate(); p.wait(); f.close()
    rows = [l.split(",") for l in open("/tmp/clk.csv").read().splitlines() if l.strip()]
    rows = rows[len(rows) // 4:]
    clk = statistics.median(float(r[0]) for r in rows) if rows else float("nan")
    pw = statistics.median(float(r[1]) for r in rows) if rows else float("nan")
    return e0.elapsed_time(e1) / k, clk, pw

fwd = lambda: fce.fused_forward(H, W, Y, "mean", handle=h)
bwd = lambda: fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h)
def step():
    o = fce.fused_forward(H, W, Y, "mean", handle=h)
    fce.fused_backward_recompute(H, W, Y, o.stats, "mean", 1.0, handle=h)
WORK = [w for w in (("fwd", fwd, 2), ("bwd", bwd, 6), ("step", step, 8))
        if w[0] in os.environ.get("PROBE_WORK", "fwd,bwd,step").split(",")]
for rep in range(2):
    for name, fn, fl in WORK:
        for x in vals:
            h.set_option(key, x)
            fn(); torch.cuda.synchronize()
            ms, clk, pw = sample(fn)
            tf = fl * n * d * v / ms / 1e9
            print(f"{name:4s} {key}={x}: {ms:7.2f} ms {tf:6.0f} TF/s at {clk:.0f} MHz {pw:.0f} W -> "
                  f"{100 * tf / (148 * 8192 * clk * 1e-6):.1f}% of clock peak", flush=True)
