"""A/B/C… of handle option sets over whole fwd+bwd steps, interleaved blocks (dev tool).
    python scripts/opt_probe.py "" "fwd_pair=1" "dh_group=2,row_chunk=8192" [--blocks 4 --steps 8]
Each option set runs on its own handle; reports median fwd / bwd / step ms per set."""
import argparse, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce

ap = argparse.ArgumentParser()
ap.add_argument("sets", nargs="+")
ap.add_argument("--blocks", type=int, default=4)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--shape", default="16384,4096,128256")
a = ap.parse_args()
n, d, v = (int(x) for x in a.shape.split(","))
H, W, Y = fce.generate_instance(n, d, v, 42)
dh = torch.empty(n, d, device="cuda")
handles = []
for s in a.sets:
    h = fce.Handle(0)
    h.set_option("validate", 0)
    for kv in filter(None, s.split(",")):
        k, x = kv.split("=")
        h.set_option(k, int(x))
    handles.append(h)


def step(h, ev=None):
    if ev: ev[0].record()
    out = fce.fused_forward(H, W, Y, "mean", handle=h)
    if ev: ev[1].record()
    g = fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
    if ev: ev[2].record()
    return out, g


ref = None
for i, h in enumerate(handles):
    for _ in range(2):
        out, gr = step(h)
    torch.cuda.synchronize()
    l = out.loss.item()
    g = (gr[0].abs().sum().item(), gr[1].abs().sum().item())
    del gr
    if ref is None:
        ref = (l, g)
    print(f"[{a.sets[i] or 'default'}] loss {l:.6f} |dH|1 {g[0]:.6e} |dW|1 {g[1]:.6e} "
          f"(rel vs set0: {abs(g[0]-ref[1][0])/ref[1][0]:.2e} {abs(g[1]-ref[1][1])/ref[1][1]:.2e})", flush=True)
res = {i: [] for i in range(len(handles))}
for b in range(a.blocks):
    order = list(range(len(handles)))
    if b % 2: order.reverse()
    for i in order:
        h = handles[i]
        step(h)
        torch.cuda.synchronize()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(a.steps)]
        for k in range(a.steps):
            step(h, evs[k])
        torch.cuda.synchronize()
        f = sum(e[0].elapsed_time(e[1]) for e in evs) / a.steps
        bw = sum(e[1].elapsed_time(e[2]) for e in evs) / a.steps
        res[i].append((f + bw, f, bw))
fl = 2.0 * n * d * v
for i, s in enumerate(a.sets):
    r = sorted(res[i])
    t, f, bw = r[len(r) // 2]
    print(f"[{s or 'default'}] step {t:.2f} ms (min {r[0][0]:.2f}) fwd {f:.2f} ({fl/f/1e9:.0f} TF/s) bwd {bw:.2f} "
          f"({3*fl/bw/1e9:.0f} TF/s) step {4*fl/t/1e9:.0f} TF/s {n/t*1e3:.0f} tok/s", flush=True)
