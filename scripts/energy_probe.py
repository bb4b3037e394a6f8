"""Energy per flop of the step's kernels vs a plain cuBLAS GEMM (dev tool).

Under the 1 kW board cap the step's speed is set by energy per flop, so this
probe loops each workload ~secs seconds and reports, from the NVML energy
counter, J per PFLOP (algorithmic flops), mean board power, median SM clock and
the tensor throughput as a fraction of the clock-scaled peak
(148 SMs x 8192 flop / clk).
    python scripts/energy_probe.py [--secs 3] [--sets "" "dh_group=2"]"""
import argparse, os, statistics, sys, threading, time
import torch
import pynvml as nv
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce

ap = argparse.ArgumentParser()
ap.add_argument("--secs", type=float, default=3.0)
ap.add_argument("--sets", nargs="*", default=[""])
ap.add_argument("--shape", default="16384,4096,128256")
ap.add_argument("--work", default="cublas,fwd,bwd,step")
ap.add_argument("--ignore", type=float, default=0.0, help="fraction of ignore_index=-100 targets")
a = ap.parse_args()
nv.nvmlInit()
dev = nv.nvmlDeviceGetHandleByIndex(int(os.environ.get("LOCAL_RANK", "0")))
n, d, v = (int(x) for x in a.shape.split(","))
H, W, Y = fce.generate_instance(n, d, v, 42, -100, a.ignore)
IGN = -100 if a.ignore > 0 else None
dh = torch.empty(n, d, device="cuda")


def measure(fn, flops):
    fn(); torch.cuda.synchronize()
    clk = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            clk.append(nv.nvmlDeviceGetClockInfo(dev, nv.NVML_CLOCK_SM))
            time.sleep(0.02)
    # settle into the power-capped state first
    t0 = time.time()
    while time.time() - t0 < 0.5:
        fn()
    torch.cuda.synchronize()
    th = threading.Thread(target=sampler); th.start()
    e_0 = nv.nvmlDeviceGetTotalEnergyConsumption(dev)
    ev0, ev1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ev0.record()
    k, t0 = 0, time.time()
    while time.time() - t0 < a.secs:
        fn(); k += 1
        if k % 4 == 0:
            torch.cuda.synchronize()
    ev1.record(); torch.cuda.synchronize()
    e_1 = nv.nvmlDeviceGetTotalEnergyConsumption(dev)
    stop.set(); th.join()
    ms = ev0.elapsed_time(ev1) / k
    joules = (e_1 - e_0) / 1e3 / k
    c = statistics.median(clk[len(clk) // 5:]) if clk else float("nan")
    tf = flops / ms / 1e9
    return (f"{ms:8.3f} ms {tf:6.0f} TF/s {joules / (flops / 1e15):6.1f} J/PFLOP "
            f"{joules / (ms / 1e3):5.0f} W  {c:5.0f} MHz  {100 * tf / (148 * 8192 * c * 1e-6):5.1f}% of clock peak")


work = a.work.split(",")
if "cublas" in work:
    A = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    B = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    C = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
    print(f"cublas 8192^3            {measure(lambda: torch.matmul(A, B, out=C), 2 * 8192 ** 3)}", flush=True)
    Hf = H[:, :d]
    Sx = torch.empty(n, 16384, device="cuda", dtype=torch.bfloat16)
    print(f"cublas H.W[:16384]^T     {measure(lambda: torch.matmul(Hf, W[:16384].t(), out=Sx), 2 * n * d * 16384)}",
          flush=True)
    hg = fce.Handle(0)
    hg.set_option("gemm_pair", 1)
    Cf = torch.empty(8192, 8192, device="cuda", dtype=torch.float32)
    print(f"fce pair gemm 8192^3     {measure(lambda: fce.gemm_bf16(A, B, out=Cf, handle=hg), 2 * 8192 ** 3)}",
          flush=True)
    hg.close()
    del A, B, C, Sx, Cf
if "copy" in work:
    # energy per byte: DRAM streaming (2 GiB copy) vs L2-resident (16 MiB copy)
    for nbytes, tag in ((2 << 30, "DRAM"), (16 << 20, "L2")):
        src = torch.empty(nbytes // 2, dtype=torch.bfloat16, device="cuda").uniform_()
        dst = torch.empty_like(src)
        reps = max(1, (256 << 20) // nbytes) if tag == "L2" else 1

        def cp():
            for _ in range(reps):
                dst.copy_(src)
        r = measure(cp, 2.0 * nbytes * reps)  # "flops" slot = bytes moved (read + write)
        print(f"copy {tag:4s} {nbytes >> 20} MiB x{reps}: {r}  (TF/s = TB/s, J/PFLOP = J/PB)", flush=True)
        del src, dst
fl = 2.0 * n * d * v
for s in a.sets:
    h = fce.Handle(0)
    h.set_option("validate", 0)
    for kv in filter(None, s.split(",")):
        k_, x = kv.split("=")
        h.set_option(k_, int(x))
    out = fce.fused_forward(H, W, Y, "mean", IGN, handle=h)
    tag = s or "default"
    if "fwd" in work:
        print(f"[{tag}] fwd  {measure(lambda: fce.fused_forward(H, W, Y, 'mean', IGN, handle=h), fl)}", flush=True)
    if "bwd" in work:
        print(f"[{tag}] bwd  {measure(lambda: fce.fused_backward_recompute(H, W, Y, out.stats, 'mean', 1.0, IGN, handle=h, dhidden=dh), 3 * fl)}", flush=True)
    if "step" in work:
        def step():
            o = fce.fused_forward(H, W, Y, "mean", IGN, handle=h)
            fce.fused_backward_recompute(H, W, Y, o.stats, "mean", 1.0, handle=h, dhidden=dh)
        print(f"[{tag}] step {measure(step, 4 * fl)}", flush=True)
    h.close()
