#!/usr/bin/env python
"""Bench of the fused linear-cross-entropy hot path (BASELINE.json metric).

One step = fused forward (loss, lse, stats) + fused backward (dH, dW) of the
Llama-3-8B lm_head shape (N=16384 tokens, D=4096, V=128256, bf16 inputs,
fp32 accumulation/outputs, mean reduction, seed-42 synthetic instance of the
reference generator), through the C-ABI of libfce.so.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl reference]

N=1: one GPU.  N>1 (launched with torchrun): vocabulary-parallel split of W
across the ranks (fce_vp_forward / fce_vp_backward: NCCL all-gather of the
per-row stats, all-reduce of dH), same total work -> "scaling": "strong".
`--impl reference` times the reference's own CPU implementation (oracle/_ref,
built from /root/reference) on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# rank 0 must print exactly one JSON line on stdout: keep NCCL's banner off it
os.environ.setdefault("NCCL_DEBUG", "WARN")

CONFIGS = {
    # name: (N, D, V, ignore_fraction)  -- BASELINE.json configs
    "small": (256, 512, 32000, 0.0),
    "llama3-8b": (16384, 4096, 128256, 0.0),
    "qwen2.5-7b": (32768, 3584, 152064, 0.25),
    "gemma2-2b": (65536, 2304, 256000, 0.0),
    "llama3-70b": (131072, 8192, 128256, 0.0),
}
CONFIG_LABEL = {
    "small": "small fp32 CPU-runnable N=256 D=512 V=32000 (bf16 grid)",
    "llama3-8b": "Llama-3-8B head N=16384 D=4096 V=128256",
    "qwen2.5-7b": "Qwen2.5-7B head N=32768 D=3584 V=152064, 25% ignore_index=-100",
    "gemma2-2b": "Gemma-2-2B head N=65536 D=2304 V=256000",
    "llama3-70b": "Llama-3-70B head N=131072 D=8192 V=128256",
}
METRIC = "fused LCE fwd+bwd tokens/sec at Llama-3-8B shape; % BF16 TC peak; peak HBM bytes"
SEED = 42


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return {"bf16_tflops": p["bf16_tflops"], "bf16_tflops_sustained": p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                "hbm_gbs": p["hbm_gbs"], "source": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0,
            "source": "fallback (B200_PROFILING.md)"}


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = f"/tmp/fce_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------- CPU reference
def cpu_reference_step(n_rows: int, d: int, v: int, frac: float, H=None, W=None, Y=None):
    """One bounded sample of the reference's own CPU path (oracle/_ref): fused_forward +
    fused_backward_recompute on the first n_rows rows at full D, V.  Returns seconds."""
    import numpy as np
    from oracle import bindings as ob
    cores = os.cpu_count() or 1
    ign = -100 if frac > 0 else None
    fwd_workers = max(1, min(cores, n_rows))
    # backward workers >= 2 each allocate a private V x D fp32 dW partial
    # (fused_backward.hpp:90-96): bound them by host memory.
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    bwd_workers = int(max(1, min(cores, n_rows, avail // (3 * v * d * 4))))
    use_ref = ob.ref_available()
    t0 = time.perf_counter()
    if use_ref:
        st, _, _ = ob.ref_forward(H, W, Y, "mean", ign, 0, fwd_workers)
        ob.ref_backward(H, W, Y, st, "mean", 1.0, ign, bwd_workers)
    else:
        st, _, _ = ob.forward(H, W, Y, "mean", ign, threads=fwd_workers)
        ob.backward(H, W, Y, st, "mean", 1.0, ign, threads=fwd_workers)
        bwd_workers = fwd_workers
    dt = time.perf_counter() - t0
    return dt, ("reference" if use_ref else "port"), max(fwd_workers, bwd_workers), fwd_workers, bwd_workers


def cpu_sample_inputs(n_rows, d, v, frac):
    from oracle import bindings as ob
    H, W, Y = ob.make_instance(n_rows, d, v, SEED, -100, frac,
                               impl="ref" if ob.ref_available() else "oracle")
    return H, W, Y


def cpu_baseline(cfg_name, budget_s=20.0):
    """Reference CPU path on this host: rows sample sized to ~budget_s of work."""
    n, d, v, frac = CONFIGS[cfg_name]
    rows = min(n, os.cpu_count() or 1, 16)  # one row per host core: every core busy
    H, W, Y = cpu_sample_inputs(64 if n >= 64 else n, d, v, frac)
    dt, kind, cores, fw, bw = cpu_reference_step(rows, d, v, frac, H[:rows], W, Y[:rows])
    if dt < budget_s / 4 and rows < n:
        rows = int(min(n, 64, max(rows + 1, rows * budget_s / 2 / max(dt, 1e-3))))
        dt, kind, cores, fw, bw = cpu_reference_step(rows, d, v, frac, H[:rows], W, Y[:rows])
    return {"value": rows / dt, "unit": "tokens/s", "cores": cores, "kind": kind,
            "sample": f"{rows} of {n} rows at full D={d}, V={v} (fused_forward + fused_backward_recompute, "
                      f"mean, seed {SEED}, bf16 grid); forward workers={fw}, backward workers={bw}; "
                      f"{dt:.1f} s wall"}


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, d, v, frac = CONFIGS[args.config]
    rows = min(n, args.ref_rows or min(os.cpu_count() or 1, 16))
    H, W, Y = cpu_sample_inputs(max(rows, 1), d, v, frac)
    for _ in range(args.warmup if args.ref_warmup else 0):
        cpu_reference_step(rows, d, v, frac, H[:rows], W, Y[:rows])
    times = []
    kind = cores = None
    for _ in range(args.steps):
        dt, kind, cores, fw, bw = cpu_reference_step(rows, d, v, frac, H[:rows], W, Y[:rows])
        times.append(dt)
    per_step = sum(times) / len(times)
    value = rows / per_step
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (bf16-grid inputs)",
            "data": "synthetic (reference splitmix64 generator, seed 42)",
            "config": {"workload": CONFIG_LABEL[args.config], "rows_per_step": rows,
                       "parallelism": "cpu threads"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": kind,
                             "sample": f"{rows} rows of the {args.config} workload per step at full D, V "
                                       f"(fwd workers={fw}, bwd workers={bw})"},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama3-8b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="fce", choices=["fce", "reference"])
    ap.add_argument("--ref-rows", type=int, default=0, help="rows per reference step (0: one per host core, <= 16)")
    ap.add_argument("--ref-warmup", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--force-vp", action="store_true",
                    help="use the native vocab-parallel (NCCL) path even on one rank (testing)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2511_17599_b200 as fce
    from paper_2511_17599_b200 import vocab_parallel as vp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.force_vp:
        dist.init_process_group("nccl", device_id=dev)
    n, d, v, frac = CONFIGS[args.config]
    ign = -100 if frac > 0 else None
    stream = torch.cuda.current_stream(dev)
    h = fce.Handle(local, stream)
    h.set_option("validate", 1)

    # ---- inputs resident in HBM (device generator == reference generator, bit for bit)
    H, W, Y = fce.generate_instance(n, d, v, SEED, -100, frac, device=local, handle=h)
    lo, hi = fce.shard_ranges(v, world)[rank]
    Ws = W[lo:hi]
    comm = vp.NativeComm.from_torch_distributed(local) if (world > 1 or args.force_vp) else None

    dh = torch.empty(n, d, dtype=torch.float32, device=dev)
    dw = torch.empty(hi - lo, d, dtype=torch.float32, device=dev)
    p, keep = fce.make_problem(H, Ws, Y, ign, lo, v)
    st = fce.Stats.empty(n, dev)
    lse = torch.empty(n, dtype=torch.float32, device=dev)
    rows = torch.empty(n, dtype=torch.float32, device=dev)
    loss = torch.empty((), dtype=torch.float32, device=dev)
    import ctypes
    lib = h.lib

    def step():
        if comm is None:
            fce._check(lib.fce_forward(h.raw, ctypes.byref(p), 0, 0, st.c(), lse.data_ptr(), rows.data_ptr(),
                                       loss.data_ptr()))
            fce._check(lib.fce_backward(h.raw, ctypes.byref(p), st.c(), 0, 1.0, None, dh.data_ptr(), d,
                                        dw.data_ptr(), d, 0))
        else:
            fce._check(lib.fce_vp_forward(h.raw, comm.ptr, ctypes.byref(p), 0, st.c(), lse.data_ptr(),
                                          rows.data_ptr(), loss.data_ptr()))
            fce._check(lib.fce_vp_backward(h.raw, comm.ptr, ctypes.byref(p), st.c(), 0, 1.0, None,
                                           dh.data_ptr(), d, dw.data_ptr(), d))

    def barrier():
        torch.cuda.synchronize(dev)
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(max(args.warmup, 3)):
        step()
    barrier()
    torch.cuda.reset_peak_memory_stats(dev)

    clocks = ClockSampler(local)
    clocks.start()
    launches0 = h.launch_count()
    h.set_option("timing", 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    kstats = {k: h.kernel_stats(k) for k in (0, 1, 2, 3)}
    h.set_option("timing", 0)
    launches = h.launch_count() - launches0
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = t.item()
    ms_step = ms_max / args.steps
    tokens_per_s = n * args.steps / (ms_max / 1e3)
    loss_val = loss.item()
    ws_cur, ws_peak = h.workspace_bytes()
    peak_torch = torch.cuda.max_memory_allocated(dev)

    # ---- end to end through the C-ABI with HOST buffers: every step copies its
    # inputs (pinned H, W shard, targets) host -> device and the loss back.  The
    # copy of step i+1 runs on a second stream while step i computes (double-
    # buffered device inputs, the usual input-prefetch pipeline); the timed
    # region spans the first copy to the last loss read.
    Hh = H.cpu().pin_memory()
    Wh = Ws.contiguous().cpu().pin_memory()
    Yh = Y.cpu().pin_memory()
    slots = [(torch.empty_like(H), torch.empty_like(Ws), torch.empty_like(Y)) for _ in range(2)]
    probs = [fce.make_problem(*sl, ign, lo, v) for sl in slots]
    loss_h = torch.empty((), dtype=torch.float32).pin_memory()
    copy_stream = torch.cuda.Stream(dev)
    ready = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]

    def enqueue_copy(i):
        s_ = i % 2
        with torch.cuda.stream(copy_stream):
            copy_stream.wait_event(free[s_])
            Hd, Wd, Yd = slots[s_]
            Hd.copy_(Hh, non_blocking=True)
            Wd.copy_(Wh, non_blocking=True)
            Yd.copy_(Yh, non_blocking=True)
            ready[s_].record(copy_stream)

    def compute(i):
        s_ = i % 2
        pe = probs[s_][0]
        stream.wait_event(ready[s_])
        if comm is None:
            fce._check(lib.fce_forward(h.raw, ctypes.byref(pe), 0, 0, st.c(), lse.data_ptr(), rows.data_ptr(),
                                       loss.data_ptr()))
            fce._check(lib.fce_backward(h.raw, ctypes.byref(pe), st.c(), 0, 1.0, None, dh.data_ptr(), d,
                                        dw.data_ptr(), d, 0))
        else:
            fce._check(lib.fce_vp_forward(h.raw, comm.ptr, ctypes.byref(pe), 0, st.c(), lse.data_ptr(),
                                          rows.data_ptr(), loss.data_ptr()))
            fce._check(lib.fce_vp_backward(h.raw, comm.ptr, ctypes.byref(pe), st.c(), 0, 1.0, None,
                                           dh.data_ptr(), d, dw.data_ptr(), d))
        free[s_].record(stream)
        loss_h.copy_(loss, non_blocking=True)

    for s_ in range(2):
        free[s_].record(stream)
    enqueue_copy(0)
    compute(0)
    barrier()
    for s_ in range(2):
        free[s_].record(stream)
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(copy_stream)
    enqueue_copy(0)
    for i in range(args.e2e_steps):
        if i + 1 < args.e2e_steps:
            enqueue_copy(i + 1)
        compute(i)
    e3.record(stream)
    barrier()
    ms_e2e = torch.tensor([e2.elapsed_time(e3)], device=dev)
    if world > 1:
        dist.all_reduce(ms_e2e, op=dist.ReduceOp.MAX)
    e2e_val = n * args.e2e_steps / (ms_e2e.item() / 1e3)
    h2d = Hh.numel() * Hh.element_size() + Wh.numel() * Wh.element_size() + Yh.numel() * 8
    d2h = 4

    if rank != 0:
        if dist.is_initialized():
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peaks = load_peaks()
    flops_step = 8.0 * n * d * v
    # dominant kernel by device time inside the timed region
    names = {0: "fce_fwd_sm100 (forward, online-LSE epilogue)", 1: "fce_bwd_grad_sm100 (recompute S, G=softmax-onehot)",
             2: "fce_bwd_gemm_sm100 (dW=G^T.H and dH+=G.W)",
             3: "fce_bwd_persistent_sm100 (recompute S -> G -> dH, dW; one launch)"}
    dom = max(kstats, key=lambda k: kstats[k][0])
    kms, kl, kfl = kstats[dom]
    per_launch_ms = kms / max(kl, 1)
    achieved = (kfl / max(kl, 1)) / (per_launch_ms / 1e3) / 1e12
    peak_sust = peaks["bf16_tflops_sustained"]
    kernels = {}
    for k, (kms_, kl_, kfl_) in kstats.items():
        if kl_:
            kernels[names[k].split(" ")[0]] = {
                "launches_per_step": kl_ / args.steps, "ms_per_step": kms_ / args.steps,
                "tflops": (kfl_ / kl_) / ((kms_ / kl_) / 1e3) / 1e12,
                "share_of_step": (kms_ / args.steps) / (ms_max / args.steps)}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(names[dom].split(" ")[0])
        except Exception:
            traffic = None

    line = {
        "metric": METRIC,
        "value": tokens_per_s,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: reference splitmix64 instance (seed 42) generated on device, bf16 grid",
        "config": {"workload": CONFIG_LABEL[args.config], "N": n, "D": d, "V": v,
                   "reduction": "mean", "ignore_fraction": frac,
                   "parallelism": f"vocab-parallel x{world}" if comm is not None else "single GPU",
                   "l2": "inputs larger than L2 (W bf16 = %.2f GB)" % (v * d * 2 / 1e9)},
        "tflops_8ndv": flops_step / (ms_step / 1e3) / 1e12,
        # per-GPU fraction of the measured bf16 peak (whole-job flops / N GPUs)
        "pct_peak_step": flops_step / (ms_step / 1e3) / 1e12 / peaks["bf16_tflops"] / world,
        "pct_peak_step_sustained": flops_step / (ms_step / 1e3) / 1e12 / peak_sust / world,
        "model_tflops_6ndv": 6.0 * n * d * v / (ms_step / 1e3) / 1e12,
        "peak_hbm_bytes": int(peak_torch + ws_peak),
        "peak_hbm_breakdown": {"torch_inputs_outputs": int(peak_torch), "library_workspace": int(ws_peak)},
        "canonical_nxv_fp32_bytes": int(n) * int(v) * 4,
        "loss": loss_val,
        "roofline": {"bound": "tensor", "kernel": names[dom], "achieved": achieved, "peak": peak_sust,
                     "unit": "TFLOP/s", "frac": achieved / peak_sust,
                     "frac_of_burst_peak": achieved / peaks["bf16_tflops"],
                     "peak_source": peaks["source"] + " bf16_tflops_sustained (kernel timed inside a long step)",
                     "traffic": traffic,
                     "algorithmic_flops_per_launch": kfl / max(kl, 1),
                     "avg_launch_ms": per_launch_ms},
        "kernels": kernels,
        "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": d2h,
                "path": "C-ABI fce_forward+fce_backward; every step copies pinned host H, W (bf16) and targets "
                        "in (copy of step i+1 overlapped with step i on a second stream) and the loss out"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config)
        except Exception as exc:  # never lose the GPU line over the CPU sample
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"failed: {exc!r}"}
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
