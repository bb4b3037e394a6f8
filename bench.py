#!/usr/bin/env python
"""Bench of the fused linear-cross-entropy hot path (BASELINE.json metric).

One step = fused forward (loss, lse, stats) + fused backward (dH, dW) of the
Llama-3-8B lm_head shape (N=16384 tokens, D=4096, V=128256, bf16 inputs,
fp32 accumulation/outputs, mean reduction, seed-42 synthetic instance of the
reference generator), through the C-ABI of libfce.so.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl reference]

N=1: one GPU.  N>1: vocabulary-parallel split of W across N ranks
(fce_vp_forward / fce_vp_backward: all-gather of the per-row stats, all-reduce
of dH), same total work -> "scaling": "strong".  Launched under torchrun the
ranks are processes over NCCL; launched plainly with --gpus N the script
re-launches itself under torch.distributed.run when the box has N GPUs, and
otherwise runs the N ranks as threads of this process over libfce's
in-process ("local") transport on the GPUs it has (the N-rank code path on a
smaller box; "parallelism" says so).
`--impl reference` times the reference's own CPU implementation (oracle/_ref,
built from /root/reference) on bounded row samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL's communicator-init lines (how a launcher verifies the N ranks) go to
# stderr; rank 0's stdout carries exactly one JSON line.
os.environ.setdefault("NCCL_DEBUG", "INFO")
os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

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
        self.path = f"/tmp/fce_clocks_{os.getpid()}_{gpu_index}.csv"

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
        pw = [float(r[3]) for r in rows if r[3].replace(".", "").isdigit()]
        loaded = [x for x in sm if x > 0.5 * max(sm)] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_median": statistics.median(pw) if pw else None}


# --------------------------------------------------------------- CPU reference
# the reference runs on row slices at full D, V; its time per call
# is t(rows) = alpha + beta * rows.  alpha is the backward's per-call fixed cost
# (allocating, zeroing and folding (workers - 1) private V x D dW partials,
# fused_backward.hpp:90-110); beta is the per-token work, which falls as
# 1 / workers.  At the workload's N the beta term dominates, so the reference
# gets every host core for both passes, and the throughput reported is the
# marginal 1 / beta tokens/s from a two-point fit, labelled "extrapolated".


def _ref_plan(cfg_name):
    """(rows pair, forward workers, backward workers) for this host."""
    n, d, v, frac = CONFIGS[cfg_name]
    cores = os.cpu_count() or 1
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:
        avail = 16 << 30
    # each backward worker past the first holds a private V x D fp32 partial
    bw = int(max(1, min(cores, avail * 0.7 // (v * d * 4))))
    # slices of 256 and 512 rows (half and all of N when N is smaller)
    rows = (256, 512) if n >= 512 else (max(1, n // 2), n)
    return rows, cores, bw


def _ref_sample(n_rows, H, W, Y, frac, fwd_workers, bwd_workers):
    from oracle import bindings as ob
    ign = -100 if frac > 0 else None
    t0 = time.perf_counter()
    if ob.ref_available():
        st, _, _ = ob.ref_forward(H[:n_rows], W, Y[:n_rows], "mean", ign, 0, fwd_workers)
        ob.ref_backward(H[:n_rows], W, Y[:n_rows], st, "mean", 1.0, ign, bwd_workers)
    else:
        st, _, _ = ob.forward(H[:n_rows], W, Y[:n_rows], "mean", ign, threads=fwd_workers)
        ob.backward(H[:n_rows], W, Y[:n_rows], st, "mean", 1.0, ign, threads=fwd_workers)
    return time.perf_counter() - t0


def _ref_inputs(cfg_name, rows):
    from oracle import bindings as ob
    n, d, v, frac = CONFIGS[cfg_name]
    H, W, Y = ob.make_instance(rows, d, v, SEED, -100, frac, impl="ref" if ob.ref_available() else "oracle")
    return H, W, Y


def _fit(samples):
    """Least-squares t = alpha + beta * rows over (rows, seconds) samples."""
    xs = [r for r, _ in samples]
    ys = [t for _, t in samples]
    mx, my = sum(xs) / len(xs), sum(ys) / len(ys)
    sxx = sum((x - mx) ** 2 for x in xs)
    beta = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx if sxx else my / mx
    alpha = my - beta * mx
    if beta <= 0:  # noise swamped the slope: fall back to the mean per-row cost
        beta, alpha = sum(ys) / sum(xs), 0.0
    return alpha, beta


def _ref_kind():
    from oracle import bindings as ob
    return "reference" if ob.ref_available() else "port"


def cpu_baseline(cfg_name):
    """The reference CPU path on this host (§8(d)): one sample at each of two row
    counts at full D, V, fit t = alpha + beta rows, value = 1 / beta."""
    n, d, v, frac = CONFIGS[cfg_name]
    rows, fw, bw = _ref_plan(cfg_name)
    H, W, Y = _ref_inputs(cfg_name, max(rows))
    samples = [(r, _ref_sample(r, H, W, Y, frac, fw, bw)) for r in rows]
    alpha, beta = _fit(samples)
    return {"value": 1.0 / beta, "unit": "tokens/s", "cores": fw, "kind": _ref_kind(),
            "sample": (f"extrapolated: reference fused_forward + fused_backward_recompute (mean, seed {SEED}, "
                       f"bf16 grid) on row slices {list(rows)} of the {cfg_name} workload at full D={d}, "
                       f"V={v}; fit t = alpha + beta*rows, value = 1/beta (alpha = {alpha:.2f} s per call, "
                       f"the backward's private dW partial fold); forward workers={fw}, backward workers={bw}; "
                       f"samples (rows, s) = " + ", ".join(f"({r}, {t:.2f})" for r, t in samples)),
            "alpha_s": alpha, "beta_s_per_row": beta, "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    n, d, v, frac = CONFIGS[args.config]
    rows, fw, bw = _ref_plan(args.config)
    H, W, Y = _ref_inputs(args.config, max(rows))
    for j in range(min(args.warmup, 1)):
        _ref_sample(rows[0], H, W, Y, frac, fw, bw)
    samples = []
    for j in range(args.steps):
        r = rows[j % 2]
        samples.append((r, _ref_sample(r, H, W, Y, frac, fw, bw)))
    alpha, beta = _fit(samples)
    value = 1.0 / beta
    per_step = sum(t for _, t in samples) / len(samples)
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32 (bf16-grid inputs)",
            "data": "synthetic (reference splitmix64 generator, seed 42)",
            "config": {"workload": CONFIG_LABEL[args.config], "N": n, "D": d, "V": v,
                       "rows_per_step": list(rows), "parallelism": f"{fw} cpu threads",
                       "value": "extrapolated marginal tokens/s = 1/beta of t = alpha + beta*rows"},
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": fw, "kind": _ref_kind(),
                             "sample": f"extrapolated: steps alternate {rows[0]} / {rows[1]} rows of the "
                                       f"{args.config} workload at full D, V (fwd workers={fw}, bwd workers={bw}); "
                                       f"fit alpha={alpha:.2f} s, beta={beta:.4f} s/row",
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- rank contexts
class DistCtx:
    """One process per GPU (torchrun, NCCL)."""

    def __init__(self, world, rank, local, force_vp):
        import torch
        import torch.distributed as dist
        from paper_2511_17599_b200 import vocab_parallel as vp
        # FCE_BENCH_TRANSPORT=ipc: libfce's own collectives over CUDA IPC peer
        # memory (ranks may share a GPU), gloo only for the launcher's barrier
        self.transport = os.environ.get("FCE_BENCH_TRANSPORT", "nccl")
        if self.transport == "ipc":
            local = local % max(torch.cuda.device_count(), 1)
        self.world, self.rank, self.device = world, rank, local
        torch.cuda.set_device(local)
        self.stream = torch.cuda.current_stream(local)
        self.dist = None
        self.comm = None
        if world > 1 or force_vp:
            if self.transport == "ipc":
                dist.init_process_group("gloo")
                self.dist = dist
                self.comm = vp.NativeComm.from_torch_distributed_ipc(local)
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
                self.dist = dist
                self.comm = vp.NativeComm.from_torch_distributed(local)

    def barrier(self):
        import torch
        torch.cuda.synchronize(self.device)
        if self.dist:
            self.dist.barrier()
        torch.cuda.synchronize(self.device)

    def max(self, x: float) -> float:
        import torch
        if not self.dist:
            return x
        t = torch.tensor([x], device="cpu" if self.transport == "ipc" else f"cuda:{self.device}")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.item()

    def close(self):
        if self.comm:
            self.comm.close()
        if self.dist:
            self.dist.barrier()
            self.dist.destroy_process_group()


class ThreadCtx:
    """N ranks as threads of one process over the in-process transport."""

    def __init__(self, world, rank, device, comm, shared):
        import torch
        self.world, self.rank, self.device, self.comm = world, rank, device, comm
        torch.cuda.set_device(device)
        self.stream = torch.cuda.Stream(device)
        self.shared = shared
        self.transport = "local"

    def barrier(self):
        import torch
        torch.cuda.synchronize(self.device)
        self.shared["barrier"].wait()
        torch.cuda.synchronize(self.device)

    def max(self, x: float) -> float:
        self.shared["vals"][self.rank] = x
        self.shared["barrier"].wait()
        m = max(self.shared["vals"])
        self.shared["barrier"].wait()
        return m

    def close(self):
        pass


# --------------------------------------------------------------- GPU arm
def bench_rank(ctx, args):
    import ctypes

    import torch

    import paper_2511_17599_b200 as fce

    world, rank, local = ctx.world, ctx.rank, ctx.device
    dev = torch.device("cuda", local)
    n, d, v, frac = CONFIGS[args.config]
    ign = -100 if frac > 0 else None
    stream = ctx.stream
    comm = ctx.comm
    with torch.cuda.stream(stream):
        h = fce.Handle(local, stream)
        h.set_option("validate", 1)
        # ---- inputs resident in HBM (device generator == reference generator, bit for bit)
        H, W, Y = fce.generate_instance(n, d, v, SEED, -100, frac, device=local, handle=h)
        n_valid = int((Y != -100).sum().item()) if ign is not None else n
        lo, hi = fce.shard_ranges(v, world)[rank]
        Ws = W[lo:hi]
        dh = torch.empty(n, d, dtype=torch.float32, device=dev)
        dw = torch.empty(hi - lo, d, dtype=torch.float32, device=dev)
        p, keep = fce.make_problem(H, Ws, Y, ign, lo, v)
        st = fce.Stats.empty(n, dev)
        lse = torch.empty(n, dtype=torch.float32, device=dev)
        rows = torch.empty(n, dtype=torch.float32, device=dev)
        loss = torch.empty((), dtype=torch.float32, device=dev)
        lib = h.lib

        def step(pe=p, dh_=dh, dw_=dw):
            if comm is None:
                fce._check(lib.fce_forward(h.raw, ctypes.byref(pe), 0, 0, st.c(), lse.data_ptr(), rows.data_ptr(),
                                           loss.data_ptr()))
                fce._check(lib.fce_backward(h.raw, ctypes.byref(pe), st.c(), 0, 1.0, None, dh_.data_ptr(), d,
                                            dw_.data_ptr(), d, 0))
            else:
                fce._check(lib.fce_vp_forward(h.raw, comm.ptr, ctypes.byref(pe), 0, st.c(), lse.data_ptr(),
                                              rows.data_ptr(), loss.data_ptr()))
                fce._check(lib.fce_vp_backward(h.raw, comm.ptr, ctypes.byref(pe), st.c(), 0, 1.0, None,
                                               dh_.data_ptr(), d, dw_.data_ptr(), d))

        for _ in range(max(args.warmup, 3)):
            step()
        ctx.barrier()
        torch.cuda.reset_peak_memory_stats(dev)

        clocks = ClockSampler(local) if rank == 0 else None
        if clocks:
            clocks.start()
        launches0 = h.launch_count()
        h.set_option("timing", 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ctx.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        ctx.barrier()
        clk = clocks.stop() if clocks else None
        ms = e0.elapsed_time(e1)
        kstats = {k: h.kernel_stats(k) for k in (0, 1, 2, 3)}
        h.set_option("timing", 0)
        launches = h.launch_count() - launches0
        ms_max = ctx.max(ms)
        ms_step = ms_max / args.steps
        tokens_per_s = n * args.steps / (ms_max / 1e3)
        loss_val = loss.item()
        ws_cur, ws_peak = h.workspace_bytes()
        peak_torch = torch.cuda.max_memory_allocated(dev)

        # ---- end to end through the C-ABI with HOST buffers: every step copies its
        # inputs (pinned H, W shard, targets) host -> device and its result back.
        # The copy of step i+1 runs on a second stream while step i computes
        # (double-buffered device inputs, the usual input-prefetch pipeline); the
        # timed region spans the first copy to the last read-back.
        #   e2e            : result = the loss (4 bytes)
        #   e2e_with_grads : result = loss + dH + this rank's dW shard, copied out on a
        #                    third stream while the next step computes (double-buffered
        #                    gradient outputs)
        Hh = H.cpu().pin_memory()
        Wh = Ws.contiguous().cpu().pin_memory()
        Yh = Y.cpu().pin_memory()
        slots = [(torch.empty_like(H), torch.empty_like(Ws), torch.empty_like(Y)) for _ in range(2)]
        probs = [fce.make_problem(*sl, ign, lo, v) for sl in slots]
        loss_h = torch.empty((), dtype=torch.float32).pin_memory()
        copy_stream = torch.cuda.Stream(dev)
        out_stream = torch.cuda.Stream(dev)
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

        def run_e2e(nsteps, grads):
            gslots = gdone = gfree = dh_h = dw_h = None
            if grads:
                gslots = [(dh, dw), (torch.empty_like(dh), torch.empty_like(dw))]
                gdone = [torch.cuda.Event() for _ in range(2)]
                gfree = [torch.cuda.Event() for _ in range(2)]
                dh_h = torch.empty(dh.shape, dtype=dh.dtype).pin_memory()
                dw_h = torch.empty(dw.shape, dtype=dw.dtype).pin_memory()
                for g in gfree:
                    g.record(stream)
            for s_ in range(2):
                free[s_].record(stream)
            ctx.barrier()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(copy_stream)
            enqueue_copy(0)
            for i in range(nsteps):
                if i + 1 < nsteps:
                    enqueue_copy(i + 1)
                s_ = i % 2
                stream.wait_event(ready[s_])
                if grads:
                    stream.wait_event(gfree[s_])
                    step(probs[s_][0], *gslots[s_])
                    gdone[s_].record(stream)
                    with torch.cuda.stream(out_stream):
                        out_stream.wait_event(gdone[s_])
                        dh_h.copy_(gslots[s_][0], non_blocking=True)
                        dw_h.copy_(gslots[s_][1], non_blocking=True)
                        gfree[s_].record(out_stream)
                else:
                    step(probs[s_][0])
                free[s_].record(stream)
                loss_h.copy_(loss, non_blocking=True)
            if grads:
                stream.wait_stream(out_stream)
            t1.record(stream)
            ctx.barrier()
            return ctx.max(t0.elapsed_time(t1))

        run_e2e(1, False)  # warm the copy path
        ms_e2e = run_e2e(args.e2e_steps, False)
        e2e_val = n * args.e2e_steps / (ms_e2e / 1e3)
        # whole-job bytes per step: every rank copies H and the targets, W is copied once in shards
        h2d = world * (n * d * 2 + n * 8) + v * d * 2
        e2e_g = None
        if not args.no_e2e_grads:
            ms_e2e_g = run_e2e(args.e2e_steps, True)
            e2e_g = {"value": n * args.e2e_steps / (ms_e2e_g / 1e3), "unit": "tokens/s",
                     "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(world * (n * d * 4 + 4) + v * d * 4),
                     "path": "as e2e, plus every step's dH and dW (fp32) copied to pinned host memory on a third "
                             "stream, overlapped with the next step (double-buffered gradients)"}
        h.close()

    if rank != 0:
        return None

    peaks = load_peaks()
    flops_step = 8.0 * n_valid * d * v
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
    traffic = _traffic_from_profile(args.config, names[dom].split(" ")[0]) if world == 1 else None
    if comm is None:
        par = "single GPU"
    elif ctx.transport == "nccl":
        par = f"vocab-parallel x{world} (NCCL, one process per GPU)"
    elif ctx.transport == "ipc":
        par = (f"vocab-parallel x{world} (IPC transport: one process per rank, libfce collectives over CUDA IPC, "
               f"{min(world, torch.cuda.device_count())} GPU(s))")
    else:
        par = (f"vocab-parallel x{world} (in-process local transport, {world} rank threads on "
               f"{args.local_gpus} GPU(s): the {world}-rank code path, not {world}-GPU throughput)")
    line = {
        "metric": METRIC,
        "value": tokens_per_s,
        "unit": "tokens/s",
        "n_gpus": world if ctx.transport == "nccl" else min(world, torch.cuda.device_count()),
        "steps": args.steps,
        "warmup": max(args.warmup, 3),
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic: reference splitmix64 instance (seed 42) generated on device, bf16 grid",
        "config": {"workload": CONFIG_LABEL[args.config], "N": n, "N_valid": n_valid, "D": d, "V": v,
                   "reduction": "mean", "ignore_fraction": frac, "ranks": world,
                   "parallelism": par,
                   "l2": "inputs larger than L2 (W bf16 = %.2f GB)" % (v * d * 2 / 1e9)},
        "tflops_8ndv": flops_step / (ms_step / 1e3) / 1e12,
        # per-GPU fraction of the measured bf16 peak (whole-job flops / N GPUs)
        "pct_peak_step": flops_step / (ms_step / 1e3) / 1e12 / peaks["bf16_tflops"] / world,
        "pct_peak_step_sustained": flops_step / (ms_step / 1e3) / 1e12 / peak_sust / world,
        "model_tflops_6ndv": 6.0 * n_valid * d * v / (ms_step / 1e3) / 1e12,
        "peak_hbm_bytes": int(peak_torch + ws_peak),
        "peak_hbm_breakdown": {"torch_inputs_outputs": int(peak_torch), "library_workspace": int(ws_peak)},
        "canonical_nxv_fp32_bytes": int(n) * int(v) * 4,
        "loss": loss_val,
        "roofline": {"bound": "tensor", "kernel": names[dom], "achieved": achieved, "peak": peak_sust,
                     "unit": "TFLOP/s", "frac": achieved / peak_sust,
                     "frac_of_burst_peak": achieved / peaks["bf16_tflops"],
                     "peak_source": peaks["source"] + " bf16_tflops_sustained (kernel timed inside a long step)",
                     "traffic": traffic["bytes"] if traffic else None,
                     "traffic_source": traffic["source"] if traffic else None,
                     "algorithmic_flops_per_launch": kfl / max(kl, 1),
                     "flops_basis": "2*N_valid*D*V per contraction (live rows only)",
                     "avg_launch_ms": per_launch_ms},
        "kernels": kernels,
        "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 4 * world,
                "path": "C-ABI fce_forward+fce_backward; every step copies pinned host H, W (bf16) and targets "
                        "in (copy of step i+1 overlapped with step i on a second stream) and the loss out"},
        "gpu_launches": int(launches),
        "clocks": clk,
    }
    if e2e_g:
        line["e2e_with_grads"] = e2e_g
    if world == 1 and not args.no_dropin:
        line["e2e_dropin_cpp"] = _dropin_e2e(n, d, v) if frac == 0 else None
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline(args.config)
        except Exception as exc:  # never lose the GPU line over the CPU sample
            line["cpu_baseline"] = {"value": None, "unit": "tokens/s", "cores": os.cpu_count(),
                                    "kind": "reference", "sample": f"failed: {exc!r}"}
    return line


def _dropin_e2e(n, d, v):
    """The drop-in C++ API (fusedce::fused_forward + fused_backward_recompute)
    with host buffers at this shape (tests/cpp/bench_dropin, built by make): the
    switch-the-include-path user's end-to-end number, uploads and owning host
    results (dH, dW) included."""
    exe = os.path.join(ROOT, "tests", "cpp", "bench_dropin")
    if not os.path.exists(exe):
        return {"value": None, "note": "tests/cpp/bench_dropin not built"}
    try:
        r = subprocess.run([exe, str(n), str(d), str(v), "2"], capture_output=True, text=True, timeout=600)
        out = [l for l in r.stdout.splitlines() if l.startswith("{")]
        return json.loads(out[-1]) if r.returncode == 0 and out else {"value": None, "note": r.stderr[-300:]}
    except Exception as exc:  # never lose the GPU line over this leg
        return {"value": None, "note": repr(exc)}


def _traffic_from_profile(cfg, kernel):
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    capture of the CURRENT sources (profiles/traffic.json records the hash of
    csrc/* it was captured on — kernels and the host launch plans; a stale
    entry is not reported)."""
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(tpath):
        return None
    try:
        data = json.load(open(tpath))
        src_hash = _source_hash()
        ent = data.get(cfg, {}).get(kernel)
        if not ent or ent.get("source_sha") != src_hash:
            return None
        return {"bytes": ent["dram_bytes"], "source": f"ncu --set full capture {ent.get('capture', '')} "
                                                      f"(dram__bytes_read.sum + dram__bytes_write.sum)"}
    except Exception:
        return None


def _source_hash():
    """Hash of the kernel sources the traffic number was measured on."""
    import hashlib
    hsh = hashlib.sha256()
    csrc = os.path.join(ROOT, "paper_2511_17599_b200", "csrc")
    for name in sorted(os.listdir(csrc)):
        if name.endswith((".cu", ".cuh", ".h", ".cpp")):
            with open(os.path.join(csrc, name), "rb") as f:
                hsh.update(f.read())
    return hsh.hexdigest()[:16]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="llama3-8b", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="fce", choices=["fce", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e-grads", action="store_true")
    ap.add_argument("--no-dropin", action="store_true", help="skip the C++ drop-in API end-to-end leg")
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "ipc", "local"],
                    help="N > 1 without torchrun: NCCL processes (needs N GPUs), IPC processes (libfce "
                         "collectives, ranks may share GPUs) or in-process local ranks")
    ap.add_argument("--force-vp", action="store_true",
                    help="use the native vocab-parallel (NCCL) path even on one rank (testing)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch

    world_env = os.environ.get("WORLD_SIZE")
    if world_env is not None:
        world = int(world_env)
        if world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
        ctx = DistCtx(world, int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
                      args.force_vp)
        line = bench_rank(ctx, args)
        ctx.close()
        if line is not None:
            print(json.dumps(line), flush=True)
        return 0

    ngpu = torch.cuda.device_count()
    args.local_gpus = min(ngpu, args.gpus)
    if args.gpus == 1:
        ctx = DistCtx(1, 0, 0, args.force_vp)
        line = bench_rank(ctx, args)
        ctx.close()
        print(json.dumps(line), flush=True)
        return 0
    use_procs = args.transport in ("nccl", "ipc") or (args.transport == "auto" and ngpu >= args.gpus)
    if use_procs:
        # one process per rank: re-launch under torch.distributed.run (rank 0 prints the line)
        env = dict(os.environ, FCE_BENCH_TRANSPORT="ipc" if args.transport == "ipc" else "nccl")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd, env=env)
    # fewer GPUs than ranks: the N ranks as threads over the in-process transport
    from paper_2511_17599_b200 import vocab_parallel as vp
    devices = [r % max(ngpu, 1) for r in range(args.gpus)]
    group = vp.LocalGroup(args.gpus)
    comms = [group.comm(r, devices[r]) for r in range(args.gpus)]
    shared = {"barrier": threading.Barrier(args.gpus), "vals": [0.0] * args.gpus}
    out, errs = [None] * args.gpus, [None] * args.gpus

    def body(r):
        try:
            out[r] = bench_rank(ThreadCtx(args.gpus, r, devices[r], comms[r], shared), args)
        except BaseException as exc:  # noqa: BLE001
            errs[r] = exc
            shared["barrier"].abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(args.gpus)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for c in comms:
        c.close()
    group.close()
    for e in errs:
        if e is not None and not isinstance(e, threading.BrokenBarrierError):
            raise e
    for e in errs:
        if e is not None:
            raise e
    print(json.dumps(out[0]), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
