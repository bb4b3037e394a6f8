"""Per-rank cost of the three vocab-parallel dH reductions on one B200 (one
rank of an in-process group; the collective itself is then a 1-rank pass over
dH): plain (all-reduce after the kernel), overlapped (vp_overlap_chunks) and
fused (vp_fused_dh: reduce-adds into the owners' accumulators inside the
kernel).  Interleaved blocks, CUDA events around fce_vp_backward.

  python scripts/vp_modes_probe.py [--n 16384 --d 4096 --v 16032]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402
from paper_2511_17599_b200 import vocab_parallel as vp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=16384)
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--v", type=int, default=16032)
ap.add_argument("--blocks", type=int, default=6)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
H, W, Y = fce.generate_instance(a.n, a.d, a.v, 42)
MODES = {"plain": {}, "overlap4": {"vp_overlap_chunks": 4, "vp_reserve_sms": 8},
         "overlap4_r4": {"vp_overlap_chunks": 4, "vp_reserve_sms": 4}, "fused": {"vp_fused_dh": 1}}


def rank_fn(r, comm, h):
    out = vp.native_forward(comm, H, W, Y, 0, a.v, "mean", None, handle=h)
    dh = torch.empty(a.n, a.d, device="cuda")
    res = {m: [] for m in MODES}
    for b in range(a.blocks):
        for m, opts in (MODES.items() if b % 2 == 0 else reversed(list(MODES.items()))):
            h.set_option("vp_overlap_chunks", 0)
            h.set_option("vp_fused_dh", 0)
            for k_, v_ in opts.items():
                h.set_option(k_, v_)
            vp.native_backward(comm, H, W, Y, 0, a.v, out.stats, "mean", 1.0, None, handle=h, dhidden=dh)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                vp.native_backward(comm, H, W, Y, 0, a.v, out.stats, "mean", 1.0, None, handle=h, dhidden=dh)
            e1.record()
            torch.cuda.synchronize()
            res[m].append(e0.elapsed_time(e1) / a.reps)
    return res


res = vp.run_ranks(1, rank_fn)[0]
for m, t in res.items():
    t = sorted(t)
    print(f"{m:12s} median {t[len(t) // 2]:.3f} ms  min {t[0]:.3f} ms  ({len(t)} blocks x {a.reps})")
