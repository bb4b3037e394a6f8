"""G-ring residency probe: the persistent backward under
several (row_chunk, band) geometries, one measured launch each after a warm-up
launch, for an ncu capture of DRAM bytes per launch:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:fce_bwd_persistent --csv python scripts/g_residency_probe.py

The G ring is 2 x row_chunk x band x 2 B.  The default plan (16384 x 3072,
192 MB) spills G to HBM; the "L2-resident" plans keep the ring <= 50 MB at the
cost of more dH passes (V / band) or more dW passes (N / row_chunk).  Per
geometry it also prints the output traffic the plan implies (dH fp32
read-modify-write per band pass, dW fp32 store + RMW per extra row chunk) so
the G-attributable rest can be read off the capture.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402

GEOMS = [(0, 0), (4096, 3072), (8192, 1536), (2048, 6144), (16384, 768)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="16384,4096,128256")
    ap.add_argument("--geoms", default="", help="rc:band[:l2_hints[:dh_group]],... (0:0 = default plan)")
    a = ap.parse_args()
    n, d, v = (int(x) for x in a.shape.split(","))
    geoms = [tuple(int(y) for y in g.split(":")) for g in a.geoms.split(",")] if a.geoms else GEOMS
    H, W, Y = fce.generate_instance(n, d, v, 42)
    dh = torch.empty(n, d, device="cuda")
    for g in geoms:
        rc, band = g[0], g[1]
        h = fce.Handle(0)
        h.set_option("validate", 0)
        if len(g) > 2:
            h.set_option("l2_hints", g[2])
        if len(g) > 3:
            h.set_option("dh_group", g[3])
        if rc:
            h.set_option("row_chunk", rc)
        if band:
            h.set_option("band_cols", band)
        out = fce.fused_forward(H, W, Y, "mean", handle=h)
        for _ in range(2):
            fce.fused_backward_recompute(H, W, Y, out.stats, "mean", 1.0, handle=h, dhidden=dh)
        torch.cuda.synchronize()
        rc_e = rc or 16384
        band_e = band or 3072
        passes_dh = -(-v // band_e)
        passes_dw = -(-n // rc_e)
        out_rw = passes_dh * n * d * 4 * 2 + v * d * 4 * (2 * passes_dw - 1)
        ring = 2 * min(rc_e, n) * band_e * 2
        print(f"geometry row_chunk={rc_e} band={band_e} l2_hints={g[2] if len(g) > 2 else 1}: ring {ring / 2**20:.0f} MiB, dH passes {passes_dh}, "
              f"dW passes {passes_dw}, output read+write bytes {out_rw / 1e9:.2f} GB", flush=True)
        h.close()


if __name__ == "__main__":
    main()
