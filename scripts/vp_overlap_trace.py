"""Device trace of the overlapped vocab-parallel backward (option
vp_overlap_chunks): when does each row chunk's dH all-reduce run relative to
the persistent kernel?  One rank of an in-process group (the collective is
then the local transport's peer-sum kernel over the chunk's rows; with k
ranks on k GPUs it would be the same stream structure).

The kernel's per-unit trace (option trace_ptr, globaltimer) gives its
timeline; the communicator stamps (option comm_trace_ptr) give, per chunk,
when the comm stream was released by the kernel's counter and when the
chunk's all-reduce finished.

  python scripts/vp_overlap_trace.py [--n 16384 --d 4096 --v 16032 --chunks 2 --reserve 8]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402
from paper_2511_17599_b200 import vocab_parallel as vp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--v", type=int, default=16032, help="per-rank vocab shard (Llama-3-8B V / 8)")
    ap.add_argument("--chunks", type=int, default=2)
    ap.add_argument("--reserve", type=int, default=8)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    H, W, Y = fce.generate_instance(a.n, a.d, a.v, 42)

    def rank_fn(r, comm, h):
        out = vp.native_forward(comm, H, W, Y, 0, a.v, "mean", None, handle=h)
        trace = torch.zeros(4 << 20, dtype=torch.int64, device="cuda")
        ctrace = torch.zeros(64, dtype=torch.int64, device="cuda")
        rows = []
        for mode in ("plain", "overlap"):
            h.set_option("vp_overlap_chunks", a.chunks if mode == "overlap" else 0)
            h.set_option("vp_reserve_sms", a.reserve)
            for rep in range(a.reps):
                trace.zero_()
                ctrace.zero_()
                h.set_option("trace_ptr", trace.data_ptr())
                h.set_option("comm_trace_ptr", ctrace.data_ptr())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                vp.native_backward(comm, H, W, Y, 0, a.v, out.stats, "mean", 1.0, None, handle=h)
                e1.record()
                torch.cuda.synchronize()
                h.set_option("trace_ptr", 0)
                h.set_option("comm_trace_ptr", 0)
                t = trace.view(-1, 8).cpu()
                k0 = int(t[t[:, 0] > 0, 0].min())   # first MMA of the launch
                k1 = int(t[t[:, 2] > 0, 2].max())   # last unit's epilogue
                c = ctrace.cpu().tolist()
                rows.append((mode, rep, e0.elapsed_time(e1), (k1 - k0) / 1e6,
                             [((c[2 * i] - k0) / 1e6, (c[2 * i + 1] - k0) / 1e6) for i in range(a.chunks)
                              if c[2 * i]]))
        return rows

    for mode, rep, ms, kms, chunks in vp.run_ranks(1, rank_fn)[0]:
        print(f"{mode:8s} rep {rep}: step {ms:.3f} ms, kernel {kms:.3f} ms, chunk all-reduce "
              f"[released, done] ms after kernel start: "
              + ", ".join(f"[{s:.3f}, {e:.3f}]" for s, e in chunks))


if __name__ == "__main__":
    main()
