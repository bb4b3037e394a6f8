"""Vocabulary-parallel parity over real ranks (one process per GPU, NCCL):

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \\
        scripts/vp_parity.py [--n 4096 --d 1024 --v 50000 --ignore 0.25]

Every rank holds its ceil-first W shard and runs fce_vp_forward /
fce_vp_backward (stats all-gather + dH all-reduce over NCCL); rank 0 then
compares the merged loss / stats, the all-reduced dH and the gathered dW shards
with the single-GPU path on the same seeded instance.  Exit code 0 = parity.
"""
import argparse
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_17599_b200 as fce  # noqa: E402
from paper_2511_17599_b200 import vocab_parallel as vp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--d", type=int, default=1024)
    ap.add_argument("--v", type=int, default=50000)
    ap.add_argument("--ignore", type=float, default=0.25)
    ap.add_argument("--reduction", default="mean")
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ign = -100 if a.ignore > 0 else None
    H, W, Y = fce.generate_instance(a.n, a.d, a.v, 42, -100, a.ignore, device=local)
    lo, hi = fce.shard_ranges(a.v, world)[rank]
    comm = vp.NativeComm.from_torch_distributed(local)
    out = vp.native_forward(comm, H, W[lo:hi], Y, lo, a.v, a.reduction, ign)
    dh, dw = vp.native_backward(comm, H, W[lo:hi], Y, lo, a.v, out.stats, a.reduction, 1.0, ign)
    torch.cuda.synchronize()
    # gather the dW shards on rank 0 (uneven shard sizes: pad to the largest)
    rows = max(h_ - l_ for l_, h_ in fce.shard_ranges(a.v, world))
    pad = torch.zeros(rows, a.d, device=dev)
    pad[: hi - lo] = dw
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    ok = True
    if rank == 0:
        ref = fce.fused_forward(H, W, Y, a.reduction, ign)
        rdh, rdw = fce.fused_backward_recompute(H, W, Y, ref.stats, a.reduction, 1.0, ign)
        gdw = torch.cat([parts[r][: h_ - l_] for r, (l_, h_) in enumerate(fce.shard_ranges(a.v, world))])
        loss_err = abs(out.loss.item() - ref.loss.item()) / max(1.0, abs(ref.loss.item()))
        dh_err = ((dh - rdh).abs().max() / rdh.abs().max()).item()
        dw_err = ((gdw - rdw).abs().max() / rdw.abs().max()).item()
        found_ok = torch.equal(out.stats.found, ref.stats.found)
        ok = loss_err < 1e-5 and dh_err < 1e-4 and dw_err < 1e-4 and found_ok
        print(f"ranks={world} loss {out.loss.item():.6f} (1-GPU {ref.loss.item():.6f}, rel {loss_err:.1e}) "
              f"dH rel-max {dh_err:.1e} dW rel-max {dw_err:.1e} found-equal {found_ok} -> "
              f"{'PARITY' if ok else 'MISMATCH'}", flush=True)
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.all_reduce(flag)
    comm.close()
    dist.destroy_process_group()
    return int(flag.item() != 0)


if __name__ == "__main__":
    sys.exit(main())
