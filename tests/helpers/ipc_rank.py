"""One rank of a multi-process job over the IPC transport (helper of
tests/test_multirank_gpu.py; not collected by pytest).

    python tests/helpers/ipc_rank.py <rank> <nranks> <id-hex> <inputs.npz> <out.npz>

Runs tp_forward + tp_backward (fce_vp_forward / fce_vp_backward) on this rank's
ceil-first vocabulary shard, then one raw all-reduce / all-gather /
reduce-scatter, and saves what it got."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2511_17599_b200 as fce  # noqa: E402
from paper_2511_17599_b200 import vocab_parallel as vp  # noqa: E402


def main():
    rank, k = int(sys.argv[1]), int(sys.argv[2])
    uid = bytes.fromhex(sys.argv[3])
    inp = np.load(sys.argv[4])
    torch.cuda.set_device(0)
    comm = vp.NativeComm.create_ipc(k, rank, 0, uid)
    assert comm.query() == (k, rank, 3)
    h = fce.Handle(0)
    H = torch.from_numpy(inp["H"]).cuda().to(torch.bfloat16)
    W = torch.from_numpy(inp["W"]).cuda().to(torch.bfloat16)
    Y = torch.from_numpy(inp["Y"]).cuda()
    ign = int(inp["ign"]) if int(inp["has_ign"]) else None
    v = W.shape[0]
    lo, hi = fce.shard_ranges(v, k)[rank]
    out = vp.native_forward(comm, H, W[lo:hi], Y, lo, v, "mean", ign, handle=h)
    if int(inp["chunks"]):
        h.set_option("vp_overlap_chunks", int(inp["chunks"]))
    if int(inp["fused"]):
        h.set_option("vp_fused_dh", 1)
    dh, dw = vp.native_backward(comm, H, W[lo:hi], Y, lo, v, out.stats, "mean", 1.0, ign, handle=h)
    # sequence-parallel backward: this rank's ceil-first position shard of dH
    plo, phi = fce.shard_ranges(H.shape[0], k)[rank]
    dh_sp, _ = vp.native_sp_vp_backward(comm, H, W[lo:hi], Y, lo, v, out.stats, phi - plo, "mean", 1.0, ign,
                                        handle=h)
    x = torch.from_numpy(inp["x"][rank]).cuda()
    s = vp.native_all_reduce(comm, x.clone(), handle=h)
    g = vp.native_all_gather(comm, torch.full((5,), float(rank), device="cuda"), handle=h)
    rs = vp.native_reduce_scatter(comm, torch.arange(k * 9, dtype=torch.float32, device="cuda") * (rank + 1),
                                  handle=h)
    torch.cuda.synchronize()
    np.savez(sys.argv[5], loss=out.loss.item(), found=out.stats.found.cpu().numpy(), lse=out.lse.cpu().numpy(),
             dh=dh.cpu().numpy(), dw=dw.cpu().numpy(), dh_sp=dh_sp.cpu().numpy(), s=s.cpu().numpy(), g=g.cpu().numpy(), rs=rs.cpu().numpy())
    h.close()
    comm.close()


if __name__ == "__main__":
    main()
