"""Vocabulary-parallel fused LCE across ranks (one process per GPU).

Two front ends over the same per-rank CUDA work:

* ``NativeComm`` / ``native_forward`` / ``native_backward`` drive the C-ABI in
  ``include/fce/fce_vp.h``: NCCL is owned by libfce.so and the collectives run
  on the handle's stream (what a C++ caller of the drop-in ``tp_forward`` /
  ``tp_backward`` gets).
* ``VocabParallel`` does the same exchange with ``torch.distributed``
  collectives, with the per-rank compute injectable.  On GPUs the compute is
  the CUDA path (``CudaCompute``); the gloo tests plug the CPU oracle in to
  check the orchestration (shard layout, gather order, dH sum) without GPUs.

Semantics follow the reference's in-process simulation
(proj/include/fusedce/parallel_sim.hpp:158-290): ceil-first contiguous W
shards, per-rank (m, a, z_target, found) partials merged in rank order
(identical stats, lse and loss on every rank), dW kept per shard, dH summed.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import paper_2511_17599_b200 as fce


# ------------------------------------------------------------------ native

class NativeComm:
    """An NCCL communicator owned by libfce.so (fce_comm_init)."""

    def __init__(self, ptr, nranks: int, rank: int, device: int):
        self.ptr = ptr
        self.nranks = nranks
        self.rank = rank
        self.device = device

    @staticmethod
    def unique_id() -> bytes:
        lib = fce.load_library()
        buf = (ctypes.c_uint8 * 128)()
        fce._check(lib.fce_comm_unique_id(buf, 128), vp=True)
        return bytes(buf)

    @classmethod
    def create(cls, nranks: int, rank: int, device: int, uid: bytes) -> "NativeComm":
        lib = fce.load_library()
        ptr = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        fce._check(lib.fce_comm_init(ctypes.byref(ptr), device, nranks, rank, buf, 128), vp=True)
        return cls(ptr, nranks, rank, device)

    @classmethod
    def create_local(cls, device: int = 0) -> "NativeComm":
        return cls.create(1, 0, device, cls.unique_id())

    @classmethod
    def from_torch_distributed(cls, device: int, group=None) -> "NativeComm":
        """Rank 0 makes the NCCL id, torch.distributed ships it to the others."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.create(world, rank, device, obj[0])

    def close(self):
        if self.ptr:
            fce.load_library().fce_comm_destroy(self.ptr)
            self.ptr = None


def native_forward(comm: NativeComm, hidden, weight_shard, targets, v_offset: int, v_total: int,
                   reduction: str = "mean", ignore_index=None, handle=None) -> fce.FusedOutput:
    """tp_forward over real ranks (fce_vp_forward)."""
    import torch
    h = handle or fce.default_handle(hidden.device.index or 0)
    p, keep = fce.make_problem(hidden, weight_shard, targets, ignore_index, v_offset, v_total)
    dev = hidden.device
    st = fce.Stats.empty(p.n, dev)
    lse = torch.empty(p.n, dtype=torch.float32, device=dev)
    rows = torch.empty(p.n, dtype=torch.float32, device=dev)
    red = torch.empty((), dtype=torch.float32, device=dev)
    fce._check(h.lib.fce_vp_forward(h.raw, comm.ptr, ctypes.byref(p), fce.REDUCTIONS[reduction],
                                    st.c(), lse.data_ptr(), rows.data_ptr(), red.data_ptr()))
    return fce.FusedOutput(rows if reduction == "none" else red, st, lse, rows)


def native_backward(comm: NativeComm, hidden, weight_shard, targets, v_offset: int, v_total: int,
                    stats: fce.Stats, reduction: str = "mean", upstream=1.0, ignore_index=None,
                    handle=None):
    """tp_backward over real ranks (fce_vp_backward) -> (dH summed over ranks, local dW shard)."""
    import torch
    h = handle or fce.default_handle(hidden.device.index or 0)
    p, keep = fce.make_problem(hidden, weight_shard, targets, ignore_index, v_offset, v_total)
    dev = hidden.device
    dh = torch.empty(p.n, p.d, dtype=torch.float32, device=dev)
    dw = torch.empty(p.v, p.d, dtype=torch.float32, device=dev)
    up_rows = None if isinstance(upstream, (int, float)) else upstream.float().contiguous()
    fce._check(h.lib.fce_vp_backward(h.raw, comm.ptr, ctypes.byref(p), stats.c(),
                                     fce.REDUCTIONS[reduction],
                                     float(upstream) if up_rows is None else 0.0,
                                     fce._ptr(up_rows), dh.data_ptr(), p.d, dw.data_ptr(), p.d))
    return dh, dw


# ------------------------------------------------------- torch.distributed

class CudaCompute:
    """Per-rank compute of the vocab-parallel step on this GPU (C-ABI kernels)."""

    def partial(self, hidden, weight_shard, targets, v_offset, v_total, ignore_index):
        st = fce.tp_rank_partial(hidden, weight_shard, v_offset, v_total, targets, ignore_index)
        return st.m, st.a, st.z_target, st.found

    def merge(self, m, a, z, f, targets, reduction, ignore_index):
        parts = [fce.Stats(m[r], a[r], z[r], f[r]) for r in range(m.shape[0])]
        out = fce.merge_rank_partials(parts, targets, reduction, ignore_index)
        return out

    def backward(self, hidden, weight_shard, targets, v_offset, v_total, stats, reduction,
                 upstream, ignore_index):
        h = fce.default_handle(hidden.device.index or 0)
        import torch
        p, keep = fce.make_problem(hidden, weight_shard, targets, ignore_index, v_offset, v_total)
        dh = torch.empty(p.n, p.d, dtype=torch.float32, device=hidden.device)
        dw = torch.empty(p.v, p.d, dtype=torch.float32, device=hidden.device)
        up_rows = None if isinstance(upstream, (int, float)) else upstream.float().contiguous()
        fce._check(h.lib.fce_backward(h.raw, ctypes.byref(p), stats.c(), fce.REDUCTIONS[reduction],
                                      float(upstream) if up_rows is None else 0.0, fce._ptr(up_rows),
                                      dh.data_ptr(), p.d, dw.data_ptr(), p.d, 0))
        return dh, dw


class VocabParallel:
    """One rank of tp_forward / tp_backward over a torch.distributed group."""

    def __init__(self, vocab: int, group=None, compute=None):
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.vocab = vocab
        self.ranges = fce.shard_ranges(vocab, self.world)
        self.lo, self.hi = self.ranges[self.rank]
        self.compute = compute or CudaCompute()

    def shard(self, weight):
        """This rank's contiguous ceil-first slice of the full W (shard_weights, parallel_sim.hpp:78-93)."""
        return weight[self.lo:self.hi]

    def forward(self, hidden, weight_shard, targets, reduction="mean", ignore_index=None):
        import torch
        import torch.distributed as dist
        if weight_shard.shape[0] != self.hi - self.lo:
            raise fce.InvalidLayout("weight shard does not match this rank's vocabulary range")
        m, a, z, f = self.compute.partial(hidden, weight_shard, targets, self.lo, self.vocab,
                                          ignore_index)
        gathered = []
        for t in (m, a, z, f):
            out = [torch.empty_like(t) for _ in range(self.world)]
            dist.all_gather(out, t.contiguous(), group=self.group)
            gathered.append(torch.stack(out))  # [rank, n]: rank order == vocab order
        return self.compute.merge(*gathered, targets, reduction, ignore_index)

    def backward(self, hidden, weight_shard, targets, stats, reduction="mean", upstream=1.0,
                 ignore_index=None):
        import torch.distributed as dist
        dh, dw = self.compute.backward(hidden, weight_shard, targets, self.lo, self.vocab, stats,
                                       reduction, upstream, ignore_index)
        dist.all_reduce(dh, group=self.group)
        return dh, dw


# ------------------------------------------------------- SP -> TP and DP
# (reference parallel_sim.hpp:294-378)

def sp_to_tp_gather(hidden_shard, positions: int, group=None):
    """Sequence-parallel -> tensor-parallel switch: every rank holds a ceil-first
    position shard of H; all-gather them into the full H (sp_to_tp_gather,
    parallel_sim.hpp:294-314).  Shards may be ragged (padded for the collective)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    ranges = fce.shard_ranges(positions, world)
    rows = max(hi - lo for lo, hi in ranges)
    pad = torch.zeros(rows, hidden_shard.shape[1], dtype=hidden_shard.dtype, device=hidden_shard.device)
    pad[: hidden_shard.shape[0]] = hidden_shard
    out = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(out, pad, group=group)
    return torch.cat([o[: hi - lo] for o, (lo, hi) in zip(out, ranges)])


def tp_to_sp_scatter(dhidden_partial, positions: int, group=None):
    """Inverse of the gather for the backward: sum the ranks' dH partials and keep
    this rank's position shard (a reduce-scatter; replaces the all-reduce when the
    caller is sequence parallel)."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    ranges = fce.shard_ranges(positions, world)
    rows = max(hi - lo for lo, hi in ranges)
    parts = []
    for lo, hi in ranges:
        p = torch.zeros(rows, dhidden_partial.shape[1], dtype=dhidden_partial.dtype, device=dhidden_partial.device)
        p[: hi - lo] = dhidden_partial[lo:hi]
        parts.append(p)
    out = torch.empty_like(parts[0])
    if dist.get_backend(group) == "gloo":  # gloo has no reduce_scatter
        full = torch.cat(parts)
        dist.all_reduce(full, group=group)
        out = full[rank * rows:(rank + 1) * rows].clone()
    else:
        dist.reduce_scatter(out, parts, group=group)
    lo, hi = ranges[rank]
    return out[: hi - lo]


class LocalCompute:
    """Per-replica fused forward + backward on this GPU (for dp_step)."""

    def step(self, hidden, weight, targets, reduction, ignore_index):
        out = fce.fused_forward(hidden, weight, targets, reduction, ignore_index)
        dh, dw = fce.fused_backward_recompute(hidden, weight, targets, out.stats, reduction, 1.0, ignore_index)
        return out.loss, dh, dw


def dp_step(hidden, weight, targets, reduction="mean", ignore_index=None, group=None, compute=None):
    """Data-parallel step (dp_step, parallel_sim.hpp:334-378): every rank runs the
    fused forward + backward on its micro-batch; loss and dW are averaged over
    ranks with all-reduce; dH stays rank-local.  Returns (loss, dH, dW)."""
    import torch
    import torch.distributed as dist
    if reduction == "none":
        raise fce.UnsupportedReduction("data-parallel loss sync requires a scalar reduction")
    world = dist.get_world_size(group)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([hidden.shape[0]], dtype=torch.int64), group=group) \
        if dist.get_backend(group) == "gloo" else None
    if dist.get_backend(group) == "gloo" and len({int(s) for s in sizes}) != 1:
        raise fce.InvalidLayout("replica micro-batches must have equal sizes")
    loss, dh, dw = (compute or LocalCompute()).step(hidden, weight, targets, reduction, ignore_index)
    loss = torch.as_tensor(loss, dtype=torch.float32, device=dw.device).reshape(1).clone()
    dist.all_reduce(loss, group=group)
    dist.all_reduce(dw, group=group)
    return loss / world, dh, dw / world
