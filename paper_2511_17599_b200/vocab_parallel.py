"""Vocabulary-parallel fused LCE across ranks (one process per GPU).

Two front ends over the same per-rank CUDA work:

* ``NativeComm`` / ``native_forward`` / ``native_backward`` /
  ``native_sp_gather`` / ``native_sp_scatter`` / ``native_dp_step`` drive the
  C-ABI in ``include/fce/fce_vp.h``: the communicator is owned by libfce.so
  (NCCL, one process per GPU; or ``LocalGroup``: k ranks as k threads of one
  process, collectives by libfce's peer-memory kernels — ``run_ranks`` runs a
  k-rank job that way on one GPU) and the collectives run on the handle's
  stream (what a C++ caller of the drop-in ``tp_forward`` / ``tp_backward``
  gets).
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

    @staticmethod
    def ipc_id() -> bytes:
        """Rendezvous id of an IPC communicator (rank 0 makes it, ships it)."""
        lib = fce.load_library()
        buf = (ctypes.c_uint8 * 128)()
        fce._check(lib.fce_comm_ipc_id(buf, 128), vp=True)
        return bytes(buf)

    @classmethod
    def create_ipc(cls, nranks: int, rank: int, device: int, uid: bytes) -> "NativeComm":
        """IPC transport: one process per rank, libfce's collectives over CUDA
        IPC peer memory (no NCCL); ranks may share a GPU."""
        lib = fce.load_library()
        ptr = ctypes.c_void_p()
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        fce._check(lib.fce_comm_init_ipc(ctypes.byref(ptr), device, nranks, rank, buf, 128), vp=True)
        return cls(ptr, nranks, rank, device)

    @classmethod
    def from_torch_distributed_ipc(cls, device: int, group=None) -> "NativeComm":
        """IPC communicator over the ranks of a torch.distributed group (any backend)."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.ipc_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls.create_ipc(world, rank, device, obj[0])

    @classmethod
    def create_local(cls, device: int = 0) -> "NativeComm":
        """A 1-rank NCCL communicator on `device`."""
        return cls.create(1, 0, device, cls.unique_id())

    def query(self):
        """(nranks, rank, transport) with transport 1 = NCCL, 2 = local, 3 = ipc."""
        lib = fce.load_library()
        k, r, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        fce._check(lib.fce_comm_query(self.ptr, ctypes.byref(k), ctypes.byref(r), ctypes.byref(t)), vp=True)
        return k.value, r.value, t.value

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


class LocalGroup:
    """In-process communicator group (fce_comm_group_create): `nranks` ranks of
    this process, each driven by its own host thread, on any devices (several
    may share one GPU).  Its collectives are libfce's own peer-memory kernels,
    so the k-rank vocab-parallel / SP / DP code runs on a single B200."""

    def __init__(self, nranks: int):
        lib = fce.load_library()
        self.nranks = nranks
        self.ptr = ctypes.c_void_p()
        fce._check(lib.fce_comm_group_create(ctypes.byref(self.ptr), nranks), vp=True)

    def comm(self, rank: int, device: int = 0) -> NativeComm:
        lib = fce.load_library()
        ptr = ctypes.c_void_p()
        fce._check(lib.fce_comm_init_local(ctypes.byref(ptr), self.ptr, device, rank), vp=True)
        return NativeComm(ptr, self.nranks, rank, device)

    def close(self):
        if self.ptr:
            fce.load_library().fce_comm_group_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_ranks(nranks: int, fn, devices=None):
    """Run ``fn(rank, comm, handle)`` for every rank of a fresh LocalGroup, each
    on its own host thread, CUDA stream and library handle (what one process
    per GPU gives each rank).  Returns the per-rank results in rank order and
    re-raises the first rank's exception.  ctypes releases the GIL inside the
    library, so the ranks meet in the collectives concurrently."""
    import threading

    import torch
    devices = devices or [0] * nranks
    for d in set(devices):
        torch.cuda.synchronize(d)  # inputs made on the default stream are ready
    group = LocalGroup(nranks)
    comms = [group.comm(r, devices[r]) for r in range(nranks)]
    results = [None] * nranks
    errors = [None] * nranks

    def body(r):
        try:
            torch.cuda.set_device(devices[r])
            stream = torch.cuda.Stream(devices[r])
            with torch.cuda.stream(stream):
                h = fce.Handle(devices[r], stream)
                try:
                    results[r] = fn(r, comms[r], h)
                    stream.synchronize()
                finally:
                    h.close()
        except BaseException as exc:  # noqa: BLE001 - handed to the caller
            errors[r] = exc

    threads = [threading.Thread(target=body, args=(r,), name=f"fce-rank{r}") for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    for c in comms:
        c.close()
    group.close()
    for e in errors:
        if e is not None:
            raise e
    return results


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
                    handle=None, dhidden=None):
    """tp_backward over real ranks (fce_vp_backward) -> (dH summed over ranks, local dW shard).
    `dhidden` may be a caller-owned fp32 [N, >= d] view (any row stride)."""
    import torch
    h = handle or fce.default_handle(hidden.device.index or 0)
    p, keep = fce.make_problem(hidden, weight_shard, targets, ignore_index, v_offset, v_total)
    dev = hidden.device
    dh = dhidden if dhidden is not None else torch.empty(p.n, p.d, dtype=torch.float32, device=dev)
    dw = torch.empty(p.v, p.d, dtype=torch.float32, device=dev)
    up_rows = None if isinstance(upstream, (int, float)) else upstream.float().contiguous()
    if up_rows is not None and up_rows.numel() != p.n:
        raise fce.InconsistentUpstream(f"per-position upstream has {up_rows.numel()} entries, expected {p.n}")
    fce._check(h.lib.fce_vp_backward(h.raw, comm.ptr, ctypes.byref(p), stats.c(),
                                     fce.REDUCTIONS[reduction],
                                     float(upstream) if up_rows is None else 0.0,
                                     fce._ptr(up_rows), dh.data_ptr(), dh.stride(0), dw.data_ptr(), p.d))
    return dh, dw


def native_sp_vp_forward(comm: NativeComm, hidden_shard, n_total: int, weight_shard, targets, v_offset: int,
                         v_total: int, reduction: str = "mean", ignore_index=None, handle=None):
    """sp_to_tp_gather + tp_forward in one call (fce_sp_vp_forward): this rank's
    position shard of H -> (the gathered full H, FusedOutput); the gather of the
    other ranks' rows overlaps K1 over this rank's rows."""
    import torch
    h = handle or fce.default_handle(hidden_shard.device.index or 0)
    d = weight_shard.shape[1]
    ld = (d + 7) // 8 * 8
    full = torch.empty(n_total, ld, dtype=torch.bfloat16, device=hidden_shard.device)[:, :d]
    x = fce._as_operand(hidden_shard, "hidden") if hidden_shard.shape[0] else hidden_shard
    p, keep = fce.make_problem(full, weight_shard, targets, ignore_index, v_offset, v_total)
    dev = hidden_shard.device
    st = fce.Stats.empty(n_total, dev)
    lse = torch.empty(n_total, dtype=torch.float32, device=dev)
    rows = torch.empty(n_total, dtype=torch.float32, device=dev)
    red = torch.empty((), dtype=torch.float32, device=dev)
    fce._check(h.lib.fce_sp_vp_forward(h.raw, comm.ptr, ctypes.byref(p), x.data_ptr() if x.shape[0] else None,
                                       x.shape[0], x.stride(0) if x.shape[0] else d, fce.REDUCTIONS[reduction],
                                       st.c(), lse.data_ptr(), rows.data_ptr(), red.data_ptr()), vp=True)
    return full, fce.FusedOutput(rows if reduction == "none" else red, st, lse, rows)


def native_sp_vp_backward(comm: NativeComm, hidden, weight_shard, targets, v_offset: int, v_total: int,
                          stats: fce.Stats, shard_rows: int, reduction: str = "mean", upstream=1.0,
                          ignore_index=None, handle=None):
    """tp_backward + the sequence-parallel reduce-scatter of dH in one call
    (fce_sp_vp_backward): -> (this rank's summed dH position shard, local dW
    shard).  Over a peer-memory transport the reduction runs inside the
    backward kernel."""
    import torch
    h = handle or fce.default_handle(hidden.device.index or 0)
    p, keep = fce.make_problem(hidden, weight_shard, targets, ignore_index, v_offset, v_total)
    dev = hidden.device
    dh = torch.empty(shard_rows, p.d, dtype=torch.float32, device=dev)
    dw = torch.empty(p.v, p.d, dtype=torch.float32, device=dev)
    up_rows = None if isinstance(upstream, (int, float)) else upstream.float().contiguous()
    fce._check(h.lib.fce_sp_vp_backward(h.raw, comm.ptr, ctypes.byref(p), stats.c(), fce.REDUCTIONS[reduction],
                                        float(upstream) if up_rows is None else 0.0, fce._ptr(up_rows),
                                        dh.data_ptr() if shard_rows else None, shard_rows, p.d, dw.data_ptr(), p.d),
               vp=True)
    return dh, dw


def native_sp_gather(comm: NativeComm, hidden_shard, n_total: int, handle=None):
    """sp_to_tp_gather (parallel_sim.hpp:294-314) through fce_sp_gather: this
    rank's position shard of H (bf16) -> the full H on every rank."""
    import torch
    h = handle or fce.default_handle(hidden_shard.device.index or 0)
    x = fce._as_operand(hidden_shard, "hidden") if hidden_shard.shape[0] else hidden_shard
    d = hidden_shard.shape[1]
    ld = (d + 7) // 8 * 8
    full = torch.empty(n_total, ld, dtype=torch.bfloat16, device=hidden_shard.device)[:, :d]
    fce._check(h.lib.fce_sp_gather(h.raw, comm.ptr, x.data_ptr() if x.shape[0] else None, x.shape[0],
                                   x.stride(0) if x.shape[0] else d, d, n_total, full.data_ptr(),
                                   full.stride(0)), vp=True)
    return full


def native_sp_scatter(comm: NativeComm, dh_partial, shard_rows: int, handle=None):
    """Reduce-scatter of full-length dH partials to this rank's position shard (fce_sp_scatter)."""
    import torch
    h = handle or fce.default_handle(dh_partial.device.index or 0)
    dh_partial = dh_partial.float()
    if dh_partial.stride(1) != 1:
        dh_partial = dh_partial.contiguous()
    n, d = dh_partial.shape
    out = torch.empty(shard_rows, d, dtype=torch.float32, device=dh_partial.device)
    fce._check(h.lib.fce_sp_scatter(h.raw, comm.ptr, dh_partial.data_ptr(), n, dh_partial.stride(0), d,
                                    out.data_ptr() if shard_rows else None, shard_rows, d), vp=True)
    return out


def native_dp_step(comm: NativeComm, hidden, weight, targets, reduction="mean", ignore_index=None,
                   want_dhidden=True, handle=None):
    """dp_step (parallel_sim.hpp:334-378) through fce_dp_step -> (loss averaged
    over replicas, local dH or None, dW averaged over replicas)."""
    import torch
    h = handle or fce.default_handle(hidden.device.index or 0)
    if reduction not in fce.REDUCTIONS:
        raise fce.UnsupportedReduction(reduction)
    p, keep = fce.make_problem(hidden, weight, targets, ignore_index)
    dev = hidden.device
    loss = torch.empty((), dtype=torch.float32, device=dev)
    dh = torch.empty(p.n, p.d, dtype=torch.float32, device=dev) if want_dhidden else None
    dw = torch.empty(p.v, p.d, dtype=torch.float32, device=dev)
    fce._check(h.lib.fce_dp_step(h.raw, comm.ptr, ctypes.byref(p), fce.REDUCTIONS[reduction], loss.data_ptr(),
                                 fce._ptr(dh), p.d, dw.data_ptr(), p.d), vp=True)
    return loss, dh, dw


def native_all_reduce(comm: NativeComm, x, handle=None):
    """In-place fp32 sum over the ranks (fce_comm_all_reduce_f32)."""
    h = handle or fce.default_handle(x.device.index or 0)
    fce._check(h.lib.fce_comm_all_reduce_f32(h.raw, comm.ptr, x.data_ptr(), x.data_ptr(), x.numel()), vp=True)
    return x


def native_all_gather(comm: NativeComm, x, handle=None):
    """[nranks, *x.shape] of every rank's x (fce_comm_all_gather)."""
    import torch
    h = handle or fce.default_handle(x.device.index or 0)
    x = x.contiguous()
    out = torch.empty((comm.nranks,) + tuple(x.shape), dtype=x.dtype, device=x.device)
    fce._check(h.lib.fce_comm_all_gather(h.raw, comm.ptr, x.data_ptr(), out.data_ptr(),
                                         x.numel() * x.element_size()), vp=True)
    return out


def native_reduce_scatter(comm: NativeComm, x, handle=None):
    """x: fp32 [nranks * m] -> this rank's [m] block of the sum over ranks."""
    import torch
    h = handle or fce.default_handle(x.device.index or 0)
    x = x.float().contiguous()
    m = x.numel() // comm.nranks
    out = torch.empty(m, dtype=torch.float32, device=x.device)
    fce._check(h.lib.fce_comm_reduce_scatter_f32(h.raw, comm.ptr, x.data_ptr(), out.data_ptr(), m), vp=True)
    return out


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
