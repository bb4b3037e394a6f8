"""B200-native fused linear-cross-entropy (arXiv 2511.17599) — Python host mirror.

The product is ``libfce.so`` (hand-written sm_100a kernels behind the C-ABI in
``include/fce/fce.h``).  This module is a thin ctypes binding over that ABI for
callers that hold torch CUDA tensors (tests, bench, the autograd op); it does
no arithmetic of its own and has no CPU path: if the library or a B200 is
missing every entry point raises.

Names mirror the reference's C++ API (``proj/include/fusedce``):
``fused_forward`` / ``fused_forward_windowed`` / ``fused_backward_recompute``
/ ``fused_forward_with_partial_grads`` / ``scale_partial_grads`` /
``tp_rank_partial`` / ``tp_forward`` / ``tp_backward``, and errors are raised
as the reference's exception types (``errors.hpp:38-47``).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfce.so")

# --------------------------------------------------------------------- errors
# Order mirrors fusedce::ErrorCode (reference errors.hpp:10-21); status = code+1.


class FusedCEError(RuntimeError):
    code = "Error"


def _mk(name):
    return type(name, (FusedCEError,), {"code": name})


DimensionMismatch = _mk("DimensionMismatch")
TargetOutOfRange = _mk("TargetOutOfRange")
UnderflowRelease = _mk("UnderflowRelease")
DuplicateTarget = _mk("DuplicateTarget")
MissingStats = _mk("MissingStats")
InconsistentUpstream = _mk("InconsistentUpstream")
UnsupportedReduction = _mk("UnsupportedReduction")
InvalidLayout = _mk("InvalidLayout")
EmptyGrid = _mk("EmptyGrid")
EmptyInput = _mk("EmptyInput")
CudaError = _mk("CudaError")
NcclError = _mk("NcclError")
InvalidArgument = _mk("InvalidArgument")

_STATUS = {
    1: DimensionMismatch, 2: TargetOutOfRange, 3: UnderflowRelease, 4: DuplicateTarget,
    5: MissingStats, 6: InconsistentUpstream, 7: UnsupportedReduction, 8: InvalidLayout,
    9: EmptyGrid, 10: EmptyInput, 100: CudaError, 101: NcclError, 102: InvalidArgument,
}

REDUCTIONS = {"mean": 0, "sum": 1, "none": 2}

# ------------------------------------------------------------------ C structs


class FceProblem(ctypes.Structure):
    _fields_ = [
        ("hidden", ctypes.c_void_p), ("ldh", ctypes.c_int64),
        ("weight", ctypes.c_void_p), ("ldw", ctypes.c_int64),
        ("n", ctypes.c_int64), ("d", ctypes.c_int64), ("v", ctypes.c_int64),
        ("v_offset", ctypes.c_int64), ("v_total", ctypes.c_int64),
        ("targets", ctypes.c_void_p),
        ("has_ignore", ctypes.c_int32), ("ignore_index", ctypes.c_int64),
    ]


class FceStats(ctypes.Structure):
    _fields_ = [("m", ctypes.c_void_p), ("a", ctypes.c_void_p),
                ("z_target", ctypes.c_void_p), ("found", ctypes.c_void_p)]


# Every symbol include/fce/fce.h and include/fce/fce_vp.h declare.
EXPORTED_SYMBOLS = [
    "fce_create", "fce_destroy", "fce_set_stream", "fce_last_error", "fce_status_string",
    "fce_set_option", "fce_workspace_bytes", "fce_launch_count", "fce_kernel_stats", "fce_forward",
    "fce_forward_partial", "fce_merge_partials", "fce_backward", "fce_backward_ex", "fce_backward_dev",
    "fce_gemm_bf16", "fce_scale",
    "fce_generate_instance", "fce_f32_to_bf16",
    "fce_comm_unique_id", "fce_comm_init", "fce_comm_ipc_id", "fce_comm_init_ipc",
    "fce_comm_group_create", "fce_comm_group_destroy",
    "fce_comm_init_local", "fce_comm_destroy", "fce_comm_query", "fce_vp_last_error", "fce_comm_scratch_bytes",
    "fce_comm_all_gather", "fce_comm_all_reduce_f32", "fce_comm_reduce_scatter_f32",
    "fce_vp_forward", "fce_vp_backward", "fce_sp_gather", "fce_sp_scatter", "fce_sp_vp_forward", "fce_sp_vp_backward",
    "fce_dp_step",
]

_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libfce.so (no GPU needed to load).  Raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: run `make` or __graft_entry__.build() first "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    F, D = ctypes.c_float, ctypes.c_double
    sig = {
        "fce_create": (I32, [ctypes.POINTER(P), I32, P]),
        "fce_destroy": (I32, [P]),
        "fce_set_stream": (I32, [P, P]),
        "fce_last_error": (ctypes.c_char_p, []),
        "fce_status_string": (ctypes.c_char_p, [I32]),
        "fce_set_option": (I32, [P, ctypes.c_char_p, I64]),
        "fce_workspace_bytes": (I32, [P, ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]),
        "fce_launch_count": (I32, [P, ctypes.POINTER(I64)]),
        "fce_kernel_stats": (I32, [P, I32, ctypes.POINTER(D), ctypes.POINTER(I64), ctypes.POINTER(D)]),
        "fce_forward": (I32, [P, ctypes.POINTER(FceProblem), I32, I64, FceStats, P, P, P]),
        "fce_forward_partial": (I32, [P, ctypes.POINTER(FceProblem), FceStats]),
        "fce_merge_partials": (I32, [P, I32, I64, I64, P, P, P, P, P, I32, I64, I32, FceStats, P, P, P]),
        "fce_backward": (I32, [P, ctypes.POINTER(FceProblem), FceStats, I32, F, P, P, I64, P, I64, I32]),
        "fce_backward_ex": (I32, [P, ctypes.POINTER(FceProblem), FceStats, I32, F, P, P, I64, I32, P, I64, I32,
                                  I32]),
        "fce_backward_dev": (I32, [P, ctypes.POINTER(FceProblem), FceStats, I32, P, P, P, I64, I32, P, I64, I32,
                                   I32]),
        "fce_scale": (I32, [P, P, I64, F]),
        "fce_gemm_bf16": (I32, [P, P, I64, I32, P, I64, I32, I64, I64, I64, P, I64, I32]),
        "fce_generate_instance": (I32, [P, I64, I64, I64, ctypes.c_uint64, P, I64, P, I64, P, I64, D, P, P]),
        "fce_f32_to_bf16": (I32, [P, P, I64, I64, I64, P, I64]),
        "fce_comm_unique_id": (I32, [P, ctypes.c_size_t]),
        "fce_comm_init": (I32, [ctypes.POINTER(P), I32, I32, I32, P, ctypes.c_size_t]),
        "fce_comm_ipc_id": (I32, [P, ctypes.c_size_t]),
        "fce_comm_init_ipc": (I32, [ctypes.POINTER(P), I32, I32, I32, P, ctypes.c_size_t]),
        "fce_comm_group_create": (I32, [ctypes.POINTER(P), I32]),
        "fce_comm_group_destroy": (I32, [P]),
        "fce_comm_init_local": (I32, [ctypes.POINTER(P), P, I32, I32]),
        "fce_comm_destroy": (I32, [P]),
        "fce_comm_query": (I32, [P, ctypes.POINTER(I32), ctypes.POINTER(I32), ctypes.POINTER(I32)]),
        "fce_comm_scratch_bytes": (I32, [P, ctypes.POINTER(ctypes.c_size_t)]),
        "fce_comm_all_gather": (I32, [P, P, P, P, ctypes.c_size_t]),
        "fce_comm_all_reduce_f32": (I32, [P, P, P, P, ctypes.c_size_t]),
        "fce_comm_reduce_scatter_f32": (I32, [P, P, P, P, ctypes.c_size_t]),
        "fce_sp_gather": (I32, [P, P, P, I64, I64, I64, I64, P, I64]),
        "fce_sp_scatter": (I32, [P, P, P, I64, I64, I64, P, I64, I64]),
        "fce_dp_step": (I32, [P, P, ctypes.POINTER(FceProblem), I32, P, P, I64, P, I64]),
        "fce_sp_vp_backward": (I32, [P, P, ctypes.POINTER(FceProblem), FceStats, I32, F, P, P, I64, I64, P, I64]),
        "fce_sp_vp_forward": (I32, [P, P, ctypes.POINTER(FceProblem), P, I64, I64, I32, FceStats, P, P, P]),
        "fce_vp_last_error": (ctypes.c_char_p, []),
        "fce_vp_forward": (I32, [P, P, ctypes.POINTER(FceProblem), I32, FceStats, P, P, P]),
        "fce_vp_backward": (I32, [P, P, ctypes.POINTER(FceProblem), FceStats, I32, F, P, P, I64, P, I64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _check(status: int, vp: bool = False):
    if status == 0:
        return
    lib = load_library()
    msg = (lib.fce_vp_last_error() if vp else lib.fce_last_error()) or b""
    raise _STATUS.get(status, FusedCEError)(msg.decode(errors="replace"))


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


# ------------------------------------------------------------------- handle

class Handle:
    """One library handle bound to a device and a CUDA stream."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        self.lib = load_library()
        self.device = device
        self._h = ctypes.c_void_p()
        s = stream if stream is not None else torch.cuda.current_stream(device)
        _check(self.lib.fce_create(ctypes.byref(self._h), device, ctypes.c_void_p(s.cuda_stream)))
        self._stream = s

    def set_stream(self, stream):
        self._stream = stream
        _check(self.lib.fce_set_stream(self._h, ctypes.c_void_p(stream.cuda_stream)))

    def set_option(self, key: str, value: int):
        _check(self.lib.fce_set_option(self._h, key.encode(), int(value)))

    def workspace_bytes(self):
        cur, peak = ctypes.c_size_t(), ctypes.c_size_t()
        _check(self.lib.fce_workspace_bytes(self._h, ctypes.byref(cur), ctypes.byref(peak)))
        return cur.value, peak.value

    def launch_count(self) -> int:
        c = ctypes.c_int64()
        _check(self.lib.fce_launch_count(self._h, ctypes.byref(c)))
        return c.value

    KERNELS = {0: "fce_fwd_sm100", 1: "fce_bwd_grad_sm100", 2: "fce_bwd_gemm_sm100",
               3: "fce_bwd_persistent_sm100"}

    def kernel_stats(self, kernel: int):
        """(total device ms, launches, algorithmic flops) since timing was enabled."""
        ms, n, fl = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _check(self.lib.fce_kernel_stats(self._h, kernel, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(fl)))
        return ms.value, n.value, fl.value

    def close(self):
        if self._h:
            self.lib.fce_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def raw(self):
        return self._h


_handles = {}


def default_handle(device: int = 0) -> Handle:
    import torch
    stream = torch.cuda.current_stream(device)
    h = _handles.get(device)
    if h is None:
        h = _handles[device] = Handle(device, stream)
    elif h._stream.cuda_stream != stream.cuda_stream:
        h.set_stream(stream)
    return h


# ------------------------------------------------------------------ problem

@dataclass
class Stats:
    """Per-row SoftmaxStats cache (reference softmax_stats.hpp:14-46)."""
    m: "object"
    a: "object"
    z_target: "object"
    found: "object"

    def c(self) -> FceStats:
        return FceStats(_ptr(self.m), _ptr(self.a), _ptr(self.z_target), _ptr(self.found))

    @staticmethod
    def empty(n: int, device) -> "Stats":
        import torch
        return Stats(torch.empty(n, dtype=torch.float32, device=device),
                     torch.empty(n, dtype=torch.float32, device=device),
                     torch.empty(n, dtype=torch.float32, device=device),
                     torch.empty(n, dtype=torch.uint8, device=device))

    def logsumexp(self):
        import torch
        return self.m + torch.log(self.a)


def _as_operand(x, name: str):
    """bf16 CUDA matrix with ld % 8 == 0 (pads a copy if needed)."""
    import torch
    if not x.is_cuda:
        raise InvalidArgument(f"{name} must be a CUDA tensor (no CPU path)")
    if x.dtype == torch.float32:
        x = x.to(torch.bfloat16)  # callers on the bf16 grid convert exactly
    if x.dtype != torch.bfloat16 or x.dim() != 2:
        raise InvalidLayout(f"{name} must be a 2-D bf16 (or bf16-grid float32) CUDA tensor")
    if x.stride(1) != 1 or x.stride(0) % 8 or x.data_ptr() % 16:
        rows, cols = x.shape
        ld = (cols + 7) // 8 * 8
        buf = torch.zeros(rows, ld, dtype=torch.bfloat16, device=x.device)
        buf[:, :cols] = x
        return buf[:, :cols]
    return x


def make_problem(hidden, weight, targets, ignore_index: Optional[int] = None,
                 v_offset: int = 0, v_total: int = 0):
    import torch
    hidden = _as_operand(hidden, "hidden")
    weight = _as_operand(weight, "weight")
    if targets.dtype != torch.int64 or not targets.is_cuda:
        targets = targets.to(device=hidden.device, dtype=torch.int64)
    targets = targets.contiguous()
    if hidden.shape[1] != weight.shape[1]:
        raise DimensionMismatch(f"hidden cols {hidden.shape[1]} != weight cols {weight.shape[1]}")
    if hidden.shape[0] != targets.numel():
        raise DimensionMismatch(f"hidden rows {hidden.shape[0]} != target count {targets.numel()}")
    p = FceProblem()
    p.hidden, p.ldh = hidden.data_ptr(), hidden.stride(0)
    p.weight, p.ldw = weight.data_ptr(), weight.stride(0)
    p.n, p.d = hidden.shape
    p.v = weight.shape[0]
    p.v_offset, p.v_total = v_offset, v_total
    p.targets = targets.data_ptr()
    p.has_ignore = 0 if ignore_index is None else 1
    p.ignore_index = 0 if ignore_index is None else int(ignore_index)
    keep = (hidden, weight, targets)
    return p, keep


@dataclass
class FusedOutput:
    """fused_forward result (reference fused_forward.hpp:21-25)."""
    loss: "object"          # 0-d tensor (mean/sum) or per-row tensor (none)
    stats: Stats
    lse: "object"
    loss_rows: "object"


def fused_forward(hidden, weight, targets, reduction: str = "mean", ignore_index=None,
                  window: int = 0, handle: Optional[Handle] = None) -> FusedOutput:
    """Fused projection + cross-entropy forward (fused_forward.hpp:161-172;
    window > 0: fused_forward_windowed, 177-195)."""
    import torch
    if reduction not in REDUCTIONS:
        raise UnsupportedReduction(reduction)
    h = handle or default_handle(hidden.device.index or 0)
    p, keep = make_problem(hidden, weight, targets, ignore_index)
    n = p.n
    dev = hidden.device
    stats = Stats.empty(n, dev)
    lse = torch.empty(n, dtype=torch.float32, device=dev)
    rows = torch.empty(n, dtype=torch.float32, device=dev)
    red = torch.empty((), dtype=torch.float32, device=dev)
    _check(h.lib.fce_forward(h.raw, ctypes.byref(p), REDUCTIONS[reduction], int(window), stats.c(),
                             _ptr(lse), _ptr(rows), _ptr(red)))
    loss = rows if reduction == "none" else red
    return FusedOutput(loss, stats, lse, rows)


def fused_forward_windowed(hidden, weight, targets, window_size: int, reduction="mean",
                           ignore_index=None, worker_count: int = 1, handle=None):
    if window_size <= 0:
        raise InvalidLayout("window size must be at least 1")
    if worker_count <= 0:
        raise InvalidLayout("worker count must be at least 1")
    return fused_forward(hidden, weight, targets, reduction, ignore_index, window_size, handle)


def fused_backward_recompute(hidden, weight, targets, stats: Stats, reduction: str = "mean",
                             upstream=1.0, ignore_index=None, handle: Optional[Handle] = None,
                             want_dhidden: bool = True, want_dweight: bool = True,
                             dhidden=None, accumulate_dhidden: bool = False, grad_dtype=None):
    """Backward by logit recompute (fused_backward.hpp:118-140) -> (dH, dW), fp32
    by default; grad_dtype=torch.bfloat16 returns bf16 gradients (fce_backward_ex:
    dW rounded straight from the accumulators, no fp32 V x D buffer).

    upstream (check_upstream, reduction.hpp:81-97): a Python number or a 0-d
    tensor for mean / sum (a CUDA 0-d tensor is read on the device:
    fce_backward_dev, no host sync), a length-N tensor for 'none'."""
    import torch
    if reduction not in REDUCTIONS:
        raise UnsupportedReduction(reduction)
    h = handle or default_handle(hidden.device.index or 0)
    p, keep = make_problem(hidden, weight, targets, ignore_index)
    dev = hidden.device
    up_rows = None
    up_dev = None
    up_scalar = 0.0
    if isinstance(upstream, (int, float)):
        up_scalar = float(upstream)
    elif reduction != "none" and upstream.numel() == 1 and upstream.dim() == 0:
        if upstream.is_cuda:
            up_dev = upstream.to(device=dev, dtype=torch.float32).reshape(()).contiguous()
        else:
            up_scalar = float(upstream.item())
    else:
        up_rows = upstream.to(device=dev, dtype=torch.float32).contiguous()
        if reduction == "none" and up_rows.numel() != p.n:
            # reference check_upstream: a per-position upstream must cover every position
            raise InconsistentUpstream(f"per-position upstream has {up_rows.numel()} entries, expected {p.n}")
    gdt = torch.float32 if grad_dtype is None else grad_dtype
    if gdt not in (torch.float32, torch.bfloat16):
        raise InvalidArgument("grad_dtype must be torch.float32 or torch.bfloat16")
    if dhidden is None and want_dhidden:
        dhidden = torch.empty(p.n, p.d, dtype=gdt, device=dev)
    dweight = torch.empty(p.v, p.d, dtype=gdt, device=dev) if want_dweight else None
    if up_dev is not None:
        code = {torch.float32: 0, torch.bfloat16: 1}
        _check(h.lib.fce_backward_dev(h.raw, ctypes.byref(p), stats.c(), REDUCTIONS[reduction], _ptr(up_dev),
                                      None, _ptr(dhidden), dhidden.stride(0) if dhidden is not None else 0,
                                      code[dhidden.dtype] if dhidden is not None else 0,
                                      _ptr(dweight), dweight.stride(0) if dweight is not None else 0,
                                      code[gdt], 1 if accumulate_dhidden else 0))
    elif gdt == torch.float32 and (dhidden is None or dhidden.dtype == torch.float32):
        _check(h.lib.fce_backward(h.raw, ctypes.byref(p), stats.c(), REDUCTIONS[reduction], up_scalar,
                                  _ptr(up_rows), _ptr(dhidden), dhidden.stride(0) if dhidden is not None else 0,
                                  _ptr(dweight), dweight.stride(0) if dweight is not None else 0,
                                  1 if accumulate_dhidden else 0))
    else:
        code = {torch.float32: 0, torch.bfloat16: 1}
        _check(h.lib.fce_backward_ex(h.raw, ctypes.byref(p), stats.c(), REDUCTIONS[reduction], up_scalar,
                                     _ptr(up_rows), _ptr(dhidden), dhidden.stride(0) if dhidden is not None else 0,
                                     code[dhidden.dtype] if dhidden is not None else 0,
                                     _ptr(dweight), dweight.stride(0) if dweight is not None else 0,
                                     code[gdt], 1 if accumulate_dhidden else 0))
    return dhidden, dweight


def fused_forward_with_partial_grads(hidden, weight, targets, reduction="mean", ignore_index=None,
                                     handle=None):
    """Alg. 3 (fused_backward.hpp:162-188): loss, stats and unscaled partial
    gradients; reduction 'none' is rejected like the reference."""
    if reduction == "none":
        raise UnsupportedReduction(
            "partial-gradient accumulation requires a scalar-upstream reduction (mean or sum)")
    out = fused_forward(hidden, weight, targets, reduction, ignore_index, handle=handle)
    dh, dw = fused_backward_recompute(hidden, weight, targets, out.stats, "sum", 1.0,
                                      ignore_index, handle)
    return out, (dh, dw)


def gemm_bf16(a, b, a_mn: bool = False, b_mn: bool = False, out=None, accumulate=False,
              handle=None):
    """C = A . B^T (fp32) on the tile kernel; A is [M, K] or, with a_mn, [K, M];
    B is [N, K] or, with b_mn, [K, N].  Test / benchmark entry of the contraction."""
    import torch
    h = handle or default_handle(a.device.index or 0)
    a = _as_operand(a, "a")
    b = _as_operand(b, "b")
    m = a.shape[1] if a_mn else a.shape[0]
    k = a.shape[0] if a_mn else a.shape[1]
    n = b.shape[1] if b_mn else b.shape[0]
    kb = b.shape[0] if b_mn else b.shape[1]
    if k != kb:
        raise DimensionMismatch(f"K mismatch {k} != {kb}")
    if out is None:
        out = torch.zeros(m, n, dtype=torch.float32, device=a.device)
    _check(h.lib.fce_gemm_bf16(h.raw, a.data_ptr(), a.stride(0), int(a_mn), b.data_ptr(), b.stride(0),
                               int(b_mn), m, n, k, out.data_ptr(), out.stride(0), int(accumulate)))
    return out


def scale_partial_grads(partials, gamma_eff: float, handle=None):
    """Alg. 4 (fused_backward.hpp:193-202): grads = gamma_eff * partials, in place."""
    dh, dw = partials
    h = handle or default_handle(dh.device.index or 0)
    for t in (dh, dw):
        if t is not None:
            _check(h.lib.fce_scale(h.raw, _ptr(t), t.numel(), float(gamma_eff)))
    return dh, dw


def generate_instance(n: int, d: int, v: int, seed: int = 42, ignore_index: int = -100,
                      ignore_fraction: float = 0.0, device=0, want_f32: bool = False,
                      handle=None):
    """Device-side make_random_instance[_with_ignores] (instance.hpp:38-85), bit-identical,
    rounded to the bf16 grid.  Returns (H bf16, W bf16, targets int64[, H f32, W f32])."""
    import torch
    h = handle or default_handle(device)
    ld = (d + 7) // 8 * 8
    H = torch.empty(n, ld, dtype=torch.bfloat16, device=device)
    W = torch.empty(v, ld, dtype=torch.bfloat16, device=device)
    Y = torch.empty(n, dtype=torch.int64, device=device)
    Hf = torch.zeros(n, ld, dtype=torch.float32, device=device) if want_f32 else None
    Wf = torch.zeros(v, ld, dtype=torch.float32, device=device) if want_f32 else None
    _check(h.lib.fce_generate_instance(h.raw, n, d, v, ctypes.c_uint64(seed & (2**64 - 1)), _ptr(H), ld,
                                       _ptr(W), ld, _ptr(Y), ignore_index, float(ignore_fraction),
                                       _ptr(Hf), _ptr(Wf)))
    out = (H[:, :d], W[:, :d], Y)
    if want_f32:
        out = out + (Hf[:, :d], Wf[:, :d])
    return out


# -------------------------------------------------- vocab parallel (one rank)

def shard_ranges(vocab: int, ranks: int) -> List[tuple]:
    """Ceil-first contiguous partition (reference exec.hpp:25-41,
    ShardLayout::tensor_parallel parallel_sim.hpp:55-57)."""
    if ranks == 0:
        raise InvalidLayout("cannot partition into 0 parts")
    if vocab < ranks:
        raise InvalidLayout(f"cannot split axis of length {vocab} across {ranks} ranks")
    base, extra = divmod(vocab, ranks)
    out, lo = [], 0
    for r in range(ranks):
        ln = base + (1 if r < extra else 0)
        out.append((lo, lo + ln))
        lo += ln
    return out


def tp_rank_partial(hidden, weight_shard, v_offset: int, v_total: int, targets,
                    ignore_index=None, handle=None) -> Stats:
    """tp_rank_partial (parallel_sim.hpp:165-181) on this GPU."""
    h = handle or default_handle(hidden.device.index or 0)
    p, keep = make_problem(hidden, weight_shard, targets, ignore_index, v_offset, v_total)
    st = Stats.empty(p.n, hidden.device)
    _check(h.lib.fce_forward_partial(h.raw, ctypes.byref(p), st.c()))
    return st


def stream_stats(h_row, weight, target, lo: int, hi: int, handle=None) -> Stats:
    """stream_stats (fused_forward.hpp:137-154): one hidden row over the vocabulary
    range [lo, hi) -> 1-row Stats; the empty range is the identity."""
    import torch
    d = weight.shape[1]
    if h_row.numel() != d:
        raise DimensionMismatch(f"hidden length {h_row.numel()} != weight cols {d}")
    if lo > hi or hi > weight.shape[0] or lo < 0:
        raise DimensionMismatch(f"vocab range [{lo}, {hi}) not contained in [0, {weight.shape[0]})")
    dev = weight.device
    if lo == hi:
        st = Stats.empty(1, dev)
        st.m.fill_(float("-inf")); st.a.zero_(); st.z_target.zero_(); st.found.zero_()
        return st
    # a target outside the range (or none) never matches: use id hi (the
    # reference's stream_stats never validates the target, it just reports
    # found = false; fused_forward.hpp:137-154)
    y = hi if target is None or not (lo <= int(target) < hi) else int(target)
    tv = torch.tensor([y], dtype=torch.int64, device=dev)
    return tp_rank_partial(h_row.reshape(1, d), weight[lo:hi], lo, max(hi + 1, weight.shape[0] + 1), tv,
                           None, handle)


def merge_rank_partials(partials: Sequence[Stats], targets, reduction="mean", ignore_index=None,
                        handle=None):
    """Rank-ordered merge (parallel_sim.hpp:214-231) of partials -> FusedOutput."""
    import torch
    dev = partials[0].m.device
    h = handle or default_handle(dev.index or 0)
    n = partials[0].m.numel()
    m = torch.stack([s.m for s in partials]).contiguous()
    a = torch.stack([s.a for s in partials]).contiguous()
    z = torch.stack([s.z_target for s in partials]).contiguous()
    f = torch.stack([s.found for s in partials]).contiguous()
    targets = targets.to(device=dev, dtype=torch.int64).contiguous()
    out = Stats.empty(n, dev)
    lse = torch.empty(n, dtype=torch.float32, device=dev)
    rows = torch.empty(n, dtype=torch.float32, device=dev)
    red = torch.empty((), dtype=torch.float32, device=dev)
    _check(h.lib.fce_merge_partials(h.raw, len(partials), n, n, _ptr(m), _ptr(a), _ptr(z), _ptr(f),
                                    _ptr(targets), 0 if ignore_index is None else 1,
                                    0 if ignore_index is None else int(ignore_index),
                                    REDUCTIONS[reduction], out.c(), _ptr(lse), _ptr(rows), _ptr(red)))
    return FusedOutput(rows if reduction == "none" else red, out, lse, rows)


__all__ = [n for n in dir() if not n.startswith("_")]
