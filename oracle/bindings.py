"""ctypes bindings of the CPU oracle (liboracle.so) and the reference build (_ref/libfce_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or the
CPU baseline, never as the product path.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libfce_ref.so")

RED = {"mean": 0, "sum": 1, "none": 2}

P = ctypes.c_void_p
SZ = ctypes.c_size_t
I64 = ctypes.c_int64
I32 = ctypes.c_int
F32 = ctypes.c_float
F64 = ctypes.c_double


class OrcStats(ctypes.Structure):
    _fields_ = [("m", ctypes.c_float), ("a", ctypes.c_float), ("z_target", ctypes.c_float),
                ("found", ctypes.c_uint8)]


STATS_DTYPE = np.dtype([("m", "<f4"), ("a", "<f4"), ("z_target", "<f4"), ("found", "u1")],
                       align=True)
assert STATS_DTYPE.itemsize == ctypes.sizeof(OrcStats)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(P)


_orc = None
_ref = None


def oracle_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_LIB):
            raise ImportError(f"{ORACLE_LIB} missing: run `make oracle/liboracle.so`")
        lib = ctypes.CDLL(ORACLE_LIB)
        lib.orc_splitmix64.restype = ctypes.c_uint64
        lib.orc_splitmix64.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        lib.orc_splitmix_unit.restype = F64
        lib.orc_splitmix_unit.argtypes = [ctypes.POINTER(ctypes.c_uint64)]
        lib.orc_round_bf16.restype = F32
        lib.orc_round_bf16.argtypes = [F32]
        lib.orc_is_bf16_value.restype = I32
        lib.orc_is_bf16_value.argtypes = [F32]
        lib.orc_make_instance.restype = I32
        lib.orc_make_instance.argtypes = [SZ, SZ, SZ, ctypes.c_uint64, I64, F64, I32, P, P, P]
        lib.orc_dot.restype = F32
        lib.orc_dot.argtypes = [P, P, SZ, SZ]
        lib.orc_stats_update.restype = None
        lib.orc_stats_update.argtypes = [ctypes.POINTER(OrcStats), F32]
        lib.orc_stats_logsumexp.restype = F32
        lib.orc_stats_logsumexp.argtypes = [ctypes.POINTER(OrcStats)]
        lib.orc_stats_loss.restype = F32
        lib.orc_stats_loss.argtypes = [ctypes.POINTER(OrcStats)]
        lib.orc_merge_stats.restype = I32
        lib.orc_merge_stats.argtypes = [ctypes.POINTER(OrcStats)] * 3
        lib.orc_partition_ranges.restype = I32
        lib.orc_partition_ranges.argtypes = [SZ, SZ, P, P]
        lib.orc_fused_forward.restype = I32
        lib.orc_fused_forward.argtypes = [P, P, SZ, SZ, SZ, SZ, P, I32, I64, I32, SZ, I32, P, P, P]
        lib.orc_rank_partial.restype = I32
        lib.orc_rank_partial.argtypes = [P, P, SZ, SZ, SZ, SZ, P, I32, I64, I32, P]
        lib.orc_fused_backward.restype = I32
        lib.orc_fused_backward.argtypes = [P, P, SZ, SZ, SZ, SZ, SZ, P, I32, I64, P, I32, F32, P, I32, P, P]
        lib.orc_reduce_losses.restype = F32
        lib.orc_reduce_losses.argtypes = [P, SZ, I32, SZ]
        _orc = lib
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            raise ImportError(f"{REF_LIB} missing (reference not built here)")
        lib = ctypes.CDLL(REF_LIB)
        lib.ref_make_instance.argtypes = [SZ, SZ, SZ, ctypes.c_uint64, I64, F64, I32, P, P, P]
        lib.ref_fused_forward.argtypes = [P, P, SZ, SZ, SZ, P, I32, I64, I32, SZ, SZ, P, P, P, P, P, P, P]
        lib.ref_fused_backward.argtypes = [P, P, SZ, SZ, SZ, P, I32, I64, P, P, P, P, I32, F32, P, SZ, P, P]
        lib.ref_partial_grads.argtypes = [P, P, SZ, SZ, SZ, P, I32, I64, I32, F32, P, P, P]
        lib.ref_tp_forward.argtypes = [P, P, SZ, SZ, SZ, P, I32, I64, SZ, I32, P, P, P, P, P, P]
        lib.ref_tp_rank_partial.argtypes = [P, P, SZ, SZ, SZ, SZ, P, I32, I64, P, P, P, P]
        lib.ref_tp_backward.argtypes = [P, P, SZ, SZ, SZ, P, I32, I64, SZ, P, P, P, P, I32, F32, P, P, P]
        lib.ref_two_stage.argtypes = [P, P, SZ, SZ, SZ, P, I32, I64, I32, F32, P, P, P, P, P]
        lib.ref_stats_example.argtypes = [P]
        for f in ("ref_make_instance", "ref_fused_forward", "ref_fused_backward", "ref_partial_grads",
                  "ref_tp_forward", "ref_tp_rank_partial", "ref_tp_backward", "ref_two_stage",
                  "ref_stats_example"):
            getattr(lib, f).restype = I32
        _ref = lib
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


def _chk(code):
    if code:
        raise OracleError(code)


# ------------------------------------------------------------------ helpers

def make_instance(n, d, v, seed=42, ignore_index=-100, ignore_fraction=0.0, round_bf16=True,
                  impl="oracle"):
    H = np.empty((n, d), np.float32)
    W = np.empty((v, d), np.float32)
    Y = np.empty(n, np.int64)
    if impl == "oracle":
        _chk(oracle_lib().orc_make_instance(n, d, v, seed, ignore_index, ignore_fraction,
                                            1 if round_bf16 else 0, _p(H), _p(W), _p(Y)))
    else:
        _chk(ref_lib().ref_make_instance(n, d, v, seed, ignore_index, ignore_fraction,
                                         1 if round_bf16 else 0, _p(H), _p(W), _p(Y)))
    return H, W, Y


def forward(H, W, Y, reduction="mean", ignore_index=None, window=0, threads=0, v_offset=0):
    """Oracle fused forward -> (stats structured array, loss_rows, loss_reduced)."""
    n, d = H.shape
    v = W.shape[0]
    H = np.ascontiguousarray(H, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    Y = np.ascontiguousarray(Y, np.int64)
    st = np.zeros(n, STATS_DTYPE)
    rows = np.zeros(n, np.float32)
    red = np.zeros(1, np.float32)
    _chk(oracle_lib().orc_fused_forward(_p(H), _p(W), n, d, v, v_offset, _p(Y),
                                        0 if ignore_index is None else 1,
                                        0 if ignore_index is None else ignore_index, RED[reduction],
                                        window, threads or os.cpu_count(), _p(st), _p(rows), _p(red)))
    return st, rows, float(red[0])


def rank_partial(H, W_shard, Y, v_offset, ignore_index=None, threads=0):
    """tp_rank_partial on the oracle -> stats structured array."""
    n, d = H.shape
    H = np.ascontiguousarray(H, np.float32)
    W_shard = np.ascontiguousarray(W_shard, np.float32)
    Y = np.ascontiguousarray(Y, np.int64)
    st = np.zeros(n, STATS_DTYPE)
    _chk(oracle_lib().orc_rank_partial(_p(H), _p(W_shard), n, d, W_shard.shape[0], v_offset, _p(Y),
                                       0 if ignore_index is None else 1,
                                       0 if ignore_index is None else ignore_index,
                                       threads or os.cpu_count(), _p(st)))
    return st


def merge(parts):
    """Rank-ordered merge_stats over a list of stats arrays (softmax_stats.hpp:52-75)."""
    lib = oracle_lib()
    n = parts[0].shape[0]
    out = np.zeros(n, STATS_DTYPE)
    for i in range(n):
        cur = OrcStats(float("-inf"), 0.0, 0.0, 0)
        for p in parts:
            q = OrcStats(float(p[i]["m"]), float(p[i]["a"]), float(p[i]["z_target"]), int(p[i]["found"]))
            nxt = OrcStats()
            _chk(lib.orc_merge_stats(ctypes.byref(cur), ctypes.byref(q), ctypes.byref(nxt)))
            cur = nxt
        out[i] = (cur.m, cur.a, cur.z_target, cur.found)
    return out


def backward(H, W, Y, stats, reduction="mean", upstream=1.0, ignore_index=None, threads=0,
             v_offset=0, want_dh=True, want_dw=True, v_total=0):
    n, d = H.shape
    v = W.shape[0]
    H = np.ascontiguousarray(H, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    Y = np.ascontiguousarray(Y, np.int64)
    st = np.ascontiguousarray(stats)
    dH = np.zeros((n, d), np.float32) if want_dh else None
    dW = np.zeros((v, d), np.float32) if want_dw else None
    up_rows = None
    up = 0.0
    if np.isscalar(upstream):
        up = float(upstream)
    else:
        up_rows = np.ascontiguousarray(upstream, np.float32)
    _chk(oracle_lib().orc_fused_backward(_p(H), _p(W), n, d, v, v_offset, v_total, _p(Y),
                                         0 if ignore_index is None else 1,
                                         0 if ignore_index is None else ignore_index, _p(st),
                                         RED[reduction], up, _p(up_rows), threads or os.cpu_count(),
                                         _p(dH), _p(dW)))
    return dH, dW


def ref_forward(H, W, Y, reduction="mean", ignore_index=None, window=0, workers=1):
    """The reference's own fused_forward (built from /root/reference)."""
    n, d = H.shape
    v = W.shape[0]
    H = np.ascontiguousarray(H, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    Y = np.ascontiguousarray(Y, np.int64)
    m = np.zeros(n, np.float32)
    a = np.zeros(n, np.float32)
    z = np.zeros(n, np.float32)
    f = np.zeros(n, np.uint8)
    rows = np.zeros(n, np.float32)
    red = np.zeros(1, np.float32)
    peak = ctypes.c_size_t()
    _chk(ref_lib().ref_fused_forward(_p(H), _p(W), n, d, v, _p(Y), 0 if ignore_index is None else 1,
                                     0 if ignore_index is None else ignore_index, RED[reduction],
                                     window, workers, _p(m), _p(a), _p(z), _p(f), _p(rows), _p(red),
                                     ctypes.byref(peak)))
    st = np.zeros(n, STATS_DTYPE)
    st["m"], st["a"], st["z_target"], st["found"] = m, a, z, f
    return st, rows, float(red[0])


def ref_backward(H, W, Y, stats, reduction="mean", upstream=1.0, ignore_index=None, workers=1):
    n, d = H.shape
    v = W.shape[0]
    H = np.ascontiguousarray(H, np.float32)
    W = np.ascontiguousarray(W, np.float32)
    Y = np.ascontiguousarray(Y, np.int64)
    m = np.ascontiguousarray(stats["m"])
    a = np.ascontiguousarray(stats["a"])
    z = np.ascontiguousarray(stats["z_target"])
    f = np.ascontiguousarray(stats["found"])
    dH = np.zeros((n, d), np.float32)
    dW = np.zeros((v, d), np.float32)
    up_rows = None
    up = 0.0
    if np.isscalar(upstream):
        up = float(upstream)
    else:
        up_rows = np.ascontiguousarray(upstream, np.float32)
    _chk(ref_lib().ref_fused_backward(_p(H), _p(W), n, d, v, _p(Y), 0 if ignore_index is None else 1,
                                      0 if ignore_index is None else ignore_index, _p(m), _p(a), _p(z),
                                      _p(f), RED[reduction], up, _p(up_rows), workers, _p(dH), _p(dW)))
    return dH, dW
