"""CPU tests of the drop-in boundary: libfce.so loads and exports every symbol
include/fce/*.h declares; status codes mirror the reference error taxonomy;
without a GPU the library refuses to run (no CPU fallback)."""
import ctypes
import glob
import os
import re

import pytest

import paper_2511_17599_b200 as fce

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# fusedce::ErrorCode declaration order, reference proj/include/fusedce/errors.hpp:10-21
REFERENCE_ERROR_ORDER = ["DimensionMismatch", "TargetOutOfRange", "UnderflowRelease",
                         "DuplicateTarget", "MissingStats", "InconsistentUpstream",
                         "UnsupportedReduction", "InvalidLayout", "EmptyGrid", "EmptyInput"]


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "fce", "*.h")):
        text = open(h).read()
        names |= set(re.findall(r"^\s*(?:fce_status|const char\*)\s+(fce_\w+)\s*\(", text, re.M))
    return names


def test_library_exports_every_declared_symbol():
    lib = fce.load_library()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, missing
    assert syms == set(fce.EXPORTED_SYMBOLS)


def test_status_codes_mirror_reference_error_order():
    lib = fce.load_library()
    for i, name in enumerate(REFERENCE_ERROR_ORDER):
        assert lib.fce_status_string(i + 1).decode() == name
        assert fce._STATUS[i + 1].__name__ == name
    assert lib.fce_status_string(0).decode() == "ok"


def test_null_handle_is_rejected():
    lib = fce.load_library()
    p = fce.FceProblem()
    st = lib.fce_forward(None, ctypes.byref(p), 0, 0, fce.FceStats(), None, None, None)
    assert st == 102  # FCE_INVALID_ARGUMENT


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = fce.load_library()
    h = ctypes.c_void_p()
    st = lib.fce_create(ctypes.byref(h), 0, None)
    assert st == 100  # FCE_CUDA_ERROR: no device, and no CPU path
    assert b"no CPU path" in lib.fce_last_error()


def test_shard_ranges_ceil_first():
    # ShardLayout::tensor_parallel / partition_ranges (parallel_sim.hpp:55-57, exec.hpp:25-41)
    assert fce.shard_ranges(128256, 8) == [(i * 16032, (i + 1) * 16032) for i in range(8)]
    assert [b - a for a, b in fce.shard_ranges(10, 4)] == [3, 3, 2, 2]
    with pytest.raises(fce.InvalidLayout):
        fce.shard_ranges(3, 4)
    with pytest.raises(fce.InvalidLayout):
        fce.shard_ranges(3, 0)


def test_sass_is_tcgen05():
    """The shipped kernels are tcgen05 / TMA (not mma.sync)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump absent")
    out = subprocess.run(["cuobjdump", "-sass", fce.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out and "UTMALDG" in out and "LDTM" in out
    assert not re.search(r"\bHMMA\b", out)


def test_headers_are_plain_c_and_link(tmp_path):
    """The boundary is a C ABI: include/fce/*.h compile as C11 (no C++ types)
    and a C program links against libfce.so and calls it (without a GPU it
    gets FCE_CUDA_ERROR, never a CPU result)."""
    import subprocess
    src = tmp_path / "abi.c"
    src.write_text(r'''
#include <stdio.h>
#include "fce/fce.h"
#include "fce/fce_vp.h"
int main(void) {
    fce_handle h = 0;
    fce_status s = fce_create(&h, 0, NULL);
    printf("%d %s\n", (int)s, fce_status_string(FCE_DIMENSION_MISMATCH));
    if (s == FCE_OK) fce_destroy(h);
    return 0;
}
''')
    exe = tmp_path / "abi"
    lib_dir = os.path.join(ROOT, "paper_2511_17599_b200")
    r = subprocess.run(["gcc", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        "-I", "/usr/local/cuda/include", str(src), "-o", str(exe), "-L", lib_dir, "-lfce",
                        f"-Wl,-rpath,{lib_dir}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    code, name = r.stdout.split()
    assert name == "DimensionMismatch"
    import torch
    assert int(code) == (0 if torch.cuda.is_available() else 100)


def test_ipc_rendezvous_ids_are_unique_names():
    """fce_comm_ipc_id needs no GPU: a POSIX shared-memory name, unique per call."""
    from paper_2511_17599_b200 import vocab_parallel as vp
    a, b = vp.NativeComm.ipc_id(), vp.NativeComm.ipc_id()
    na, nb = a.split(b"\0")[0].decode(), b.split(b"\0")[0].decode()
    assert na.startswith("/fce_ipc_") and nb.startswith("/fce_ipc_") and na != nb
    assert len(a) == 128


def test_comm_entry_points_reject_null_handles():
    lib = fce.load_library()
    assert lib.fce_vp_forward(None, None, None, 0, fce.FceStats(), None, None, None) == 102
    assert lib.fce_sp_vp_backward(None, None, None, fce.FceStats(), 0, 1.0, None, None, 0, 0, None, 0) == 102
    assert lib.fce_dp_step(None, None, None, 0, None, None, 0, None, 0) == 102
    g = ctypes.c_void_p()
    assert lib.fce_comm_group_create(ctypes.byref(g), 0) == 8      # FCE_INVALID_LAYOUT
    assert lib.fce_comm_group_create(ctypes.byref(g), 65) == 8
    assert lib.fce_comm_group_create(ctypes.byref(g), 2) == 0
    assert lib.fce_comm_group_destroy(g) == 0
