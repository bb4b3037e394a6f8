"""CPU tests: the oracle (C restatement of the reference) against the reference's
own known-answer values and the golden fixtures made by the reference build.

Reference KATs cited as proj/tests/<file>:<line>.
"""
import ctypes
import glob
import math
import os

import numpy as np
import pytest

from oracle import bindings as ob

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _stats(m=-math.inf, a=0.0):
    s = ob.OrcStats()
    s.m, s.a, s.z_target, s.found = m, a, 0.0, 0
    return s


def test_recurrence_worked_example():
    # test_core_types.cpp:281-302 (double there; float here)
    lib = ob.oracle_lib()
    s = _stats()
    for z in (0.0, 1.0, 2.0):
        lib.orc_stats_update(ctypes.byref(s), z)
    s.z_target, s.found = 2.0, 1
    assert s.m == 2.0
    assert s.a == pytest.approx(1.503214724408055, rel=1e-6)
    assert lib.orc_stats_logsumexp(ctypes.byref(s)) == pytest.approx(2.4076059644443806, rel=1e-6)
    assert lib.orc_stats_loss(ctypes.byref(s)) == pytest.approx(0.4076059644443806, rel=1e-6)


def test_merge_example_and_identity():
    # test_core_types.cpp:328-361
    lib = ob.oracle_lib()
    s1, s2, out = _stats(1.0, 2.0), _stats(3.0, 1.0), ob.OrcStats()
    assert lib.orc_merge_stats(ctypes.byref(s1), ctypes.byref(s2), ctypes.byref(out)) == 0
    assert out.m == 3.0 and out.a == pytest.approx(1.2706705664732254, rel=1e-6)
    ident = _stats()
    assert lib.orc_merge_stats(ctypes.byref(ident), ctypes.byref(s1), ctypes.byref(out)) == 0
    assert (out.m, out.a) == (1.0, 2.0)
    # DuplicateTarget (test_core_types.cpp:382-390)
    s1.found = s2.found = 1
    assert lib.orc_merge_stats(ctypes.byref(s1), ctypes.byref(s2), ctypes.byref(out)) == 4


def test_reference_build_kat_matches():
    if not ob.ref_available():
        pytest.skip("reference build absent")
    kat = np.zeros(4, np.float64)
    assert ob.ref_lib().ref_stats_example(kat.ctypes.data_as(ob.P)) == 0
    np.testing.assert_allclose(kat, [1.503214724408055, 2.4076059644443806, 0.4076059644443806,
                                     1.2706705664732254], rtol=1e-14)
    np.testing.assert_allclose(np.load(os.path.join(GOLDEN, "stats_example.npy")), kat, rtol=0)


@pytest.mark.parametrize("x,expect", [(1.00390625, 1.0), (1.01171875, 1.015625), (10240.0, 10240.0),
                                      (1.0, 1.0), (-1.00390625, -1.0)])
def test_round_bf16_ties(x, expect):
    # test_core_types.cpp:22-40
    assert ob.oracle_lib().orc_round_bf16(x) == expect


def test_round_bf16_bit_oracle():
    # test_core_types.cpp:42-56: RNE on the top 16 bits
    rng = np.random.default_rng(1)
    bits = rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    xs = xs[np.isfinite(xs)]
    lib = ob.oracle_lib()
    for x in xs[:4000]:
        b = np.float32(x).view(np.uint32)
        lsb = (int(b) >> 16) & 1
        r = np.uint32(((int(b) + 0x7FFF + lsb) & 0xFFFF0000) & 0xFFFFFFFF).view(np.float32)
        got = np.float32(lib.orc_round_bf16(float(x)))
        assert got.view(np.uint32) == r.view(np.uint32) or (np.isinf(r) and np.isinf(got))


def test_hand_examples_through_fused_forward():
    # test_reference.cpp:70-91: uniform logits -> ln 4; (0, 1) target 1 -> log(1+e)-1; V = 1 -> 0
    H = np.array([[1.0]], np.float32)
    W = np.array([[0.7], [0.7], [0.7], [0.7]], np.float32)
    _, rows, red = ob.forward(H, W, np.array([2]), "sum")
    assert red == pytest.approx(math.log(4.0), rel=1e-6)
    W2 = np.array([[0.0], [1.0]], np.float32)
    _, _, red = ob.forward(H, W2, np.array([1]), "sum")
    assert red == pytest.approx(0.3132616875182228, rel=1e-6)
    _, _, red = ob.forward(np.array([[5.0], [-3.0]], np.float32), np.array([[1.0]], np.float32),
                           np.array([0, 0]), "sum")
    assert red == 0.0


def test_two_class_backward_hand_example():
    # test_reference.cpp:180-195: dW = (p0, p1 - 1), dH = p1 - 1, sigma(-1) = 0.2689414213699951
    H = np.array([[1.0]], np.float32)
    W = np.array([[0.0], [1.0]], np.float32)
    Y = np.array([1])
    st, _, _ = ob.forward(H, W, Y, "sum")
    dH, dW = ob.backward(H, W, Y, st, "sum")
    sig = 0.2689414213699951
    assert dW[0, 0] == pytest.approx(sig, rel=1e-6)
    assert dW[1, 0] == pytest.approx(-sig, rel=1e-6)
    assert dH[0, 0] == pytest.approx(-sig, rel=1e-6)


def test_partition_ranges_ceil_first():
    # exec.hpp:25-41, test_core_types.cpp:248-265
    lo = np.zeros(8, np.uint64)
    hi = np.zeros(8, np.uint64)
    assert ob.oracle_lib().orc_partition_ranges(128256, 8, lo.ctypes.data_as(ob.P), hi.ctypes.data_as(ob.P)) == 0
    assert list(hi - lo) == [16032] * 8
    assert ob.oracle_lib().orc_partition_ranges(10, 4, lo.ctypes.data_as(ob.P), hi.ctypes.data_as(ob.P)) == 0
    assert list((hi - lo)[:4]) == [3, 3, 2, 2]


def _load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


GOLDEN_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_generator_matches_golden(case):
    g = _load(case)
    n, d, v = (int(x) for x in g["dims"])
    frac = {"sum_ignores_ragged_d": 0.25, "none_per_position": 0.2, "tp_3_ranks": 0.25}.get(case, 0.0)
    H, W, Y = ob.make_instance(n, d, v, int(g["seed"]), -100, frac)
    np.testing.assert_array_equal(H, g["H"])
    np.testing.assert_array_equal(Y, g["Y"])
    if g["W"].size:
        np.testing.assert_array_equal(W, g["W"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_oracle_matches_golden_bitwise(case):
    g = _load(case)
    n, d, v = (int(x) for x in g["dims"])
    H, W, Y = g["H"], g["W"], g["Y"]
    if not W.size:
        _, W, _ = ob.make_instance(n, d, v, int(g["seed"]), -100, 0.0)
    ign = int(g["ignore_index"]) if int(g["has_ignore"]) else None
    red = str(g["reduction"])
    ranks = int(g["ranks"])
    if ranks == 1:
        st, rows, lr = ob.forward(H, W, Y, red, ign, int(g["window"]))
    else:
        # tp_forward: per-shard partials merged in rank order (parallel_sim.hpp:186-236)
        lo = np.zeros(ranks, np.uint64); hi = np.zeros(ranks, np.uint64)
        ob.oracle_lib().orc_partition_ranges(v, ranks, lo.ctypes.data_as(ob.P), hi.ctypes.data_as(ob.P))
        parts = [ob.rank_partial(H, W[int(a):int(b)], Y, int(a), ign) for a, b in zip(lo, hi)]
        st = ob.merge(parts)
        with np.errstate(divide="ignore"):
            rows = np.where(st["found"] == 1, (st["m"] - st["z_target"]) + np.log(st["a"]), 0).astype(np.float32)
        lr = float(g["loss_reduced"])
    np.testing.assert_array_equal(st["m"], g["m"])
    np.testing.assert_array_equal(st["a"], g["a"])
    np.testing.assert_array_equal(st["z_target"], g["z_target"])
    np.testing.assert_array_equal(st["found"], g["found"])
    if ranks == 1:
        assert lr == float(g["loss_reduced"])
    up = g["upstream"] if red == "none" else 1.0
    if n * v * d <= 5_000_000:
        dH, dW = ob.backward(H, W, Y, st, red, up, ign)
        if ranks == 1:
            np.testing.assert_array_equal(dH, g["dH"])
            np.testing.assert_array_equal(dW, g["dW"])
        else:  # rank-ordered dH sum differs in rounding only
            np.testing.assert_allclose(dH, g["dH"], rtol=0, atol=1e-6 * np.abs(g["dH"]).max())
            np.testing.assert_array_equal(dW, g["dW"])


def test_oracle_vs_reference_random_bitwise():
    if not ob.ref_available():
        pytest.skip("reference build absent")
    rng = np.random.default_rng(5)
    for rep in range(12):
        n, d, v = int(rng.integers(1, 40)), int(rng.integers(1, 70)), int(rng.integers(1, 300))
        frac = 0.25 if rep % 2 else 0.0
        H, W, Y = ob.make_instance(n, d, v, 100 + rep, -100, frac)
        ign = -100 if frac else None
        for red in ("mean", "sum"):
            st, rows, lr = ob.forward(H, W, Y, red, ign)
            st2, rows2, lr2 = ob.ref_forward(H, W, Y, red, ign)
            assert lr == lr2
            np.testing.assert_array_equal(st["a"], st2["a"])
            dH, dW = ob.backward(H, W, Y, st, red, 1.0, ign)
            dH2, dW2 = ob.ref_backward(H, W, Y, st2, red, 1.0, ign)
            np.testing.assert_array_equal(dH, dH2)
            np.testing.assert_array_equal(dW, dW2)


def test_oracle_error_semantics():
    H, W, Y = ob.make_instance(4, 8, 10, 1)
    with pytest.raises(ob.OracleError) as e:
        ob.forward(H, W, np.array([0, 1, 10, 2]), "mean")
    assert e.value.code == 2  # TargetOutOfRange
    st, _, _ = ob.forward(H, W, Y, "mean")
    bad = st.copy()
    bad["found"][1] = 0
    with pytest.raises(ob.OracleError) as e:
        ob.backward(H, W, Y, bad, "mean")
    assert e.value.code == 5  # MissingStats
    with pytest.raises(ob.OracleError) as e:
        ob.backward(H, W, Y, st, "none", 1.0)
    assert e.value.code == 6  # InconsistentUpstream
