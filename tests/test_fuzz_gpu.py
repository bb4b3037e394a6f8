"""Randomised parity sweep: ragged shapes x ignore fractions x reductions x
handle options (kernel variants, chunk geometries) against the CPU oracle."""
import numpy as np
import pytest
import torch

import paper_2511_17599_b200 as fce
from oracle import bindings as ob
from test_parity_gpu import check_forward, check_grads, to_dev

pytestmark = pytest.mark.gpu

OPTION_SETS = [
    {},
    {"fwd_mc": 1},
    {"fwd_pair": 1},
    {"skip_ignored": 0},
    {"row_chunk": 256, "band_cols": 512},
    {"row_chunk": 512, "band_cols": 256, "dh_group": 3},
    {"bwd_epi_warps": 8},
    {"bwd_tma_epi": 0},
    {"bwd_tma_epi": 1},
    {"bwd_tma_epi": 2},
    {"splits": 3},
]


@pytest.mark.parametrize("case", range(120))
def test_random_case(cuda, case):
    rng = np.random.default_rng(7000 + case)
    n = int(rng.integers(1, 1200))
    d = int(rng.integers(1, 260))
    v = int(rng.integers(1, 4000))
    frac = [0.0, 0.3, 0.9][case % 3]
    red = ["mean", "sum", "none"][(case // 3) % 3]
    opts = OPTION_SETS[case % len(OPTION_SETS)]
    H, W, Y = ob.make_instance(n, d, v, 100 + case, -100, frac)
    ign = -100 if frac > 0 else None
    st, rows, lred = ob.forward(H, W, Y, red, ign)
    Hd, Wd, Yd = to_dev(H, W, Y)
    h = fce.Handle(0)
    for k, x in opts.items():
        h.set_option(k, x)
    out = fce.fused_forward(Hd, Wd, Yd, red, ign, handle=h)
    check_forward(out, st, rows, lred, Y, ign, red)
    up = rng.uniform(0.25, 2.0, n).astype(np.float32) if red == "none" else 1.5
    dH, dW = ob.backward(H, W, Y, st, red, up, ign)
    upd = torch.from_numpy(up).cuda() if red == "none" else 1.5
    dh, dw = fce.fused_backward_recompute(Hd, Wd, Yd, out.stats, red, upd, ign, handle=h)
    check_grads(dh, dw, dH, dW, Y, ign)
    h.close()


@pytest.mark.parametrize("case", range(30))
def test_random_vocab_parallel_case(cuda, case):
    """Simulated vocabulary-parallel ranks (tp_rank_partial / rank-ordered merge /
    per-shard backward summed into dH) on random shapes, shard counts, ignore
    fractions and windows, against the oracle."""
    from test_parity_gpu import _tp_backward
    rng = np.random.default_rng(9000 + case)
    n = int(rng.integers(1, 700))
    d = int(rng.integers(1, 200))
    v = int(rng.integers(2, 3000))
    ranks = int(rng.integers(2, min(9, v + 1)))
    frac = [0.0, 0.4][case % 2]
    red = ["mean", "sum"][(case // 2) % 2]
    H, W, Y = ob.make_instance(n, d, v, 300 + case, -100, frac)
    ign = -100 if frac > 0 else None
    st, rows, lred = ob.forward(H, W, Y, red, ign)
    Hd, Wd, Yd = to_dev(H, W, Y)
    parts = [fce.tp_rank_partial(Hd, Wd[lo:hi], lo, v, Yd, ign) for lo, hi in fce.shard_ranges(v, ranks)]
    out = fce.merge_rank_partials(parts, Yd, red, ign)
    check_forward(out, st, rows, lred, Y, ign, red)
    dH, dW = ob.backward(H, W, Y, st, red, 1.0, ign)
    dh, dw = _tp_backward(Hd, Wd, Yd, out.stats, red, 1.0, ign, ranks)
    check_grads(dh, dw, dH, dW, Y, ign)
    if case % 3 == 0:
        window = int(rng.integers(1, v + 1))
        stw, rowsw, lredw = ob.forward(H, W, Y, red, ign, window)
        outw = fce.fused_forward_windowed(Hd, Wd, Yd, window, red, ign)
        check_forward(outw, stw, rowsw, lredw, Y, ign, red)
