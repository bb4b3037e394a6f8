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
    {"bwd_epi_warps": 4},
    {"bwd_tma_epi": 0},
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
