"""Multi-rank C-ABI (include/fce/fce_vp.h) with k > 1 real ranks on one B200.

The ranks are k host threads of this process, each with its own CUDA stream,
library handle and communicator of one in-process group (the "local"
transport: libfce's own peer-memory collectives).  Every rank runs exactly the
code a one-process-per-GPU NCCL job runs — fce_vp_forward / fce_vp_backward /
fce_sp_gather / fce_sp_scatter / fce_dp_step — and the results are checked
against the CPU oracle's restatement of the reference's tp_forward /
tp_backward / sp_to_tp_gather / dp_step (parallel_sim.hpp:165-378) on the same
bf16-grid inputs.  Tolerances as tests/test_parity_gpu.py: loss / lse 1e-3
relative, dH / dW 1e-2 relative max-norm, found flags and ignored rows exact.
"""
import os

import numpy as np
import pytest
import torch

import paper_2511_17599_b200 as fce
from paper_2511_17599_b200 import vocab_parallel as vp
from oracle import bindings as ob

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-3
GRAD_RTOL = 1e-2


def relmax(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = np.abs(ref).max()
    return float(np.abs(got - ref).max() / scale) if scale else float(np.abs(got).max())


def bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda().to(torch.bfloat16)


def vp_step(k, H, W, Y, ign, reduction, upstream=1.0, strided_dh=False):
    """k-rank tp_forward + tp_backward; returns per-rank (out, dH, dW shard)."""
    n, d = H.shape
    v = W.shape[0]
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    up = upstream if np.isscalar(upstream) else torch.from_numpy(np.asarray(upstream, np.float32)).cuda()
    ranges = fce.shard_ranges(v, k)

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        out = vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, reduction, ign, handle=h)
        dh_buf = None
        if strided_dh:
            dh_buf = torch.full((n, d + 12), 7.0, dtype=torch.float32, device="cuda")[:, :d]
        dh, dw = vp.native_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, out.stats, reduction, up, ign,
                                    handle=h, dhidden=dh_buf)
        if strided_dh:
            # columns past d belong to the caller: untouched
            assert torch.all(dh_buf.as_strided((n, 12), (d + 12, 1), d) == 7.0)
        return out, dh, dw

    return vp.run_ranks(k, rank_fn)


@pytest.mark.parametrize("k,reduction,ign,frac,strided", [
    (2, "sum", None, 0.0, True),
    (3, "mean", -100, 0.25, False),
    (8, "none", -1, 0.2, False),
    (5, "mean", None, 0.0, False),
])
def test_vocab_parallel_k_ranks_match_oracle(cuda, k, reduction, ign, frac, strided):
    n, d, v = 200, 136, 1500
    H, W, Y = ob.make_instance(n, d, v, 11 + k, -100 if ign is None else ign, frac)
    rng = np.random.default_rng(k)
    upstream = rng.standard_normal(n).astype(np.float32) if reduction == "none" else 1.0
    res = vp_step(k, H, W, Y, ign, reduction, upstream, strided)
    st, rows, lred = ob.forward(H, W, Y, reduction, ign)
    dH, dW = ob.backward(H, W, Y, st, reduction, upstream, ign)
    valid = np.ones(n, bool) if ign is None else Y != ign
    lse_ref = st["m"] + np.log(np.where(valid, st["a"], 1))
    out0 = res[0][0]
    for r, (out, dh, dw) in enumerate(res):
        # every rank holds the same merged stats / loss (rank-ordered merge)
        np.testing.assert_array_equal(out.stats.found.cpu().numpy(), st["found"])
        np.testing.assert_array_equal(out.stats.m.cpu().numpy(), out0.stats.m.cpu().numpy())
        np.testing.assert_array_equal(out.loss_rows.cpu().numpy(), out0.loss_rows.cpu().numpy())
        lse = out.lse.cpu().numpy()
        assert np.max(np.abs(lse[valid] - lse_ref[valid]) / np.maximum(1, np.abs(lse_ref[valid]))) < LOSS_RTOL
        got_rows = out.loss_rows.cpu().numpy()
        assert np.all(got_rows[~valid] == 0.0)
        assert np.max(np.abs(got_rows - rows) / np.maximum(1, np.abs(rows))) < LOSS_RTOL
        if reduction != "none":
            assert abs(out.loss.item() - lred) <= LOSS_RTOL * max(1.0, abs(lred))
        # dH: the all-reduced sum over the k shards, identical on every rank
        dh_np = dh.cpu().numpy()
        assert relmax(dh_np, dH) < GRAD_RTOL, (r, relmax(dh_np, dH))
        np.testing.assert_array_equal(dh_np, res[0][1].cpu().numpy())
        if ign is not None:
            assert np.all(dh_np[~valid] == 0.0)
    # dW stays sharded: the concatenation of the rank shards is the full dW
    dw_all = np.concatenate([x[2].cpu().numpy() for x in res])
    assert dw_all.shape == dW.shape
    assert relmax(dw_all, dW) < GRAD_RTOL


def test_vocab_parallel_matches_single_rank_path(cuda):
    n, d, v = 256, 264, 2048
    H, W, Y = ob.make_instance(n, d, v, 3, -100, 0.1)
    res = vp_step(4, H, W, Y, -100, "mean")
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    one = fce.fused_forward(Hd, Wd, Yd, "mean", -100)
    dh1, dw1 = fce.fused_backward_recompute(Hd, Wd, Yd, one.stats, "mean", 1.0, -100)
    out, dh, _ = res[0]
    np.testing.assert_array_equal(out.stats.found.cpu().numpy(), one.stats.found.cpu().numpy())
    assert abs(out.loss.item() - one.loss.item()) <= 1e-5 * abs(one.loss.item())
    assert relmax(dh.cpu().numpy(), dh1.cpu().numpy()) < 1e-3
    dw_all = torch.cat([x[2] for x in res]).cpu().numpy()
    assert relmax(dw_all, dw1.cpu().numpy()) < 1e-3


def test_vocab_parallel_target_errors_raise_on_every_rank(cuda):
    n, d, v = 64, 72, 600
    H, W, Y = ob.make_instance(n, d, v, 5)
    Y = Y.copy()
    Y[7] = v + 3  # outside [0, V): every rank's validation rejects it before any collective
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    ranges = fce.shard_ranges(v, 3)
    caught = []

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        try:
            vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, "mean", None, handle=h)
        except fce.TargetOutOfRange:
            caught.append(r)

    vp.run_ranks(3, rank_fn)
    assert sorted(caught) == [0, 1, 2]


def test_comm_query_and_collectives_are_rank_ordered(cuda):
    k = 5
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal(1003).astype(np.float32) * 10 ** r for r in range(k)]
    ref = xs[0].copy()
    for x in xs[1:]:
        ref = (ref + x).astype(np.float32)  # sequential fp32 adds in rank order

    def rank_fn(r, comm, h):
        assert comm.query() == (k, r, 2)
        x = torch.from_numpy(xs[r]).cuda()
        s = vp.native_all_reduce(comm, x.clone(), handle=h)
        g = vp.native_all_gather(comm, torch.full((3,), float(r), device="cuda"), handle=h)
        big = torch.arange(k * 7, dtype=torch.float32, device="cuda") * (r + 1)
        rs = vp.native_reduce_scatter(comm, big, handle=h)
        return s.cpu().numpy(), g.cpu().numpy(), rs.cpu().numpy()

    res = vp.run_ranks(k, rank_fn)
    tot = sum(range(1, k + 1))
    for r, (s, g, rs) in enumerate(res):
        np.testing.assert_array_equal(s, ref)  # bit-exact: the local transport sums in rank order
        np.testing.assert_array_equal(g, np.repeat(np.arange(k, dtype=np.float32)[:, None], 3, 1))
        np.testing.assert_array_equal(rs, np.arange(r * 7, r * 7 + 7, dtype=np.float32) * tot)


@pytest.mark.parametrize("k,sizes", [(3, None), (4, [5, 0, 40, 19])])
def test_sp_gather_and_scatter(cuda, k, sizes):
    n, d = 64, 40
    rng = np.random.default_rng(k)
    H = ob.make_instance(n, d, 10, 1)[0]
    if sizes is None:
        ranges = fce.shard_ranges(n, k)
    else:
        edges = np.concatenate([[0], np.cumsum(sizes)])
        ranges = [(int(edges[i]), int(edges[i + 1])) for i in range(k)]
    parts = [rng.standard_normal((n, d)).astype(np.float32) for _ in range(k)]
    Hd = bf16(H)

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        full = vp.native_sp_gather(comm, Hd[lo:hi], n, handle=h)
        shard = vp.native_sp_scatter(comm, torch.from_numpy(parts[r]).cuda(), hi - lo, handle=h)
        return full.float().cpu().numpy(), shard.cpu().numpy()

    res = vp.run_ranks(k, rank_fn)
    total = parts[0].copy()
    for p_ in parts[1:]:
        total = (total + p_).astype(np.float32)
    for r, (full, shard) in enumerate(res):
        np.testing.assert_array_equal(full, H)  # bf16-grid H gathers exactly, in position order
        lo, hi = ranges[r]
        np.testing.assert_array_equal(shard, total[lo:hi])


def test_sp_gather_rejects_bad_layouts(cuda):
    n, d = 30, 16
    H = bf16(ob.make_instance(n, d, 10, 1)[0])
    errs = {}

    def rank_fn(r, comm, h):
        try:  # rows do not add up to n
            vp.native_sp_gather(comm, H[:10], n + 5, handle=h)
        except fce.DimensionMismatch:
            errs.setdefault("rows", []).append(r)
        try:  # widths disagree (sp_to_tp_gather: "hidden shards disagree on width")
            vp.native_sp_gather(comm, H[:15, : 8 + 8 * r], n, handle=h)
        except fce.InvalidLayout:
            errs.setdefault("width", []).append(r)

    vp.run_ranks(2, rank_fn)
    assert sorted(errs["rows"]) == [0, 1] and sorted(errs["width"]) == [0, 1]


@pytest.mark.parametrize("k,reduction", [(2, "mean"), (3, "sum")])
def test_dp_step_matches_oracle(cuda, k, reduction):
    n, d, v = 96, 104, 900
    W = ob.make_instance(n, d, v, 100)[1]
    reps = [ob.make_instance(n, d, v, 200 + r, -100, 0.2) for r in range(k)]
    Wd = bf16(W)

    def rank_fn(r, comm, h):
        H, _, Y = reps[r]
        loss, dh, dw = vp.native_dp_step(comm, bf16(H), Wd, torch.from_numpy(Y).cuda(), reduction, -100, handle=h)
        return loss.item(), dh.cpu().numpy(), dw.cpu().numpy()

    res = vp.run_ranks(k, rank_fn)
    losses, dws, dhs = [], [], []
    for r in range(k):
        H, _, Y = reps[r]
        st, _, lred = ob.forward(H, W, Y, reduction, -100)
        dH, dW_ = ob.backward(H, W, Y, st, reduction, 1.0, -100)
        losses.append(lred)
        dws.append(dW_)
        dhs.append(dH)
    loss_ref = sum(losses) / k
    dw_ref = sum(dws) / k
    for r, (loss, dh, dw) in enumerate(res):
        assert abs(loss - loss_ref) <= LOSS_RTOL * max(1.0, abs(loss_ref))
        assert relmax(dw, dw_ref) < GRAD_RTOL
        assert relmax(dh, dhs[r]) < GRAD_RTOL  # dH stays rank-local
        np.testing.assert_array_equal(dw, res[0][2])


def test_dp_step_rejects_unequal_micro_batches_and_none(cuda):
    d, v = 40, 300
    W = bf16(ob.make_instance(4, d, v, 1)[1])
    got = {}

    def rank_fn(r, comm, h):
        n = 32 + 16 * r
        H, _, Y = ob.make_instance(n, d, v, r)
        try:
            vp.native_dp_step(comm, bf16(H), W, torch.from_numpy(Y).cuda(), "mean", handle=h)
        except fce.InvalidLayout:
            got.setdefault("sizes", []).append(r)
        try:
            vp.native_dp_step(comm, bf16(H), W, torch.from_numpy(Y).cuda(), "none", handle=h)
        except fce.UnsupportedReduction:
            got.setdefault("none", []).append(r)

    vp.run_ranks(2, rank_fn)
    assert sorted(got["sizes"]) == [0, 1] and sorted(got["none"]) == [0, 1]


@pytest.mark.parametrize("k,chunks", [(1, 2), (2, 2), (3, 3), (4, 2)])
def test_overlapped_dh_all_reduce_matches_oracle(cuda, k, chunks):
    """Option vp_overlap_chunks: the backward runs in row chunks and each
    chunk's dH all-reduce is released from the communicator's stream by the
    kernel's own completion counter while later chunks compute.  Results equal
    the oracle (and the unchunked path) on every rank."""
    n, d, v = 1024, 136, 3000
    H, W, Y = ob.make_instance(n, d, v, 40 + k, -100, 0.0)
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    ranges = fce.shard_ranges(v, k)

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        out = vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, "mean", None, handle=h)
        h.set_option("vp_overlap_chunks", chunks)
        h.set_option("vp_reserve_sms", 16)
        dh, dw = vp.native_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, out.stats, "mean", 1.0, None, handle=h)
        h.set_option("vp_overlap_chunks", 0)
        dh0, dw0 = vp.native_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, out.stats, "mean", 1.0, None, handle=h)
        return dh, dw, dh0, dw0

    res = vp.run_ranks(k, rank_fn)
    st, _, _ = ob.forward(H, W, Y, "mean")
    dH, dW = ob.backward(H, W, Y, st, "mean", 1.0)
    for dh, dw, dh0, dw0 in res:
        assert relmax(dh.cpu().numpy(), dH) < GRAD_RTOL
        assert relmax(dh.cpu().numpy(), dh0.cpu().numpy()) < 1e-3
        np.testing.assert_array_equal(dh.cpu().numpy(), res[0][0].cpu().numpy())
    dw_all = np.concatenate([x[1].cpu().numpy() for x in res])
    assert relmax(dw_all, dW) < GRAD_RTOL


@pytest.mark.parametrize("case", range(8))
def test_random_multirank_cases(cuda, case):
    """Randomised k-rank vocab-parallel steps (k, shapes, reduction, ignore
    sentinel, overlap option) against the oracle on every rank."""
    rng = np.random.default_rng(500 + case)
    k = int(rng.integers(2, 7))
    n = int(rng.integers(1, 700))
    d = int(rng.integers(1, 300))
    v = int(rng.integers(k, 3000))
    red = ("mean", "sum", "none")[case % 3]
    ign = (None, -100, -1, -5)[case % 4]
    frac = 0.0 if ign is None else float(rng.uniform(0.05, 0.5))
    chunks = 2 if (case % 2 and ign is None and n >= 512) else 0
    H, W, Y = ob.make_instance(n, d, v, 900 + case, -100 if ign is None else ign, frac)
    up = rng.standard_normal(n).astype(np.float32) if red == "none" else 1.0
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    upd = torch.from_numpy(up).cuda() if red == "none" else 1.0
    ranges = fce.shard_ranges(v, k)

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        h.set_option("vp_overlap_chunks", chunks)
        out = vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, red, ign, handle=h)
        dh, dw = vp.native_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, out.stats, red, upd, ign, handle=h)
        return out, dh, dw

    res = vp.run_ranks(k, rank_fn)
    st, rows, lred = ob.forward(H, W, Y, red, ign)
    dH, dW = ob.backward(H, W, Y, st, red, up, ign)
    for out, dh, dw in res:
        np.testing.assert_array_equal(out.stats.found.cpu().numpy(), st["found"])
        got = out.loss_rows.cpu().numpy()
        assert np.max(np.abs(got - rows) / np.maximum(1, np.abs(rows))) < LOSS_RTOL
        if red != "none":
            assert abs(out.loss.item() - lred) <= LOSS_RTOL * max(1.0, abs(lred))
        assert relmax(dh.cpu().numpy(), dH) < GRAD_RTOL
    assert relmax(np.concatenate([x[2].cpu().numpy() for x in res]), dW) < GRAD_RTOL


@pytest.mark.parametrize("k,ign,chunks,fused", [(2, None, 0, 0), (3, -100, 0, 0), (4, None, 2, 0), (3, None, 0, 1),
                                                (8, None, 0, 1)])
def test_ipc_transport_multiprocess(cuda, tmp_path, k, ign, chunks, fused):
    """k separate processes (all on this GPU) over the IPC transport: CUDA IPC
    mappings of each rank's registered buffer, cross-process events and a
    shared-memory barrier — the one-process-per-rank data path without NCCL.
    Every rank's loss / stats / dH and the concatenated dW shards against the
    oracle; the raw collectives bit-exact against rank-ordered sums."""
    import subprocess
    import sys
    n, d, v = 600 if chunks else 300, 136, 2500
    H, W, Y = ob.make_instance(n, d, v, 70 + k, -100, 0.2 if ign is not None else 0.0)
    rng = np.random.default_rng(k)
    x = rng.standard_normal((k, 777)).astype(np.float32)
    inp = tmp_path / "in.npz"
    np.savez(inp, H=H, W=W, Y=Y, ign=-100, has_ign=int(ign is not None), x=x, chunks=chunks, fused=fused)
    uid = vp.NativeComm.ipc_id().hex()
    helper = os.path.join(os.path.dirname(os.path.abspath(__file__)), "helpers", "ipc_rank.py")
    env = dict(os.environ, FCE_LOCAL_TIMEOUT_S="300")
    procs = [subprocess.Popen([sys.executable, helper, str(r), str(k), uid, str(inp), str(tmp_path / f"out{r}.npz")],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(k)]
    logs = [p.communicate(timeout=600)[0] for p in procs]
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    outs = [np.load(tmp_path / f"out{r}.npz") for r in range(k)]
    st, rows, lred = ob.forward(H, W, Y, "mean", ign)
    dH, dW = ob.backward(H, W, Y, st, "mean", 1.0, ign)
    ref_s = x[0].copy()
    for r in range(1, k):
        ref_s = (ref_s + x[r]).astype(np.float32)
    tot = sum(range(1, k + 1))
    for r, o in enumerate(outs):
        np.testing.assert_array_equal(o["found"], st["found"])
        assert abs(float(o["loss"]) - lred) <= LOSS_RTOL * max(1.0, abs(lred))
        assert relmax(o["dh"], dH) < GRAD_RTOL
        if not fused:  # in-kernel peer reduction adds in arrival order
            np.testing.assert_array_equal(o["dh"], outs[0]["dh"])
        np.testing.assert_array_equal(o["s"], ref_s)
        np.testing.assert_array_equal(o["g"], np.repeat(np.arange(k, dtype=np.float32)[:, None], 5, 1))
        np.testing.assert_array_equal(o["rs"], np.arange(r * 9, r * 9 + 9, dtype=np.float32) * tot)
    assert relmax(np.concatenate([o["dw"] for o in outs]), dW) < GRAD_RTOL
    assert relmax(np.concatenate([o["dh_sp"] for o in outs]), dH) < GRAD_RTOL  # SP shards, fused reduce-scatter


@pytest.mark.parametrize("k,red", [(2, "mean"), (3, "sum"), (8, "none")])
def test_fused_dh_reduction_in_kernel(cuda, k, red):
    """Option vp_fused_dh: every rank's dH tiles are TMA-reduce-added straight
    into the owning rank's accumulator (peer memory) inside the backward; the
    full dH on every rank equals the oracle."""
    n, d, v = 700, 136, 2000
    H, W, Y = ob.make_instance(n, d, v, 300 + k)
    up = np.linspace(0.5, 1.5, n).astype(np.float32) if red == "none" else 1.0
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    upd = torch.from_numpy(up).cuda() if red == "none" else 1.0
    ranges = fce.shard_ranges(v, k)

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        out = vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, red, None, handle=h)
        h.set_option("vp_fused_dh", 1)
        return vp.native_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, out.stats, red, upd, None, handle=h)

    res = vp.run_ranks(k, rank_fn)
    st, _, _ = ob.forward(H, W, Y, red)
    dH, dW = ob.backward(H, W, Y, st, red, up)
    for dh, _ in res:
        assert relmax(dh.cpu().numpy(), dH) < GRAD_RTOL
    assert relmax(np.concatenate([x[1].cpu().numpy() for x in res]), dW) < GRAD_RTOL


@pytest.mark.parametrize("k,sizes,ign", [(3, None, None), (4, [70, 0, 500, 130], None), (2, [333, 367], -100)])
def test_sp_vp_backward_reduce_scatter(cuda, k, sizes, ign):
    """fce_sp_vp_backward: rank r gets the summed dH rows of its position shard
    (ragged, unaligned and empty shards; fused in the kernel without ignore,
    local dH + reduce-scatter with it) and its dW shard."""
    n, d, v = 700, 72, 1500
    H, W, Y = ob.make_instance(n, d, v, 410 + k, -100, 0.2 if ign is not None else 0.0)
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    vr = fce.shard_ranges(v, k)
    if sizes is None:
        pr = fce.shard_ranges(n, k)
    else:
        e = np.concatenate([[0], np.cumsum(sizes)])
        pr = [(int(e[i]), int(e[i + 1])) for i in range(k)]

    def rank_fn(r, comm, h):
        lo, hi = vr[r]
        out = vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, "mean", ign, handle=h)
        return vp.native_sp_vp_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, out.stats, pr[r][1] - pr[r][0], "mean",
                                        1.0, ign, handle=h)

    res = vp.run_ranks(k, rank_fn)
    st, _, _ = ob.forward(H, W, Y, "mean", ign)
    dH, dW = ob.backward(H, W, Y, st, "mean", 1.0, ign)
    got = np.concatenate([x[0].cpu().numpy() for x in res])
    assert got.shape == dH.shape
    assert relmax(got, dH) < GRAD_RTOL
    if ign is not None:
        assert np.all(got[Y == ign] == 0.0)
    assert relmax(np.concatenate([x[1].cpu().numpy() for x in res]), dW) < GRAD_RTOL


def test_sp_vp_backward_fallbacks(cuda):
    """fce_sp_vp_backward where the in-kernel reduction does not apply: a
    1-rank NCCL communicator (no peer memory) and a width whose fp32 rows are
    not 16-byte multiples (d % 4 != 0) on the local transport — local dH, then
    the reduce-scatter; vp_fused_dh falls back the same way."""
    n, d, v = 300, 70, 900
    H, W, Y = ob.make_instance(n, d, v, 77)
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    st, _, _ = ob.forward(H, W, Y, "mean")
    dH, dW = ob.backward(H, W, Y, st, "mean", 1.0)
    comm = vp.NativeComm.create_local(device=0)
    out = vp.native_forward(comm, Hd, Wd, Yd, 0, v, "mean")
    dh, dw = vp.native_sp_vp_backward(comm, Hd, Wd, Yd, 0, v, out.stats, n, "mean", 1.0)
    comm.close()
    assert relmax(dh.cpu().numpy(), dH) < GRAD_RTOL and relmax(dw.cpu().numpy(), dW) < GRAD_RTOL
    ranges = fce.shard_ranges(v, 2)
    pr = fce.shard_ranges(n, 2)

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        o = vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, "mean", None, handle=h)
        h.set_option("vp_fused_dh", 1)
        full, _ = vp.native_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, o.stats, "mean", 1.0, None, handle=h)
        shard, dw_r = vp.native_sp_vp_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, o.stats, pr[r][1] - pr[r][0],
                                               "mean", 1.0, None, handle=h)
        return full.cpu().numpy(), shard.cpu().numpy(), dw_r.cpu().numpy()

    res = vp.run_ranks(2, rank_fn)
    for full, _, _ in res:
        assert relmax(full, dH) < GRAD_RTOL
    assert relmax(np.concatenate([x[1] for x in res]), dH) < GRAD_RTOL
    assert relmax(np.concatenate([x[2] for x in res]), dW) < GRAD_RTOL


@pytest.mark.parametrize("k,sizes,ign", [(3, None, None), (4, [130, 0, 400, 170], -100)])
def test_sp_vp_forward_then_backward(cuda, k, sizes, ign):
    """SP -> TP -> SP: fce_sp_vp_forward (H all-gather overlapped with K1 on the
    rank's own rows) then fce_sp_vp_backward (dH reduce-scatter in the kernel);
    every rank's gathered H is bit-exact, stats / loss / dH shards / dW shards
    match the oracle."""
    n, d, v = 700, 136, 1800
    H, W, Y = ob.make_instance(n, d, v, 520 + k, -100, 0.25 if ign is not None else 0.0)
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    vr = fce.shard_ranges(v, k)
    if sizes is None:
        pr = fce.shard_ranges(n, k)
    else:
        e = np.concatenate([[0], np.cumsum(sizes)])
        pr = [(int(e[i]), int(e[i + 1])) for i in range(k)]

    def rank_fn(r, comm, h):
        lo, hi = vr[r]
        full, out = vp.native_sp_vp_forward(comm, Hd[pr[r][0]:pr[r][1]], n, Wd[lo:hi], Yd, lo, v, "mean", ign,
                                            handle=h)
        dh, dw = vp.native_sp_vp_backward(comm, full, Wd[lo:hi], Yd, lo, v, out.stats, pr[r][1] - pr[r][0],
                                          "mean", 1.0, ign, handle=h)
        return full.float().cpu().numpy(), out.loss.item(), out.stats.found.cpu().numpy(), dh.cpu().numpy(), \
            dw.cpu().numpy()

    res = vp.run_ranks(k, rank_fn)
    st, _, lred = ob.forward(H, W, Y, "mean", ign)
    dH, dW = ob.backward(H, W, Y, st, "mean", 1.0, ign)
    for full, loss, found, _, _ in res:
        np.testing.assert_array_equal(full, H)
        np.testing.assert_array_equal(found, st["found"])
        assert abs(loss - lred) <= LOSS_RTOL * max(1.0, abs(lred))
    assert relmax(np.concatenate([x[3] for x in res]), dH) < GRAD_RTOL
    assert relmax(np.concatenate([x[4] for x in res]), dW) < GRAD_RTOL


def test_ranks_with_different_problems_fail_instead_of_hanging(cuda):
    """With validation on, fce_vp_forward cross-checks (N, d, V_total, ignore)
    across the ranks before any size-dependent collective."""
    d, v = 72, 600
    W = bf16(ob.make_instance(4, d, v, 1)[1])
    ranges = fce.shard_ranges(v, 2)
    got = []

    def rank_fn(r, comm, h):
        n = 64 + 32 * r
        H, _, Y = ob.make_instance(n, d, v, r)
        lo, hi = ranges[r]
        try:
            vp.native_forward(comm, bf16(H), W[lo:hi], torch.from_numpy(Y).cuda(), lo, v, "mean", handle=h)
        except fce.DimensionMismatch:
            got.append(r)

    vp.run_ranks(2, rank_fn)
    assert sorted(got) == [0, 1]


def test_ranks_with_different_backward_modes_fail_instead_of_hanging(cuda):
    n, d, v = 256, 72, 600
    H, W, Y = ob.make_instance(n, d, v, 3)
    Hd, Wd, Yd = bf16(H), bf16(W), torch.from_numpy(Y).cuda()
    ranges = fce.shard_ranges(v, 2)
    got = []

    def rank_fn(r, comm, h):
        lo, hi = ranges[r]
        out = vp.native_forward(comm, Hd, Wd[lo:hi], Yd, lo, v, "mean", handle=h)
        h.set_option("vp_fused_dh", r)  # rank 1 asks for the in-kernel reduction, rank 0 does not
        try:
            vp.native_backward(comm, Hd, Wd[lo:hi], Yd, lo, v, out.stats, "mean", 1.0, handle=h)
        except fce.InvalidArgument:
            got.append(r)

    vp.run_ranks(2, rank_fn)
    assert sorted(got) == [0, 1]
