"""World-size-2/3 gloo tests (CPU) of the vocab-parallel orchestration in
paper_2511_17599_b200.vocab_parallel.VocabParallel: shard layout, all-gather of
per-rank (m, a, z_target, found) partials in rank order, ordered merge, dH
all-reduce, dW kept per shard.  The per-rank compute is the CPU oracle here
(test infrastructure); on GPUs it is the CUDA path.  Expected values: the
reference's own tp_forward / tp_backward (golden fixture tp_3_ranks) and the
single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class OracleCompute:
    """CPU stand-in for CudaCompute (tests only)."""

    def partial(self, hidden, weight_shard, targets, v_offset, v_total, ignore_index):
        from oracle import bindings as ob
        st = ob.rank_partial(hidden.numpy(), weight_shard.numpy(), targets.numpy(), v_offset,
                             ignore_index, threads=1)
        return (torch.from_numpy(st["m"].copy()), torch.from_numpy(st["a"].copy()),
                torch.from_numpy(st["z_target"].copy()), torch.from_numpy(st["found"].copy()))

    def merge(self, m, a, z, f, targets, reduction, ignore_index):
        from oracle import bindings as ob
        parts = []
        for r in range(m.shape[0]):
            s = np.zeros(m.shape[1], ob.STATS_DTYPE)
            s["m"], s["a"], s["z_target"], s["found"] = m[r].numpy(), a[r].numpy(), z[r].numpy(), f[r].numpy()
            parts.append(s)
        return ob.merge(parts)

    def backward(self, hidden, weight_shard, targets, v_offset, v_total, stats, reduction,
                 upstream, ignore_index):
        from oracle import bindings as ob
        dh, dw = ob.backward(hidden.numpy(), weight_shard.numpy(), targets.numpy(), stats, reduction,
                             upstream, ignore_index, threads=1, v_offset=v_offset,
                             v_total=v_total)
        return torch.from_numpy(dh), torch.from_numpy(dw)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2511_17599_b200.vocab_parallel import VocabParallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _body(rank, world, case, q)
    except Exception as e:  # surface the failure instead of hanging the queue
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def _body(rank, world, case, q):
    from paper_2511_17599_b200.vocab_parallel import VocabParallel
    if True:
        g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
        H, W, Y = (torch.from_numpy(g[k]) for k in ("H", "W", "Y"))
        ign = int(g["ignore_index"]) if int(g["has_ignore"]) else None
        vp = VocabParallel(W.shape[0], compute=OracleCompute())
        st = vp.forward(H, vp.shard(W), Y, str(g["reduction"]), ign)
        dh, dw = vp.backward(H, vp.shard(W), Y, st, str(g["reduction"]), 1.0, ign)
        q.put((rank, vp.lo, vp.hi, st["m"], st["a"], st["z_target"], st["found"], dh.numpy(), dw.numpy()))


def _run(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for r in res:
        assert not (isinstance(r[1], str) and r[1] == "error"), r
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    return sorted(res, key=lambda r: r[0])


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_vocab_parallel_matches_reference_tp(world):
    case = "tp_3_ranks"
    g = dict(np.load(os.path.join(GOLDEN, case + ".npz")))
    res = _run(world, case)
    v = g["W"].shape[0]
    # shards tile [0, V) contiguously, ceil-first
    assert [r[1] for r in res] == [0] + [r[2] for r in res[:-1]] and res[-1][2] == v
    for rank, lo, hi, m, a, z, f, dh, dw in res:
        # every rank holds the same merged stats == the reference's tp_forward
        np.testing.assert_array_equal(f, g["found"])
        np.testing.assert_allclose(m, g["m"], rtol=0, atol=0)
        if world == 3:  # same shard layout as the fixture: bit-identical merge
            np.testing.assert_array_equal(a, g["a"])
        else:
            np.testing.assert_allclose(a, g["a"], rtol=1e-5)
        np.testing.assert_allclose(dh, g["dH"], rtol=0, atol=1e-6 * np.abs(g["dH"]).max())
        np.testing.assert_allclose(dw, g["dW"][lo:hi], rtol=0, atol=1e-6 * np.abs(g["dW"]).max())


def _sp_dp_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import bindings as ob
        from paper_2511_17599_b200 import shard_ranges
        from paper_2511_17599_b200.vocab_parallel import dp_step, sp_to_tp_gather, tp_to_sp_scatter
        H, W, Y = ob.make_instance(30, 12, 90, 5)
        lo, hi = shard_ranges(30, world)[rank]
        Hf = sp_to_tp_gather(torch.from_numpy(H[lo:hi]), 30)
        # reduce-scatter of per-rank dH partials gives each rank the sum of its rows
        part = torch.full((30, 12), float(rank + 1))
        mine = tp_to_sp_scatter(part, 30)

        class OracleStep:
            def step(self, hidden, weight, targets, reduction, ignore_index):
                st, _, l = ob.forward(hidden.numpy(), weight.numpy(), targets.numpy(), reduction, ignore_index,
                                      threads=1)
                dh, dw = ob.backward(hidden.numpy(), weight.numpy(), targets.numpy(), st, reduction, 1.0,
                                     ignore_index, threads=1)
                return l, torch.from_numpy(dh), torch.from_numpy(dw)

        dlo, dhi = rank * 15, rank * 15 + 15  # equal micro-batches for DP
        loss, dh, dw = dp_step(torch.from_numpy(H[dlo:dhi]), torch.from_numpy(W), torch.from_numpy(Y[dlo:dhi]),
                               "mean", None, compute=OracleStep())
        q.put((rank, Hf.numpy(), mine.numpy(), float(loss), dw.numpy()))
    except Exception as e:
        q.put((rank, "error", repr(e)))
        raise
    finally:
        dist.destroy_process_group()


def test_gloo_sp_gather_and_dp_step():
    from oracle import bindings as ob
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sp_dp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(world)], key=lambda r: r[0])
    for p in procs:
        p.join(60)
    for r in res:
        assert not (isinstance(r[1], str) and r[1] == "error"), r
    H, W, Y = ob.make_instance(30, 12, 90, 5)
    for rank, Hf, mine, loss, dw in res:
        np.testing.assert_array_equal(Hf, H)  # SP -> TP gather restores H exactly
        np.testing.assert_array_equal(mine, np.full((15, 12), 3.0, np.float32))  # 1 + 2 summed
    # DP with equal micro-batches and mean reduction == the mean over replicas
    l0 = ob.forward(H[:15], W, Y[:15], "mean")[2]
    l1 = ob.forward(H[15:], W, Y[15:], "mean")[2]
    assert abs(res[0][3] - (l0 + l1) / 2) < 1e-6 and res[0][3] == res[1][3]
    np.testing.assert_array_equal(res[0][4], res[1][4])  # every rank holds the same averaged dW
