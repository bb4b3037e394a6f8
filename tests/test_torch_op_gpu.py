"""The PyTorch autograd op over the C-ABI against a plain PyTorch fp32 reference."""
import numpy as np
import pytest
import torch

import paper_2511_17599_b200 as fce
from paper_2511_17599_b200.torch_op import canonical_linear_cross_entropy, fused_linear_cross_entropy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("reduction,ign", [("mean", None), ("sum", -100), ("none", -100)])
def test_autograd_matches_torch_fp32(cuda, reduction, ign):
    H, W, Y = fce.generate_instance(300, 136, 2000, 11, -100, 0.2 if ign is not None else 0.0)
    H = H.clone().requires_grad_(True)
    W = W.clone().requires_grad_(True)
    loss = fused_linear_cross_entropy(H, W, Y, reduction, ign)
    g = torch.linspace(0.5, 1.5, 300, device="cuda") if reduction == "none" else torch.tensor(1.0, device="cuda")
    loss.backward(g)
    Hr = H.detach().float().requires_grad_(True)
    Wr = W.detach().float().requires_grad_(True)
    ref = canonical_linear_cross_entropy(Hr, Wr, Y, reduction, ign)
    ref.backward(g)
    assert torch.allclose(loss.float(), ref, rtol=1e-3, atol=1e-5)
    for got, exp in ((H.grad, Hr.grad), (W.grad, Wr.grad)):
        err = ((got.float() - exp).abs().max() / exp.abs().max()).item()
        assert err < 2e-2, err  # bf16 gradient storage + bf16 G


def test_no_nxv_allocation(cuda):
    """Peak memory of fwd+bwd stays far below the N x V logits (fp32)."""
    n, d, v = 4096, 1024, 65536
    h = fce.Handle(0)
    H, W, Y = fce.generate_instance(n, d, v, 3, handle=h)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    out = fce.fused_forward(H, W, Y, handle=h)
    dh, dw = fce.fused_backward_recompute(H, W, Y, out.stats, handle=h)
    torch.cuda.synchronize()
    extra = torch.cuda.max_memory_allocated() - base
    ws = h.workspace_bytes()[1]
    nxv = n * v * 4
    # outputs dH + dW (fp32) dominate; the library's own scratch is ~1/30 of N x V
    assert ws < nxv / 8, (ws, nxv)
    assert extra - dh.numel() * 4 - dw.numel() * 4 < nxv / 8, (extra, nxv)
    h.close()


def test_custom_op_registration_opcheck(cuda):
    """fce::lce_forward / fce::lce_backward pass torch.library.opcheck (schema,
    fake kernels, autograd registration)."""
    from paper_2511_17599_b200.torch_op import lce_backward, lce_forward
    H, W, Y = fce.generate_instance(200, 72, 900, 13, -100, 0.2)
    H = H.clone().requires_grad_(True)
    W = W.clone().requires_grad_(True)
    torch.library.opcheck(lce_forward, (H, W, Y, 0, -100, True))
    loss, m, a, z, f = lce_forward(H.detach(), W.detach(), Y, 0, -100, True)
    torch.library.opcheck(lce_backward, (H.detach(), W.detach(), Y, m, a, z, f, torch.tensor(1.0, device="cuda"),
                                         0, -100, True, True, True))


def test_torch_compile_traces_the_op(cuda):
    """A compiled training step keeps the op as one opaque call and matches eager."""
    H, W, Y = fce.generate_instance(256, 128, 3000, 17, -100, 0.1)

    def step(h, w, y):
        return fused_linear_cross_entropy(h, w, y, "mean", -100) * 2.0

    compiled = torch.compile(step, backend="aot_eager", fullgraph=True)
    outs = []
    for fn in (step, compiled):
        h = H.clone().requires_grad_(True)
        w = W.clone().requires_grad_(True)
        loss = fn(h, w, Y)
        loss.backward()
        outs.append((loss.detach(), h.grad, w.grad))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_loss_module_with_batch_dims(cuda):
    """FusedLinearCrossEntropyLoss on [B, T, D] hidden states matches the
    canonical torch loss (ignore_index -100) and trains an lm_head."""
    from paper_2511_17599_b200.torch_op import FusedLinearCrossEntropyLoss
    torch.manual_seed(0)
    B, T, D, V = 3, 70, 96, 1500
    hidden = (torch.randn(B, T, D, device="cuda") / D ** 0.5).to(torch.bfloat16).requires_grad_(True)
    head = torch.nn.Linear(D, V, bias=False, device="cuda", dtype=torch.bfloat16)
    targets = torch.randint(0, V, (B, T), device="cuda")
    targets[:, :10] = -100
    loss = FusedLinearCrossEntropyLoss()(hidden, head.weight, targets)
    loss.backward()
    ref = canonical_linear_cross_entropy(hidden.detach().float().reshape(-1, D), head.weight.detach().float(),
                                         targets.reshape(-1), "mean", -100)
    assert abs(loss.item() - ref.item()) <= 1e-3 * abs(ref.item())
    assert head.weight.grad is not None and head.weight.grad.dtype == torch.bfloat16
    assert hidden.grad.shape == (B, T, D)
    per_tok = FusedLinearCrossEntropyLoss("none")(hidden.detach(), head.weight.detach(), targets)
    assert per_tok.shape == (B, T) and torch.all(per_tok[:, :10] == 0)


def test_autograd_step_is_cuda_graph_capturable(cuda):
    """loss.backward() through the custom op inside torch.cuda.graph: the scalar
    upstream is read on the device (fce_backward_dev), so with validation off
    the whole autograd step is stream-ordered and replays with new inputs."""
    import paper_2511_17599_b200 as fce
    from oracle import bindings as ob
    n, d, v = 192, 136, 1500
    H, W, Y = ob.make_instance(n, d, v, 21, -100, 0.2)
    h = fce.default_handle(0)
    h.set_option("validate", 0)
    try:
        hid = torch.from_numpy(H).cuda().to(torch.bfloat16).requires_grad_()
        w = torch.from_numpy(W).cuda().to(torch.bfloat16).requires_grad_()
        y = torch.from_numpy(Y).cuda()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):  # warm-up on the capture stream (allocator, workspaces)
            for _ in range(2):
                hid.grad = w.grad = None
                loss = fused_linear_cross_entropy(hid, w, y, "mean", -100)
                loss.backward()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        hid.grad = w.grad = None
        with torch.cuda.graph(g):
            loss = fused_linear_cross_entropy(hid, w, y, "mean", -100)
            loss.backward()
        # new inputs in place, replay, compare with the oracle
        H2, W2, Y2 = ob.make_instance(n, d, v, 22, -100, 0.2)
        with torch.no_grad():
            hid.copy_(torch.from_numpy(H2).cuda().to(torch.bfloat16))
            w.copy_(torch.from_numpy(W2).cuda().to(torch.bfloat16))
            y.copy_(torch.from_numpy(Y2).cuda())
        g.replay()
        torch.cuda.synchronize()
        st, _, lred = ob.forward(H2, W2, Y2, "mean", -100)
        dH, dW = ob.backward(H2, W2, Y2, st, "mean", 1.0, -100)
        assert abs(loss.item() - lred) <= 1e-3 * abs(lred)
        gh = hid.grad.float().cpu().numpy()
        gw = w.grad.float().cpu().numpy()
        assert np.abs(gh - dH).max() / np.abs(dH).max() < 2e-2
        assert np.abs(gw - dW).max() / np.abs(dW).max() < 2e-2
    finally:
        h.set_option("validate", 1)
