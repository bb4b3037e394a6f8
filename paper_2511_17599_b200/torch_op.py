"""PyTorch caller of the fused LCE C-ABI (the paper's integration
point is the lm_head + cross-entropy of a training step).

    loss = fused_linear_cross_entropy(hidden, weight, targets, ignore_index=-100)
    loss.backward()          # dH, dW from the persistent sm_100a backward

hidden [N, D] and weight [V, D] are bf16 (or fp32 on the bf16 grid) CUDA
tensors; gradients are returned in the inputs' dtype.  No N x V tensor is ever
allocated; all arithmetic runs in libfce.so.
"""
from __future__ import annotations

import torch

import paper_2511_17599_b200 as fce


class _FusedLCE(torch.autograd.Function):
    @staticmethod
    def forward(ctx, hidden, weight, targets, reduction, ignore_index):
        out = fce.fused_forward(hidden.detach(), weight.detach(), targets, reduction, ignore_index)
        ctx.save_for_backward(hidden, weight, targets, out.stats.m, out.stats.a, out.stats.z_target,
                              out.stats.found)
        ctx.reduction = reduction
        ctx.ignore_index = ignore_index
        return out.loss

    @staticmethod
    def backward(ctx, grad_out):
        hidden, weight, targets, m, a, z, f = ctx.saved_tensors
        stats = fce.Stats(m, a, z, f)
        if ctx.reduction == "none":
            upstream = grad_out.float().contiguous()
        else:
            upstream = float(grad_out.item())
        want_h, want_w = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        dh, dw = fce.fused_backward_recompute(hidden.detach(), weight.detach(), targets, stats, ctx.reduction,
                                              upstream, ctx.ignore_index, want_dhidden=want_h or not want_w,
                                              want_dweight=want_w)
        dh = dh.to(hidden.dtype) if (want_h and dh is not None) else None
        dw = dw.to(weight.dtype) if (want_w and dw is not None) else None
        return dh, dw, None, None, None


def fused_linear_cross_entropy(hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor,
                               reduction: str = "mean", ignore_index=None) -> torch.Tensor:
    """Loss of softmax(hidden @ weight.T) against targets without the logits."""
    if reduction not in fce.REDUCTIONS:
        raise fce.UnsupportedReduction(reduction)
    return _FusedLCE.apply(hidden, weight, targets, reduction, ignore_index)


def canonical_linear_cross_entropy(hidden, weight, targets, reduction="mean", ignore_index=None):
    """The two-stage baseline (lm_head GEMM + cross-entropy) the paper compares
    against (Table 2 "canonical"); materialises the N x V logits."""
    logits = hidden @ weight.t()
    return torch.nn.functional.cross_entropy(
        logits.float(), targets, reduction=reduction,
        ignore_index=-100 if ignore_index is None else ignore_index)
