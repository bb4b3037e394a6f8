"""PyTorch caller of the fused LCE C-ABI (the paper's integration
point is the lm_head + cross-entropy of a training step).

    loss = fused_linear_cross_entropy(hidden, weight, targets, ignore_index=-100)
    loss.backward()          # dH, dW from the persistent sm_100a backward

hidden [N, D] and weight [V, D] are bf16 (or fp32 on the bf16 grid) CUDA
tensors; gradients are returned in the inputs' dtype.  No N x V tensor is ever
allocated; all arithmetic runs in libfce.so.

The forward and backward are registered as ``torch.library`` custom ops
(``fce::lce_forward`` / ``fce::lce_backward``) with fake (meta) kernels and an
autograd formula, so ``torch.compile`` traces through a model that calls them
and keeps them as opaque calls into the library (no graph break, no
re-implementation by the compiler).
"""
from __future__ import annotations

from typing import Tuple

import torch

import paper_2511_17599_b200 as fce

_RED = {"mean": 0, "sum": 1, "none": 2}
_RED_NAME = {v: k for k, v in _RED.items()}


@torch.library.custom_op("fce::lce_forward", mutates_args=())
def lce_forward(hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor, reduction: int,
                ignore_index: int, has_ignore: bool) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor,
                                                               torch.Tensor, torch.Tensor]:
    """-> (loss: 0-d (mean / sum) or [N] (none), m, a, z_target, found)."""
    out = fce.fused_forward(hidden, weight, targets, _RED_NAME[reduction],
                            ignore_index if has_ignore else None)
    st = out.stats
    return out.loss.clone() if reduction == 2 else out.loss, st.m, st.a, st.z_target, st.found


@lce_forward.register_fake
def _(hidden, weight, targets, reduction, ignore_index, has_ignore):
    n = hidden.shape[0]
    loss = hidden.new_empty((n,) if reduction == 2 else (), dtype=torch.float32)
    f32 = hidden.new_empty((n,), dtype=torch.float32)
    return loss, f32, torch.empty_like(f32), torch.empty_like(f32), hidden.new_empty((n,), dtype=torch.uint8)


@torch.library.custom_op("fce::lce_backward", mutates_args=())
def lce_backward(hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor, m: torch.Tensor,
                 a: torch.Tensor, z_target: torch.Tensor, found: torch.Tensor, grad_out: torch.Tensor,
                 reduction: int, ignore_index: int, has_ignore: bool, want_dhidden: bool,
                 want_dweight: bool) -> Tuple[torch.Tensor, torch.Tensor]:
    """-> (dH, dW) in the inputs' dtypes (empty tensors for gradients not wanted)."""
    stats = fce.Stats(m, a, z_target, found)
    if reduction == 2:
        upstream = grad_out.float().contiguous()
    else:
        # read on the device (fce_backward_dev): no host sync, CUDA-graph capturable
        upstream = grad_out.float().reshape(())
    # gradients come out of the library in the parameters' dtype (bf16 dW is
    # rounded straight from the tensor-core accumulators)
    gdt = torch.bfloat16 if weight.dtype == torch.bfloat16 else torch.float32
    dh, dw = fce.fused_backward_recompute(hidden, weight, targets, stats, _RED_NAME[reduction], upstream,
                                          ignore_index if has_ignore else None,
                                          want_dhidden=want_dhidden or not want_dweight,
                                          want_dweight=want_dweight, grad_dtype=gdt)
    dh = dh.to(hidden.dtype) if (want_dhidden and dh is not None) else hidden.new_empty((0,))
    dw = dw.to(weight.dtype) if (want_dweight and dw is not None) else weight.new_empty((0,))
    return dh, dw


@lce_backward.register_fake
def _(hidden, weight, targets, m, a, z_target, found, grad_out, reduction, ignore_index, has_ignore,
      want_dhidden, want_dweight):
    dh = torch.empty_like(hidden) if want_dhidden else hidden.new_empty((0,))
    dw = torch.empty_like(weight) if want_dweight else weight.new_empty((0,))
    return dh, dw


def _setup_context(ctx, inputs, output):
    hidden, weight, targets, reduction, ignore_index, has_ignore = inputs
    _, m, a, z, f = output
    ctx.save_for_backward(hidden, weight, targets, m, a, z, f)
    ctx.reduction = reduction
    ctx.ignore_index = ignore_index
    ctx.has_ignore = has_ignore


def _backward(ctx, grad_loss, _gm, _ga, _gz, _gf):
    hidden, weight, targets, m, a, z, f = ctx.saved_tensors
    want_h, want_w = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
    dh, dw = lce_backward(hidden, weight, targets, m, a, z, f, grad_loss, ctx.reduction, ctx.ignore_index,
                          ctx.has_ignore, want_h, want_w)
    return (dh if want_h else None), (dw if want_w else None), None, None, None, None


lce_forward.register_autograd(_backward, setup_context=_setup_context)


def fused_linear_cross_entropy(hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor,
                               reduction: str = "mean", ignore_index=None) -> torch.Tensor:
    """Loss of softmax(hidden @ weight.T) against targets without the logits."""
    if reduction not in fce.REDUCTIONS:
        raise fce.UnsupportedReduction(reduction)
    loss, *_ = lce_forward(hidden, weight, targets.to(torch.int64), _RED[reduction],
                           0 if ignore_index is None else int(ignore_index), ignore_index is not None)
    return loss


class FusedLinearCrossEntropyLoss(torch.nn.Module):
    """Drop-in for ``F.cross_entropy(hidden @ lm_head.weight.T, targets)`` in a
    training step: ``loss = FusedLinearCrossEntropyLoss()(hidden, lm_head.weight, targets)``.
    hidden may carry leading batch dims ([B, T, D] is flattened to [B*T, D])."""

    def __init__(self, reduction: str = "mean", ignore_index: int = -100):
        super().__init__()
        if reduction not in fce.REDUCTIONS:
            raise fce.UnsupportedReduction(reduction)
        self.reduction = reduction
        self.ignore_index = ignore_index

    def forward(self, hidden: torch.Tensor, weight: torch.Tensor, targets: torch.Tensor) -> torch.Tensor:
        lead = hidden.shape[:-1]
        loss = fused_linear_cross_entropy(hidden.reshape(-1, hidden.shape[-1]), weight, targets.reshape(-1),
                                          self.reduction, self.ignore_index)
        return loss.reshape(lead) if self.reduction == "none" else loss


def canonical_linear_cross_entropy(hidden, weight, targets, reduction="mean", ignore_index=None):
    """The two-stage baseline (lm_head GEMM + cross-entropy) the paper compares
    against (Table 2 "canonical"); materialises the N x V logits."""
    logits = hidden @ weight.t()
    return torch.nn.functional.cross_entropy(
        logits.float(), targets, reduction=reduction,
        ignore_index=-100 if ignore_index is None else ignore_index)
