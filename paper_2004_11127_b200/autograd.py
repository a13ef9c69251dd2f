"""torch.autograd integration of the Gaussian Genred Sum (Sec. 2 "Backpropagation":
"users can seamlessly backprop through KeOps calls using torch.autograd.grad() and .backward()").

Every gradient is itself a Genred call into libgenred (the derivative of a
reduction is another reduction), using the role swap of the transposed reduction (SPEC S:206,
S:389 -- SURVEY.md 8(f) row 1):

    a_i = sum_j K_ij b_j ,  K_ij = exp(-|x_i - y_j|^2 / sigma^2),  cotangent g_i:
    dL/dx_i = sum_j (-2/sigma^2)(x_i - y_j) K_ij <b_j, g_i>      = GAUSS_GRADX(x, y; b, g)
    dL/db_j = sum_i K_ij g_i                                     = GAUSS sum over i   (x <-> y, b := g)
    dL/dy_j = sum_i (-2/sigma^2)(y_j - x_i) K_ij <g_i, b_j>      = GAUSS_GRADX(y, x; g, b)

The last two come out of ONE fused GAUSS_SUM_GRADX launch on the swapped roles.  This module is
glue only (argument routing); no arithmetic of the method happens here.
"""
from __future__ import annotations

import torch

from . import genred


class GaussSum(torch.autograd.Function):
    """a = GaussSum.apply(x, y, b, sigma): x (M, D), y (N, D), b (N, E) fp32 CUDA tensors."""

    @staticmethod
    def forward(ctx, x, y, b, sigma: float):
        x, y, b = x.contiguous(), y.contiguous(), b.contiguous()
        ctx.save_for_backward(x, y, b)
        ctx.sigma = float(sigma)
        return genred.eval("gauss", "sum", x, y, b, scale=ctx.sigma)

    @staticmethod
    def backward(ctx, g):
        x, y, b = ctx.saved_tensors
        g = g.contiguous().to(torch.float32)
        gx = gy = gb = None
        if ctx.needs_input_grad[0]:
            gx = genred.eval("gauss_gradx", "sum", x, y, b, g, scale=ctx.sigma)
        if ctx.needs_input_grad[1] or ctx.needs_input_grad[2]:
            # transposed reduction: rows are the y_j, the reduced axis is i, signal g, cotangent b
            gb, gy = genred.eval("gauss_sum_gradx", "sum", y, x, g, b, scale=ctx.sigma)
        return gx, gy, gb, None


def gauss_sum(x, y, b, sigma: float):
    """Differentiable a_i = sum_j exp(-|x_i - y_j|^2 / sigma^2) b_j (all three inputs)."""
    return GaussSum.apply(x, y, b, sigma)


class LogSumExp(torch.autograd.Function):
    """a = LogSumExp.apply(x, y, h, eps): a_i = log sum_j exp(-|x_i - y_j|^2/eps + h_j) (fp64 out).

    Backward = two GENRED_LSE_GRAD reductions with the saved a as the
    max shift (softmax weights p_ij = exp(F_ij - a_i), never above 1):
        dL/dx_i = g_i sum_j p_ij (-2/eps)(x_i - y_j)            rows x, alpha = -a, beta = h
        dL/dh_j = sum_i g_i p_ij, dL/dy_j = sum_i g_i p_ij (-2/eps)(y_j - x_i)
                                                                rows y, alpha = h, beta = -a, sig = g
    """

    @staticmethod
    def forward(ctx, x, y, h, eps: float):
        x, y = x.contiguous(), y.contiguous()
        h = None if h is None else h.contiguous().to(torch.float32)
        a = genred.eval("sqdist", "lse", x, y, h, scale=float(eps), out_dtype="float64")
        ctx.save_for_backward(x, y, h if h is not None else torch.empty(0, device=x.device), a)
        ctx.has_h = h is not None
        ctx.eps = float(eps)
        return a

    @staticmethod
    def backward(ctx, g):
        x, y, h, a = ctx.saved_tensors
        h = h if ctx.has_h else None
        g32 = g.contiguous().to(torch.float32)
        neg_a = (-a).contiguous()                        # the max shift (argument marshalling)
        h64 = None if h is None else h.to(torch.float64).contiguous()
        gx = gy = gh = None
        if ctx.needs_input_grad[0]:
            _, gx = genred.eval("lse_grad", "sum", x, y, None, g32, scale=ctx.eps,
                                row_shift=neg_a, col_shift=h64)
        if ctx.needs_input_grad[1] or ctx.needs_input_grad[2]:
            gh, gy = genred.eval("lse_grad", "sum", y, x, g32, None, scale=ctx.eps,
                                 row_shift=h64, col_shift=neg_a)
        return gx, gy, (gh if ctx.has_h else None), None


def logsumexp(x, y, h, eps: float):
    """Differentiable a_i = log sum_j exp(-|x_i - y_j|^2 / eps + h_j) (in x, y and h)."""
    return LogSumExp.apply(x, y, h, eps)
