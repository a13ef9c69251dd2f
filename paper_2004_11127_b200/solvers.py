"""Workloads on top of the Genred kernels ("k-means
clustering", "interface with the iterative linear solvers ... solve large kernel
linear systems efficiently").

* ``gauss_cg``: matrix-free conjugate gradients for (K + alpha I) x = b with K_ij =
  exp(-|p_i - p_j|^2 / sigma^2) (kernel ridge / GP / Kriging systems).  Every product K v is one
  libgenred Gaussian Sum over the same points (optionally block-sparse ``ranges``); the O(N)
  vector updates run as torch device ops (plumbing: they are not Genred reductions).
* ``kmeans``: Lloyd iterations whose assignment step is libgenred ArgKMin with K = 1 (ties to the
  lowest centroid index, R7) and whose update is a device scatter-add.
"""
from __future__ import annotations

import torch

from . import genred


def gauss_matvec(p, v, sigma: float, ranges=None):
    """K v with K_ij = exp(-|p_i - p_j|^2 / sigma^2): one Genred Sum (v: (N, E))."""
    return genred.eval("gauss", "sum", p, p, v.contiguous(), scale=sigma, ranges=ranges)


def gauss_cg(p, b, sigma: float, alpha: float, tol: float = 1e-6, max_iter: int = 500, x0=None,
             ranges=None, graph: bool = False, check_every: int = 8):
    """Solve (K + alpha I) x = b by conjugate gradients (K is SPD for distinct points, alpha > 0).

    p: (N, D) fp32 CUDA points, b: (N,) or (N, E) right-hand side.  Residual norms are tracked in
    fp64; matvecs run in libgenred (fp32 data, fp64 tile accumulation).  Returns (x, info).

    graph=True captures one CG iteration (the Genred matvec launches + the vector updates) in a
    CUDA graph and replays it, testing convergence every ``check_every`` iterations (one host
    sync per check instead of one per iteration); the arithmetic is identical."""
    if graph:
        return _gauss_cg_graph(p, b, sigma, alpha, tol, max_iter, x0, ranges, check_every)
    squeeze = b.dim() == 1
    B = (b[:, None] if squeeze else b).to(torch.float32).contiguous()
    X = torch.zeros_like(B) if x0 is None else (x0[:, None] if squeeze else x0).clone().float()
    r = B - (gauss_matvec(p, X, sigma, ranges) + alpha * X) if x0 is not None else B.clone()
    d = r.clone()
    rr = (r.double() * r.double()).sum(0)
    bnorm = torch.sqrt((B.double() * B.double()).sum(0))
    it = 0
    for it in range(1, max_iter + 1):
        Ad = gauss_matvec(p, d, sigma, ranges) + alpha * d
        step = rr / (d.double() * Ad.double()).sum(0)
        X = X + step.float() * d
        r = r - step.float() * Ad
        rr_new = (r.double() * r.double()).sum(0)
        if bool(torch.all(torch.sqrt(rr_new) <= tol * bnorm)):
            rr = rr_new
            break
        d = r + (rr_new / rr).float() * d
        rr = rr_new
    info = {"iterations": it, "rel_residual": (torch.sqrt(rr) / bnorm).max().item()}
    return (X[:, 0] if squeeze else X), info


def _gauss_cg_graph(p, b, sigma, alpha, tol, max_iter, x0, ranges, check_every):
    squeeze = b.dim() == 1
    B = (b[:, None] if squeeze else b).to(torch.float32).contiguous()
    X = torch.zeros_like(B) if x0 is None else (x0[:, None] if squeeze else x0).clone().float().contiguous()
    r = B - (gauss_matvec(p, X, sigma, ranges) + alpha * X) if x0 is not None else B.clone()
    d = r.clone()
    rr = (r.double() * r.double()).sum(0)
    bnorm = torch.sqrt((B.double() * B.double()).sum(0))
    done = torch.zeros((), dtype=torch.bool, device=B.device)

    def iteration():
        # once converged, the step and the direction update are frozen (masked), so replays
        # past convergence leave X unchanged: same result as stopping at the first hit
        Ad = gauss_matvec(p, d, sigma, ranges) + alpha * d
        step = torch.where(done, torch.zeros_like(rr), rr / (d.double() * Ad.double()).sum(0))
        X.add_(step.float() * d)
        r.sub_(step.float() * Ad)
        rr_new = (r.double() * r.double()).sum(0)
        hit = torch.all(torch.sqrt(rr_new) <= tol * bnorm)
        beta = torch.where(done | hit, torch.zeros_like(rr), rr_new / rr)
        d.mul_(beta.float()).add_(r)
        rr.copy_(torch.where(done, rr, rr_new))
        done.logical_or_(hit)

    side = torch.cuda.Stream(device=B.device)
    side.wait_stream(torch.cuda.current_stream(B.device))
    with torch.cuda.stream(side):                       # warm-up outside the capture
        state = [t.clone() for t in (X, r, d, rr, done)]
        iteration()
        for t, v in zip((X, r, d, rr, done), state):
            t.copy_(v)
    torch.cuda.current_stream(B.device).wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        iteration()
    it = 0
    while it < max_iter:
        n = min(check_every, max_iter - it)
        for _ in range(n):
            g.replay()
        it += n
        if bool(done.item()):
            break
    info = {"iterations": it, "rel_residual": (torch.sqrt(rr) / bnorm).max().item(), "graph": True,
            "converged": bool(done.item())}
    return (X[:, 0] if squeeze else X), info


def kmeans(x, k: int, iters: int = 10, init=None):
    """Lloyd's algorithm.  x: (N, D) fp32 CUDA.  Returns (labels (N,) int64, centroids (k, D),
    objective per iteration).  Assignment = libgenred ArgKMin K=1 (exact distances)."""
    N, D = x.shape
    c = (x[:k].clone() if init is None else init.clone().float()).contiguous()
    hist = []
    labels = None
    for _ in range(iters):
        d, j = genred.eval("sqdist", "argkmin", x, c, K=1)
        labels = j[:, 0]
        hist.append(float(d.double().sum().item()))
        # centroid update: deterministic segment sums (sort by label, fp64 prefix sums) instead of
        # fp64 atomics into k bins (contended and order-dependent)
        order = torch.argsort(labels, stable=True)
        counts = torch.bincount(labels, minlength=k)
        ends = torch.cumsum(counts, 0)
        xs = x[order].double().t().contiguous()                 # (D, N): scan along rows
        pref = torch.cat([torch.zeros((D, 1), dtype=torch.float64, device=x.device),
                          torch.cumsum(xs, 1)], 1)
        sums = (pref[:, ends] - pref[:, ends - counts]).t()
        keep = counts > 0
        c = torch.where(keep[:, None], (sums / counts.clamp_min(1)[:, None].double()).float(), c).contiguous()
    return labels, c, hist
