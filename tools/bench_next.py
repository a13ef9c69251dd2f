"""Measurements for the SURVEY.md 8(f) rows built on the kernels (one JSON line per item).

Not the driver's bench (bench.py measures the BASELINE.json metric); these put numbers next to
the 'next' rows: autograd backward of the Gaussian Sum, LSE backward, block-sparse ranges, kernel
CG solve and k-means.  CUDA-event timing after warm-up; synthetic seeded inputs.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_11127_b200 import genred, solvers  # noqa: E402
from paper_2004_11127_b200.autograd import gauss_sum, logsumexp  # noqa: E402


def timed(fn, reps=3, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def main():
    lines = []
    # 1. Gaussian Sum forward + backward in x, y, b (3 Genred launches: fwd, gradx, fused swapped)
    M = N = 100_000
    x = dev(synth.uniform3(M, 1)).requires_grad_(True); y = dev(synth.uniform3(N, 2)).requires_grad_(True)
    b = dev(synth.signal(N, 3)).requires_grad_(True); g = dev(synth.cotangent(M, 4))

    def fb():
        a = gauss_sum(x, y, b, 0.5)
        a.backward(g)
        return a
    ms, _ = timed(fb)
    lines.append({"item": "8(f)1 autograd Gaussian Sum fwd+bwd (x, y, b)", "M": M, "N": N, "ms": ms,
                  "pair_evals_per_s": 3 * M * N / (ms * 1e-3), "launches_per_step": "fwd + gradx + fused(swapped)"})
    # 2. LSE forward + backward (C3 shape)
    M = N = 1_000_000
    x = dev(synth.uniform3(M, 1003)).requires_grad_(True); y = dev(synth.gmm3(N, 2003)).requires_grad_(True)
    h = torch.zeros(N, device="cuda", requires_grad=True); gg = torch.ones(M, dtype=torch.float64, device="cuda")

    def lb():
        a = logsumexp(x, y, h, 0.05)
        a.backward(gg)
        return a
    ms, _ = timed(lb, reps=2, warm=1)
    lines.append({"item": "8(f)2 LSE fwd+bwd (x, y, h), C3 shape", "M": M, "N": N, "ms": ms,
                  "pair_evals_per_s": 3 * M * N / (ms * 1e-3)})
    # 3. block-sparse ranges vs dense on clustered points
    rng = np.random.default_rng(7)
    C, per = 1000, 1000
    cen = rng.uniform(0, 1, (C, 3))
    pts = np.concatenate([cen[c] + 0.01 * rng.standard_normal((per, 3)) for c in range(C)]).astype(np.float32)
    bounds = np.arange(C + 1) * per
    sigma, thr = 0.02, 0.1
    ri, sl, rj = [], [], []
    for c in range(C):
        ri.append((bounds[c], bounds[c + 1]))
        near = np.nonzero(np.linalg.norm(cen - cen[c], axis=1) < thr)[0]
        rj.extend((bounds[k], bounds[k + 1]) for k in near)
        sl.append(len(rj))
    ranges = (np.array(ri, np.int64), np.array(sl, np.int64), np.array(rj, np.int64))
    admissible = sum((e - s) for s, e in rj) * per
    P = dev(pts); B = dev(synth.signal(len(pts), 5))
    ms_s, a_s = timed(lambda: genred.eval("gauss", "sum", P, P, B, scale=sigma, ranges=ranges), reps=3)
    ms_d, a_d = timed(lambda: genred.eval("gauss", "sum", P, P, B, scale=sigma), reps=2, warm=1)
    rel = (torch.abs(a_s - a_d).max() / a_d.abs().max()).item()
    lines.append({"item": "8(f)3 block-sparse ranges, 1e6 clustered points", "clusters": C,
                  "admissible_pair_fraction": admissible / len(pts) ** 2, "ms_ranges": ms_s, "ms_dense": ms_d,
                  "speedup": ms_d / ms_s, "admissible_pairs_per_s": admissible / (ms_s * 1e-3),
                  "max_rel_diff_vs_dense": rel})
    # 4. kernel CG solve
    N = 100_000
    p = dev(synth.uniform3(N, 11)); rhs = dev(synth.signal(N, 12, signed=True)[:, 0])
    solvers.gauss_cg(p, rhs, 0.05, 0.1, tol=1e-6, max_iter=3)                 # warm-up (plan, scratch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    xs, info = solvers.gauss_cg(p, rhs, 0.05, 0.1, tol=1e-6, max_iter=1000)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    lines.append({"item": "8(f)4 CG (K + 0.1 I) x = b, Gaussian sigma=0.05", "N": N, "ms": ms,
                  "iterations": info["iterations"], "rel_residual": info["rel_residual"],
                  "ms_per_iteration": ms / max(info["iterations"], 1)})
    solvers.gauss_cg(p, rhs, 0.05, 0.1, tol=1e-6, max_iter=16, graph=True)      # capture warm-up
    torch.cuda.synchronize()
    e0.record()
    xg, ginfo = solvers.gauss_cg(p, rhs, 0.05, 0.1, tol=1e-6, max_iter=1000, graph=True)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    lines.append({"item": "8(f)4 CG as above, one iteration captured in a CUDA graph", "N": N, "ms": ms,
                  "iterations": ginfo["iterations"], "rel_residual": ginfo["rel_residual"],
                  "ms_per_iteration": ms / max(ginfo["iterations"], 1),
                  "bitwise_equal_to_eager": bool(torch.equal(xg, xs))})
    # 5. k-means
    N, k = 1_000_000, 1000
    xk = dev(synth.gmm3(N, 13))
    solvers.kmeans(xk, k, iters=1)                                             # warm-up (plan, scratch)
    torch.cuda.synchronize()
    e0.record()
    labels, c, hist = solvers.kmeans(xk, k, iters=10)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    lines.append({"item": "8(f)4 k-means N=1e6 D=3 k=1000, 10 Lloyd iterations", "ms": ms,
                  "ms_per_iteration": ms / 10, "objective_first_last": [hist[0], hist[-1]],
                  "assign_pairs_per_s": N * k * 10 / (ms * 1e-3)})
    for l in lines:
        print(json.dumps(l), flush=True)


if __name__ == "__main__":
    main()
