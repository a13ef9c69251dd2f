"""Parity metrics (DESIGN.md Sec. 3 readings R4, R6, R8) shared by the GPU tests and bench.py.

Pure comparison logic: no method arithmetic.  The expected values always come from oracle/.
"""
from __future__ import annotations

import numpy as np

SUM_TOL = 1e-5        # north star: max relative error <= 1e-5 for Sum and gradient (R4 metric)
LSE_TOL = 1e-6        # north star: <= 1e-6 absolute on LSE (fp64 output, R6)
GAP_TOL = 1e-6        # north star: index exactness required where the oracle's gap > 1e-6 (R8)

# (what, rows that passed only thanks to a conditioning floor (R4c / R6b), rows checked): every
# use of a floor is recorded and tests/conftest.py prints the totals at the end of the session.
FLOOR_LOG: list = []


def r4_error(gpu, orc, denom, floor: float = 1e-30) -> np.ndarray:
    """err = |a - o| / S with S = sum_j |term_ij| per coordinate (R4); rows with S < floor
    (complete fp32 underflow, R13) use an absolute floor."""
    gpu = np.asarray(gpu, np.float64)
    return np.abs(gpu - orc) / np.maximum(denom, floor)


def assert_sum_parity(gpu, orc, denom, tol: float = SUM_TOL, what: str = "", cond=None, D: int = 3):
    """R4: |a - o| <= tol S.  cond = (C, T) from oracle.gauss_sum / gauss_gradx(..., cond=True)
    applies reading R4c (randomized cases only; the benchmark workloads keep the plain bar):
    |a - o| <= max(tol S, (D + 6) 2^-24 C) + T -- C_i = sum_j |term_ij| u_ij bounds the effect of
    rounding each exponent u_ij by (D + 6) fp32 ulps (the D squares and their sum, s = sqrt(log2 e)
    / sigma, s^2 and the product), T_i = the terms below 2^-100 (fp32's normal range)."""
    if cond is not None:
        C, T = (np.asarray(v, np.float64) for v in cond)
        excess = np.maximum(np.abs(np.asarray(gpu, np.float64) - orc) - T, 0.0)
        scale = np.maximum(np.maximum(denom, (D + 6) * 2.0 ** -24 * C / tol), 1e-30)
        err = excess / scale
        plain = r4_error(gpu, orc, denom)
        rows_plain = plain.reshape(plain.shape[0], -1).max(1) > tol if plain.size else np.zeros(0, bool)
        FLOOR_LOG.append((what, int(rows_plain.sum()), int(rows_plain.size)))
    else:
        err = r4_error(gpu, orc, denom)
    worst = float(err.max()) if err.size else 0.0
    assert np.all(np.isfinite(np.asarray(gpu, np.float64))), f"{what}: non-finite GPU output"
    assert worst <= tol, f"{what}: max R4 error {worst:.3e} > {tol:.0e} at {np.unravel_index(err.argmax(), err.shape)}"
    return worst


def assert_lse_parity(gpu, orc, tol: float = LSE_TOL, rel: bool = False, what: str = "",
                      cond=None, D: int = 3, half_ulp_f32: bool = False):
    """|a - o| <= 1e-6 (R6).  rel=True adds the fp32 floor of reading R6b: (D + 2) 2^-24 C_i with
    C_i = sum_j p_ij (|x_i - y_j|^2/eps + |h_j|) from oracle.lse(..., cond=True) (the exponent
    magnitudes of the dominant terms, each rounded by a few ulps in fp32), or 3 2^-24 |o| when
    cond is not given; the benchmark workloads are held to the plain 1e-6 bar."""
    gpu = np.asarray(gpu, np.float64)
    both_inf = np.isneginf(gpu) & np.isneginf(orc)
    err = np.where(both_inf, 0.0, np.abs(gpu - orc))
    if half_ulp_f32:
        # fp32 output: the bar is 1e-6 + 1/2 ulp_f32(a_i) -- the rounding of the
        # exact result to fp32 alone costs up to half an ulp
        o32 = np.abs(np.where(np.isfinite(orc), orc, 0.0)).astype(np.float32)
        half_ulp = 0.5 * (np.nextafter(o32, np.float32(np.inf)) - o32).astype(np.float64)
        err = err - half_ulp
    if rel:
        mag = np.where(np.isfinite(orc), np.abs(orc), 0.0)
        if cond is not None:
            mag = np.maximum(mag, (D + 2) / 3.0 * np.asarray(cond, np.float64))
        FLOOR_LOG.append((what, int(np.sum(err > tol)), int(err.size)))
        err = err - 3.0 * 2.0 ** -24 * mag
    worst = float(err.max()) if err.size else 0.0
    assert worst <= tol, f"{what}: max |LSE error| {worst:.3e} > {tol:.0e}"
    return worst


def argk_check(gpu_d, gpu_j, orc_d_k1, orc_j_k1, K: int, gap_tol: float = GAP_TOL,
               dist_tol: float = 1e-6, what: str = ""):
    """R8: orc_* hold the oracle's K+1 best (d, j).  Position k's index must match where the
    relative gaps on both sides of it exceed gap_tol; elsewhere only the distance is checked.
    Returns (#checked index positions, #distance-only positions)."""
    gpu_d = np.asarray(gpu_d, np.float64)
    od, oj = orc_d_k1[:, :K + 1], orc_j_k1[:, :K + 1]
    M = od.shape[0]
    n_idx = n_dist = 0
    for i in range(M):
        d = od[i]
        for k in range(K):
            if oj[i, k] < 0:                       # padding (K > N)
                assert gpu_j[i, k] == -1 and np.isinf(gpu_d[i, k]), f"{what}: row {i} pad"
                continue
            lo = np.inf if k == 0 else (d[k] - d[k - 1]) / max(d[k], 1e-300)
            hi = np.inf if (k + 1 >= d.shape[0] or not np.isfinite(d[k + 1])) else \
                (d[k + 1] - d[k]) / max(d[k + 1], 1e-300)
            if lo > gap_tol and hi > gap_tol:
                assert gpu_j[i, k] == oj[i, k], f"{what}: row {i} pos {k}: j {gpu_j[i, k]} != {oj[i, k]}"
                n_idx += 1
            else:
                n_dist += 1
            assert abs(gpu_d[i, k] - d[k]) <= dist_tol * d[k] + 1e-30, \
                f"{what}: row {i} pos {k}: d {gpu_d[i, k]} vs {d[k]}"
    return n_idx, n_dist
