"""Pins for the fp64 oracle (oracle/genred_oracle.c) against things other than itself.

Each test names the pin (P1..P8, SURVEY.md Sec. 8(c) / DESIGN.md Sec. 4) and the paper/SPEC passage.
None of these tests re-types the oracle's formula and compares it with itself: they use closed
forms of separable lattices, invariants (antisymmetry, bounds, linearity, translation,
permutation), finite differences of a *different* oracle function, brute-force full sorts and
the worked examples in tests/golden/.
"""
import math

import numpy as np
import pytest

import oracle
import synth

# --------------------------------------------------------------------------------------------
# P1 + P2: worked examples (tests/golden/spec_worked_examples.json, each entry carries its cite)
# --------------------------------------------------------------------------------------------


def _f(v):
    return float(v) if not isinstance(v, str) else float(v.replace("inf", "inf"))


def test_golden_gauss_sum(golden):
    for ex in golden["gauss_sum"]:
        a, den = oracle.gauss_sum(np.array(ex["x"], np.float32), np.array(ex["y"], np.float32),
                                  np.array(ex["b"], np.float32), sigma=ex["sigma"])
        np.testing.assert_allclose(a, ex["expected"], rtol=1e-15, err_msg=ex["cite"])
        np.testing.assert_allclose(den, np.abs(ex["expected"]), rtol=1e-15)


def test_golden_gauss_gradx(golden):
    for ex in golden["gauss_gradx"]:
        G, _ = oracle.gauss_gradx(np.array(ex["x"], np.float32), np.array(ex["y"], np.float32),
                                  np.array(ex["b"], np.float32), np.array(ex["g"], np.float32),
                                  sigma=ex["sigma"])
        np.testing.assert_allclose(G, ex["expected"], rtol=1e-15, atol=1e-300, err_msg=ex["cite"])


def test_golden_sqdist(golden):
    for ex in golden["sqdist_sum"]:
        a, _ = oracle.sqdist_sum(np.array(ex["x"], np.float32), np.array(ex["y"], np.float32),
                                 np.array(ex["b"], np.float32))
        assert a[0, 0] == ex["expected"][0][0], ex["cite"]


def test_golden_lse(golden):
    for ex in golden["lse"]:
        y = np.array(ex["y"], np.float32).reshape(-1, 3)
        h = None if ex["h"] is None else np.array(ex["h"], np.float64)
        a, m = oracle.lse(np.array(ex["x"], np.float32), y, h, eps=ex["eps"])
        exp = [_f(v) for v in ex["expected"]]
        if math.isinf(exp[0]):
            assert a[0] == -math.inf, ex["cite"]
        else:
            np.testing.assert_allclose(a, exp, rtol=1e-15, err_msg=ex["cite"])


def test_golden_argkmin(golden):
    for ex in golden["argkmin"]:
        x = np.array(ex["x"], np.float32)
        y = np.array(ex["y"], np.float32).reshape(-1, x.shape[1])
        d, j = oracle.argkmin(x, y, ex["K"])
        assert j.tolist() == ex["expected_idx"], ex["cite"]
        np.testing.assert_array_equal(d, np.array([[_f(v) for v in r] for r in ex["expected_d"]]))


def test_single_point_all_reductions():
    """P1 (north star "a single point gives exp(0)*b"): M=N=1, x=y."""
    x = np.array([[0.3, -0.2, 0.9]], np.float32)
    b = np.array([[1.75]], np.float32)
    a, _ = oracle.gauss_sum(x, x, b, sigma=0.5)
    assert a[0, 0] == np.float64(np.float32(1.75))
    G, _ = oracle.gauss_gradx(x, x, b, None, sigma=0.5)
    assert np.all(G == 0.0)
    l, m = oracle.lse(x, x, np.array([0.625]), eps=0.05)
    assert l[0] == 0.625 and m[0] == 0.625
    d, j = oracle.argkmin(x, x, 1)
    assert d[0, 0] == 0.0 and j[0, 0] == 0


# --------------------------------------------------------------------------------------------
# P3: separable-lattice closed forms (exact products of 1-D sums)
# --------------------------------------------------------------------------------------------

def _lattice(shape, seed):
    rng = np.random.default_rng(seed)
    nodes = [np.sort(rng.uniform(-0.2, 1.2, n)).astype(np.float32).astype(np.float64) for n in shape]
    # dyadic weights / biases -> their products and sums are exact in fp32 (no rounding of b, h)
    w = [rng.choice([0.25, 0.5, 1.0, 2.0, 4.0], size=n) for n in shape]
    hd = [rng.choice([-1.0, -0.5, 0.0, 0.25, 0.75], size=n) for n in shape]
    grids = np.meshgrid(*nodes, indexing="ij")
    y = np.stack([g.reshape(-1) for g in grids], axis=1)
    wg = np.meshgrid(*w, indexing="ij")
    b = np.prod(np.stack([g.reshape(-1) for g in wg], 1), axis=1)
    hg = np.meshgrid(*hd, indexing="ij")
    h = np.sum(np.stack([g.reshape(-1) for g in hg], 1), axis=1)
    assert np.all(b.astype(np.float32) == b) and np.all(h.astype(np.float32) == h)
    return nodes, w, hd, y.astype(np.float32), b.astype(np.float32), h.astype(np.float32)


@pytest.mark.parametrize("shape,sigma", [((7, 6, 5), 0.5), ((10, 10, 10), 0.3), ((4, 9, 3), 1.7),
                                         ((13, 1, 1), 0.5)])
def test_lattice_gauss_sum_and_grad(shape, sigma):
    nodes, w, _, y, b, _ = _lattice(shape, 11)
    rng = np.random.default_rng(5)
    x = rng.uniform(-0.3, 1.3, (64, 3)).astype(np.float32)
    g = rng.standard_normal((64, 1)).astype(np.float32)
    X = x.astype(np.float64)
    s2 = sigma * sigma
    # per-axis factors S_d(x) = sum_k w_d(k) e^{-(x_d-g_dk)^2/s2},  T_d = sum_k w_d(k) (-2/s2)(x_d-g_dk) e^{...}
    S = np.stack([(w[d][None, :] * np.exp(-(X[:, d:d + 1] - nodes[d][None, :]) ** 2 / s2)).sum(1)
                  for d in range(3)], 1)
    T = np.stack([(w[d][None, :] * (-2 / s2) * (X[:, d:d + 1] - nodes[d][None, :])
                   * np.exp(-(X[:, d:d + 1] - nodes[d][None, :]) ** 2 / s2)).sum(1) for d in range(3)], 1)
    Tabs = np.stack([(w[d][None, :] * (2 / s2) * np.abs(X[:, d:d + 1] - nodes[d][None, :])
                      * np.exp(-(X[:, d:d + 1] - nodes[d][None, :]) ** 2 / s2)).sum(1) for d in range(3)], 1)
    a_cf = S.prod(1)
    a, den = oracle.gauss_sum(x, y, b, sigma=sigma)
    np.testing.assert_allclose(a[:, 0], a_cf, rtol=1e-13)
    np.testing.assert_allclose(den[:, 0], a_cf, rtol=1e-13)
    G_cf = np.stack([T[:, d] * np.prod(np.delete(S, d, axis=1), axis=1) for d in range(3)], 1) * g
    den_cf = np.stack([Tabs[:, d] * np.prod(np.delete(S, d, axis=1), axis=1) for d in range(3)], 1) * np.abs(g)
    G, gden = oracle.gauss_gradx(x, y, b, g, sigma=sigma)
    assert np.all(np.abs(G - G_cf) <= 1e-13 * den_cf + 1e-300)
    np.testing.assert_allclose(gden, den_cf, rtol=1e-13)


@pytest.mark.parametrize("shape,eps", [((7, 6, 5), 0.05), ((10, 10, 10), 0.5), ((3, 8, 6), 0.01)])
def test_lattice_lse(shape, eps):
    nodes, _, hd, y, _, h = _lattice(shape, 23)
    rng = np.random.default_rng(7)
    x = rng.uniform(-0.3, 1.3, (64, 3)).astype(np.float32)
    X = x.astype(np.float64)
    # LSE_i = sum_d log sum_k exp(-(x_d - g_dk)^2/eps + h_d(k))
    parts = []
    for d in range(3):
        F = -(X[:, d:d + 1] - nodes[d][None, :]) ** 2 / eps + hd[d][None, :]
        mx = F.max(1, keepdims=True)
        parts.append(mx[:, 0] + np.log(np.exp(F - mx).sum(1)))
    a_cf = np.sum(parts, axis=0)
    a, _ = oracle.lse(x, y, h, eps=eps)
    np.testing.assert_allclose(a, a_cf, rtol=1e-13, atol=1e-12)


@pytest.mark.parametrize("shape,sigma", [((7, 6, 5), 0.5), ((5, 5, 4), 1.1)])
def test_lattice_signed_b_denominator(shape, sigma):
    """P3 with SIGNED separable weights b_j = w1(k1) w2(k2) w3(k3), w_d(k) in +-{1/4 .. 4}:
    a_i = prod_d sum_k w_d(k) e_dk, and the R4 denominator S_i = sum_j |b_j| e_ij = prod_d
    sum_k |w_d(k)| e_dk (|prod w| = prod |w|): pins O1/O2's denominators as sums of |terms|,
    not |sum of terms| (signed terms cancel in a_i, never in S_i)."""
    rng = np.random.default_rng(31)
    nodes = [np.sort(rng.uniform(-0.2, 1.2, n)).astype(np.float32).astype(np.float64) for n in shape]
    w = [rng.choice([0.25, 0.5, 1.0, 2.0, 4.0], size=n) * rng.choice([-1.0, 1.0], size=n) for n in shape]
    for d in range(3):
        w[d][0], w[d][-1] = abs(w[d][0]), -abs(w[d][-1])        # both signs on every axis
    grids = np.meshgrid(*nodes, indexing="ij")
    y = np.stack([q.reshape(-1) for q in grids], 1).astype(np.float32)
    wg = np.meshgrid(*w, indexing="ij")
    b = np.prod(np.stack([q.reshape(-1) for q in wg], 1), axis=1).astype(np.float32)
    x = rng.uniform(-0.3, 1.3, (48, 3)).astype(np.float32)
    X = x.astype(np.float64)
    s2 = sigma * sigma
    e = [np.exp(-(X[:, d:d + 1] - nodes[d][None, :]) ** 2 / s2) for d in range(3)]
    S = np.stack([(w[d][None, :] * e[d]).sum(1) for d in range(3)], 1)
    Sabs = np.stack([(np.abs(w[d])[None, :] * e[d]).sum(1) for d in range(3)], 1)
    a, den = oracle.gauss_sum(x, y, b, sigma=sigma)
    assert np.all(np.abs(a[:, 0] - S.prod(1)) <= 1e-13 * Sabs.prod(1))
    np.testing.assert_allclose(den[:, 0], Sabs.prod(1), rtol=1e-13)
    assert np.any(np.abs(S.prod(1)) < 0.5 * Sabs.prod(1))       # the case really cancels
    # gradient: |T_d| with |w| and |x - g| in the d-th factor, |w| in the others
    Tabs = np.stack([(np.abs(w[d])[None, :] * (2 / s2) * np.abs(X[:, d:d + 1] - nodes[d][None, :])
                      * e[d]).sum(1) for d in range(3)], 1)
    G, gden = oracle.gauss_gradx(x, y, b, None, sigma=sigma)
    gden_cf = np.stack([Tabs[:, d] * np.prod(np.delete(Sabs, d, axis=1), axis=1) for d in range(3)], 1)
    np.testing.assert_allclose(gden, gden_cf, rtol=1e-13)


def test_lattice_centre_gradient_is_zero():
    """P3: x at the centre of a symmetric lattice with symmetric weights -> grad = 0."""
    g1 = np.array([-1.0, -0.5, 0.0, 0.5, 1.0], np.float32)
    grids = np.meshgrid(g1, g1, g1, indexing="ij")
    y = np.stack([q.reshape(-1) for q in grids], 1).astype(np.float32)
    x = np.zeros((1, 3), np.float32)
    G, den = oracle.gauss_gradx(x, y, None, None, sigma=0.7)
    assert np.all(np.abs(G) <= 1e-15 * den)


# --------------------------------------------------------------------------------------------
# P4: invariants
# --------------------------------------------------------------------------------------------

def test_lse_bounds():
    """North star: max_j F_ij <= LSE_i <= max_j F_ij + log N."""
    x = synth.uniform3(200, 1); y = synth.gmm3(3000, 2)
    h = np.random.default_rng(3).standard_normal(3000)
    for eps in (0.05, 0.5, 5.0):
        a, m = oracle.lse(x, y, h, eps=eps)
        assert np.all(m <= a) and np.all(a <= m + math.log(3000) + 1e-12)


def test_gradient_antisymmetry_sums_to_zero():
    """P4: y = x, b = g = 1 -> sum_i G_i = 0 (pair terms are antisymmetric in (i, j))."""
    x = synth.gmm3(400, 9)
    G, den = oracle.gauss_gradx(x, x, None, None, sigma=0.5)
    tot = G.sum(0)
    assert np.all(np.abs(tot) <= 1e-13 * den.sum(0))
    assert np.max(np.abs(G)) > 1.0          # non-trivial individual rows


def test_lse_equals_log_gauss_sum():
    """P4: with eps = sigma^2 and h = log b, LSE_i = log(sum_j b_j e^{-|x-y|^2/sigma^2})."""
    rng = np.random.default_rng(4)
    x = synth.uniform3(50, 4); y = synth.uniform3(700, 5)
    h = rng.uniform(-2, 2, 700)
    b = np.exp(h)                           # fp64, passed to the oracle as fp64
    sigma = 0.37
    a, _ = oracle.lse(x, y, h, eps=sigma * sigma)
    s, _ = oracle.gauss_sum(x, y, b, sigma=sigma)
    np.testing.assert_allclose(a, np.log(s[:, 0]), rtol=0, atol=1e-13)


def test_linearity_in_b():
    x = synth.uniform3(40, 6); y = synth.uniform3(500, 7)
    rng = np.random.default_rng(8)
    b1 = rng.standard_normal((500, 2)); b2 = rng.standard_normal((500, 2)); lam = -1.7
    a1, d1 = oracle.gauss_sum(x, y, b1, sigma=0.5)
    a2, d2 = oracle.gauss_sum(x, y, b2, sigma=0.5)
    a3, _ = oracle.gauss_sum(x, y, lam * b1 + b2, sigma=0.5)
    assert np.all(np.abs(a3 - (lam * a1 + a2)) <= 1e-14 * (abs(lam) * d1 + d2))


def test_translation_and_permutation_invariance():
    rng = np.random.default_rng(10)
    x = synth.uniform3(30, 10).astype(np.float64); y = synth.uniform3(400, 11).astype(np.float64)
    b = rng.random(400); h = rng.standard_normal(400)
    t = np.array([3.25, -7.5, 0.125])
    a0, _ = oracle.gauss_sum(x, y, b, sigma=0.5)
    at, _ = oracle.gauss_sum(x + t, y + t, b, sigma=0.5)
    np.testing.assert_allclose(at, a0, rtol=1e-13)
    perm = rng.permutation(400)
    ap, _ = oracle.gauss_sum(x, y[perm], b[perm], sigma=0.5)
    np.testing.assert_allclose(ap, a0, rtol=1e-14)
    l0, _ = oracle.lse(x, y, h, eps=0.05)
    lp, _ = oracle.lse(x, y[perm], h[perm], eps=0.05)
    np.testing.assert_allclose(lp, l0, rtol=0, atol=1e-13)
    d0, j0 = oracle.argkmin(x, y, 5)
    dp, jp = oracle.argkmin(x, y[perm], 5)
    np.testing.assert_array_equal(perm[jp], j0)
    np.testing.assert_array_equal(dp, d0)


def test_row_subset_matches_full():
    x = synth.uniform3(100, 12); y = synth.uniform3(300, 13); b = synth.signal(300, 14)
    rows = np.array([97, 3, 3, 50, 0])
    a, _ = oracle.gauss_sum(x, y, b, sigma=0.5)
    ar, _ = oracle.gauss_sum(x, y, b, sigma=0.5, rows=rows)
    np.testing.assert_array_equal(ar, a[rows])
    l, _ = oracle.lse(x, y, None, eps=0.05)
    lr, _ = oracle.lse(x, y, None, eps=0.05, rows=rows)
    np.testing.assert_array_equal(lr, l[rows])
    d, j = oracle.argkmin(x, y, 4)
    dr, jr = oracle.argkmin(x, y, 4, rows=rows)
    np.testing.assert_array_equal(jr, j[rows])


def test_wide_bandwidth_limit_is_plain_sum():
    """sigma -> infinity: exp(-d^2/sigma^2) -> 1, so a_i -> sum_j b_j (textbook sum)."""
    x = synth.uniform3(5, 1); y = synth.uniform3(1000, 2); b = synth.signal(1000, 3, signed=True)
    a, _ = oracle.gauss_sum(x, y, b, sigma=1e9)
    np.testing.assert_allclose(a[:, 0], np.sum(b.astype(np.float64)), rtol=1e-12)


# --------------------------------------------------------------------------------------------
# P5: finite differences of O1 pin O2 (including the <b_j, g_i> contraction for E > 1)
# --------------------------------------------------------------------------------------------

@pytest.mark.parametrize("E", [1, 3])
def test_gradient_finite_differences(E):
    rng = np.random.default_rng(15 + E)
    M, N, D, sigma = 12, 80, 3, 0.5
    x = rng.uniform(0, 1, (M, D)); y = rng.uniform(0, 1, (N, D))
    b = rng.standard_normal((N, E)); g = rng.standard_normal((M, E))
    G, den = oracle.gauss_gradx(x, y, b, g, sigma=sigma)
    hstep = 1e-5 * sigma
    for d in range(D):
        xp = x.copy(); xp[:, d] += hstep
        xm = x.copy(); xm[:, d] -= hstep
        ap, _ = oracle.gauss_sum(xp, y, b, sigma=sigma)
        am, _ = oracle.gauss_sum(xm, y, b, sigma=sigma)
        fd = ((ap - am) * g).sum(1) / (2 * hstep)
        assert np.all(np.abs(G[:, d] - fd) <= 1e-8 * den[:, d]), (d, np.abs(G[:, d] - fd) / den[:, d])


# --------------------------------------------------------------------------------------------
# P6 + P7: ArgKMin against brute-force full sorts; ties
# --------------------------------------------------------------------------------------------

@pytest.mark.parametrize("M,N,D,K", [(8, 13, 3, 4), (5, 64, 5, 64), (6, 10, 2, 13), (4, 1, 1, 3),
                                     (3, 40, 7, 1)])
def test_argkmin_brute_force(M, N, D, K):
    rng = np.random.default_rng(M * 1000 + N)
    # coarse grid values -> many exact ties, exercising the (d, j) order
    x = rng.integers(0, 4, (M, D)).astype(np.float32)
    y = rng.integers(0, 4, (N, D)).astype(np.float32)
    d, j = oracle.argkmin(x, y, K)
    for i in range(M):
        dist = [sum((float(x[i, k]) - float(y[q, k])) ** 2 for k in range(D)) for q in range(N)]
        order = sorted(range(N), key=lambda q: (dist[q], q))[:K]
        exp_j = order + [-1] * (K - len(order))
        exp_d = [dist[q] for q in order] + [math.inf] * (K - len(order))
        assert j[i].tolist() == exp_j
        assert d[i].tolist() == exp_d


def test_argkmin_lattice_ties():
    """P7: query at a node of the 5x5x5 integer lattice: node, then its 6 unit neighbours in
    ascending j, then the d^2=2 ring starting from its lowest index."""
    g = np.arange(5, dtype=np.float32)
    grids = np.meshgrid(g, g, g, indexing="ij")
    y = np.stack([q.reshape(-1) for q in grids], 1)
    x = np.array([[2, 2, 2]], np.float32)
    d, j = oracle.argkmin(x, y, 8)
    assert j[0].tolist() == [62, 37, 57, 61, 63, 67, 87, 32]
    assert d[0].tolist() == [0, 1, 1, 1, 1, 1, 1, 2]


def test_argkmin_duplicates_lower_index_first():
    y = np.array([[0.5, 0.5, 0.5], [0.1, 0.1, 0.1], [0.5, 0.5, 0.5], [0.9, 0.9, 0.9]], np.float32)
    d, j = oracle.argkmin(np.array([[0.5, 0.5, 0.5]], np.float32), y, 3)
    assert j[0].tolist()[:2] == [0, 2]


# --------------------------------------------------------------------------------------------
# P8: SqDist Sum against its expanded closed form
# --------------------------------------------------------------------------------------------

def test_sqdist_sum_closed_form():
    rng = np.random.default_rng(17)
    x = synth.uniform3(30, 17).astype(np.float64); y = synth.gmm3(900, 18).astype(np.float64)
    b = rng.standard_normal(900)
    a, den = oracle.sqdist_sum(x, y, b)
    cf = (x * x).sum(1) * b.sum() - 2 * x @ (b[:, None] * y).sum(0) + (b * (y * y).sum(1)).sum()
    scale = (x * x).sum(1) * np.abs(b).sum() + 2 * np.abs(x) @ (np.abs(b)[:, None] * np.abs(y)).sum(0) \
        + (np.abs(b) * (y * y).sum(1)).sum()
    assert np.all(np.abs(a[:, 0] - cf) <= 1e-13 * scale)


# --------------------------------------------------------------------------------------------
# Degenerate cases (R11): N = 0 gives neutral outputs
# --------------------------------------------------------------------------------------------

def test_empty_reduction_axis():
    x = synth.uniform3(3, 1); y = np.zeros((0, 3), np.float32)
    a, _ = oracle.gauss_sum(x, y, np.zeros((0, 1), np.float32), sigma=0.5)
    assert np.all(a == 0.0)
    l, _ = oracle.lse(x, y, None, eps=0.05)
    assert np.all(l == -math.inf)
    d, j = oracle.argkmin(x, y, 2)
    assert np.all(j == -1) and np.all(d == math.inf)


# --------------------------------------------------------------------------------------------
# O6 (LSE backward): pinned by the softmax identity and finite differences
# of O3 in x, y and h
# --------------------------------------------------------------------------------------------

def test_softmax_grad_is_lse_gradient():
    rng = np.random.default_rng(31)
    M, N, D, eps = 9, 40, 3, 0.3
    x = rng.random((M, D)); y = rng.random((N, D)); h = rng.standard_normal(N)
    g = rng.standard_normal(M)
    a, _ = oracle.lse(x, y, h, eps=eps)
    S, G, dS, dG = oracle.softmax_grad(x, y, alpha=-a, beta=h, eps=eps)
    np.testing.assert_allclose(S, 1.0, rtol=1e-13)                 # softmax weights sum to 1
    step = 1e-6
    for d in range(D):                                              # d a_i / d x_i
        xp = x.copy(); xp[:, d] += step
        xm = x.copy(); xm[:, d] -= step
        fd = (oracle.lse(xp, y, h, eps=eps)[0] - oracle.lse(xm, y, h, eps=eps)[0]) / (2 * step)
        assert np.all(np.abs(G[:, d] - fd) <= 1e-7 * dG[:, d] + 1e-9)
    # transposed: d/dh_j sum_i g_i a_i = sum_i g_i p_ij ;  d/dy_j = G of the swapped call
    Sh, Gy, dSh, dGy = oracle.softmax_grad(y, x, alpha=h, beta=-a, sig=g, eps=eps)
    for j in (0, 7, 39):
        hp = h.copy(); hp[j] += step
        hm = h.copy(); hm[j] -= step
        fd = (g * (oracle.lse(x, y, hp, eps=eps)[0] - oracle.lse(x, y, hm, eps=eps)[0])).sum() / (2 * step)
        assert abs(Sh[j] - fd) <= 1e-7 * dSh[j] + 1e-9
        for d in range(D):
            yp = y.copy(); yp[j, d] += step
            ym = y.copy(); ym[j, d] -= step
            fd = (g * (oracle.lse(x, yp, h, eps=eps)[0] - oracle.lse(x, ym, h, eps=eps)[0])).sum() / (2 * step)
            assert abs(Gy[j, d] - fd) <= 1e-7 * dGy[j, d] + 1e-9


def test_lse_conditioning_closed_forms():
    """oracle_lse_cond (the R6b metric's C_i): one j gives C = |x-y|^2/eps + |h|; equal exponents
    give the plain average of the magnitudes."""
    x = np.array([[0.1, 0.2, 0.3]]); y = np.array([[0.4, 0.0, 0.3]])
    a, _, c = oracle.lse(x, y, np.array([-2.5]), eps=0.1, cond=True)
    assert abs(c[0] - (0.13 / 0.1 + 2.5)) < 1e-12
    y2 = np.array([[0.1, 0.2, 0.3], [0.1, 0.2, 0.3]])
    a, _, c = oracle.lse(x, y2, np.array([1.0, -1.0]), eps=0.1, cond=True)
    p = np.exp(np.array([1.0, -1.0]) - a[0])
    assert abs(c[0] - (p[0] * 1.0 + p[1] * 1.0)) < 1e-12


def test_gauss_conditioning_by_bandwidth_derivative():
    """oracle_gauss_cond (the R4c metric's cond, tail) against the oracle's own denominators on a
    different route: S(lam) = sum_j |b_j| exp(-lam u_ij) is the O1 denominator at sigma/sqrt(lam),
    so cond = -dS/dlam at lam = 1; the O2 denominator is lam A(lam), so cond = den - d den/dlam.
    tail = the denominator restricted to the j with u log2(e) >= 100 (a y subset)."""
    rng = np.random.default_rng(7)
    x = rng.random((9, 3)) * 2.0
    y = rng.random((40, 3)) * 2.0
    b = rng.standard_normal((40, 2))
    g = rng.standard_normal((9, 2))
    sigma, h = 0.7, 1e-5
    _, den, cond, tail = oracle.gauss_sum(x, y, b, sigma=sigma, cond=True)
    Sp = oracle.gauss_sum(x, y, b, sigma=sigma / np.sqrt(1 + h))[1]
    Sm = oracle.gauss_sum(x, y, b, sigma=sigma / np.sqrt(1 - h))[1]
    np.testing.assert_allclose(cond, -(Sp - Sm) / (2 * h), rtol=1e-6)
    assert np.all(tail == 0.0)                      # u <= 12/0.49 ~ 24 < 100 / log2(e)
    _, dg, cg, tg = oracle.gauss_gradx(x, y, b, g, sigma=sigma, cond=True)
    Ap = oracle.gauss_gradx(x, y, b, g, sigma=sigma / np.sqrt(1 + h))[1]
    Am = oracle.gauss_gradx(x, y, b, g, sigma=sigma / np.sqrt(1 - h))[1]
    np.testing.assert_allclose(cg, dg - (Ap - Am) / (2 * h), rtol=1e-6, atol=1e-12 * dg.max())
    assert np.all(tg == 0.0)
    # deep tail: y far enough that some u log2(e) >= 100 (u >= 69.3), the rest near
    sig = 0.1
    xn = x * 0.05
    yf = np.concatenate([y * 0.05, 1.5 + y * 0.05], 0)   # 40 near (u <= 3), 40 at 470 <= u <= 675
    bf = np.concatenate([b, b], 0)
    _, den2, _, tail2 = oracle.gauss_sum(xn, yf, bf, sigma=sig, cond=True)
    far = oracle.gauss_sum(xn, yf[40:], bf[40:], sigma=sig)[1]
    assert np.all(far > 0) and np.all(tail2 < 1e-200 * den2)
    np.testing.assert_array_equal(tail2, far)
    _, _, _, tgf = oracle.gauss_gradx(xn, yf, bf, g, sigma=sig, cond=True)
    np.testing.assert_array_equal(tgf, oracle.gauss_gradx(xn, yf[40:], bf[40:], g, sigma=sig)[1])
    # moderately deep: one j at u log2(e) = 110 contributes exactly its term to tail and den
    x1 = np.zeros((1, 1)); y1 = np.array([[np.sqrt(110 / 1.4426950408889634)]]); b1 = np.ones((1, 1))
    _, d1, c1, t1 = oracle.gauss_sum(x1, y1, b1, sigma=1.0, cond=True)
    assert t1[0, 0] == d1[0, 0] > 0 and np.isclose(c1[0, 0], d1[0, 0] * 110 / 1.4426950408889634)


def test_softmax_conditioning_identities():
    """oracle_softmax_cond (R4c for O6) on routes other than its own loop: with alpha = beta = 0,
    condS = -dS/dlam and condG = denG - d denG/dlam for eps -> eps/lam (O6's denominators); a
    constant alpha_i = c > 0 multiplies every term by e^c and adds c to each magnitude, so
    cond(c) = e^c (cond(0) + c den(0)); tail = the denominators over the deep-tail y subset."""
    rng = np.random.default_rng(8)
    x = rng.random((7, 2)); y = rng.random((30, 2)); sig = rng.standard_normal(30); coef = rng.standard_normal(7)
    eps, h = 0.3, 1e-5
    S, G, dS, dG, cS, cG, tS, tG = oracle.softmax_grad(x, y, sig=sig, coef=coef, eps=eps, cond=True)
    Sp, _, dSp, dGp = oracle.softmax_grad(x, y, sig=sig, coef=coef, eps=eps / (1 + h))
    Sm, _, dSm, dGm = oracle.softmax_grad(x, y, sig=sig, coef=coef, eps=eps / (1 - h))
    np.testing.assert_allclose(cS, -(dSp - dSm) / (2 * h), rtol=1e-6)
    np.testing.assert_allclose(cG, dG - (dGp - dGm) / (2 * h), rtol=1e-6, atol=1e-12 * dG.max())
    assert np.all(tS == 0) and np.all(tG == 0)
    c = 0.75
    _, _, dS1, dG1, cS1, cG1, _, _ = oracle.softmax_grad(x, y, alpha=np.full(7, c), sig=sig, coef=coef,
                                                         eps=eps, cond=True)
    np.testing.assert_allclose(cS1, np.exp(c) * (cS + c * dS), rtol=1e-12)
    np.testing.assert_allclose(cG1, np.exp(c) * (cG + c * dG), rtol=1e-12)
    beta = np.concatenate([np.zeros(15), np.full(15, -80.0)])      # second half: z log2 e <= -100
    r = oracle.softmax_grad(x, y, beta=beta, sig=sig, coef=coef, eps=eps, cond=True)
    sub = oracle.softmax_grad(x, y[15:], beta=beta[15:], sig=sig[15:], coef=coef, eps=eps)
    np.testing.assert_array_equal(r[6], sub[2])
    np.testing.assert_array_equal(r[7], sub[3])
