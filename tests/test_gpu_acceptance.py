"""SURVEY.md 8(c) "Parity acceptance per config", at the BASELINE.json sizes, through the C ABI.

| Cfg | rows vs the oracle                        | extra full-scale checks (no oracle needed)        |
|-----|-------------------------------------------|----------------------------------------------------|
| C1  | all 1000 (b ~ U and b ~ N(0,1); U3, GMM3) | P3 on a 10x10x10 lattice                           |
| C2  | all 1e5, Sum and grad                     | P4 sum_i grad_i = 0 with y = x                      |
| C3  | seeded 4096, plain 1e-6 (fp64 output)     | all rows: LSE bounds vs the GPU's own ArgKMin;     |
|     | + fp32 output at 1e-6 + 1/2 ulp           | LSE(h = log b, eps = sigma^2) = log GaussSum      |
| C4  | seeded 2000                               | R17 certificate: rare exact rescans                |
| C5  | 1024 = 8 blocks of 128 (8 shards), U3     | P3 lattice 200x200x250 as y (1e5 query rows; Sum   |
|     | and GMM3                                  | and gradient); i-shards bitwise across G=1,2,4,8   |

Closed forms (P3) are computed here in fp64 from the lattice's 1-D factors (PAPER.md:166-167,
the Gaussian formula; separability of exp over coordinates) -- not by the oracle, and not by
the GPU.  Bars: R4 <= 1e-5 (Sum/gradient), 1e-6 absolute (LSE), R8 (ArgKMin); no conditioning
floor anywhere in this file (the benchmark workloads keep the plain bars).
"""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.parity import SUM_TOL, LSE_TOL, argk_check, assert_lse_parity, assert_sum_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

LOG2E = 1.4426950408889634


@pytest.fixture(scope="module")
def G():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2004_11127_b200 import genred
    genred.context(0)
    return genred


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.detach().cpu().numpy()


def shard_rows(M, G_, per, seed):
    """`per` seeded rows from each of the G_ contiguous i-shards of bench.py's partition
    (dist.shard_range on the 1024-row tile, 8(e))."""
    from paper_2004_11127_b200.dist import ISHARD_ALIGN, shard_range
    rng = np.random.default_rng(seed)
    out = []
    for r in range(G_):
        lo, hi = shard_range(M, G_, r, align=ISHARD_ALIGN)
        out.append(np.sort(rng.choice(np.arange(lo, hi), size=per, replace=False)))
    return np.concatenate(out)


# ---- separable lattices (P3) -----------------------------------------------------------------

def lattice(shape, lo=0.0, hi=1.0, seed=5):
    """y on a tensor grid (fp32 nodes), separable dyadic weights b_j = prod_d w_d(k_d) (exact in
    fp32, so b carries no rounding) and separable biases h_j = sum_d h_d(k_d)."""
    rng = np.random.default_rng(seed)
    nodes = [np.linspace(lo, hi, n).astype(np.float32).astype(np.float64) for n in shape]
    w = [rng.choice([0.25, 0.5, 1.0, 2.0], size=n) for n in shape]
    hd = [rng.choice([-0.5, -0.25, 0.0, 0.25, 0.5], size=n) for n in shape]
    grids = np.meshgrid(*nodes, indexing="ij")
    y = np.stack([g.reshape(-1) for g in grids], 1).astype(np.float32)
    wg = np.meshgrid(*w, indexing="ij")
    b = np.prod(np.stack([g.reshape(-1) for g in wg], 1), axis=1).astype(np.float32)
    hg = np.meshgrid(*hd, indexing="ij")
    h = np.sum(np.stack([g.reshape(-1) for g in hg], 1), axis=1).astype(np.float32)
    return nodes, w, hd, y, b.reshape(-1, 1), h


def lattice_gauss(x, nodes, w, sigma):
    """a_i = prod_d S_d, S_d = sum_k w_d(k) e^{-(x_id - g_dk)^2 / sigma^2}; the gradient's d-th
    component replaces S_d by T_d = sum_k w_d(k) (-2/sigma^2)(x_id - g_dk) e^{...}, and its R4
    denominator by |T|_d (|x - g| in place of (x - g))."""
    X = x.astype(np.float64)
    s2 = sigma * sigma
    S, T, Ta = [], [], []
    for d in range(X.shape[1]):
        diff = X[:, d:d + 1] - nodes[d][None, :]
        e = w[d][None, :] * np.exp(-diff * diff / s2)
        S.append(e.sum(1)); T.append(((-2.0 / s2) * diff * e).sum(1)); Ta.append(((2.0 / s2) * np.abs(diff) * e).sum(1))
    S, T, Ta = np.stack(S, 1), np.stack(T, 1), np.stack(Ta, 1)
    a = S.prod(1)
    rest = np.stack([np.prod(np.delete(S, d, axis=1), axis=1) for d in range(X.shape[1])], 1)
    return a, T * rest, Ta * rest


def lattice_lse(x, nodes, hd, eps):
    """LSE_i = sum_d log sum_k exp(-(x_id - g_dk)^2/eps + h_d(k)) (max-shifted per axis)."""
    X = x.astype(np.float64)
    tot = np.zeros(X.shape[0])
    for d in range(X.shape[1]):
        F = -(X[:, d:d + 1] - nodes[d][None, :]) ** 2 / eps + hd[d][None, :]
        m = F.max(1)
        tot += m + np.log(np.exp(F - m[:, None]).sum(1))
    return tot


# ---- C1 ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("dist", ["U3", "GMM3"])
@pytest.mark.parametrize("signed", [False, True])
def test_c1_all_rows(G, dist, signed):
    c = synth.config(1); sd = synth.seeds(1)
    x = synth.points(dist, c.M, sd["x"]); y = synth.points(dist, c.N, sd["y"])
    b = synth.signal(c.N, sd["b"], signed=signed)
    a = G.eval("gauss", "sum", dev(x), dev(y), dev(b), scale=c.scale)
    o, den = oracle.gauss_sum(x, y, b, sigma=c.scale)
    assert_sum_parity(host(a), o, den, what=f"C1 {dist} signed={signed} (all rows)")


def test_c1_lattice_10x10x10(G):
    """P3 at C1's size: y = a 10x10x10 lattice over [0,1]^3, all 1000 rows of C1's x."""
    c = synth.config(1); sd = synth.seeds(1)
    nodes, w, _, y, b, _ = lattice((10, 10, 10))
    x = synth.uniform3(c.M, sd["x"])
    a_cf, G_cf, Gden_cf = lattice_gauss(x, nodes, w, c.scale)
    a = host(G.eval("gauss", "sum", dev(x), dev(y), dev(b), scale=c.scale, out_dtype="float64"))
    assert_sum_parity(a[:, 0], a_cf, a_cf, what="C1 lattice sum")
    gr = host(G.eval("gauss_gradx", "sum", dev(x), dev(y), dev(b), scale=c.scale, out_dtype="float64"))
    assert_sum_parity(gr, G_cf, Gden_cf, what="C1 lattice grad")


# ---- C2 ---------------------------------------------------------------------------------------

def test_c2_all_rows_sum_and_grad(G):
    c = synth.config(2); sd = synth.seeds(2)
    x = synth.uniform3(c.M, sd["x"]); y = synth.uniform3(c.N, sd["y"]); b = synth.signal(c.N, sd["b"])
    s, gr = G.eval("gauss_sum_gradx", "sum", dev(x), dev(y), dev(b), None, scale=c.scale)
    os_, dens = oracle.gauss_sum(x, y, b, sigma=c.scale)
    og, deng = oracle.gauss_gradx(x, y, b, None, sigma=c.scale)
    assert_sum_parity(host(s), os_, dens, what="C2 sum (all rows, fused)")
    assert_sum_parity(host(gr), og, deng, what="C2 grad (all rows, fused)")
    # the separate kernels (GAUSS, GAUSS_GRADX) on the same inputs
    s2 = G.eval("gauss", "sum", dev(x), dev(y), dev(b), scale=c.scale)
    g2 = G.eval("gauss_gradx", "sum", dev(x), dev(y), dev(b), scale=c.scale)
    assert_sum_parity(host(s2), os_, dens, what="C2 sum (all rows, separate)")
    assert_sum_parity(host(g2), og, deng, what="C2 grad (all rows, separate)")


def test_c2_gradient_sums_to_zero_when_y_is_x(G):
    """P4 antisymmetry at C2's size: y = x, b = g = 1 -> sum_i G_i = 0 exactly (term_ij =
    -term_ji).  By R4 each row errs by <= 1e-5 S_i, so |sum_i G_i| <= 1e-5 sum_i S_i; the
    denominators S_i = sum_j |term_ij| come from the oracle."""
    c = synth.config(2); sd = synth.seeds(2)
    x = synth.uniform3(c.M, sd["x"])
    for formula in ("gauss_gradx", "gauss_sum_gradx"):
        res = G.eval(formula, "sum", dev(x), dev(x), None, None, scale=c.scale, out_dtype="float64")
        gr = host(res[1] if isinstance(res, tuple) else res).astype(np.float64)
        if formula == "gauss_gradx":
            _, den = oracle.gauss_gradx(x, x, None, None, sigma=c.scale)
            S = den.sum(0)
        tot = gr.sum(0)
        assert np.all(np.abs(tot) <= SUM_TOL * S), (formula, tot / S)


# ---- C3 ---------------------------------------------------------------------------------------

def _c3():
    c = synth.config(3); sd = synth.seeds(3)
    return c, synth.uniform3(c.M, sd["x"]), synth.gmm3(c.N, sd["y"])


def test_c3_4096_rows_plain_bar_and_f32_output(G):
    c, x, y = _c3()
    rows = np.sort(np.random.default_rng(8).choice(c.M, size=4096, replace=False))
    o, _ = oracle.lse(x, y, None, eps=c.scale, rows=rows)
    a = host(G.eval("sqdist", "lse", dev(x), dev(y), None, scale=c.scale, out_dtype="float64"))
    assert_lse_parity(a[rows], o, what="C3 lse fp64 (4096 rows, plain 1e-6)")
    a32 = host(G.eval("sqdist", "lse", dev(x), dev(y), None, scale=c.scale, out_dtype="float32"))
    assert a32.dtype == np.float32
    assert_lse_parity(a32[rows], o, half_ulp_f32=True, what="C3 lse fp32 (1e-6 + 1/2 ulp)")
    # all rows: max_j F <= LSE <= max_j F + log N, max_j F from the GPU's own ArgKMin K = 1
    d, _ = G.eval("sqdist", "argkmin", dev(x), dev(y), K=1)
    fmax = -host(d)[:, 0].astype(np.float64) / c.scale
    assert np.all(a >= fmax - 1e-5) and np.all(a <= fmax + math.log(c.N) + 1e-5)


def test_c3_lse_of_log_b_is_log_gauss_sum(G):
    """P4 cross-path check on all 1e6 rows: LSE with h = log b and eps = sigma^2 equals
    log(GaussSum(b)) (b > 0).  Bars: LSE within 1e-6, GaussSum within 1e-5 relative (R4 with
    b > 0), so |LSE - log Sum| <= 1e-6 - log(1 - 1e-5)."""
    c, x, y = _c3()
    b = synth.signal(c.N, synth.seeds(3)["b"])
    b = np.maximum(b, np.float32(1e-6))                       # log b finite
    h = np.log(b.astype(np.float64)).astype(np.float32)
    bh = np.exp(h.astype(np.float64)).astype(np.float32)      # b as the LSE sees it (fp32 h)
    sigma = math.sqrt(c.scale)
    lse = host(G.eval("sqdist", "lse", dev(x), dev(y), dev(h), scale=c.scale, out_dtype="float64"))
    gs = host(G.eval("gauss", "sum", dev(x), dev(y), dev(bh.reshape(-1, 1)), scale=sigma, out_dtype="float64"))[:, 0]
    err = np.abs(lse - np.log(gs))
    assert err.max() <= LSE_TOL - math.log1p(-SUM_TOL), err.max()


def test_c3_lattice_lse(G):
    """P3 for the LSE at C3's size: y = a 100x100x100 lattice (1e6 points), 1e5 query rows, h
    separable (dyadic per-axis biases) or zero; LSE = sum_d log sum_k exp(...) in fp64."""
    c, x, _ = _c3()
    nodes, _, hd, y, _, h = lattice((100, 100, 100), 0.0, 1.0, seed=17)
    xq = x[:100_000]
    for with_h in (False, True):
        hh = hd if with_h else [np.zeros_like(v) for v in hd]
        cf = lattice_lse(xq, nodes, hh, c.scale)
        a = host(G.eval("sqdist", "lse", dev(xq), dev(y), dev(h) if with_h else None, scale=c.scale,
                        out_dtype="float64"))
        assert_lse_parity(a, cf, what=f"C3 lattice lse h={with_h}")


# ---- C4 ---------------------------------------------------------------------------------------

def test_c4_2000_rows(G):
    c = synth.config(4); sd = synth.seeds(4)
    x = synth.mnist784(c.M, sd["x"]); y = synth.mnist784(c.N, sd["y"])
    d, j = G.eval("sqdist", "argkmin", dev(x), dev(y), K=c.K)
    plan = G.last_plan()
    assert plan["path"] == 1 and 0 <= plan["fallback_rows"] <= c.M // 100   # R17: rare rescans
    rows = np.sort(np.random.default_rng(10).choice(c.M, size=2000, replace=False))
    od, oj = oracle.argkmin(x, y, c.K + 1, rows=rows)
    n_idx, n_dist = argk_check(host(d)[rows], host(j)[rows], od, oj, c.K, what="C4 (2000 rows)")
    assert n_idx >= 0.95 * len(rows) * c.K


# ---- C5 ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("dist", ["U3", "GMM3"])
def test_c5_1024_rows_over_8_shards(G, dist):
    c = synth.config(5); sd = synth.seeds(5)
    x = synth.points(dist, c.M, sd["x"]); y = synth.points(dist, c.N, sd["y"]); b = synth.signal(c.N, sd["b"])
    a = host(G.eval("gauss", "sum", dev(x), dev(y), dev(b), scale=c.scale))
    rows = shard_rows(c.M, 8, 128, 9)
    o, den = oracle.gauss_sum(x, y, b, sigma=c.scale, rows=rows)
    assert_sum_parity(a[rows], o, den, what=f"C5 {dist} (1024 rows, 8 shards x 128)")


def test_c5_lattice_200x200x250(G):
    """P3 at C5's N: y = a 200x200x250 lattice (N = 1e7) over [0,1]^3, 1e5 query rows of C5's x;
    the Gaussian Sum and its x-gradient against the separable closed forms (all rows)."""
    c = synth.config(5); sd = synth.seeds(5)
    nodes, w, _, y, b, _ = lattice((200, 200, 250), seed=21)
    assert y.shape[0] == c.N
    x = synth.uniform3(100_000, sd["x"])
    a_cf, G_cf, Gden_cf = lattice_gauss(x, nodes, w, c.scale)
    a = host(G.eval("gauss", "sum", dev(x), dev(y), dev(b), scale=c.scale, out_dtype="float64"))
    assert_sum_parity(a[:, 0], a_cf, a_cf, what="C5 lattice sum")
    gr = host(G.eval("gauss_gradx", "sum", dev(x), dev(y), dev(b), scale=c.scale, out_dtype="float64"))
    assert_sum_parity(gr, G_cf, Gden_cf, what="C5 lattice grad")


@pytest.mark.parametrize("split", [1, 3])
def test_ishard_bitwise_across_1_2_4_8(G, split):
    """8(e): with the same (forced) j-split and shard boundaries on the 1024-row tile
    (dist.ISHARD_ALIGN, as bench.py partitions) every i-shard computes its rows with exactly the
    unsharded arithmetic, so the outputs are bitwise equal for G = 1, 2, 4, 8 (each shard run as
    its own call, as a rank would)."""
    M, N = 1_000_003, 200_000
    x = synth.uniform3(M, 151); y = synth.uniform3(N, 152); b = synth.signal(N, 153)
    yd, bd = dev(y), dev(b)
    from paper_2004_11127_b200.dist import ISHARD_ALIGN, shard_range
    full = host(G.eval("gauss", "sum", dev(x), yd, bd, scale=0.5, split_j=split))
    for Gn in (2, 4, 8):
        rg = [shard_range(M, Gn, r, align=ISHARD_ALIGN) for r in range(Gn)]
        parts = [host(G.eval("gauss", "sum", dev(x[lo:hi]), yd, bd, scale=0.5, split_j=split)) for lo, hi in rg]
        np.testing.assert_array_equal(np.concatenate(parts), full, err_msg=f"G={Gn}")
    lf = host(G.eval("sqdist", "lse", dev(x[:300_000]), yd, None, scale=0.05, out_dtype="float64", split_j=split))
    for Gn in (2, 4, 8):
        rg = [shard_range(300_000, Gn, r, align=ISHARD_ALIGN) for r in range(Gn)]
        parts = [host(G.eval("sqdist", "lse", dev(x[lo:hi]), yd, None, scale=0.05, out_dtype="float64",
                             split_j=split)) for lo, hi in rg]
        np.testing.assert_array_equal(np.concatenate(parts), lf, err_msg=f"lse G={Gn}")
