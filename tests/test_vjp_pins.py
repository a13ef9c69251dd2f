"""Pins of the transposed-reduction reading: the
gradients of the Gaussian Sum with respect to y and b are Genred reductions over i with the
roles of x and y swapped.  CPU-only: checked with the fp64 oracle by an adjoint identity and by
finite differences, so the GPU autograd path can be compared with these oracle calls."""
import numpy as np

import oracle


def _data(seed, M=13, N=17, D=3, E=2):
    rng = np.random.default_rng(seed)
    x = rng.random((M, D)); y = rng.random((N, D))
    b = rng.standard_normal((N, E)); g = rng.standard_normal((M, E))
    return x, y, b, g


def test_adjoint_identity_b():
    """<g, K b> = <K^T g, b>, with K^T g = gauss_sum(y, x, g)."""
    x, y, b, g = _data(1)
    Kb, _ = oracle.gauss_sum(x, y, b, sigma=0.4)
    KTg, _ = oracle.gauss_sum(y, x, g, sigma=0.4)
    np.testing.assert_allclose((g * Kb).sum(), (b * KTg).sum(), rtol=1e-13)


def test_y_gradient_is_swapped_gradx():
    """d/dy_j sum_i <g_i, a_i> (central differences of O1) = gauss_gradx(y, x; b=g, g=b)."""
    x, y, b, g = _data(2)
    sigma, h = 0.4, 1e-6
    Gy, den = oracle.gauss_gradx(y, x, g, b, sigma=sigma)
    for d in range(3):
        for j in range(y.shape[0]):
            yp = y.copy(); yp[j, d] += h
            ym = y.copy(); ym[j, d] -= h
            ap, _ = oracle.gauss_sum(x, yp, b, sigma=sigma)
            am, _ = oracle.gauss_sum(x, ym, b, sigma=sigma)
            fd = ((ap - am) * g).sum() / (2 * h)
            assert abs(Gy[j, d] - fd) <= 1e-7 * den[j, d] + 1e-9
