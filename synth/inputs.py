"""Seeded synthetic workloads shaped like the paper's benchmarks (no method arithmetic here).

PAPER.md:182-183 (Sec. 4): "a Gaussian kernel matrix-vector product with a growing number of
points N in dimension D=3", float32.  The paper does not state the point distribution, M, E,
sigma or b; the recipe below is this build's reading:

* ``U3``    : uniform [0,1)^3.
* ``GMM3``  : 32 isotropic Gaussian components, means ~ U[0.15,0.85]^3, std 0.04, equal weights.
* signal b  : U[0,1) (default, positive) or N(0,1) (``signed``).
* cotangent g : 1 (default) or N(0,1).
* ``MNIST784``: 28x28 "digit-like" images: 10 class prototypes made of 2-4 Gaussian-blob strokes;
  each sample rolls its prototype by up to +-3 px, 70 % get one extra stroke, stroke pixels are
  scaled by U(0.6,1.4) plus N(0,0.15) noise, then clipped to [0,1] and quantised to k/255.
* ``LAT``   : tensor-product lattices (used by the closed-form pins).

Seeds for configuration c: x 1000+c, y 2000+c, b 3000+c, g 4000+c.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration (shapes and parameters only)."""
    cid: int
    name: str
    formula: str          # "gauss", "gauss_gradx", "sqdist"
    reduction: str        # "sum", "lse", "argkmin"
    M: int
    N: int
    D: int
    E: int = 1
    scale: float = 0.5    # sigma (Gaussian) or eps (LSE)
    K: int = 1
    x_dist: str = "U3"
    y_dist: str = "U3"
    extra: tuple = field(default_factory=tuple)   # e.g. ("gauss_gradx",) computed in the same step


CONFIGS = {
    1: Config(1, "C1 Gaussian Sum M=N=1000 D=3 E=1 sigma=0.5", "gauss", "sum", 1000, 1000, 3, 1, 0.5),
    2: Config(2, "C2 Gaussian Sum + grad_x M=N=1e5 D=3 E=1 sigma=0.5", "gauss", "sum",
              100_000, 100_000, 3, 1, 0.5, extra=("gauss_gradx",)),
    3: Config(3, "C3 LSE softmin M=N=1e6 D=3 eps=0.05", "sqdist", "lse", 1_000_000, 1_000_000, 3, 1,
              0.05, x_dist="U3", y_dist="GMM3"),
    4: Config(4, "C4 ArgKMin K=10 M=1e4 N=6e4 D=784", "sqdist", "argkmin", 10_000, 60_000, 784, 1,
              1.0, K=10, x_dist="MNIST784", y_dist="MNIST784"),
    5: Config(5, "C5 Gaussian Sum M=N=1e7 D=3 E=1 sigma=0.5 (i-sharded 1/2/4/8)", "gauss", "sum",
              10_000_000, 10_000_000, 3, 1, 0.5),
    # Cedge: the memory-bound low-N, high-M edge; N in {1, 2, 4, 8, 16, 32}
    6: Config(6, "Cedge Gaussian Sum M=2^28 N=8 D=3 E=1 sigma=0.5 (HBM-bound)", "gauss", "sum",
              1 << 28, 8, 3, 1, 0.5),
    # the north star's "gradient form" alone: C2's shape with the x-gradient only (GAUSS_GRADX)
    9: Config(9, "C2g Gaussian grad_x only M=N=1e5 D=3 E=1 sigma=0.5", "gauss_gradx", "sum",
              100_000, 100_000, 3, 1, 0.5),
    # the j-shard regime of SURVEY.md 8(e) (M << N; north star (d)): y, b sharded over ranks
    7: Config(7, "Cj Gaussian Sum M=1e4 N=1e8 D=3 E=1 sigma=0.5 (j-sharded)", "gauss", "sum",
              10_000, 100_000_000, 3, 1, 0.5),
    8: Config(8, "Cj LSE M=1e4 N=1e8 D=3 eps=0.05 (j-sharded)", "sqdist", "lse",
              10_000, 100_000_000, 3, 1, 0.05),
}


def config(cid: int) -> Config:
    return CONFIGS[cid]


def seeds(cid: int) -> dict:
    return {"x": 1000 + cid, "y": 2000 + cid, "b": 3000 + cid, "g": 4000 + cid}


def uniform3(n: int, seed: int, D: int = 3) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.random((n, D)).astype(np.float32)


def uniform3_rows(n: int, seed: int, lo: int, hi: int, D: int = 3) -> np.ndarray:
    """Rows [lo, hi) of uniform3(n, seed, D), drawn without generating the others (PCG64
    advance: each float64 consumes one 64-bit output), so a j-shard makes only its slice."""
    assert 0 <= lo <= hi <= n
    rng = np.random.default_rng(seed)
    rng.bit_generator.advance(lo * D)
    return rng.random((hi - lo, D)).astype(np.float32)


def signal_rows(n: int, seed: int, lo: int, hi: int, E: int = 1) -> np.ndarray:
    """Rows [lo, hi) of signal(n, seed, E) (the U[0,1) signal), as uniform3_rows."""
    return uniform3_rows(n, seed, lo, hi, E)


def gmm3(n: int, seed: int, D: int = 3, ncomp: int = 32, std: float = 0.04) -> np.ndarray:
    rng = np.random.default_rng(seed)
    means = rng.uniform(0.15, 0.85, size=(ncomp, D))
    comp = rng.integers(0, ncomp, size=n)
    pts = means[comp] + std * rng.standard_normal((n, D))
    return pts.astype(np.float32)


def signal(n: int, seed: int, E: int = 1, signed: bool = False) -> np.ndarray:
    rng = np.random.default_rng(seed)
    v = rng.standard_normal((n, E)) if signed else rng.random((n, E))
    return v.astype(np.float32)


def cotangent(n: int, seed: int | None, E: int = 1) -> np.ndarray:
    if seed is None:
        return np.ones((n, E), dtype=np.float32)
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, E)).astype(np.float32)


def _stroke_image(rng, npts: int = None) -> np.ndarray:
    """One random Gaussian-blob stroke (a polyline of 2-3 segments) on a 28x28 canvas."""
    yy, xx = np.mgrid[0:28, 0:28].astype(np.float64)
    npts = npts or int(rng.integers(2, 4))
    ctrl = rng.uniform(5.0, 23.0, size=(npts + 1, 2))
    width = rng.uniform(0.9, 1.4)
    img = np.zeros((28, 28))
    for a, b in zip(ctrl[:-1], ctrl[1:]):
        ab = b - a
        t = ((yy - a[0]) * ab[0] + (xx - a[1]) * ab[1]) / max(ab @ ab, 1e-9)
        t = np.clip(t, 0.0, 1.0)
        dy = yy - (a[0] + t * ab[0])
        dx = xx - (a[1] + t * ab[1])
        img = np.maximum(img, np.exp(-(dy * dy + dx * dx) / (2 * width * width)))
    img[img < 0.12] = 0.0
    return img


def mnist784(n: int, seed: int, proto_seed: int = 784) -> np.ndarray:
    """MNIST-shaped synthetic images, flattened to n x 784, values k/255 in [0,1]."""
    prng = np.random.default_rng(proto_seed)          # shared class prototypes across x and y
    protos = []
    for _ in range(10):
        img = np.zeros((28, 28))
        for _ in range(int(prng.integers(2, 5))):
            img = np.maximum(img, _stroke_image(prng))
        protos.append(img)
    protos = np.stack(protos)
    extra_bank = np.stack([_stroke_image(prng) for _ in range(256)])

    rng = np.random.default_rng(seed)
    out = np.empty((n, 784), dtype=np.float32)
    chunk = 8192
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        cls = rng.integers(0, 10, size=m)
        sy = rng.integers(-3, 4, size=m)
        sx = rng.integers(-3, 4, size=m)
        add = rng.random(m) < 0.7
        pick = rng.integers(0, extra_bank.shape[0], size=m)
        scale = rng.uniform(0.6, 1.4, size=m)
        imgs = protos[cls].copy()
        imgs = np.where(add[:, None, None], np.maximum(imgs, extra_bank[pick]), imgs)
        for k in range(m):                              # per-sample roll by (sy, sx)
            imgs[k] = np.roll(imgs[k], (sy[k], sx[k]), axis=(0, 1))
        mask = imgs > 0
        noise = 0.15 * rng.standard_normal(imgs.shape)
        imgs = np.where(mask, imgs * scale[:, None, None] + noise, 0.0)
        imgs = np.clip(imgs, 0.0, 1.0)
        imgs = np.round(imgs * 255.0) / 255.0
        out[s:s + m] = imgs.reshape(m, 784).astype(np.float32)
    return out


def lattice_nodes(shape, spacing=None, origin=None) -> list:
    """Per-axis node coordinates g_{d,k} of a tensor-product lattice, rounded to fp32."""
    spacing = spacing or [1.0] * len(shape)
    origin = origin or [0.0] * len(shape)
    return [(origin[d] + spacing[d] * np.arange(n)).astype(np.float32) for d, n in enumerate(shape)]


def points(kind: str, n: int, seed: int, D: int = 3) -> np.ndarray:
    if kind == "U3":
        return uniform3(n, seed, D)
    if kind == "GMM3":
        return gmm3(n, seed, D)
    if kind == "MNIST784":
        return mnist784(n, seed)
    raise ValueError(kind)
