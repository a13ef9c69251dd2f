"""Seeded synthetic inputs shared by the oracle-side tests and the CUDA path.

This module holds NO arithmetic of the method (no kernels, distances, reductions): only point
clouds, signals and the configuration table (BASELINE.json ``configs``) as shapes and seeds.
Recipe: SURVEY.md Sec. 8(d) "Synthetic generators", restated in DESIGN.md Sec. 5.

All generators draw in fp64 with numpy ``default_rng(seed)`` (PCG64) and return fp32 arrays.
"""
from .inputs import (  # noqa: F401
    CONFIGS, Config, config, seeds,
    uniform3, uniform3_rows, signal_rows, gmm3, signal, cotangent, mnist784, lattice_nodes, points,
)
