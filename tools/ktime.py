"""Kernel-only timing of one Genred call shape (main kernel, CUDA events via genred_profile).

  python tools/ktime.py CASE [CASE ...]      CASE = name:formula:reduction:M:N:scale[:dist]
  e.g. fused:gauss_sum_gradx:sum:100000:100000:0.5   gradx:gauss_gradx:sum:200000:200000:0.5
       lse:sqdist:lse:1000000:1000000:0.05:gmm        direct:gauss:sum:2000000:2000000:0.05

Prints min / median main-kernel ms over 7 timed calls (3 warm-up) and pairs/clk/SM at 1965 MHz.
GENRED_LIB selects a library variant (tools/variants.sh).
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2004_11127_b200 import genred  # noqa: E402


def run(case: str) -> None:
    parts = case.split(":")
    name, formula, red, M, N, scale = parts[:6]
    dist = parts[6] if len(parts) > 6 else "u"
    M, N, scale = int(float(M)), int(float(N)), float(scale)
    x = torch.from_numpy(synth.uniform3(M, 1)).cuda()
    y = torch.from_numpy(synth.gmm3(N, 2) if dist.startswith("gmm") else synth.uniform3(N, 2)).cuda()
    b = torch.from_numpy(synth.signal(N, 3)).cuda() if red == "sum" else None
    if red == "lse" and "h" in dist:                      # LSE with a bias h ~ N(0, 1)
        import numpy as np
        b = torch.from_numpy(np.random.default_rng(4).standard_normal(N).astype(np.float32)).cuda()
    kw = dict(scale=scale)
    if red == "lse":
        kw["out_dtype"] = "float64"
    for _ in range(3):
        genred.eval(formula, red, x, y, b, **kw)
    genred.profile(True)
    for _ in range(7):
        genred.eval(formula, red, x, y, b, **kw)
    ms = genred.profile_read()
    genred.profile(False)
    lib = os.path.basename(os.environ.get("GENRED_LIB", "libgenred.so"))
    print(f"{lib:28s} {name:10s} min {min(ms):9.3f} ms  med {statistics.median(ms):9.3f} ms  "
          f"pairs/clk/SM {M * N / (min(ms) * 1e-3) / (148 * 1.965e9):6.2f}  plan {genred.last_plan()}", flush=True)


if __name__ == "__main__":
    for c in sys.argv[1:]:
        run(c)
