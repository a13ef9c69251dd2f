"""One genred_eval of a chosen workload, for ncu captures (`ncu ... python tools/profile_run.py`).

Not a benchmark (numbers under ncu are never bench values); it only launches the kernels.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_11127_b200 import genred  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="gauss",
                    choices=["gauss", "gradx", "fused", "lse", "lse_h", "argk"])
    ap.add_argument("--M", type=int, default=1_000_000)
    ap.add_argument("--N", type=int, default=1_000_000)
    ap.add_argument("--K", type=int, default=10)
    ap.add_argument("--D", type=int, default=3)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--scale", type=float, default=None, help="sigma (Gaussian) / eps (LSE)")
    a = ap.parse_args()
    if a.D == 784:
        x = torch.from_numpy(synth.mnist784(a.M, 1)).cuda()
        y = torch.from_numpy(synth.mnist784(a.N, 2)).cuda()
    else:
        x = torch.from_numpy(synth.uniform3(a.M, 1, a.D)).cuda()
        y = torch.from_numpy(synth.uniform3(a.N, 2, a.D)).cuda()
    b = torch.from_numpy(synth.signal(a.N, 3)).cuda()
    h = torch.from_numpy(np.random.default_rng(4).standard_normal(a.N).astype(np.float32)).cuda()
    for _ in range(a.reps):
        if a.what == "gauss":
            genred.eval("gauss", "sum", x, y, b, scale=a.scale or 0.5)
        elif a.what == "gradx":
            genred.eval("gauss_gradx", "sum", x, y, b, scale=0.5)
        elif a.what == "fused":
            genred.eval("gauss_sum_gradx", "sum", x, y, b, scale=0.5)
        elif a.what == "lse":
            genred.eval("sqdist", "lse", x, y, None, scale=a.scale or 0.05, out_dtype="float64")
        elif a.what == "lse_h":
            genred.eval("sqdist", "lse", x, y, h, scale=a.scale or 0.05, out_dtype="float64")
        else:
            genred.eval("sqdist", "argkmin", x, y, K=a.K)
    torch.cuda.synchronize()
    print("plan", genred.last_plan(), "launches", genred.launch_count())


if __name__ == "__main__":
    main()
