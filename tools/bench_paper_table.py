"""The paper's one published benchmark on this path, re-run on B200:
Gaussian Sum a_i = sum_j exp(-|x_i - y_j|^2) b_j (sigma = 1, reading R1), D = 3, M = N in
{1e4, 1e5, 1e6}, fp32.  Reports the device-resident time per genred_eval (CUDA events, median of
repeats after warm-up) and the end-to-end time from host numpy arrays (H2D + kernels + D2H), next
to the paper's PyKeOps / KeOps++ times on an RTX 2080 Ti (context, not a target)."""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_11127_b200 import genred  # noqa: E402

PAPER = {10_000: (0.7, 0.4), 100_000: (15.0, 14.6), 1_000_000: (1390.0, 1380.0)}   # ms: PyKeOps, KeOps++


def main():
    for n, reps in ((10_000, 200), (100_000, 50), (1_000_000, 5)):
        x = synth.uniform3(n, 1); y = synth.uniform3(n, 2); b = synth.signal(n, 3)
        xd, yd, bd = (torch.from_numpy(a).cuda() for a in (x, y, b))
        out = torch.empty((n, 1), device="cuda")
        for _ in range(3):
            genred.eval("gauss", "sum", xd, yd, bd, scale=1.0, out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            genred.eval("gauss", "sum", xd, yd, bd, scale=1.0, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        plan = genred.last_plan()
        te = []
        for _ in range(max(3, reps // 10)):
            t0 = time.perf_counter()
            genred.eval("gauss", "sum", x, y, b, scale=1.0)                 # host arrays in and out
            te.append((time.perf_counter() - t0) * 1e3)
        ms = statistics.median(ts)
        print(json.dumps({"N": n, "device_ms": ms, "pairs_per_s": n * n / (ms * 1e-3),
                          "e2e_host_ms": statistics.median(te),
                          "paper_pykeops_ms_2080ti": PAPER[n][0], "paper_keopspp_ms_2080ti": PAPER[n][1],
                          "speedup_vs_pykeops_device": PAPER[n][0] / ms,
                          "plan": {k: plan[k] for k in ("split_j", "rows_per_cta", "ctas", "path")}}),
              flush=True)


if __name__ == "__main__":
    main()
