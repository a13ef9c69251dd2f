"""A/B of the Gaussian Sum paths (tensor-core exponent vs FP32 expanded) at M = N = n."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synth
from paper_2004_11127_b200 import genred as G
import oracle

def run(n, reps, tc):
    os.environ["GENRED_GAUSS_TC"] = "1" if tc else "0"
    x = torch.from_numpy(synth.uniform3(n, 1005)).cuda(); y = torch.from_numpy(synth.uniform3(n, 2005)).cuda()
    b = torch.from_numpy(synth.signal(n, 3005)).cuda()
    a = G.eval("gauss", "sum", x, y, b, scale=0.5)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        a = G.eval("gauss", "sum", x, y, b, scale=0.5)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rows = np.arange(0, n, max(1, n // 64))
    o, den = oracle.gauss_sum(x.cpu().numpy(), y.cpu().numpy(), b.cpu().numpy(), sigma=0.5, rows=rows)
    err = float(np.max(np.abs(a.cpu().numpy()[rows].astype(np.float64).ravel() - o.ravel()) / den.ravel()))
    print(json.dumps({"n": n, "tc": tc, "path": G.last_plan()["path"], "ms": ms,
                      "pairs_per_s": n * n / (ms * 1e-3), "max_rel_err_sampled": err}), flush=True)

for n, reps in [(1_000_000, 5), (4_000_000, 2)]:
    run(n, reps, True)
    run(n, reps, False)
