"""Small invocations of every libgenred kernel family, for compute-sanitizer (one tool per run):
    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2004_11127_b200 import genred  # noqa: E402
from paper_2004_11127_b200.autograd import gauss_sum, logsumexp  # noqa: E402

d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
x = d(synth.uniform3(1500, 1)); y = d(synth.uniform3(1100, 2)); b = d(synth.signal(1100, 3))
for split in (0, 3):
    genred.eval("gauss", "sum", x, y, b, scale=0.5, split_j=split)
    genred.eval("gauss", "sum", x, y, b, scale=0.05, split_j=split)          # direct path
    genred.eval("gauss_sum_gradx", "sum", x, y, b, None, scale=0.5, split_j=split)
    genred.eval("sqdist", "lse", x, y, None, scale=0.05, out_dtype="float64", split_j=split)
    genred.eval("sqdist", "argkmin", x, y, K=5, split_j=split)
ri = np.array([[0, 700], [700, 1500]], np.int64); sl = np.array([1, 3], np.int64)
rj = np.array([[0, 333], [0, 500], [600, 1100]], np.int64)
genred.eval("gauss", "sum", x, y, b, scale=0.5, ranges=(ri, sl, rj))
xa = x.clone().requires_grad_(True); ya = y.clone().requires_grad_(True); ba = b.clone().requires_grad_(True)
gauss_sum(xa, ya, ba, 0.5).sum().backward()
logsumexp(xa, ya, None, 0.1).sum().backward()
X = d(synth.mnist784(300, 4)); Y = d(synth.mnist784(700, 5))
genred.eval("sqdist", "argkmin", X, Y, K=10)
torch.cuda.synchronize()
print("sanitize_run ok", genred.launch_count())
