"""Main-kernel time of the LSE backward (softmax-weighted gradient) at M = N = n (default 4e5)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2004_11127_b200 import genred
n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 400_000
x = torch.from_numpy(synth.uniform3(n, 1)).cuda(); y = torch.from_numpy(synth.gmm3(n, 2)).cuda()
h = torch.from_numpy(np.random.default_rng(3).standard_normal(n).astype(np.float32)).cuda()
a = genred.eval("sqdist", "lse", x, y, h, scale=0.05, out_dtype="float64")
g = torch.ones(n, dtype=torch.float32, device="cuda")
f = lambda: genred.eval("lse_grad", "sum", x, y, None, g, scale=0.05, out_dtype="float64",
                        row_shift=-a, col_shift=h.double())
for _ in range(2): f()
genred.profile(True)
for _ in range(5): f()
ms = min(genred.profile_read()); genred.profile(False)
print(os.path.basename(os.environ.get("GENRED_LIB", "libgenred.so")), "lse_grad", n, f"{ms:.3f} ms",
      f"{n * n / (ms * 1e-3) / (148 * 1.965e9):.2f} pairs/clk/SM", genred.last_plan(), flush=True)
