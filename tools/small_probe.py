"""Launch-level timing of one small Gaussian Sum (N = 1e4): total device time vs the kernels."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000
x, y, b = (torch.from_numpy(a).cuda() for a in (synth.uniform3(n, 1), synth.uniform3(n, 2), synth.signal(n, 3)))
out = torch.empty((n, 1), device="cuda")
for _ in range(20):
    genred.eval("gauss", "sum", x, y, b, scale=1.0, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    genred.eval("gauss", "sum", x, y, b, scale=1.0, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print("host enqueue us/call", (t1 - t0) / 200 * 1e6, "wall us/call", (t2 - t0) / 200 * 1e6, genred.last_plan())
