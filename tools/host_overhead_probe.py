"""Host-side cost per genred call (small problem): full Python binding vs a prebuilt Args struct."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred
n = 1000
x, y, b = (torch.from_numpy(a).cuda() for a in (synth.uniform3(n, 1), synth.uniform3(n, 2), synth.signal(n, 3)))
out = torch.empty((n, 1), device="cuda")
for _ in range(50): genred.eval("gauss", "sum", x, y, b, scale=0.5, out=out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000): genred.eval("gauss", "sum", x, y, b, scale=0.5, out=out)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("binding: enqueue us/call %.1f, wall us/call %.1f" % ((t1 - t0) / 2000 * 1e6, (t2 - t0) / 2000 * 1e6))
a = genred.Args(); a.abi_version = genred.ABI_VERSION
a.formula, a.reduction = genred.FORMULAS["gauss"], genred.REDUCTIONS["sum"]
a.M, a.N, a.D, a.E, a.K, a.scale = n, n, 3, 1, 1, 0.5
a.x, a.y, a.b, a.out = x.data_ptr(), y.data_ptr(), b.data_ptr(), out.data_ptr()
s = torch.cuda.current_stream()
for _ in range(50): genred.eval_args(a, stream=s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(2000): genred.eval_args(a, stream=s)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print("prebuilt args: enqueue us/call %.1f, wall us/call %.1f" % ((t1 - t0) / 2000 * 1e6, (t2 - t0) / 2000 * 1e6))
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(500): genred.eval("gauss", "sum", x, y, b, scale=0.5, out=out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(8)
