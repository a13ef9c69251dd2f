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
# per-call GPU time with the enqueue taken out: the same call captured once in a CUDA graph
g = torch.cuda.CUDAGraph()
cs = torch.cuda.Stream()
cs.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cs):
    for _ in range(5): genred.eval_args(a, stream=cs)
torch.cuda.current_stream().wait_stream(cs)
torch.cuda.synchronize()
with torch.cuda.graph(g):
    genred.eval_args(a, stream=torch.cuda.current_stream())
for _ in range(20): g.replay()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(2000): g.replay()
e1.record(); torch.cuda.synchronize()
print("graph replay: device us/call %.2f" % (e0.elapsed_time(e1) / 2000 * 1e3))
ref = out.clone(); genred.eval("gauss", "sum", x, y, b, scale=0.5, out=out); torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
print("graph result bitwise equal:", bool(torch.equal(ref, out)))
e0.record()
for _ in range(2000): genred.eval_args(a, stream=torch.cuda.current_stream())
e1.record(); torch.cuda.synchronize()
print("eager prebuilt: device us/call %.2f" % (e0.elapsed_time(e1) / 2000 * 1e3))
