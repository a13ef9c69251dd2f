"""Python-side cost of one C1 call through the binding: genred.eval, eval_args, bound_call, and a
trivial ctypes call (genred_launch_count) for the ctypes floor."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred
n = 1000
x, y, b = (torch.from_numpy(a).cuda() for a in (synth.uniform3(n, 1), synth.uniform3(n, 2), synth.signal(n, 3)))
out = torch.empty((n, 1), device="cuda")
s = torch.cuda.current_stream()
args, _, keep = genred.prepare("gauss", "sum", x, y, b, None, scale=0.5, out=out)
call = genred.bound_call(args, s)
lib = genred.load(); ctx = genred.context()
for name, f in (("eval", lambda: genred.eval("gauss", "sum", x, y, b, scale=0.5, out=out)),
                ("eval_args", lambda: genred.eval_args(args, stream=s)),
                ("bound_call", call),
                ("ctypes floor (genred_launch_count)", lambda: lib.genred_launch_count(ctx))):
    for _ in range(100): f()
    torch.cuda.synchronize()
    K = 3000
    t0 = time.perf_counter()
    for _ in range(K): f()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"{name:38s} enqueue us/call {(t1 - t0) / K * 1e6:6.2f}  wall us/call {(t2 - t0) / K * 1e6:6.2f}", flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for K in (20, 200):
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(K): call()
    e1.record(s); torch.cuda.synchronize()
    print(f"bound_call x{K}: event us/call {e0.elapsed_time(e1) / K * 1e3:.2f}")
