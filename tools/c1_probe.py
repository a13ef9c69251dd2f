"""C1 step timing outside bench.py's harness (same inputs, same prepared call) to locate overhead."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
from paper_2004_11127_b200 import genred
torch.cuda.set_device(0)
w = bench.workload(1); c = w["cfg"]
x, y, b = bench.make_inputs(w, "U3")
dev = torch.device("cuda", 0)
xd, yd, bd = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, y, b))
out = torch.empty((c.M, 1), dtype=torch.float32, device=dev)
s = torch.cuda.current_stream(dev)
args, _, keep = genred.prepare("gauss", "sum", xd, yd, bd, None, scale=c.scale, K=1, out=out, out_dtype="float32", j_offset=0)
call = genred.bound_call(args, s, 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for label, warm in (("cold", 5), ("warm", 2000)):
    for _ in range(warm): call()
    for K in (20, 200, 2000):
        torch.cuda.synchronize(); e0.record(s)
        for _ in range(K): call()
        e1.record(s); torch.cuda.synchronize()
        print(f"{label} x{K}: {e0.elapsed_time(e1) / K * 1e3:.2f} us/call", flush=True)
print(genred.last_plan())
# bench.py's sequence around the timed region, one piece at a time
def loop(tag, K=20):
    torch.cuda.synchronize(); e0.record(s)
    for _ in range(K): call()
    e1.record(s); torch.cuda.synchronize()
    print(f"{tag} x{K}: {e0.elapsed_time(e1) / K * 1e3:.2f} us/call", flush=True)
loop("baseline")
genred.profile(False, 0); loop("after profile(False)")
genred.launch_count(0); loop("after launch_count")
smp = bench.ClockSampler(0).start(); loop("sampler running"); loop("sampler running", 200); smp.stop()
genred.profile(True, 0); loop("profile(True)"); genred.profile_read(0); genred.profile(False, 0)
loop("after profile pass")
