import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, time
from paper_2004_11127_b200 import solvers, genred
x = torch.from_numpy(synth.gmm3(1_000_000, 13)).cuda()
solvers.kmeans(x, 1000, iters=2); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); l, c, h = solvers.kmeans(x, 1000, iters=10); e1.record(); torch.cuda.synchronize()
print("kmeans ms/iter", e0.elapsed_time(e1)/10, h[0], h[-1])
c = c.contiguous()
e0.record()
for _ in range(10): genred.eval("sqdist", "argkmin", x, c, K=1)
e1.record(); torch.cuda.synchronize()
print("argkmin ms", e0.elapsed_time(e1)/10, genred.last_plan())
