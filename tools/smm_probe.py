"""Kernel breakdown of the small-M Gaussian Sum (one call per M)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred
N = 10_000_000
y = torch.from_numpy(synth.uniform3(N, 2)).cuda(); b = torch.from_numpy(synth.signal(N, 3)).cuda()
for M in [int(v) for v in sys.argv[1:]] or [1, 256]:
    x = torch.from_numpy(synth.uniform3(M, 1)).cuda()
    genred.eval("gauss", "sum", x, y, b, scale=0.5)
    torch.cuda.synchronize()
    print(M, genred.last_plan())
