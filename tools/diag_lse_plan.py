"""Planner check: LSE M = 1e4 against N = 1e8 (the j-shard config 8 on one rank)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred, dist as gdist
x = torch.from_numpy(synth.uniform3(10000, 1)).cuda()
for N in (10_000_000, 100_000_000):
    y = torch.from_numpy(synth.uniform3(N, 2)).cuda()
    genred.eval("sqdist", "lse", x, y, None, scale=0.05, out_dtype="float64"); print(N, "eval", genred.last_plan(), flush=True)
    st = torch.empty((10000, 2), dtype=torch.float64, device="cuda")
    genred.eval("sqdist", "lse", x, y, None, scale=0.05, out_dtype="float64", lse_state=st); print(N, "eval+state", genred.last_plan(), flush=True)
    gdist.jshard_eval("sqdist", "lse", x, y, None, scale=0.05); print(N, "jshard", genred.last_plan(), flush=True)
    del y
