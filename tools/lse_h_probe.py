"""LSE with and without h (M = N = 1e6, D = 3): pairs/s of the main kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2004_11127_b200 import genred
n = 1_000_000
x = torch.from_numpy(synth.uniform3(n, 1)).cuda(); y = torch.from_numpy(synth.gmm3(n, 2)).cuda()
h = torch.from_numpy((np.random.default_rng(3).standard_normal(n) * 2).astype(np.float32)).cuda()
for name, hh in (("h=0", None), ("h random", h)):
    for _ in range(2): genred.eval("sqdist", "lse", x, y, hh, scale=0.05, out_dtype="float64")
    genred.profile(True)
    for _ in range(3): genred.eval("sqdist", "lse", x, y, hh, scale=0.05, out_dtype="float64")
    ms = min(genred.profile_read()); genred.profile(False)
    print(name, "kernel ms", round(ms, 2), "pairs/clk/SM", round(n * n / (ms * 1e-3) / (148 * 1.965e9), 2))
