"""Main-kernel time of one shape across forced j-splits (planner check)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred
M = N = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100000
formula = sys.argv[2] if len(sys.argv) > 2 else "gauss"
x = torch.from_numpy(synth.uniform3(M, 1)).cuda(); y = torch.from_numpy(synth.uniform3(N, 2)).cuda()
b = torch.from_numpy(synth.signal(N, 3)).cuda()
for S in [0, 3, 6, 9, 12, 18, 24]:
    for _ in range(3): genred.eval(formula, "sum", x, y, b, scale=0.5, split_j=S)
    genred.profile(True)
    for _ in range(5): genred.eval(formula, "sum", x, y, b, scale=0.5, split_j=S)
    ms = min(genred.profile_read()); genred.profile(False)
    pl = genred.last_plan()
    print(f"S={S:3d} -> split {pl['split_j']:3d} ctas {pl['ctas']:5d}  {ms:.4f} ms  {M*N/(ms*1e-3)/(148*1.965e9):.2f} pairs/clk/SM", flush=True)
