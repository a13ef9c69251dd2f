python - > gpurun_out/sweep.txt 2>&1 <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2004_11127_b200 import genred
for formula, M in (("gauss", 100000), ("gauss_sum_gradx", 100000), ("gauss", 300000)):
    x = torch.from_numpy(synth.uniform3(M, 1)).cuda(); y = torch.from_numpy(synth.uniform3(M, 2)).cuda(); b = torch.from_numpy(synth.signal(M, 3)).cuda()
    res = []
    for S in (0, 6, 9, 12, 15, 18, 21, 24, 27, 30, 36):
        for _ in range(2): genred.eval(formula, "sum", x, y, b, scale=0.5, split_j=S)
        genred.profile(True)
        for _ in range(5): genred.eval(formula, "sum", x, y, b, scale=0.5, split_j=S)
        ms = min(genred.profile_read()); genred.profile(False)
        pl = genred.last_plan()
        res.append(f"S{pl['split_j']}:{M*M/(ms*1e-3)/(148*1.965e9):.2f}")
    print(formula, M, " ".join(res), flush=True)
PY
