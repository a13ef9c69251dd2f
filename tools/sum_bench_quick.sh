# quick kernel-only timings of the Gaussian Sum (C5-like 1e6 x 1e6 slice) and the fused Sum+grad (C2)
python - <<'PY'
import torch, synth
from paper_2004_11127_b200 import genred
for (name, M, formula) in (("gauss 1e6", 1_000_000, "gauss"), ("fused 1e5", 100_000, "gauss_sum_gradx")):
    x = torch.from_numpy(synth.uniform3(M, 1)).cuda(); y = torch.from_numpy(synth.uniform3(M, 2)).cuda()
    b = torch.from_numpy(synth.signal(M, 3)).cuda()
    for _ in range(2): genred.eval(formula, "sum", x, y, b, scale=0.5)
    genred.profile(True)
    for _ in range(5): genred.eval(formula, "sum", x, y, b, scale=0.5)
    ms = genred.profile_read(); genred.profile(False)
    print("quick", name, "ms", round(min(ms), 3), "pairs/clk/SM", round(M * M / (min(ms) * 1e-3) / (148 * 1.965e9), 2))
PY
