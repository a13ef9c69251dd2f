# Gaussian Sum (M = N = 1e6) main-kernel time across library variants (VARS or build/var/*.so).
for lib in ${VARS:-build/var/libgenred_*.so}; do
GENRED_LIB=$lib python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2004_11127_b200 import genred
n = 1_000_000
x = torch.from_numpy(synth.uniform3(n, 1)).cuda(); y = torch.from_numpy(synth.uniform3(n, 2)).cuda()
b = torch.from_numpy(synth.signal(n, 3)).cuda()
for _ in range(2): genred.eval("gauss", "sum", x, y, b, scale=0.5)
genred.profile(True)
for _ in range(3): genred.eval("gauss", "sum", x, y, b, scale=0.5)
ms = min(genred.profile_read())
print("lib", os.environ["GENRED_LIB"], "ms", round(ms, 2), "pairs/clk/SM", round(n * n / (ms * 1e-3) / (148 * 1.965e9), 2))
PY
done
