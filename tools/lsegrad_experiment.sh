# LSE backward kernel (GENRED_LSE_GRAD) timing across library variants (VARS or build/var/*.so).
for lib in ${VARS:-build/var/libgenred_*.so}; do
GENRED_LIB=$lib python - <<'PY'
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import synth
from paper_2004_11127_b200 import genred
n = 1_000_000
x = torch.from_numpy(synth.uniform3(n, 1)).cuda(); y = torch.from_numpy(synth.gmm3(n, 2)).cuda()
h = torch.from_numpy(np.random.default_rng(3).standard_normal(n)).cuda()
a = torch.zeros(n, dtype=torch.float64, device="cuda") - 5.0
g = torch.ones(n, device="cuda")
f = lambda: genred.eval("lse_grad", "sum", x, y, None, g, scale=0.05, out_dtype="float64", row_shift=a, col_shift=h)
for _ in range(2): f()
genred.profile(True)
for _ in range(3): f()
ms = min(genred.profile_read())
print("lib", os.environ["GENRED_LIB"], "ms", round(ms, 2), "pairs/clk/SM", round(n * n / (ms * 1e-3) / (148 * 1.965e9), 2), genred.last_plan()["rows_per_cta"])
PY
done
