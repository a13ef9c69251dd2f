for lib in ${VARS:-build/var/libgenred_*.so}; do
  GENRED_LIB=$lib python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2004_11127_b200 import genred
M = N = 1_000_000
x = torch.from_numpy(synth.uniform3(M, 1003)).cuda(); y = torch.from_numpy(synth.gmm3(N, 2003)).cuda()
for _ in range(2): genred.eval("sqdist", "lse", x, y, None, scale=0.05, out_dtype="float64")
genred.profile(True)
for _ in range(3): genred.eval("sqdist", "lse", x, y, None, scale=0.05, out_dtype="float64")
ms = genred.profile_read()
print("lib", os.environ["GENRED_LIB"], "ms", [round(v,2) for v in ms], "pairs/clk/SM", round(M*N / (min(ms) * 1e-3) / (148 * 1.965e9), 2), genred.last_plan()["split_j"])
PY
done
