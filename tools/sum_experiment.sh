for d in 0 1 2; do
  GENRED_SUM_DBG=$d python - <<'PY'
import os, torch, synth
from paper_2004_11127_b200 import genred
x = torch.from_numpy(synth.uniform3(1_000_000, 1)).cuda(); y = torch.from_numpy(synth.uniform3(1_000_000, 2)).cuda()
b = torch.from_numpy(synth.signal(1_000_000, 3)).cuda()
for _ in range(2): genred.eval("gauss", "sum", x, y, b, scale=0.5)
genred.profile(True)
for _ in range(3): genred.eval("gauss", "sum", x, y, b, scale=0.5)
ms = genred.profile_read()
print("dbg", os.environ["GENRED_SUM_DBG"], "kernel ms", ms, "pairs/clk/SM", 1e12 / (min(ms) * 1e-3) / (148 * 1.965e9), "plan", genred.last_plan())
PY
done
