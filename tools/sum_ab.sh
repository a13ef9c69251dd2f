# A/B of Gaussian Sum kernel variants on the same box (M = N = 2e6, interleaved runs)
for rep in 1 2; do
for lib in ${VARS:-build/var/libgenred_*.so}; do
GENRED_LIB=$lib python - <<'PY'
import os, torch, synth
from paper_2004_11127_b200 import genred
M = 2_000_000
x = torch.from_numpy(synth.uniform3(M, 1)).cuda(); y = torch.from_numpy(synth.uniform3(M, 2)).cuda(); b = torch.from_numpy(synth.signal(M, 3)).cuda()
for _ in range(2): genred.eval("gauss", "sum", x, y, b, scale=0.5)
genred.profile(True)
for _ in range(3): genred.eval("gauss", "sum", x, y, b, scale=0.5)
ms = genred.profile_read()
print("lib", os.environ["GENRED_LIB"], "ms", round(min(ms), 2), "pairs/clk/SM", round(M*M/(min(ms)*1e-3)/(148*1.965e9), 3))
PY
done
done
