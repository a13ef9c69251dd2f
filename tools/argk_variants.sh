# ArgKMin (small D) main-kernel time across library variants: M = 1e5, N = 1e7 (K = 1 and 10).
for lib in ${VARS:-build/var/libgenred_*.so}; do
GENRED_LIB=$lib python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2004_11127_b200 import genred
M, N = 100_000, 10_000_000
x = torch.from_numpy(synth.uniform3(M, 1)).cuda(); y = torch.from_numpy(synth.uniform3(N, 2)).cuda()
for K in (1, 10):
    for _ in range(2): genred.eval("sqdist", "argkmin", x, y, K=K)
    genred.profile(True)
    for _ in range(2): genred.eval("sqdist", "argkmin", x, y, K=K)
    ms = min(genred.profile_read()); genred.profile(False)
    print("lib", os.environ["GENRED_LIB"], "K", K, "ms", round(ms, 2), "pairs/clk/SM", round(M * N / (ms * 1e-3) / (148 * 1.965e9), 2))
PY
done
