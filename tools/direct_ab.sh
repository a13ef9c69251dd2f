# A/B of the direct-form Gaussian kernels across library variants (narrow sigma: the box rules
# the expanded form out).  VARS = the .so files; interleaved reps.
for rep in 1 2; do
for lib in ${VARS:-build/var/libgenred_*.so}; do
GENRED_LIB=$lib python - <<'PY'
import os, torch, synth
from paper_2004_11127_b200 import genred
M = 2_000_000
x = torch.from_numpy(synth.uniform3(M, 1)).cuda(); y = torch.from_numpy(synth.uniform3(M, 2)).cuda(); b = torch.from_numpy(synth.signal(M, 3)).cuda()
out = []
for name, red, args in (("sum s=.05", "gauss", {}), ("sum+grad s=.05", "gauss_sum_gradx", {})):
    for _ in range(2): genred.eval(red, "sum", x, y, b, scale=0.05)
    genred.profile(True)
    for _ in range(3): genred.eval(red, "sum", x, y, b, scale=0.05)
    ms = genred.profile_read()
    out.append(f"{name} {min(ms):.2f} ms path {genred.last_plan()['path'] if hasattr(genred, 'last_plan') else '?'}")
xe = torch.from_numpy(synth.uniform3(1 << 27, 4)).cuda(); ye = y[:8].contiguous(); be = b[:8].contiguous()
for _ in range(2): genred.eval("gauss", "sum", xe, ye, be, scale=0.5)
genred.profile(True)
for _ in range(5): genred.eval("gauss", "sum", xe, ye, be, scale=0.5)
ms = genred.profile_read()
out.append(f"edge N=8 M=2^27 {min(ms):.3f} ms")
print(os.path.basename(os.environ["GENRED_LIB"]), " | ".join(out))
PY
done
done
