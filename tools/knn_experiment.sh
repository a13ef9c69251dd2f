for d in 0 1 2 3; do
  GENRED_KNN_DBG=$d python - <<'PY'
import os, torch, synth
from paper_2004_11127_b200 import genred
x = torch.from_numpy(synth.mnist784(10000, 1)).cuda(); y = torch.from_numpy(synth.mnist784(60000, 2)).cuda()
for _ in range(2): genred.eval("sqdist", "argkmin", x, y, K=10)
genred.profile(True)
for _ in range(3): genred.eval("sqdist", "argkmin", x, y, K=10)
print("dbg", os.environ["GENRED_KNN_DBG"], "kernel ms", genred.profile_read())
PY
done
