for d in 0 4; do
GENRED_KNN_DBG=$d python - <<'PY'
import os, numpy as np, torch, oracle
from paper_2004_11127_b200 import genred
rng = np.random.default_rng(1332)
M, N, D, K = 300, 1000, 32, 10
x = rng.random((M, D)).astype(np.float32); y = rng.random((N, D)).astype(np.float32)
dd, j = genred.eval("sqdist", "argkmin", torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), K=K)
od, oj = oracle.argkmin(x, y, K)
bad = np.nonzero((j.cpu().numpy() != oj).any(1))[0]
print("dbg", os.environ["GENRED_KNN_DBG"], "bad rows", len(bad), bad[:10], "fallback", genred.last_plan()["fallback_rows"])
PY
done
