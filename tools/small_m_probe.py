"""M << N: Gaussian Sum and LSE with few rows against a large N (pairs/s per shape)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred
N = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
y = torch.from_numpy(synth.uniform3(N, 2)).cuda(); b = torch.from_numpy(synth.signal(N, 3)).cuda()
for M in (1, 16, 64, 65, 256, 1024, 2048, 16384):
    x = torch.from_numpy(synth.uniform3(M, 1)).cuda()
    for red in ("sum", "lse"):
        f = (lambda: genred.eval("gauss", "sum", x, y, b, scale=0.5)) if red == "sum" else \
            (lambda: genred.eval("sqdist", "lse", x, y, None, scale=0.05, out_dtype="float64"))
        for _ in range(3): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        pl = genred.last_plan()
        print(json.dumps({"M": M, "N": N, "red": red, "ms": round(ms, 4), "pairs_per_s": M * N / (ms * 1e-3),
                          "split": pl["split_j"], "rows_per_cta": pl["rows_per_cta"], "ctas": pl["ctas"]}), flush=True)
