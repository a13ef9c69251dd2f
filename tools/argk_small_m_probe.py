"""ArgKMin (small D) with few query rows against a large N."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2004_11127_b200 import genred
N = 10_000_000
y = torch.from_numpy(synth.uniform3(N, 2)).cuda()
for M in (1, 100, 1000, 10000, 100000):
    x = torch.from_numpy(synth.uniform3(M, 1)).cuda()
    for K in (1, 10):
        f = lambda: genred.eval("sqdist", "argkmin", x, y, K=K)
        for _ in range(2): f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3): f()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        pl = genred.last_plan()
        print(json.dumps({"M": M, "K": K, "ms": round(ms, 3), "pairs_per_s": M * N / (ms * 1e-3),
                          "split": pl["split_j"], "rows_per_cta": pl["rows_per_cta"], "ctas": pl["ctas"]}), flush=True)
