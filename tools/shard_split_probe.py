"""Main-kernel time of one i-shard of C5 (M = 1e7 / G rows against N = 1e7) at the planner's
j-split and at forced ones (the split-major wave rule)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2004_11127_b200 import genred as G  # noqa: E402

Gs = int(sys.argv[1]) if len(sys.argv) > 1 else 8
M = 10_000_000 // Gs
x = torch.from_numpy(synth.uniform3(M, 1)).cuda()
y = torch.from_numpy(synth.uniform3(10_000_000, 2)).cuda()
b = torch.from_numpy(synth.signal(10_000_000, 3)).cuda()
for split in [0] + [int(v) for v in sys.argv[2:]]:
    G.eval("gauss", "sum", x, y, b, scale=0.5, split_j=split)
    G.profile(True)
    for _ in range(2):
        G.eval("gauss", "sum", x, y, b, scale=0.5, split_j=split)
    ms = G.profile_read()
    G.profile(False)
    p = G.last_plan()
    print(f"G={Gs} M={M} split_j={split} -> split {p['split_j']} ctas {p['ctas']} kernel ms {min(ms):.1f} "
          f"pairs/clk/SM {M * 1e7 / (min(ms) * 1e-3) / (148 * 1.965e9):.2f}", flush=True)
