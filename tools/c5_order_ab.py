"""C5 main-kernel time with the split-major CTA order on and off (option split_major)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2004_11127_b200 import genred as G  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
x = torch.from_numpy(synth.uniform3(M, 1)).cuda()
y = torch.from_numpy(synth.uniform3(10_000_000, 2)).cuda()
b = torch.from_numpy(synth.signal(10_000_000, 3)).cuda()
for sm in (1, 0, 1, 0):
    G.set_option("split_major", sm)
    G.eval("gauss", "sum", x, y, b, scale=0.5)
    G.profile(True)
    for _ in range(2):
        G.eval("gauss", "sum", x, y, b, scale=0.5)
    ms = G.profile_read()
    G.profile(False)
    print(f"M={M} split_major={sm} split={G.last_plan()['split_j']} kernel ms {[round(v, 1) for v in ms]}", flush=True)
