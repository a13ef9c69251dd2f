"""Tile-centred form of the Gaussian Sum (R18j): parity against the oracle on a few shapes and the
pair-loop time against the direct form.

  python tools/local_check.py [parity] [time]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2004_11127_b200 import genred as G  # noqa: E402
from tests.parity import r4_error  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def parity():
    rng = np.random.default_rng(5)
    cases = [
        ("u3 s0.25", synth.uniform3(20000, 1), synth.uniform3(30001, 2), synth.signal(30001, 3), 0.25),
        ("u3 s0.15 mixed", synth.uniform3(20000, 1), synth.uniform3(30001, 2), synth.signal(30001, 3), 0.15),
        ("u3 s0.05", synth.uniform3(4000, 1), synth.uniform3(400000, 2), synth.signal(400000, 3), 0.05),
        ("gmm s0.05", synth.gmm3(6000, 1), synth.gmm3(60000, 2), synth.signal(60000, 3, signed=True), 0.05),
        ("far 1000", (synth.uniform3(8000, 1) + 1000).astype(np.float32),
         (synth.uniform3(40000, 2) + 1000).astype(np.float32), synth.signal(40000, 3), 0.2),
    ]
    y = rng.random((50000, 2)).astype(np.float32)
    cases.append(("D2 s0.05", rng.random((3000, 2)).astype(np.float32), y, synth.signal(50000, 4), 0.05))
    y = rng.random((70000, 1)).astype(np.float32)
    cases.append(("D1 s0.01", rng.random((3000, 1)).astype(np.float32), y, synth.signal(70000, 5), 0.01))
    yo = synth.uniform3(30000, 7)
    yo[::101] *= 40.0                                   # outliers: wide tiles stay direct
    cases.append(("outliers", synth.uniform3(5000, 8), yo, synth.signal(30000, 9), 0.25))
    G.set_option("local_form", 2)
    for name, x, y, b, sig in cases:
        a = G.eval("gauss", "sum", dev(x), dev(y), dev(b), scale=sig)
        plan = G.last_plan()
        lt = G.last_tiles()
        t0 = time.time()
        o, den = oracle.gauss_sum(x, y, b, sigma=sig)
        err = r4_error(a.cpu().numpy(), o, den)
        print(f"{name:16s} M={len(x):6d} N={len(y):7d} path={plan['path']} split={plan['split_j']} "
              f"tiles={lt} maxR4={err.max():.3e} meanR4={err.mean():.2e} (oracle {time.time() - t0:.1f}s)",
              flush=True)
    G.set_option("local_form", 1)


def lse_parity():
    rng = np.random.default_rng(7)
    cases = [
        ("lse u3 e0.05", synth.uniform3(4000, 1), synth.uniform3(400000, 2), None, 0.05),
        ("lse u3 e0.05 h", synth.uniform3(4000, 1), synth.uniform3(400000, 2),
         rng.standard_normal(400000).astype(np.float32), 0.05),
        ("lse u3 e0.2 h3", synth.uniform3(20000, 3), synth.uniform3(30001, 4),
         (3 * rng.standard_normal(30001)).astype(np.float32), 0.2),
        ("lse gmm e0.01", synth.gmm3(5000, 5), synth.gmm3(100000, 6), None, 0.01),
        ("lse far e0.1", (synth.uniform3(5000, 7) + 1000).astype(np.float32),
         (synth.uniform3(60000, 8) + 1000).astype(np.float32), None, 0.1),
        ("lse D2 e0.01", rng.random((3000, 2)).astype(np.float32), rng.random((100000, 2)).astype(np.float32),
         None, 0.01),
        ("lse D1 e1e-4", rng.random((3000, 1)).astype(np.float32), rng.random((70000, 1)).astype(np.float32),
         rng.standard_normal(70000).astype(np.float32), 1e-4),
    ]
    G.set_option("local_form", 2)
    for name, x, y, h, eps in cases:
        a = G.eval("sqdist", "lse", dev(x), dev(y), dev(h) if h is not None else None, scale=eps,
                   out_dtype="float64")
        plan = G.last_plan()
        lt = G.last_tiles()
        o, _ = oracle.lse(x, y, h, eps=eps)
        err = np.abs(a.cpu().numpy() - o)
        print(f"{name:16s} M={len(x):6d} N={len(y):7d} path={plan['path']} split={plan['split_j']} "
              f"tiles={lt} maxabs={err.max():.3e} mean={err.mean():.2e}", flush=True)
    G.set_option("local_form", 1)


def lse_timing():
    for (M, N, eps, hz) in [(1_000_000, 1_000_000, 0.05, True), (1_000_000, 1_000_000, 0.05, False)]:
        x = dev(synth.uniform3(M, 1)); y = dev(synth.uniform3(N, 2))
        h = None if hz else dev(np.random.default_rng(4).standard_normal(N).astype(np.float32))
        for lf in (0, 1):
            G.set_option("local_form", lf)
            for _ in range(2):
                G.eval("sqdist", "lse", x, y, h, scale=eps, out_dtype="float64")
            torch.cuda.synchronize()
            G.profile(True)
            t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(3):
                G.eval("sqdist", "lse", x, y, h, scale=eps, out_dtype="float64")
            t1.record(); torch.cuda.synchronize()
            ms = G.profile_read()
            G.profile(False)
            plan = G.last_plan()
            lt = G.last_tiles()
            print(f"LSE M={M} N={N} eps={eps} h={'0' if hz else 'N(0,1)'} local_form={lf} path={plan['path']} "
                  f"tiles={lt} split={plan['split_j']} kernel {min(ms):.2f} ms step {t0.elapsed_time(t1) / 3:.2f} ms "
                  f"pairs/clk/SM {M * N / (min(ms) * 1e-3) / (148 * 1.965e9):.2f}", flush=True)
    G.set_option("local_form", 1)


def grad_timing():
    for formula in ("gauss_sum_gradx", "gauss_gradx"):
        M = N = 1_000_000
        x = dev(synth.uniform3(M, 1)); y = dev(synth.uniform3(N, 2)); b = dev(synth.signal(N, 3))
        for lf in (0, 1):
            G.set_option("local_form", lf)
            for _ in range(2):
                G.eval(formula, "sum", x, y, b, scale=0.05)
            torch.cuda.synchronize()
            G.profile(True)
            for _ in range(3):
                G.eval(formula, "sum", x, y, b, scale=0.05)
            ms = G.profile_read()
            G.profile(False)
            plan = G.last_plan()
            print(f"{formula} M=N=1e6 sigma=0.05 local_form={lf} path={plan['path']} tiles={G.last_tiles()} "
                  f"kernel {min(ms):.2f} ms pairs/clk/SM {M * N / (min(ms) * 1e-3) / (148 * 1.965e9):.2f}", flush=True)
    G.set_option("local_form", 1)


def timing():
    for (M, N, sig) in [(2_000_000, 2_000_000, 0.05), (1_000_000, 1_000_000, 0.05), (1_000_000, 1_000_000, 0.1)]:
        x = dev(synth.uniform3(M, 1)); y = dev(synth.uniform3(N, 2)); b = dev(synth.signal(N, 3))
        for lf in (0, 1):
            G.set_option("local_form", lf)
            for _ in range(2):
                G.eval("gauss", "sum", x, y, b, scale=sig)
            torch.cuda.synchronize()
            G.profile(True)
            t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
            t0.record()
            for _ in range(3):
                G.eval("gauss", "sum", x, y, b, scale=sig)
            t1.record(); torch.cuda.synchronize()
            ms = G.profile_read()
            G.profile(False)
            plan = G.last_plan()
            lt = G.last_tiles()
            step = t0.elapsed_time(t1) / 3
            print(f"M={M} N={N} sigma={sig} local_form={lf} path={plan['path']} tiles={lt} "
                  f"kernel {min(ms):.2f} ms step {step:.2f} ms pairs/clk/SM {M * N / (min(ms) * 1e-3) / (148 * 1.965e9):.2f}",
                  flush=True)
    G.set_option("local_form", 1)


if __name__ == "__main__":
    what = sys.argv[1:] or ["parity", "time"]
    if "parity" in what:
        parity()
    if "time" in what:
        timing()
    if "lse" in what:
        lse_parity()
    if "lsetime" in what:
        lse_timing()
    if "gradtime" in what:
        grad_timing()
