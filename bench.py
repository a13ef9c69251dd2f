#!/usr/bin/env python
"""bench.py -- pair-evaluations/s of the Genred hot path on B200 (BASELINE.json ``metric``).

Default workload (N=1): configuration C5 of BASELINE.json, the one the metric is quoted on:
Gaussian Genred Sum a_i = sum_j exp(-|x_i - y_j|^2/sigma^2) b_j, M = N = 1e7, D = 3, E = 1,
sigma = 0.5, x, y ~ U[0,1)^3, b ~ U[0,1) (synthetic, seeded).

A step = one genred_eval (pack j-records -> pair-loop kernel -> fixed-order merge) over the whole
problem.  With --gpus N (torchrun, one process per GPU, NCCL) the i-range is sharded: each step
broadcasts y and b from rank 0 and every rank reduces its M/N rows (strong scaling of the fixed
1e14-pair problem; no reduction collective is needed, north star (d)).

Timing: W warm-up steps; then K steps bracketed by barrier + cuda synchronize, CUDA events on
the launching stream, max over ranks.  Inputs (280 MB) exceed the 126 MB L2, so no flush.
Extra keys: roofline (dominant kernel, live CUDA-event timing through genred_profile: inside the
timed region for steps >= 5 ms, else over a second pass of the same K steps -- kernel_timing),
cpu_baseline (the fp64 oracle on a bounded row sample; at N > 1 on 128 seeded rows of EACH shard
gathered to rank 0, with max_r4_err_vs_gpu), per_rank (N > 1: every rank's plan and kernel time),
e2e (host buffers through the C ABI's host mode, H2D + D2H inside the timed region), clocks (NVML
sampled during the timed region), gpu_launches (libgenred kernels launched in the timed region,
all ranks).  NCCL runs with NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=INIT (communicator rank counts).

``--mode jshard`` (configs 7, 8: M = 1e4 against N = 1e8, Gaussian Sum / LSE): the j-shard path of
SURVEY.md 8(e) -- each rank draws its slice of y, a step is the public dist.jshard_eval (local
reduction + fp64 all-reduce, or (m, s) all-gather + genred_combine_lse).

``--impl reference``: there is no reference implementation (PAPER.md only); the reference arm
is the fp64 oracle (oracle/) timed on this host's cores on a bounded row sample of the same
workload -- a deliberately slow baseline, not a target.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "pair-evals/sec (M·N/s) Gaussian Genred Sum D=3 at 1/2/4/8 B200; % FP32/MUFU peak"
UNIT = "pairs/s"
SMS = 148
MUFU_PER_CLK_SM = 16          # MUFU.EX2 lanes per clock per SM (sm_100)
FP32_PER_CLK_SM = 128         # FP32 lanes per clock per SM (FFMA/FADD/FMUL; FFMA2 counts 2)


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def workload(cid: int) -> dict:
    """Per-config step definition: formula, algorithmic FP32 lane-ops and exps per pair (D=3)."""
    c = synth.config(cid)
    if cid in (1, 5):  # expanded form: u = 2x'.y' - |y'|^2 (3 FFMA) + acc (1 FFMA) = 4 lane-ops;
        #                and 1/8 of the exponentials on the FP32 pipe (degree-5 polynomial: 8 lane-ops
        #                each): MUFU 7/8 and FP32 4 + 8/8 = 5 per pair
        return dict(cfg=c, formula="gauss", reduction="sum", fp32=5, mufu=7 / 8, out_dtype="float32")
    if cid == 2:   # Sum + gradient, one fused pass, expanded form: u (3 FFMA) + S0 += e b (1 FFMA)
        #            + S += e (b y') (3 FFMA, b y' packed with the j-records) = 7 lane-ops; the peak
        #            is the MUFU's either way (min(16/1, 128/7) = 16 pairs/clk/SM)
        return dict(cfg=c, formula="gauss_sum_gradx", reduction="sum", fp32=7, mufu=1,
                    out_dtype="float32")
    if cid == 9:   # the x-gradient alone (GAUSS_GRADX), expanded form: u (3) + S0 += e b' (1) +
        #            S += e (b' y') (3) = 7 lane-ops, as the fused kernel (the Sum column is S0)
        return dict(cfg=c, formula="gauss_gradx", reduction="sum", fp32=7, mufu=1, out_dtype="float32")
    if cid == 7:   # j-sharded Gaussian Sum (M << N): as C5 per rank, fp64 partials all-reduced
        return dict(cfg=c, formula="gauss", reduction="sum", fp32=5, mufu=7 / 8, out_dtype="float64")
    if cid == 8:   # j-sharded LSE: as C3 per rank, (m, s) states all-gathered and combined
        return dict(cfg=c, formula="sqdist", reduction="lse", fp32=8, mufu=1, out_dtype="float64")
    if cid == 3:   # raw diff (3) + |d|^2 (3) + t = fma(-c,|d|^2,-m) (1) + s += e (1) = 8; at C3's
        #            size the tile-centred form runs (R18j): w - m' (1) + 2x''.y'' (3) + s += e (1)
        #            = 5 (set from the plan below); the peak is the MUFU's either way
        return dict(cfg=c, formula="sqdist", reduction="lse", fp32=8, mufu=1, out_dtype="float64")
    if cid == 6:   # Cedge: N tiny -> 12 B of x read + 4 B of a written per row (HBM-bound)
        return dict(cfg=c, formula="gauss", reduction="sum", fp32=None, mufu=None, out_dtype="float32",
                    hbm=True)
    if cid == 4:   # k-NN, D=784: 3xTF32 tcgen05 contraction (tensor-bound)
        return dict(cfg=c, formula="sqdist", reduction="argkmin", fp32=None, mufu=None,
                    out_dtype="float32")
    raise SystemExit(f"config {cid} is not benchmarked yet")


def alu_peak_pairs(fp32: int, mufu: int, mhz: float) -> float:
    """Pairs/s ceiling of the FP32 + MUFU pipes for an algorithmic mix."""
    per_clk = min(MUFU_PER_CLK_SM / mufu, FP32_PER_CLK_SM / fp32)
    return per_clk * SMS * mhz * 1e6


class ClockSampler:
    """NVML SM-clock / throttle-reason sampler running during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int, period: float = 0.2):
        self.device, self.period = device, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self

        def run():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for bit, name in self.REASONS.items():
                        if r & bit and bit != 0x1:
                            self.reasons.add(name)
                except Exception:
                    pass
                self._stop.wait(self.period)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()
        return self

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join()
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def ncu_traffic(cid: int, n: int = 0):
    """dram read+write bytes per launch of the dominant kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    if cid == 6:
        return d.get(f"C6_N{n}")
    return d.get(f"C{cid}")


def cpu_model() -> str:
    """The host CPU's model name (what `lscpu` reports as "Model name")."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(w: dict, x, y, b, rows: np.ndarray, gpu_rows=None) -> dict:
    """The fp64 oracle as it stands, on a bounded row sample of the same workload."""
    import oracle
    c = w["cfg"]
    t0 = time.perf_counter()
    if w["reduction"] == "argkmin":
        od, oj = oracle.argkmin(x, y, c.K, rows=rows)
        dt = time.perf_counter() - t0
        res = {"value": len(rows) * c.N / dt, "unit": UNIT, "cores": oracle.num_threads(),
               "cpu_model": cpu_model(), "kind": "oracle", "seconds": round(dt, 3),
               "sample": f"{len(rows)} seeded rows x all N={c.N}, D={c.D} (fp64 direct differences)"}
        if gpu_rows is not None:
            res["index_match_frac_vs_gpu"] = float(np.mean(np.asarray(gpu_rows) == oj))
        return res
    if w["reduction"] == "lse":
        o, _ = oracle.lse(x, y, None, eps=c.scale, rows=rows)
        den = None
    elif w["formula"] == "gauss_sum_gradx":
        o, den = oracle.gauss_sum(x, y, b, sigma=c.scale, rows=rows)
        oracle.gauss_gradx(x, y, b, None, sigma=c.scale, rows=rows)
    elif w["formula"] == "gauss_gradx":
        o, den = oracle.gauss_gradx(x, y, b, None, sigma=c.scale, rows=rows)
    else:
        o, den = oracle.gauss_sum(x, y, b, sigma=c.scale, rows=rows)
    dt = time.perf_counter() - t0
    res = {"value": len(rows) * c.N / dt, "unit": UNIT, "cores": oracle.num_threads(),
           "cpu_model": cpu_model(), "kind": "oracle", "seconds": round(dt, 3),
           "sample": f"{len(rows)} seeded rows x all N={c.N} (fp64, OpenMP, Neumaier)"}
    if gpu_rows is not None:
        if den is not None:
            err = np.abs(np.asarray(gpu_rows, np.float64).reshape(o.shape) - o) / np.maximum(den, 1e-30)
            res["max_r4_err_vs_gpu"] = float(err.max())
        else:
            res["max_abs_err_vs_gpu"] = float(np.abs(np.asarray(gpu_rows, np.float64).reshape(o.shape) - o).max())
    return res


def make_inputs(w: dict, dist_kind: str):
    c = w["cfg"]
    sd = synth.seeds(c.cid)
    xk = dist_kind if w["reduction"] != "lse" else c.x_dist
    yk = dist_kind if w["reduction"] != "lse" else c.y_dist
    if c.cid == 4:
        xk = yk = "MNIST784"
    x = synth.points(xk, c.M, sd["x"], c.D)
    y = synth.points(yk, c.N, sd["y"], c.D)
    b = synth.signal(c.N, sd["b"], c.E) if w["reduction"] == "sum" else None
    return x, y, b


def run_reference(args, rank: int, world: int) -> None:
    if rank != 0:
        return
    import oracle
    oracle.set_num_threads(os.cpu_count() or 1)     # the other ranks exit: all host cores are ours
    w = workload(args.config)
    c = w["cfg"]
    x, y, b = make_inputs(w, args.dist)
    ref_pairs = args.ref_pairs or (1e9 if w["reduction"] != "argkmin" else 1e9 / c.D)
    rows_per_step = max(1, min(c.M, int(ref_pairs // c.N)))
    rng = np.random.default_rng(12345)

    def step():
        rows = np.sort(rng.choice(c.M, size=rows_per_step, replace=False))
        if w["reduction"] == "argkmin":
            oracle.argkmin(x, y, c.K, rows=rows)
        elif w["reduction"] == "lse":
            oracle.lse(x, y, None, eps=c.scale, rows=rows)
        elif w["formula"] == "gauss_sum_gradx":
            oracle.gauss_sum(x, y, b, sigma=c.scale, rows=rows)
            oracle.gauss_gradx(x, y, b, None, sigma=c.scale, rows=rows)
        elif w["formula"] == "gauss_gradx":
            oracle.gauss_gradx(x, y, b, None, sigma=c.scale, rows=rows)
        else:
            oracle.gauss_sum(x, y, b, sigma=c.scale, rows=rows)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    pairs = rows_per_step * c.N * args.steps
    value = pairs / dt
    cores = oracle.num_threads()
    sample = f"{rows_per_step} seeded rows x all N={c.N} per step (fp64 oracle, OpenMP)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": c.name, "M": c.M, "N": c.N, "D": c.D, "E": c.E, "scale": c.scale,
                   "dist": args.dist, "parallelism": "host cores (rank 0 only)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "cpu_model": cpu_model(),
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def gather_rows(dist, world: int, dev, t):
    """All-gather equal-shaped 2-D tensors from every rank; every rank gets them concatenated in
    rank order (gloo: through host memory)."""
    if world == 1:
        return t
    import torch
    if dist.get_backend() == "gloo":
        t = t.cpu()
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return torch.cat(parts, 0)


def shard_parity_sample(dist, world: int, rank: int, lo: int, res, per: int, seed: int = 777):
    """`per` seeded rows of this rank's output shard `res` (global rows lo + local), gathered to
    every rank: returns (global row indices [world*per], values [world*per, C] fp64)."""
    import torch
    Ml = res.shape[0]
    per = min(per, Ml)
    lrows = np.sort(np.random.default_rng(seed + rank).choice(Ml, size=per, replace=False))
    vals = res[torch.from_numpy(lrows).to(res.device)].to(torch.float64).reshape(per, -1)
    both = torch.cat([torch.from_numpy(lrows + lo).to(res.device, torch.float64)[:, None], vals], 1)
    both = gather_rows(dist, world, res.device, both).cpu().numpy()
    return both[:, 0].astype(np.int64), both[:, 1:]


def run_jshard(args, rank: int, world: int, local: int, w: dict) -> None:
    """j-shard mode (north star (d) "a j-sharded mode for M << N"): rank r owns
    y[rN/G:(r+1)N/G] (and b), every rank holds all M rows of x, and one step = the public
    dist.jshard_eval: the local Genred reduction, then the combine across ranks (Sum: fp64
    all_reduce; LSE: all_gather of the (m, s) states + genred_combine_lse).  Each rank draws only
    its slice of y (synth.uniform3_rows)."""
    import torch
    import torch.distributed as dist
    from paper_2004_11127_b200 import dist as gdist, genred

    c = w["cfg"]
    M, N = c.M, c.N
    sd = synth.seeds(c.cid)
    lo, hi = N * rank // world, N * (rank + 1) // world
    x = synth.uniform3(M, sd["x"])
    yl = synth.uniform3_rows(N, sd["y"], lo, hi)
    bl = synth.signal_rows(N, sd["b"], lo, hi) if w["reduction"] == "sum" else None
    dev = torch.device("cuda", local)
    xd = torch.from_numpy(x).to(dev)
    yd = torch.from_numpy(yl).to(dev)
    bd = torch.from_numpy(bl).to(dev) if bl is not None else None
    stream = torch.cuda.current_stream(dev)

    def step():
        return gdist.jshard_eval(w["formula"], w["reduction"], xd, yd, bd, None, scale=c.scale,
                                 j_offset=lo, out_dtype="float64")

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def reduce(v: float, op) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    for _ in range(args.warmup):
        res = step()
    barrier()
    plan = genred.last_plan(local)
    sampler = ClockSampler(local).start()
    genred.profile(True, local)
    l0 = genred.launch_count(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        res = step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    launches = genred.launch_count(local) - l0
    kms = genred.profile_read(local)
    genred.profile(False, local)
    barrier()
    ms_local = ev0.elapsed_time(ev1)
    ms_total = reduce(ms_local, dist.ReduceOp.MAX if world > 1 else None)
    launches = int(reduce(float(launches), dist.ReduceOp.SUM if world > 1 else None))
    ms_step = ms_total / args.steps
    value = M * N * args.steps / (ms_total * 1e-3)
    kmean_local = statistics.mean(kms) if kms else float("nan")
    kmean = reduce(kmean_local, dist.ReduceOp.MAX if world > 1 else None)
    peaks = measured_peaks()
    mhz_max = float(peaks.get("sm_max_mhz", clocks.get("sm_max_mhz") or 1965.0))
    peak = alu_peak_pairs(w["fp32"], w["mufu"], mhz_max)
    achieved = M * (hi - lo) / (kmean * 1e-3)
    roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tpair/s",
                "frac": achieved / peak, "traffic": None,
                "kernel": f"{w['formula']}/{w['reduction']} pair loop (one rank's j-slice)",
                "kernel_ms": kmean, "share_of_step": kmean / ms_step if world == 1 else None,
                "peak_basis": f"min({MUFU_PER_CLK_SM}/{w['mufu']:g} MUFU, {FP32_PER_CLK_SM}/{w['fp32']} FP32)"
                              f" pairs/clk/SM x {SMS} SMs x {mhz_max:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)",
                "pairs_per_launch": M * (hi - lo)}
    mine = [float(rank), float(lo), float(hi), float(plan["split_j"]), float(plan["rows_per_cta"]),
            float(plan["ctas"]), float(kmean_local), float(ms_local / args.steps)]
    per_rank = gather_rows(dist, world, dev, torch.tensor([mine], dtype=torch.float64, device=dev))

    # end to end: pinned host x, y-slice, b-slice -> device, jshard_eval, merged result -> host
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(x).pin_memory()
        yh = torch.from_numpy(yl).pin_memory()
        bh = torch.from_numpy(bl).pin_memory() if bl is not None else None
        oh = torch.empty(tuple(res.shape), dtype=res.dtype).pin_memory()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            xd.copy_(xh, non_blocking=True)
            yd.copy_(yh, non_blocking=True)
            if bh is not None:
                bd.copy_(bh, non_blocking=True)
            r = step()
            oh.copy_(r, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        e2e_ms = reduce(e0.elapsed_time(e1), dist.ReduceOp.MAX if world > 1 else None)
        h2d = xh.numel() * 4 + yh.numel() * 4 + (bh.numel() * 4 if bh is not None else 0)
        d2h = oh.numel() * oh.element_size()
        e2e = {"value": M * N * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(reduce(float(h2d), dist.ReduceOp.SUM if world > 1 else None)),
               "d2h_bytes_per_step": int(reduce(float(d2h), dist.ReduceOp.SUM if world > 1 else None)),
               "ms_per_step": e2e_ms / args.steps, "api": "dist.jshard_eval (public API) from pinned host buffers"}

    # parity: the merged rows against the fp64 oracle over ALL of y (rank 0 draws the full y)
    cpu = None
    if rank == 0 and not args.no_cpu:
        import oracle
        oracle.set_num_threads(os.cpu_count() or 1)
        y = synth.uniform3(N, sd["y"])
        b = synth.signal(N, sd["b"]) if w["reduction"] == "sum" else None
        rows = np.sort(np.random.default_rng(777).choice(M, size=min(args.parity_rows, M), replace=False))
        cpu = cpu_baseline(w, x, y, b, rows, gpu_rows=res.cpu().numpy()[rows])
        cpu["sample"] = f"{len(rows)} seeded rows (after the cross-rank combine) x all N={N}"

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": c.name, "M": M, "N": N, "D": c.D, "E": c.E, "scale": c.scale,
                       "dist": "x U3, y U3", "b": "U[0,1)" if bl is not None else None,
                       "parallelism": f"jshard{world}" if world > 1 else "single (j-shard path, 1 rank)",
                       "combine": "all_reduce fp64 (Sum)" if w["reduction"] == "sum"
                                  else "all_gather (m, s) + genred_combine_lse",
                       "l2": "y slice larger than L2 at G <= 8 (1.2 GB / G); no flush",
                       "split_j": plan["split_j"], "rows_per_cta": plan["rows_per_cta"], "ctas": plan["ctas"]},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches,
            "per_rank": [dict(zip(("rank", "j_lo", "j_hi", "split_j", "rows_per_cta", "ctas", "kernel_ms",
                                   "step_ms"), [int(v) if k < 6 else round(v, 4) for k, v in enumerate(r)]))
                         for r in per_rank.tolist()],
        }
        print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=0, help="BASELINE config (default 5; 7 with --mode jshard)")
    ap.add_argument("--mode", default="ishard", choices=["ishard", "jshard"],
                    help="multi-GPU partition (SURVEY.md 8(e)): i-shard (default) or j-shard (M << N)")
    ap.add_argument("--parity-rows", type=int, default=128,
                    help="N>1 / j-shard: seeded rows per rank checked against the oracle on rank 0")
    ap.add_argument("--dist", default="U3", choices=["U3", "GMM3"])
    ap.add_argument("--cpu-rows", type=int, default=0, help="oracle sample rows (cpu_baseline); 0 = auto")
    ap.add_argument("--ref-pairs", type=float, default=0, help="oracle pairs per reference step (0 = auto)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="testing only: gloo lets several ranks share one GPU (--one-device)")
    ap.add_argument("--one-device", action="store_true", help="testing only: every rank uses cuda:0")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--edge-n", type=int, default=0, help="config 6 (Cedge): N (default 8)")
    ap.add_argument("--shape", default="", help="testing only: M,N override of the config's sizes "
                    "(the line's config.workload then names the override)")
    ap.add_argument("--scale", type=float, default=0.0, help="override sigma / eps (e.g. 0.05: the "
                    "Gaussian Sum's direct form, reading R18e); config.workload names the override")
    args = ap.parse_args()
    if not args.config:
        args.config = 7 if args.mode == "jshard" else 5
    if args.mode == "jshard" and args.config not in (7, 8):
        raise SystemExit("--mode jshard runs the j-shard configs 7 (Gaussian Sum) or 8 (LSE)")
    if args.edge_n:
        if args.config != 6:
            raise SystemExit("--edge-n applies to --config 6")
        import dataclasses
        synth.CONFIGS[6] = dataclasses.replace(synth.CONFIGS[6], N=args.edge_n,
                                               name=f"Cedge Gaussian Sum M=2^28 N={args.edge_n} D=3 E=1 sigma=0.5 (HBM-bound)")

    if args.shape:
        import dataclasses
        Mo, No = (int(float(v)) for v in args.shape.split(","))
        c0 = synth.CONFIGS[args.config]
        synth.CONFIGS[args.config] = dataclasses.replace(c0, M=Mo, N=No,
                                                         name=f"{c0.name} [test override M={Mo} N={No}]")
    if args.scale:
        import dataclasses
        c0 = synth.CONFIGS[args.config]
        synth.CONFIGS[args.config] = dataclasses.replace(c0, scale=args.scale,
                                                         name=f"{c0.name} [scale override {args.scale}]")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2004_11127_b200 import genred

    if args.one_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            # communicator evidence: NCCL's INIT lines name every rank ("nranks N") in the log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    w = workload(args.config)
    c = w["cfg"]
    if args.mode == "jshard":
        run_jshard(args, rank, world, local, w)
        if world > 1:
            dist.destroy_process_group()
        return
    M, N = c.M, c.N
    # i-shard rows: boundaries on the 1024-row tile (dist.ISHARD_ALIGN), so the shards' rows are
    # bitwise the unsharded ones for the same j-split
    from paper_2004_11127_b200.dist import ISHARD_ALIGN, shard_range
    lo, hi = shard_range(M, world, rank, align=ISHARD_ALIGN)
    x, y, b = make_inputs(w, args.dist)
    xl = np.ascontiguousarray(x[lo:hi])
    dev = torch.device("cuda", local)
    xd = torch.from_numpy(xl).to(dev)
    yd = torch.from_numpy(y).to(dev) if rank == 0 else torch.empty(y.shape, dtype=torch.float32, device=dev)
    bd = None
    if b is not None:
        bd = torch.from_numpy(b).to(dev) if rank == 0 else torch.empty(b.shape, dtype=torch.float32, device=dev)
    Ml = hi - lo
    argk = w["reduction"] == "argkmin"
    out_shape = (Ml,) if w["reduction"] == "lse" else ((Ml, c.K) if argk else
                                                       ((Ml, c.D) if w["formula"] == "gauss_gradx" else (Ml, c.E)))
    out = torch.empty(out_shape, dtype=getattr(torch, w["out_dtype"]), device=dev)
    out_idx = torch.empty((Ml, c.K), dtype=torch.int64, device=dev) if argk else None
    out_grad = torch.empty((Ml, c.D), dtype=torch.float32, device=dev) \
        if w["formula"] == "gauss_sum_gradx" else None
    stream = torch.cuda.current_stream(dev)

    # the call is marshalled once (genred.prepare); each step is then one genred_eval through the
    # C ABI on the resident buffers, with no per-step Python argument building (C1 is
    # launch-latency bound and the binding's marshalling alone costs ~6 us per call)
    step_args, _, _keep = genred.prepare(w["formula"], w["reduction"], xd, yd, bd, None, scale=c.scale,
                                         K=c.K, out=out, out_dtype=w["out_dtype"], out_grad=out_grad,
                                         out_idx=out_idx, j_offset=0)

    call = genred.bound_call(step_args, stream, local)   # ctypes arguments converted once

    def step():
        if world > 1:                                   # X1: y (and b) broadcast once per step
            dist.broadcast(yd, src=0)
            if bd is not None:
                dist.broadcast(bd, src=0)
        call()

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---------------- device-resident timed region ----------------
    # Per-kernel CUDA events (genred_profile) time the dominant kernel for the roofline.  For
    # steps of >= 5 ms they are recorded inside the timed region itself; for launch-bound steps
    # (C1: ~6 us of device time per call) two extra events per call would inflate the step they
    # measure, so the timed region runs without them and the same K steps are then re-run with
    # them (the "kernel_timing" key says which).
    for _ in range(args.warmup):
        step()
    barrier()
    # the decision times the LAST warm-up step only (the first call allocates scratch)
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0.record(stream)
    step()
    w1.record(stream)
    barrier()
    inline_prof = max_over_ranks(w0.elapsed_time(w1)) >= 5.0
    plan = genred.last_plan(local)
    tiles = genred.last_tiles(local) if plan.get("path") == 3 else (0, 0)
    sampler = ClockSampler(local)
    if not os.environ.get("BENCH_NO_SAMPLER"):
        sampler.start()
    genred.profile(inline_prof, local)
    l0 = genred.launch_count(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    launches = genred.launch_count(local) - l0
    if not inline_prof:
        barrier()
        genred.profile(True, local)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize(dev)
    kms = genred.profile_read(local)
    genred.profile(False, local)
    barrier()
    kernel_timing = ("CUDA events around the main kernel inside the timed region" if inline_prof else
                     "CUDA events around the main kernel over a second pass of the same K steps "
                     "(the timed region runs without per-kernel events: the step is launch-bound)")
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    launches = int(sum_over_ranks(launches))
    ms_step = ms_total / args.steps
    value = M * N * args.steps / (ms_total * 1e-3)

    # dominant kernel roofline (this rank's launches; the slowest rank bounds the job)
    kmean_local = statistics.mean(kms) if kms else float("nan")
    kmean = max_over_ranks(kmean_local)
    peaks = measured_peaks()
    mhz_max = float(peaks.get("sm_max_mhz", clocks.get("sm_max_mhz") or 1965.0))
    if argk:
        plan["fallback_rows"] = genred.last_plan(local)["fallback_rows"]
    traffic = ncu_traffic(args.config, N)
    if argk:
        # tensor-bound: 3xTF32 = three tf32 GEMMs of 2*M*N*D flops each, against the measured
        # bf16 dense peak x the nominal tf32/bf16 ratio 1/2 (B200_PROFILING.md)
        bf16 = float(peaks.get("bf16_tflops", 1590.0))
        peak_t = bf16 * 0.5
        flops = 3 * 2.0 * Ml * N * c.D
        achieved_t = flops / (kmean * 1e-3) / 1e12
        roofline = {"bound": "tensor", "achieved": achieved_t, "peak": peak_t, "unit": "TFLOP/s",
                    "frac": achieved_t / peak_t, "traffic": traffic,
                    "kernel": "knn_tc_kernel (tcgen05 kind::tf32, 3xTF32)", "kernel_ms": kmean,
                    "share_of_step": kmean / ms_step if world == 1 else None,
                    "peak_basis": f"bf16_tflops {bf16:.1f} (MEASURED_PEAKS.json, burst) x 0.5 (tf32/bf16 nominal)",
                    "flops_per_launch": flops, "exact_fp32_equivalent_flops": 2.0 * Ml * N * c.D}
    elif w.get("hbm"):
        # HBM-bound edge: algorithmic bytes = x read (D fp32) + a written (E fp32) per row, plus
        # the packed j-records once (L2-resident afterwards)
        hbm = float(peaks.get("hbm_gbs", 6541.0))
        nbytes = Ml * (c.D + c.E) * 4 + N * (c.D + 1 + c.E) * 4
        achieved_b = nbytes / (kmean * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": achieved_b, "peak": hbm, "unit": "GB/s",
                    "frac": achieved_b / hbm, "traffic": traffic,
                    "kernel": "gauss/sum pair loop (direct form, tiny N)", "kernel_ms": kmean,
                    "share_of_step": kmean / ms_step if world == 1 else None,
                    "peak_basis": "HBM copy bandwidth (MEASURED_PEAKS.json)",
                    "bytes_per_launch": nbytes}
    else:
        # the Gaussian Sum's form is decided on the device (bounding box, reading R18b): the
        # direct form on raw differences runs 8 FP32 lane-ops per pair instead of 4 (same peak)
        if w["formula"] == "gauss" and plan.get("path") == 0 and not w.get("hbm"):
            w = dict(w, fp32=8, mufu=1)                      # (no polynomial share in the direct form)
        peak = alu_peak_pairs(w["fp32"], w["mufu"], mhz_max)
        basis_extra = ""
        if w["formula"] in ("gauss", "sqdist") and plan.get("path") == 3:
            # tile-centred form (R18j): centred tiles run the expanded mix (Sum: 4 FP32 lane-ops
            # + 1 of the polynomial exp share, 7/8 MUFU; LSE: FADD + 3 FFMA + 1 accumulate, 1
            # MUFU), the others the direct one (8 FP32 + 1 MUFU); the ceiling is the
            # pair-weighted harmonic mix of the two
            f_loc = tiles[0] / max(tiles[1], 1)
            loc_mix = (5, 7 / 8) if w["formula"] == "gauss" else (5, 1)
            p_loc = alu_peak_pairs(*loc_mix, mhz_max)
            p_dir = alu_peak_pairs(8, 1, mhz_max)
            peak = 1.0 / (f_loc / p_loc + (1.0 - f_loc) / p_dir)
            w = dict(w, fp32=loc_mix[0], mufu=loc_mix[1])
            basis_extra = (f"; tile-centred form: {tiles[0]} of {tiles[1]} tiles centred (this mix), "
                           f"the rest direct (16/1 MUFU, 128/8 FP32), harmonic mix")
        achieved = Ml * N / (kmean * 1e-3)
        roofline = {"bound": "alu", "achieved": achieved / 1e12, "peak": peak / 1e12, "unit": "Tpair/s",
                    "frac": achieved / peak, "traffic": traffic,
                    "kernel": f"{w['formula']}/{w['reduction']} pair loop", "kernel_ms": kmean,
                    "share_of_step": kmean / ms_step if world == 1 else None,
                    "peak_basis": f"min({MUFU_PER_CLK_SM}/{w['mufu']:g} MUFU, {FP32_PER_CLK_SM}/{w['fp32']} FP32)"
                                  f" pairs/clk/SM x {SMS} SMs x {mhz_max:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)"
                                  + basis_extra,
                    "pairs_per_launch": Ml * N}

    roofline["kernel_timing"] = kernel_timing

    # ---------------- end-to-end: host buffers through the C ABI (H2D + D2H inside) ----------------
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(xl).pin_memory()
        yh = torch.from_numpy(y).pin_memory()
        bh = torch.from_numpy(b).pin_memory() if b is not None else None
        oh = torch.empty(out_shape, dtype=getattr(torch, w["out_dtype"])).pin_memory()
        gh = torch.empty((Ml, c.D), dtype=torch.float32).pin_memory() if out_grad is not None else None
        ih = torch.empty((Ml, c.K), dtype=torch.int64).pin_memory() if argk else None
        a = genred.Args()
        a.abi_version = genred.ABI_VERSION
        a.formula, a.reduction = genred.FORMULAS[w["formula"]], genred.REDUCTIONS[w["reduction"]]
        a.memory = genred.MEM_HOST
        a.M, a.N, a.D, a.E, a.K, a.scale = Ml, N, c.D, c.E, 1, c.scale
        a.x, a.y = xh.data_ptr(), yh.data_ptr()
        a.b = bh.data_ptr() if bh is not None else None
        a.out = oh.data_ptr()
        a.out_dtype = genred.F64 if w["out_dtype"] == "float64" else genred.F32
        a.out_grad = gh.data_ptr() if gh is not None else None
        a.out_idx = ih.data_ptr() if ih is not None else None
        a.K = c.K
        genred.eval_args(a, stream=stream)                      # warm the staging buffers
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            genred.eval_args(a, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        e2e_ms = max_over_ranks(e0.elapsed_time(e1))
        h2d = xh.numel() * 4 + yh.numel() * 4 + (bh.numel() * 4 if bh is not None else 0)
        d2h = oh.numel() * oh.element_size() + (gh.numel() * 4 if gh is not None else 0) + \
            (ih.numel() * 8 if ih is not None else 0)
        e2e = {"value": M * N * args.steps / (e2e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(sum_over_ranks(h2d)),
               "d2h_bytes_per_step": int(sum_over_ranks(d2h)),
               "ms_per_step": e2e_ms / args.steps, "api": "genred_eval(memory=GENRED_MEM_HOST)"}

    # ---------------- per-rank plan and main-kernel time (all ranks -> rank 0) ----------------
    mine = [float(rank), float(lo), float(hi), float(plan["split_j"]), float(plan["rows_per_cta"]),
            float(plan["ctas"]), float(kmean_local), float(ev0.elapsed_time(ev1) / args.steps)]
    per_rank = gather_rows(dist, world, dev, torch.tensor([mine], dtype=torch.float64, device=dev))
    per_rank = [dict(zip(("rank", "row_lo", "row_hi", "split_j", "rows_per_cta", "ctas", "kernel_ms",
                          "step_ms"), [int(v) if k < 6 else round(v, 4) for k, v in enumerate(r)]))
                for r in per_rank.tolist()]

    # ---------------- fp64 oracle on the host cores ----------------
    # N = 1: a row sample sized for ~15 s of host work.  N > 1: `--parity-rows` seeded rows from
    # EACH rank's shard are gathered to rank 0 and checked there, so every sharded line carries
    # its own parity evidence (the oracle's rows/s is then timed on that sample).
    cpu = None
    if not args.no_cpu:
        res = (out_idx if argk else out)
        if world == 1:
            nrows = args.cpu_rows or max(16, min(M, 4_000_000, int(3e10 // (N * (c.D if argk else 1)))))
            rows = np.sort(np.random.default_rng(777).choice(M, size=min(nrows, M), replace=False))
            gpu_rows = res.cpu().numpy()[rows]
        else:
            per = min(args.parity_rows, Ml)
            rows, gpu_rows = shard_parity_sample(dist, world, rank, lo, res, per)
            if argk:
                gpu_rows = gpu_rows.astype(np.int64)
        if rank == 0:
            import oracle
            oracle.set_num_threads(os.cpu_count() or 1)
            cpu = cpu_baseline(w, x, y, b, rows, gpu_rows=gpu_rows)
            if world > 1:
                cpu["sample"] = f"{per} seeded rows of each of the {world} shards (all gathered to rank 0) x all N={N}"

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": c.name, "M": M, "N": N, "D": c.D, "E": c.E, "scale": c.scale,
                       "dist": ("MNIST784" if argk else args.dist) if w["reduction"] != "lse"
                               else f"x {c.x_dist}, y {c.y_dist}",
                       "b": "U[0,1)" if b is not None else None,
                       "parallelism": f"ishard{world}" if world > 1 else "single",
                       "l2": ("inputs larger than L2 (280 MB vs 126 MB); no flush" if c.cid == 5 else
                              "x larger than L2 (3.2 GB vs 126 MB); no flush") if c.cid in (5, 6) else
                             "inputs re-read from HBM/L2 each step; no flush",
                       "split_j": plan["split_j"], "rows_per_cta": plan["rows_per_cta"],
                       "ctas": plan["ctas"], "K": c.K if argk else None,
                       "form": {0: "direct", 1: "tensor", 2: "expanded",
                                3: f"tile-centred ({tiles[0]} of {tiles[1]} tiles)"}.get(plan.get("path")),
                       "fallback_rows": plan.get("fallback_rows")},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches,
        }
        if world > 1:
            line["per_rank"] = per_rank
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
