"""Multi-GPU Genred: one process per GPU, torch.distributed (NCCL) for the plumbing.

SURVEY.md Sec. 8(e).  Eq. (1) shards along either axis:

* ``ishard_eval`` (default, north star (d)): rank r owns rows [rM/G, (r+1)M/G) of x; y and b are
  broadcast once from ``src`` (collective X1) and every rank runs libgenred on its rows.  No
  reduction is needed.  Per-row arithmetic is bitwise that of the single-GPU run only when every
  shard runs the same j-split (pass the same ``split_j`` to all ranks: the automatic planner
  chooses it from the local M), the shard boundaries are multiples of ``ISHARD_ALIGN`` rows
  (``shard_range(M, G, r, align=ISHARD_ALIGN)``) and every shard takes the same form (shards of a
  problem with max(M, N) > 4096 all take the pair-loop kernels; the one-launch small-problem path
  takes the direct form).
* ``jshard_eval`` (M << N): rank r owns [rN/G, (r+1)N/G) of y and b; every rank reduces all M rows
  over its slice and the monoid states are merged:
    Sum      fp64 partials -> all_reduce(SUM)                                        (X3)
    LSE      (m, s) states -> all_gather -> genred_combine_lse (max-rescale)           (X4)
    ArgKMin  K (d, j) per row with j_offset -> all_gather -> genred_merge_topk          (X5)

The evaluator and combiners default to the libgenred binding; the CPU (gloo) tests inject
host-side stand-ins to exercise the partitioning and collective wiring without a GPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


# Row tile of the Sum / LSE row-tile kernels (8 warps x 32 threads x 4 rows).  A row's arithmetic
# depends on its slot in its row tile (the expanded Gaussian Sum evaluates the exponentials of the
# last row slot of a thread on the FP32 pipe for every other record pair), so i-shards whose
# boundaries are multiples of it compute their rows bitwise as the unsharded call does (given the
# same j-split).
ISHARD_ALIGN = 1024


def shard_range(n: int, world: int, rank: int, align: int = 1) -> tuple:
    """Contiguous shard [lo, hi) of n items for `rank` of `world`, balanced to within `align` items,
    with every boundary but the last a multiple of `align`."""
    def b(r):
        return n if r >= world else min(n, (n * r // world) // align * align)
    return b(rank), b(rank + 1)


def _default_fns():
    from . import genred
    return {"eval": genred.eval, "combine_lse": genred.combine_lse, "merge_topk": genred.merge_topk}


def ishard_eval(formula: str, reduction: str, x_local, y, b=None, g_local=None, *, scale=1.0, K=1,
                src: int = 0, group=None, fns=None, gather: bool = False, **kw):
    """Evaluate this rank's rows.  ``y``/``b`` must be allocated on every rank; they are
    broadcast from ``src`` first.  With gather=True the full output is all-gathered (X2)."""
    fns = fns or _default_fns()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(y, src=src, group=group)
        if b is not None:
            dist.broadcast(b, src=src, group=group)
    res = fns["eval"](formula, reduction, x_local, y, b, g_local, scale=scale, K=K, **kw)
    if not gather or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return res
    outs = res if isinstance(res, tuple) else (res,)
    gathered = []
    world = dist.get_world_size(group)
    for t in outs:
        # shards differ by at most one row: pad to the largest, gather, trim (gloo and NCCL both
        # want equal sizes)
        sizes = [torch.zeros(1, dtype=torch.int64, device=t.device) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device), group=group)
        sizes = [int(v.item()) for v in sizes]
        mx = max(sizes)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad, group=group)
        gathered.append(torch.cat([p[:n] for p, n in zip(parts, sizes)], 0))
    return tuple(gathered) if isinstance(res, tuple) else gathered[0]


def jshard_eval(formula: str, reduction: str, x, y_local, b_local=None, g=None, *, scale=1.0, K=1,
                j_offset: int = 0, group=None, fns=None, out_dtype: str = "float32"):
    """Reduce all rows of x over this rank's slice of y, then merge across ranks."""
    fns = fns or _default_fns()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    M = x.shape[0]
    if reduction == "sum":
        part = fns["eval"](formula, reduction, x, y_local, b_local, g, scale=scale, out_dtype="float64")
        parts = part if isinstance(part, tuple) else (part,)
        for t in parts:
            if world > 1:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        if out_dtype == "float32":
            parts = tuple(t.float() for t in parts)
        return parts if isinstance(part, tuple) else parts[0]
    if reduction == "lse":
        state = torch.empty((M, 2), dtype=torch.float64, device=x.device)
        fns["eval"](formula, reduction, x, y_local, b_local, None, scale=scale, out_dtype="float64",
                    lse_state=state)
        states = [torch.empty_like(state) for _ in range(world)]
        if world > 1:
            dist.all_gather(states, state, group=group)
        else:
            states = [state]
        return fns["combine_lse"](torch.stack(states), out_dtype=out_dtype)
    if reduction == "argkmin":
        d, j = fns["eval"](formula, reduction, x, y_local, None, None, K=K, j_offset=j_offset)
        ds = [torch.empty_like(d) for _ in range(world)]
        js = [torch.empty_like(j) for _ in range(world)]
        if world > 1:
            dist.all_gather(ds, d, group=group)
            dist.all_gather(js, j, group=group)
        else:
            ds, js = [d], [j]
        return fns["merge_topk"](torch.stack(ds), torch.stack(js))
    raise ValueError(reduction)


def dist_eval(formula: str, reduction: str, x, y, b=None, g=None, *, mode: str = "ishard", **kw):
    """SURVEY.md 8(b)'s ``genred.dist_eval``: ``mode="ishard"`` -> ishard_eval (x: this rank's
    rows, y/b broadcast from ``src``), ``mode="jshard"`` -> jshard_eval (y/b: this rank's j-slice,
    partial results merged across ranks)."""
    if mode == "ishard":
        return ishard_eval(formula, reduction, x, y, b, g, **kw)
    if mode == "jshard":
        return jshard_eval(formula, reduction, x, y, b, g, **kw)
    raise ValueError(f"mode must be 'ishard' or 'jshard', not {mode!r}")
