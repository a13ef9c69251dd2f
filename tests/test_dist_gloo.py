"""Multi-process (world_size 2, gloo, CPU) tests of the i-shard / j-shard orchestration in
paper_2004_11127_b200/dist.py: partition ranges, broadcast/all-gather wiring, j_offset and the
monoid merges.  The per-rank evaluator and the combiners are host stand-ins
built on the fp64 oracle (the GPU kernels are covered by tests/test_gpu_parity.py), so this
checks the plumbing, not the kernels."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

LN2 = math.log(2.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_fns():
    import oracle

    def ev(formula, reduction, x, y, b=None, g=None, *, scale=1.0, K=1, out_dtype="float32",
           lse_state=None, j_offset=0, **kw):
        X, Y = x.numpy(), y.numpy()
        if reduction == "sum":
            a, _ = oracle.gauss_sum(X, Y, None if b is None else b.numpy(), sigma=scale)
            return torch.from_numpy(a)
        if reduction == "lse":
            a, m = oracle.lse(X, Y, None if b is None else b.numpy(), eps=scale)
            if lse_state is not None:
                lse_state[:, 0] = torch.from_numpy(m / LN2)
                lse_state[:, 1] = torch.from_numpy(np.exp(a - m))
            return torch.from_numpy(a)
        d, j = oracle.argkmin(X, Y, K)
        j = np.where(j >= 0, j + j_offset, -1)
        return torch.from_numpy(d.astype(np.float32)), torch.from_numpy(j)

    def combine(states, out_dtype="float64"):
        S = states.numpy()
        m = S[:, :, 0].max(0)
        s = (S[:, :, 1] * np.exp2(S[:, :, 0] - m)).sum(0)
        return torch.from_numpy(LN2 * (m + np.log2(s)))

    def merge(d, j):
        G, M, K = d.shape
        D, J = d.numpy(), j.numpy()
        od = np.full((M, K), np.inf, np.float32); oj = np.full((M, K), -1, np.int64)
        for i in range(M):
            cand = sorted((float(D[g, i, k]), int(J[g, i, k])) for g in range(G) for k in range(K) if J[g, i, k] >= 0)
            for k, (dd, jj) in enumerate(cand[:K]):
                od[i, k], oj[i, k] = dd, jj
        return torch.from_numpy(od), torch.from_numpy(oj)

    return {"eval": ev, "combine_lse": combine, "merge_topk": merge}


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import synth
        from paper_2004_11127_b200.dist import dist_eval, ishard_eval, jshard_eval, shard_range
        fns = _cpu_fns()
        M, N = 37, 53
        x = torch.from_numpy(synth.uniform3(M, 1)); y = torch.from_numpy(synth.gmm3(N, 2))
        b = torch.from_numpy(synth.signal(N, 3))
        # i-shard: y, b only valid on rank 0 before the broadcast
        lo, hi = shard_range(M, world, rank)
        yb = y.clone() if rank == 0 else torch.zeros_like(y)
        bb = b.clone() if rank == 0 else torch.zeros_like(b)
        a_i = ishard_eval("gauss", "sum", x[lo:hi].contiguous(), yb, bb, scale=0.5, fns=fns, gather=True)
        # j-shard
        jlo, jhi = shard_range(N, world, rank)
        ys, bs = y[jlo:jhi].contiguous(), b[jlo:jhi].contiguous()
        a_s = dist_eval("gauss", "sum", x, ys, bs, mode="jshard", scale=0.5, fns=fns, out_dtype="float64")
        a_l = jshard_eval("sqdist", "lse", x, ys, None, scale=0.05, fns=fns)
        d_k, j_k = jshard_eval("sqdist", "argkmin", x, ys, K=4, j_offset=jlo, fns=fns)
        # bench.py's j-shard inputs: each rank draws only its slice of y (PCG64 advance)
        assert np.array_equal(synth.uniform3_rows(N, 5, jlo, jhi), synth.uniform3(N, 5)[jlo:jhi])
        # bench.py's N > 1 parity sample: seeded rows of each rank's shard, gathered in rank order
        import bench
        full = torch.arange(M * 2, dtype=torch.float32).reshape(M, 2)
        rows, vals = bench.shard_parity_sample(dist, world, rank, lo, full[lo:hi].contiguous(), per=5)
        plan = bench.gather_rows(dist, world, None, torch.tensor([[float(rank), float(hi - lo)]], dtype=torch.float64))
        q.put((rank, a_i.numpy(), a_s.numpy(), a_l.numpy(), d_k.numpy(), j_k.numpy(), rows, vals,
               plan.numpy()))
    finally:
        dist.destroy_process_group()


def test_ishard_jshard_world2():
    import oracle
    import synth
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    M, N = 37, 53
    x = synth.uniform3(M, 1); y = synth.gmm3(N, 2); b = synth.signal(N, 3)
    a_ref, _ = oracle.gauss_sum(x, y, b, sigma=0.5)
    l_ref, _ = oracle.lse(x, y, None, eps=0.05)
    d_ref, j_ref = oracle.argkmin(x, y, 4)
    full = np.arange(M * 2, dtype=np.float64).reshape(M, 2)
    for rank, a_i, a_s, a_l, d_k, j_k, rows, vals, plan in res:
        assert len(rows) == 5 * world and len(set(rows.tolist())) == 5 * world
        for r in range(world):                                        # 5 rows from each shard
            lo, hi = M * r // world, M * (r + 1) // world
            assert np.all((rows[5 * r:5 * r + 5] >= lo) & (rows[5 * r:5 * r + 5] < hi))
        np.testing.assert_array_equal(vals, full[rows])
        np.testing.assert_array_equal(plan[:, 0], np.arange(world))
        np.testing.assert_array_equal(a_i, a_ref)                      # i-shard: same rows, same numbers
        np.testing.assert_allclose(a_s, a_ref, rtol=1e-13)            # j-shard Sum: fp64 all-reduce
        np.testing.assert_allclose(a_l, l_ref, rtol=0, atol=1e-12)    # j-shard LSE: max-rescale merge
        np.testing.assert_array_equal(j_k, j_ref)                     # j-shard ArgKMin: offsets + merge
        np.testing.assert_allclose(d_k, d_ref.astype(np.float32))


def test_shard_range_partitions():
    from paper_2004_11127_b200.dist import shard_range
    for n in (0, 1, 7, 10_000_000):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[k][1] == rs[k + 1][0] for k in range(w - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
