"""Multi-rank (N > 1) host logic on CPU, world_size 2 over gloo.

The device path shards A by rows: rank p owns rows
[p·rpr, (p+1)·rpr) of A (rpr a multiple of 256), each pass computes its rows of
A·V in two K windows -- its own operand chunk while the all-gather of the others is in
flight, then the rest -- all-gathers the next fp16 operand planes laid out [world][s][rpr] with
each rank's per-column maxima in a tail of its chunk (merged after the gather, so every rank picks
the same plane scale without a separate all-reduce) and sum-reduces the
row-separable fp64 trace partials once per estimate; CholeskyQR2/projection Grams are
sum-reduced. These tests run that exact protocol with the fp64 oracle as the compute
and torch.distributed (gloo) as the transport, and check it against the unsharded
oracle; the device implementation of the same protocol is exercised on one GPU by
tests/test_gpu_sharded.py.
"""
import math
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def test_shard_rows_partition(R):
    for n in (2, 255, 256, 1000, 100000, 400001):
        for world in (1, 2, 3, 4, 8):
            spans = [R.shard_rows(n, world, r) for r in range(world)]
            rpr = spans[0][2]
            assert rpr % 256 == 0 and all(s[2] == rpr for s in spans)
            cover = 0
            for r, (row0, rows, _) in enumerate(spans):
                assert row0 == min(n, r * rpr) and rows >= 0
                assert row0 == cover
                cover += rows
            assert cover == n
            if world == 1:
                assert spans[0] == (0, n, ((n + 255) // 256) * 256)
    with pytest.raises(R.RenyiError):
        R.shard_rows(10, 2, 2)


def _worker(rank, world, port, n, out_path):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch

    import paper_2205_07426_b200 as R
    from oracle import oracle as orc

    x = orc.fill_gaussian(5, n, 6)
    a = orc.build_kernel(x, math.sqrt(6.0))
    row0, rows, rpr = R.shard_rows(n, world, rank)
    a_p = a[row0:row0 + rows, :]  # this rank's rows of A
    s_q, s_g, m, alpha = 4, 10, 20, 1.5
    # probes: every rank draws only its rows, from the same per-column streams
    S_full = R.gaussian_panel(n, s_q, 3, "hutchpp-sketch")
    G_full = R.gaussian_panel(n, s_g, 3, "hutchpp-probe")
    S, G = S_full[row0:row0 + rows], G_full[row0:row0 + rows]

    own = np.arange(row0, row0 + rows)
    rest = np.r_[np.arange(row0 + rows, n), np.arange(0, row0)]  # the other chunks, wrapping at n

    def product(local, cols, colmax=None):
        """A_p · V with the device schedule: the all-gather of V's chunks (each with a tail carrying the
        rank's column maxima of V) in flight while the rank's own K window (its own chunk) is
        multiplied, then the other window once the gather lands. Returns (A_p V, max over ranks of
        the column maxima) -- the maxima need no all-reduce of their own."""
        chunk = torch.zeros((cols, rpr + 1), dtype=torch.float64)
        chunk[:, :rows] = torch.from_numpy(np.ascontiguousarray(local.T))
        if colmax is not None:
            chunk[:, rpr] = torch.from_numpy(np.asarray(colmax, dtype=np.float64))
        planes = [torch.zeros_like(chunk) for _ in range(world)]
        work = dist.all_gather(planes, chunk, async_op=True)
        y = a_p[:, own] @ local  # own window: no remote data needed
        work.wait()
        full = torch.cat([p[:, :rpr] for p in planes], dim=1)[:, :n].numpy().T
        merged = np.max(np.stack([p[:, rpr].numpy() for p in planes]), axis=0)
        return y + a_p[:, rest] @ full[rest], merged  # second window summed after the first (epilogue order)

    def allreduce(arr, op=dist.ReduceOp.SUM):
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64))
        dist.all_reduce(t, op=op)
        return t.numpy()

    # sketch pass and CholeskyQR2 with summed Grams
    Y, _ = product(S, s_q)
    g = allreduce(Y.T @ Y)
    w, v = np.linalg.eigh(g)
    keep = w > 1e-13 * w.max()
    Q1 = Y @ (v[:, keep] / np.sqrt(w[keep]))
    r2 = np.linalg.cholesky(allreduce(Q1.T @ Q1)).T
    Q = Q1 @ np.linalg.inv(r2)
    W = G - Q @ allreduce(Q.T @ G)
    X0 = np.hstack([Q, W])
    # Chebyshev passes on [0,1]: T_{k+1} = 2(2 A T_k - T_k) - T_{k-1}; per-pass column maxima
    c, safe_v = orc.spec_coeffs(orc.Spec("chebyshev", alpha, m, 0.0, 1.0))
    scale, center = 2.0 / safe_v, 1.0
    dots = [allreduce(np.einsum("ij,ij->j", X0, X0))]
    ax0, _ = product(X0, X0.shape[1])
    tp, tc = X0, scale * ax0 - center * X0
    local_dots = [np.einsum("ij,ij->j", X0, tc)]
    colmax = np.abs(tc).max(axis=0) if rows else np.zeros(X0.shape[1])
    for _ in range(2, m + 1):
        atc, cmax = product(tc, tc.shape[1], colmax)  # cmax: global maxima of tc, gathered with tc
        assert np.array_equal(cmax, allreduce(colmax, dist.ReduceOp.MAX))
        tn = 2 * (scale * atc - center * tc) - tp
        local_dots.append(np.einsum("ij,ij->j", X0, tn))
        colmax = np.abs(tn).max(axis=0)
        tp, tc = tc, tn
    dots += [allreduce(d) for d in local_dots]  # one reduction per estimate in the device path
    tr = 0.5 * c[0] * dots[0] + sum(c[k] * dots[k] for k in range(1, m + 1))
    k_rank = int(keep.sum())
    value = tr[:k_rank].sum() + tr[k_rank:].sum() / s_g
    np.save(out_path.format(rank=rank), np.array([value, k_rank, cmax.max()]))
    dist.destroy_process_group()


def test_gloo_world2_sharded_protocol_matches_unsharded(tmp_path):
    from oracle import oracle as orc

    import paper_2205_07426_b200 as R

    n = 600  # rpr = 512: rank 1 holds a short last chunk
    out = str(tmp_path / "r{rank}.npy")
    port = 29500 + os.getpid() % 1000
    mp.start_processes(_worker, args=(2, port, n, out), nprocs=2, join=True, start_method="spawn")
    v0, v1 = np.load(out.format(rank=0)), np.load(out.format(rank=1))
    assert np.array_equal(v0, v1)  # identical on every rank
    x = orc.fill_gaussian(5, n, 6)
    a = orc.build_kernel(x, math.sqrt(6.0))
    ref = orc.hutchpp(orc.Spec("chebyshev", 1.5, 20, 0.0, 1.0), a, 4, 10,
                      sketch=R.gaussian_panel(n, 4, 3, "hutchpp-sketch"),
                      probes=R.gaussian_panel(n, 10, 3, "hutchpp-probe"))
    assert int(v0[1]) == ref["sketch_rank"]
    assert abs(v0[0] - ref["value"]) <= 1e-10 * abs(ref["value"])


def test_bench_reference_arm_under_torchrun_gloo():
    """bench.py --impl reference under a 2-rank launch: rank 0 prints one JSON line, rank 1 exits 0."""
    port = 28500 + os.getpid() % 1000
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), "--impl",
           "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--samples", "3000"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    import json

    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 0
