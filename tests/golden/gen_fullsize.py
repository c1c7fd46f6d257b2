#!/usr/bin/env python
"""Generates tests/golden/fullsize.json: fp64 oracle results for BASELINE.json's configurations
at their FULL sizes (n = 20k, 50k, 100k, 400k), for tests/test_gpu_fullsize_parity.py.

TEST INFRASTRUCTURE. Runs once, on this container's host cores (hours of CPU for config 4):

    ORACLE_NATIVE=1 python tests/golden/gen_fullsize.py [c2 c3 c5 c4]

Inputs are the seeded synthetic workloads (workloads.py, reference RNG drawn through the oracle,
so the GPU box regenerates them bit for bit through the product library). Config 2 runs the
oracle's dense estimator (A = 3.2 GB fp64, the reference's own cost structure); configs 3-5 run
the same restated estimator over KernelBlocksOp, which recomputes kernel entries block by block
(the fp64 A would be 20 GB, 80 GB x 3 and 1.28 TB). Probes are the reference's seeded streams
(hutchpp.cpp:13-22, Rademacher for config 2 per BASELINE.json) — the device draws the same
streams (Gaussian ones with CUDA's log/sin/cos, <= 2 ulp from glibc).
"""
from __future__ import annotations

import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from workloads import bf16, f32, gaussian, mi_inputs, mixture10  # noqa: E402

SEED = 2205  # bench.py's default seed: the bench's config-4/5 results are comparable too
OUT = Path(__file__).resolve().parent / "fullsize.json"
PROBE_COLS = 4  # per-probe quadratic forms x^T f(A) x on these seeded Gaussian columns


def _load():
    return json.loads(OUT.read_text()) if OUT.exists() else {}


def _save(key, rec):
    d = _load()
    d[key] = rec
    OUT.write_text(json.dumps(d, indent=1, sort_keys=True) + "\n")


def _est(e):
    keep = ("entropy", "trace", "low_rank_part", "residual_part", "sketch_rank", "queries_used", "u", "v",
            "iterations_used", "s", "m", "method")
    return {k: e[k] for k in keep}


def c2():
    n, d = 20000, 32
    x = f32(gaussian(n, d, SEED, "X", "oracle"))
    sigma = math.sqrt(d)
    params = dict(alpha=1.5, method="chebyshev", s=60, m=40, seed=SEED, bounds=(0.0, 1.0),
                  probe_kind="rademacher", s_q=20, s_g=40)
    t = time.time()
    a = O.build_kernel(x, sigma)
    est = O.estimate(a, **params)
    probes = O.probe_panel(n, PROBE_COLS, SEED, "fullsize-probe")
    traces = O.apply_panel(O.Spec("chebyshev", 1.5, 40, 0.0, 1.0), a, probes)
    qf = [float(probes[:, j] @ traces[:, j]) for j in range(PROBE_COLS)]
    del a
    return dict(n=n, d=d, sigma=sigma, seed=SEED, inputs="X = f32(gaussian(n, d, seed, 'X'))", precision="fp32",
                params={k: v for k, v in params.items()}, estimate=_est(est),
                probe_label="fullsize-probe", probe_spec=["chebyshev", 1.5, 40, 0.0, 1.0], probe_traces=qf,
                oracle="dense (reference cost structure)", seconds=time.time() - t)


def c3():
    n, d = 50000, 64
    x = f32(mixture10(n, d, SEED, "oracle"))
    sigma = math.sqrt(d)
    params = dict(alpha=0.5, method="taylor", s=100, m=30, seed=SEED, probe_kind="gaussian", s_q=0, s_g=100)
    t = time.time()
    op = O.KernelBlocksOp(x, sigma)
    est = op.estimate(**params)
    probes = O.probe_panel(n, PROBE_COLS, SEED, "fullsize-probe")
    spec = ["taylor", 0.5, 30, 0.0, est["v"]]
    qf = op.matfun_traces(O.Spec(*spec), probes)
    return dict(n=n, d=d, sigma=sigma, seed=SEED, inputs="X = f32(mixture10(n, d, seed))", precision="fp32",
                params=params, estimate=_est(est), probe_label="fullsize-probe", probe_spec=spec,
                probe_traces=[float(v) for v in qf], oracle="matrix-free blocks", seconds=time.time() - t)


def c4():
    n = 100000
    x, y = mi_inputs(n, SEED, gen="oracle")
    x, y = f32(x), f32(y)
    sx, sy = 4.0, math.sqrt(8.0)
    params = dict(alpha=1.01, method="chebyshev", s=90, m=60, bounds=(0.0, 1.0), probe_kind="gaussian")
    t = time.time()
    # the three terms' passes served together (one A/B block evaluation per sweep) and Hutch++'s
    # Q and W panels through one apply_panel: the same estimator and blocks as
    # blocks_mutual_information up to BLAS summation order (1e-14, tests/test_oracle_fullsize.py)
    O.set_merge_panels(True)
    try:
        mi = O.lockstep_mutual_information(x, sx, y, sy, seed=SEED, **params)
    finally:
        O.set_merge_panels(False)
    terms = {k: _est(v) for k, v in mi.pop("terms").items()}
    return dict(n=n, dx=16, dy=8, sigma_x=sx, sigma_y=sy, seed=SEED,
                inputs="X, Y = f32(mi_inputs(n, seed)) (Y = X W + 0.5 noise)", precision="fp32",
                params=dict(params, seed=SEED), mi=mi, terms=terms, oracle="matrix-free blocks, three terms in lockstep, Q and W merged",
                seconds=time.time() - t)


def c5():
    n, d = 400000, 128
    x = bf16(gaussian(n, d, SEED, "X", "oracle"))
    sigma = math.sqrt(d)
    params = dict(alpha=3.0, method="int", s=120, seed=SEED, probe_kind="gaussian")
    t = time.time()
    op = O.KernelBlocksOp(x, sigma)
    est = op.estimate(**params)
    return dict(n=n, d=d, sigma=sigma, seed=SEED, inputs="X = bf16(gaussian(n, d, seed, 'X'))", precision="mf",
                params=params, estimate=_est(est), oracle="matrix-free blocks", seconds=time.time() - t)


def main():
    if os.environ.get("ORACLE_NATIVE") != "1":
        print("note: ORACLE_NATIVE=1 selects the -march=native oracle build (same results, faster)")
    which = sys.argv[1:] or ["c2", "c3", "c5", "c4"]
    for name in which:
        t = time.time()
        rec = globals()[name]()
        _save(name, rec)
        print(f"{name}: {time.time() - t:.0f} s", json.dumps(rec)[:400], flush=True)


if __name__ == "__main__":
    main()
