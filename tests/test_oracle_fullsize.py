"""The full-size oracle paths (tests/golden/gen_fullsize.py) against the dense oracle at small n.

GaussOp recomputes kernel entries with the reference's arithmetic (bit-identical entries) and
KernelBlocksOp does the same in BLAS blocks with a vectorised exp (<= 2 ulp); both run the same
restated estimator as the dense path, so they must agree with it to rounding.
"""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O

N, D = 900, 6


@pytest.fixture(scope="module")
def data():
    x = O.fill_gaussian(31, N, D)
    y = O.fill_gaussian(32, N, 3)
    a, b = O.build_kernel(x, 2.0), O.build_kernel(y, 1.5)
    return x, y, a, b, O.hadamard_joint(a, b)


def test_exp_nonpos_ulp():
    xs = -np.concatenate([np.linspace(0, 50, 200001), np.linspace(50, 745.3, 100001), [708.39, 744.44, 745.13]])
    dot = np.ascontiguousarray(xs / 2)
    sq = np.zeros(len(xs))
    out = np.empty(len(xs))
    O.lib().oracle_kernel_block(O._p(dot), 1, len(xs), O._p(sq[:1]), O._p(sq), 1.0, 1.0, 1.0, 0, O._p(out))
    ref = np.array([math.exp(v) for v in xs])
    nz = ref > 0
    ulp = np.abs(out[nz] - ref[nz]) / np.spacing(ref[nz])
    assert ulp.max() <= 2.0
    assert np.array_equal(out[~nz], ref[~nz])


@pytest.mark.parametrize("block", [128, 512])
def test_matrix_free_products(data, block):
    x, y, a, b, j = data
    v = O.probe_panel(N, 9, 3, "p")
    for dense, args in ((a, (x, 2.0)), (j, (x, 2.0, y, 1.5))):
        ref = O.matmul_panel(dense, v)
        got = O.mf_matmul(args[0], args[1], v, *args[2:])
        assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()
        op = O.KernelBlocksOp(*args, block=block)
        got = op.mul(np.ascontiguousarray(v))
        assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("kw", [
    dict(alpha=1.5, method="chebyshev", s=40, m=20, seed=5, bounds=(0.0, 1.0), probe_kind="rademacher", s_q=8, s_g=16),
    dict(alpha=0.5, method="taylor", s=40, m=12, seed=6, probe_kind="gaussian", s_q=0, s_g=40),
    dict(alpha=3.0, method="int", s=40, seed=7),
    dict(alpha=1.3, method="auto", s=40, m=15, seed=9),
])
def test_matrix_free_estimates(data, kw):
    x, y, a, b, j = data
    ref = O.estimate(a, **kw)
    for got in (O.mf_estimate(x, 2.0, **kw), O.KernelBlocksOp(x, 2.0, block=256).estimate(**kw)):
        assert got["entropy"] == pytest.approx(ref["entropy"], rel=1e-12)
        assert got["v"] == pytest.approx(ref["v"], rel=1e-12)
        assert got["iterations_used"] == ref["iterations_used"]
        assert got["sketch_rank"] == ref["sketch_rank"]


def test_matrix_free_mutual_information(data):
    x, y, a, b, j = data
    kw = dict(alpha=1.01, method="chebyshev", s=40, m=30, seed=11, bounds=(0.0, 1.0))
    ref = O.mutual_information(a, b, **dict(kw))
    got = O.blocks_mutual_information(x, 2.0, y, 1.5, block=256, **dict(kw))
    for key in ("value", "vars_entropy", "target_entropy", "joint_entropy"):
        assert got[key] == pytest.approx(ref[key], rel=1e-10, abs=1e-12)


def test_lockstep_mutual_information(data):
    """The config-4 fixture's scheduling (three terms served by one block sweep, Hutch++'s Q and W
    through one apply_panel) changes only BLAS summation order (wider panels)."""
    x, y, a, b, j = data
    kw = dict(alpha=1.01, method="chebyshev", s=40, m=30, seed=11, bounds=(0.0, 1.0))
    ref = O.blocks_mutual_information(x, 2.0, y, 1.5, block=256, **dict(kw))
    O.set_merge_panels(True)
    try:
        got = O.lockstep_mutual_information(x, 2.0, y, 1.5, block=256, **dict(kw))
    finally:
        O.set_merge_panels(False)
    for key in ("value", "vars_entropy", "target_entropy", "joint_entropy"):
        assert got[key] == pytest.approx(ref[key], rel=1e-12)
    assert got["terms"]["joint"]["queries_used"] == ref["terms"]["joint"]["queries_used"]


def test_matrix_free_probe_traces(data):
    x, y, a, b, j = data
    spec = O.Spec("chebyshev", 1.5, 25, 0.0, 1.0)
    q = O.probe_panel(N, 4, 2, "fullsize-probe")
    ref = np.einsum("ij,ij->j", q, O.apply_panel(spec, a, q))
    np.testing.assert_allclose(O.mf_matfun_traces(spec, x, 2.0, q), ref, rtol=1e-12)
    np.testing.assert_allclose(O.KernelBlocksOp(x, 2.0, block=256).matfun_traces(spec, q), ref, rtol=1e-12)


def test_fullsize_fixture_shape():
    """The committed fixture file (when present) names its inputs and carries finite results."""
    f = Path(__file__).resolve().parent / "golden" / "fullsize.json"
    if not f.exists():
        pytest.skip("tests/golden/fullsize.json not generated yet")
    d = json.loads(f.read_text())
    for name, rec in d.items():
        assert rec["seed"] == 2205 and rec["n"] in (20000, 50000, 100000, 400000), name
        vals = [rec["mi"]["value"]] if "mi" in rec else [rec["estimate"]["entropy"], rec["estimate"]["trace"]]
        assert all(np.isfinite(vals)), name
