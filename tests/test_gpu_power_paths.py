"""The single-column paths of the power iteration (proj/src/spectrum.cpp:25-49) and matvec
(proj/src/ops.cpp:73-85) on the device:
* fp32 kernels run s = 1 passes through the upper-triangle product (symv.cu): same products as the
  tensor-core block product (RB_SYMV=0) up to summation order, and the oracle's fp64 A·x to the fp32 bar,
  at sizes on and off the 128-row tile grid;
* the speculative schedule (the next pass queued before the host reads the current pass's dots, its
  normalisation computed on the device; RB_SPECULATE=0 turns it off) is bitwise the synchronous loop:
  same Rayleigh quotients, iteration counts and convergence flags, shifted runs included."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def context(R, monkeypatch, **env):
    for key, val in env.items():
        monkeypatch.setenv(key, val)
    ctx = R.Context(0)  # the engine reads RB_SYMV / RB_SPECULATE when the context is created
    for key in env:
        monkeypatch.delenv(key)
    return ctx


@pytest.mark.parametrize("n", [50, 128, 129, 300, 1000, 2500])
def test_symv_matvec_matches_oracle_and_tensor_path(R, orc, monkeypatch, n):
    d = 7
    x = f32(orc.fill_gaussian(900 + n, n, d))
    v = orc.fill_gaussian(77 + n, n, 1)[:, 0]
    sigma = math.sqrt(d)
    ref = orc.build_kernel(x, sigma) @ v
    ys = R.ops.matvec(R.build_kernel(x, R.GaussianKernel(sigma), "fp32", ctx=context(R, monkeypatch)), v)
    yt = R.ops.matvec(R.build_kernel(x, R.GaussianKernel(sigma), "fp32",
                                     ctx=context(R, monkeypatch, RB_SYMV="0")), v)
    scale = np.max(np.abs(ref))
    # fp32 outputs of a sum with cancellation (x is signed): both paths within 2e-6 of the fp64 product
    assert np.max(np.abs(ys - ref)) <= 2e-6 * scale
    assert np.max(np.abs(yt - ref)) <= 2e-6 * scale


def test_symv_power_iteration_matches_tensor_path(R, orc, monkeypatch):
    n = 3000
    x = f32(orc.mixture_samples(n, 6, 17))
    opts = R.PowerOptions(max_iters=200, tol=1e-6, seed=3)
    out = []
    for env in ({}, {"RB_SYMV": "0"}):
        k = R.build_kernel(x, R.GaussianKernel(1.0), "fp32", ctx=context(R, monkeypatch, **env))
        out.append(R.estimate_bounds(k, opts))
    ref = orc.estimate_bounds(orc.build_kernel(x, 1.0), max_iters=200, tol=1e-6, seed=3)
    for b in out:
        assert b.v == pytest.approx(ref["v"], rel=1e-5)
        assert b.u == pytest.approx(ref["u"], rel=1e-4, abs=1e-9)


@pytest.mark.parametrize("prec,n", [("fp32", 300), ("fp32", 2600), ("fp64", 700)])
def test_speculative_power_iteration_is_bitwise_the_synchronous_loop(R, orc, monkeypatch, prec, n):
    x = f32(orc.mixture_samples(n, 8, 29))
    ks = [R.build_kernel(x, R.GaussianKernel(1.0), prec, ctx=context(R, monkeypatch, RB_SPECULATE=flag))
          for flag in ("0", "1")]
    cases = [(R.PowerOptions(max_iters=1, tol=1e-16, seed=1), 0.0),
             (R.PowerOptions(max_iters=2, tol=1e-16, seed=2), 0.0),
             (R.PowerOptions(max_iters=60, tol=1e-16, seed=3), 0.0),   # budget exhausted
             (R.PowerOptions(max_iters=500, tol=1e-7, seed=4), 0.0),   # converges early
             (R.PowerOptions(max_iters=300, tol=1e-7, seed=5), 0.9)]   # shifted (0.9 I - A)
    for opts, shift in cases:
        a, b = (R.power_method(k, opts, shift) for k in ks)
        assert (a.rayleigh, a.iterations, a.converged) == (b.rayleigh, b.iterations, b.converged), (opts, shift)
    a, b = (R.estimate_bounds(k, R.PowerOptions(max_iters=400, tol=1e-8, seed=6)) for k in ks)
    assert (a.u, a.v, a.iterations_used, a.u_converged, a.v_converged) == \
        (b.u, b.v, b.iterations_used, b.u_converged, b.v_converged)
