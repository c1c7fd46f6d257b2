"""The reference's spectrum and Hutch++ known-answer tests (proj/tests/test_spectrum.cpp:63-121,
proj/tests/test_hutchpp.cpp:138-153) through the device power iteration and Hutch++ -- extreme
iteration budgets and tolerances included (5000 iterations at tol 1e-12, tol 1e-16, one iteration)."""
import math

import numpy as np
import pytest

from fixtures import mixture_kernel, oracle_trace_power, random_unit_trace_spd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dctx(R):
    return R.Context(0)


def test_sandwich_property(R, orc, dctx):  # test_spectrum.cpp:63-80
    for rep in range(6):
        n = 40 + 32 * rep
        a = random_unit_trace_spd(n, 43 + rep, orc, floor=0.1)
        eigs = np.linalg.eigvalsh(a)
        k = R.NormalizedKernel.from_matrix(a, "fp64", ctx=dctx)
        b = R.estimate_bounds(k, R.PowerOptions(max_iters=5000, tol=1e-12, seed=100 + rep))
        assert b.u <= eigs.min() + 1e-6 and b.v >= eigs.max() - 1e-6
        assert b.u <= b.v and b.u <= 1.0 / n + 1e-12 and b.v >= 1.0 / n - 1e-12


def test_rayleigh_never_degrades(R, orc, dctx):  # test_spectrum.cpp:82-95
    k = R.NormalizedKernel.from_matrix(random_unit_trace_spd(60, 44, orc), "fp64", ctx=dctx)
    prev = 0.0
    for iters in (1, 2, 5, 10, 25, 50, 100):
        r = R.power_method(k, R.PowerOptions(max_iters=iters, tol=1e-16, seed=11))
        assert r.rayleigh >= prev - 1e-15
        prev = r.rayleigh


def test_nonconvergence_is_diagnostic(R, orc, dctx):  # test_spectrum.cpp:97-108
    k = R.NormalizedKernel.from_matrix(random_unit_trace_spd(50, 46, orc), "fp64", ctx=dctx)
    b = R.estimate_bounds(k, R.PowerOptions(max_iters=1, tol=1e-14))
    assert not b.v_converged
    assert 1.0 / 50 <= b.v <= 1.0


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_clamp_invariants(R, orc, dctx, prec):  # test_spectrum.cpp:110-121
    x = orc.fill_gaussian(45, 30, 3)
    k = R.build_kernel(x, R.GaussianKernel(0.4), prec, ctx=dctx)
    b = R.estimate_bounds(k)
    assert 1.0 / 30 <= b.v <= 1.0 and 0.0 <= b.u <= 1.0 / 30


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_concentration_frozen_budget(R, orc, dctx, prec):  # test_hutchpp.cpp:138-153
    eps, delta, c = 0.1, 0.1, 4.0
    s = (int(math.ceil(c / eps)) + 3) // 4 * 4
    x = orc.mixture_samples(300, 6, 31)
    exact = oracle_trace_power(orc.build_kernel(x, 1.0), 2.0)
    k = R.build_kernel(x, R.GaussianKernel(1.0), prec, ctx=dctx)
    f = R.MatrixFunctionSpec.int_power(2)
    misses = sum(abs(R.hutchpp(f, k, R.SketchConfig(s=s, seed=seed)).value - exact) > eps * exact
                 for seed in range(200))
    assert misses <= delta * 200
