"""build_kernel(X, PolynomialKernel{degree, offset}) on the device (proj/src/kernel.cpp:35-72,
proj/src/ops.cpp:22-28,58-64) against the pinned oracle: the normalised matrix itself, the
reference's error contract, and the estimators on top of it (the reference's rank-deficient
polynomial fixtures, test_entropy.cpp:121-131 and acceptance criterion 6). Probes are drawn on the
host (bitwise the reference's) so fp64 estimates meet the 1e-9 contract on identical probes."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dup(orc, key, n, d, ndup):
    x = orc.fill_gaussian(key, n, d)
    x[n - ndup:] = x[:ndup]  # duplicates force u = 0
    return x


@pytest.mark.parametrize("degree,offset", [(2, 1.0), (3, 0.5), (1, 0.0), (4, 2.0)])
def test_polynomial_kernel_matrix(R, orc, degree, offset):
    x = orc.fill_gaussian(31 + degree, 777, 6)
    ref = orc.build_kernel_polynomial(x, degree, offset)
    ctx = R.Context(0)
    a64 = R.build_kernel(x, R.PolynomialKernel(degree, offset), "fp64", ctx=ctx).matrix()
    assert np.array_equal(a64, a64.T)  # the reference mirrors each pair
    assert np.all(np.diag(a64) == 1.0 / x.shape[0])
    np.testing.assert_allclose(a64, ref, rtol=1e-12, atol=1e-15 * np.abs(ref).max())
    a32 = R.build_kernel(x, R.PolynomialKernel(degree, offset), "fp32", ctx=ctx).matrix()
    assert np.max(np.abs(a32 - ref)) <= 2e-6 * np.abs(ref).max()


def test_polynomial_kernel_errors(R):
    ctx = R.Context(0)
    x = np.zeros((3, 2))
    x[1] = [1.0, 0.0]
    x[2] = [0.0, 1.0]
    for prec in ("fp64", "fp32"):
        with pytest.raises(R.RenyiError) as e:  # test_kernel.cpp:65-71
            R.build_kernel(x, R.PolynomialKernel(2, 0.0), prec, ctx=ctx)
        assert e.value.kind == "zero_diagonal" and "kernel diagonal entry 0 is not positive" in str(e.value)
        with pytest.raises(R.RenyiError) as e:  # test_kernel.cpp:73-77
            R.build_kernel(np.array([[1e200], [-1e200]]), R.PolynomialKernel(2, 1.0), prec, ctx=ctx)
        assert e.value.kind == "non_finite" and "non-finite" in str(e.value)
    for deg, off in ((0, 1.0), (2, -0.5)):
        with pytest.raises(R.RenyiError) as e:
            R.build_kernel(np.ones((4, 2)), R.PolynomialKernel(deg, off), "fp64", ctx=ctx)
        assert e.value.kind == "invalid_argument"
    with pytest.raises(R.RenyiError) as e:
        R.build_kernel(np.array([[np.nan], [1.0]]), R.PolynomialKernel(2, 1.0), "fp64", ctx=ctx)
    assert e.value.kind == "non_finite" and "sample matrix" in str(e.value)


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_rank_deficient_polynomial_chebyshev(R, orc, prec, tol):  # test_entropy.cpp:121-131
    x = _dup(orc, 65, 120, 4, 30)
    a = orc.build_kernel_polynomial(x, 2, 1.0)
    exact = orc.entropy_exact(a, 2.5)
    b = orc.estimate_bounds(a)
    kw = dict(alpha=2.5, method="chebyshev", s=64, m=30, seed=3, bounds=(0.0, b["v"]))
    ref = orc.estimate(a, **kw)
    ctx = R.Context(0)
    ctx.set_probe_source("host")
    k = R.build_kernel(x, R.PolynomialKernel(2, 1.0), prec, ctx=ctx)
    est = R.estimate(k, R.EstimatorParams(alpha=2.5, method="chebyshev", s=64, m=30, seed=3,
                                          bounds=R.SpectrumBounds(u=0.0, v=b["v"])))
    assert est.entropy == pytest.approx(ref["entropy"], rel=tol)
    assert abs(est.entropy - exact) <= 1e-2 * abs(exact)
    bd = R.estimate_bounds(k)  # device power iteration on the polynomial kernel
    assert bd.v == pytest.approx(b["v"], rel=1e-9 if prec == "fp64" else 1e-5)
    assert bd.rank_deficient == b["rank_deficient"]


def test_acceptance_rank_deficient_polynomial(R, orc):  # acceptance.cpp:230-254 (criterion 6)
    x = _dup(orc, 888, 400, 8, 100)
    a = orc.build_kernel_polynomial(x, 2, 1.0)
    exact = orc.entropy_exact(a, 2.5)
    ctx = R.Context(0)
    k = R.build_kernel(x, R.PolynomialKernel(2, 1.0), "fp64", ctx=ctx)
    bounds = R.estimate_bounds(k, R.PowerOptions(seed=5))
    assert bounds.rank_deficient
    worst = 0.0
    for seed in range(20):
        est = R.estimate(k, R.EstimatorParams(alpha=2.5, method="chebyshev", s=64, m=30, seed=seed,
                                              bounds=R.SpectrumBounds(u=0.0, v=bounds.v)))
        worst = max(worst, abs(est.entropy - exact) / abs(exact))
    assert worst <= 1e-2


def test_polynomial_mutual_information_fused(R, orc):
    """MI over two polynomial kernels: the fp32 fused pass forms n·A∘B on the fly like for Gaussians."""
    n = 1500
    x, y = orc.fill_gaussian(5, n, 6), orc.fill_gaussian(6, n, 3)
    a, b = orc.build_kernel_polynomial(x, 2, 1.0), orc.build_kernel_polynomial(y, 3, 0.5)
    kw = dict(alpha=1.5, method="chebyshev", s=40, m=30, seed=9, bounds=(0.0, 1.0))
    ref = orc.mutual_information(a, b, **dict(kw))
    ctx = R.Context(0)
    ctx.set_probe_source("host")
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=40, m=30, seed=9, bounds=R.SpectrumBounds(u=0.0, v=1.0))
    for prec, tol in (("fp64", 1e-9), ("fp32", 1e-4)):
        ka = R.build_kernel(x, R.PolynomialKernel(2, 1.0), prec, ctx=ctx)
        kb = R.build_kernel(y, R.PolynomialKernel(3, 0.5), prec, ctx=ctx)
        mi = R.mutual_information([ka], kb, p)
        for key in ("vars_entropy", "target_entropy", "joint_entropy"):
            assert getattr(mi, key) == pytest.approx(ref[key], rel=tol), (prec, key)


def test_raw_ops_seam(R, orc):
    """ops::gaussian_gram / polynomial_gram / hadamard_scaled (proj/include/renyi/ops.hpp:12-33) on the
    device: the reference's KATs (test_ops.cpp:39-56, 69-76) and the oracle, unnormalised."""
    ctx = R.Context(0)
    x = orc.fill_gaussian(12, 23, 3)
    g = R.ops.gaussian_gram(x, 1.3, ctx=ctx)
    d2 = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
    np.testing.assert_allclose(g, np.exp(-d2 / (2 * 1.3 * 1.3)), rtol=1e-12, atol=0)
    p = R.ops.polynomial_gram(x, 3, 0.5, ctx=ctx)
    np.testing.assert_allclose(p, (x @ x.T + 0.5) ** 3, rtol=1e-12, atol=0)
    x = orc.fill_gaussian(13, 640, 5)
    g = R.ops.gaussian_gram(x, 1.0, ctx=ctx)
    assert np.array_equal(g, g.T) and np.all(np.diag(g) == 1.0)
    np.testing.assert_allclose(g, orc.gaussian_gram(x, 1.0), rtol=1e-13, atol=1e-300)
    p = R.ops.polynomial_gram(x, 2, 1.0, ctx=ctx)
    assert np.array_equal(p, p.T)
    np.testing.assert_allclose(p, orc.polynomial_gram(x, 2, 1.0), rtol=1e-12, atol=1e-12 * np.abs(p).max())
    a, b = orc.fill_gaussian(1, 300, 7), orc.fill_gaussian(2, 300, 7)
    assert np.array_equal(R.ops.hadamard_scaled(a, b, 2.5, ctx=ctx), 2.5 * (a * b))


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_hadamard_joint_of_three_is_permutation_invariant(R, orc, prec):
    """hadamard_joint over three kernels (kernel.cpp:74-101; test_kernel.cpp:113-127): a canonical
    content order makes every permutation bitwise identical; fp64 matches the oracle to rounding."""
    ctx = R.Context(0)
    xs = [orc.fill_gaussian(24 + v, 300, 2) for v in range(3)]
    ks = [R.build_kernel(x, R.GaussianKernel(1.0), prec, ctx=ctx) for x in xs]
    j = R.hadamard_joint(ks).matrix()
    for perm in ((2, 0, 1), (1, 2, 0), (0, 2, 1)):
        assert np.array_equal(R.hadamard_joint([ks[p] for p in perm]).matrix(), j)
    ref = orc.hadamard_joint_n([orc.build_kernel(x, 1.0) for x in xs])
    tol = 1e-14 if prec == "fp64" else 2e-6
    assert np.max(np.abs(j - ref)) <= tol * np.abs(ref).max()
    assert abs(np.trace(j) - 1.0) <= 1e-12
    # joint entropy over three variables (measures.cpp:15-21) on top of it
    p = R.EstimatorParams(alpha=2.0, method="int", s=40, seed=1)
    e = R.joint_entropy(ks, p)
    assert np.isfinite(e.entropy)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_measures_permutation_invariant(R, orc, prec):  # test_measures.cpp:112-130
    ctx = R.Context(0)
    ks = [R.build_kernel(orc.fill_gaussian(80 + i, 250, dd), R.GaussianKernel(1.0), prec, ctx=ctx)
          for i, dd in enumerate((2, 3, 1))]
    a, b, c = ks
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=16, m=20, seed=4, bounds=R.SpectrumBounds(u=0.0, v=1.0))
    r1 = R.joint_entropy([a, b, c], p).entropy
    r2 = R.joint_entropy([b, c, a], p).entropy
    assert r1 == r2
    if prec == "fp64":
        ex = R.EstimatorParams(alpha=1.5, method="exact")
        assert R.joint_entropy([a, b, c], ex).entropy == R.joint_entropy([c, a, b], ex).entropy
