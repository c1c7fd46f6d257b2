"""Parity of the B200 path (through the C ABI) against the pinned fp64 oracle on
identical inputs and probes. Tolerances (north_star): fp64 configuration within
1e-9 relative, fp32 configuration within 1e-4 relative, on traces, entropies and
MI terms; elementwise checks on A and A·V are tighter and stated per test."""
import math

import numpy as np
import pytest

from conftest import rel
from fixtures import mixture_kernel, oracle_trace_power, random_low_rank_psd, random_unit_trace_spd

pytestmark = pytest.mark.gpu

TOL = {"fp64": 1e-9, "fp32": 1e-4}


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


# ------------------------------------------------------------------ Gram construction (K1+K2)
@pytest.mark.parametrize("n,d,sigma", [(2, 3, 1.0), (3, 1, 1.0), (129, 7, 0.8), (1001, 10, math.sqrt(10)),
                                       (2048, 32, math.sqrt(32))])
def test_build_kernel_parity(R, orc, n, d, sigma):
    x = orc.fill_gaussian(1000 + n, n, d)
    a64 = R.build_kernel(x, R.GaussianKernel(sigma), precision="fp64").matrix()
    ref = orc.build_kernel(x, sigma)
    assert np.max(np.abs(a64 - ref)) <= 4e-16 / n * 8  # ~1 ulp of 1/n scale entries
    assert np.array_equal(a64, a64.T) and np.all(np.diag(a64) == 1.0 / n)
    xs = f32(x)
    a32 = R.build_kernel(xs, R.GaussianKernel(sigma), precision="fp32").matrix()
    ref32 = orc.build_kernel(xs, sigma)
    assert np.max(np.abs(a32 - ref32)) * n <= 2e-6  # fp32 distance/exp + 22-bit split storage
    assert np.array_equal(a32, a32.T)


def test_kernel_kats_on_device(R):  # test_kernel.cpp:25-50
    for prec, tol in (("fp64", 1e-15), ("fp32", 1e-6)):
        k = R.build_kernel(np.array([[0.3, -1.2, 0.7], [0.3, -1.2, 0.7]]), R.GaussianKernel(1.0), prec).matrix()
        np.testing.assert_allclose(k, 0.5, rtol=tol)
        k = R.build_kernel(np.array([[0.0], [1e6], [2e6], [3e6]]), R.GaussianKernel(1.0), prec).matrix()
        assert np.max(np.abs(k - np.eye(4) / 4)) <= 1e-15
        k = R.build_kernel(np.array([[0.0], [1.0], [2.0]]), R.GaussianKernel(1.0), prec).matrix()
        assert k[0, 1] == pytest.approx(math.exp(-0.5) / 3, rel=tol)
        assert k[0, 2] == pytest.approx(math.exp(-2.0) / 3, rel=tol)


def test_kernel_errors_on_device(R):  # test_kernel.cpp:65-83
    with pytest.raises(R.RenyiError) as e:
        R.build_kernel(np.array([[1.0, 2.0]]), R.GaussianKernel(1.0))
    assert e.value.kind == "invalid_argument"
    with pytest.raises(R.RenyiError) as e:
        R.build_kernel(np.array([[np.inf], [1.0]]), R.GaussianKernel(1.0))
    assert e.value.kind == "non_finite"
    with pytest.raises(R.RenyiError) as e:
        R.build_kernel(np.array([[0.0], [1.0]]), R.GaussianKernel(-1.0))
    assert e.value.kind == "invalid_argument"


def test_hadamard_joint_parity(R, orc):  # kernel.cpp:74-101, test_kernel.cpp:85-127
    n = 700
    x, y = orc.fill_gaussian(5, n, 4), orc.fill_gaussian(6, n, 2)
    ax, ay = orc.build_kernel(x, 2.0), orc.build_kernel(y, 1.5)
    ref = orc.hadamard_joint(ax, ay)
    for prec, tol in (("fp64", 1e-15), ("fp32", 2e-6)):
        kx = R.build_kernel(x if prec == "fp64" else f32(x), R.GaussianKernel(2.0), prec)
        ky = R.build_kernel(y if prec == "fp64" else f32(y), R.GaussianKernel(1.5), prec)
        j = R.hadamard_joint([kx, ky]).matrix()
        fused = R.build_joint_kernel(x if prec == "fp64" else f32(x), R.GaussianKernel(2.0),
                                     y if prec == "fp64" else f32(y), R.GaussianKernel(1.5), prec).matrix()
        r = orc.hadamard_joint(orc.build_kernel(f32(x), 2.0), orc.build_kernel(f32(y), 1.5)) if prec == "fp32" else ref
        assert np.max(np.abs(j - r)) * n <= tol * 4
        assert np.max(np.abs(fused - r)) * n <= tol * 4
        assert abs(np.trace(fused) - 1.0) <= 1e-12
    eye = R.NormalizedKernel.from_matrix(np.eye(5) / 5)
    assert np.max(np.abs(R.hadamard_joint([eye, eye]).matrix() - np.eye(5) / 5)) <= 1e-15
    with pytest.raises(R.RenyiError) as e:
        R.hadamard_joint([R.NormalizedKernel.from_matrix(np.eye(4) / 4), eye])
    assert e.value.kind == "size_mismatch"


# ------------------------------------------------------------------ block product (K6)
@pytest.mark.parametrize("n,s", [(2, 1), (127, 8), (129, 17), (1000, 30), (2049, 68), (1500, 128), (777, 129),
                                 (640, 300)])
def test_matmul_panel_parity(R, orc, n, s):
    x = orc.fill_gaussian(77 + n, n, 6)
    v = orc.fill_gaussian(88 + s, n, s)
    a = orc.build_kernel(x, 2.0)
    ref = orc.matmul_panel(a, v)
    y64 = R.ops.matmul_panel(R.build_kernel(x, R.GaussianKernel(2.0), "fp64"), v)
    assert rel(y64, ref) <= 1e-13
    a32 = orc.build_kernel(f32(x), 2.0)
    y32 = R.ops.matmul_panel(R.build_kernel(f32(x), R.GaussianKernel(2.0), "fp32"), v)
    assert rel(y32, orc.matmul_panel(a32, v)) <= 2e-6


def test_matmul_arbitrary_matrix_and_matvec(R, orc):
    # non-kernel input (NormalizedKernel(Matrix)): wide dynamic range, negative entries
    a = random_unit_trace_spd(300, 11, orc, 0.05)
    v = orc.fill_gaussian(12, 300, 9)
    for prec, tol in (("fp64", 1e-13), ("fp32", 2e-6)):
        k = R.NormalizedKernel.from_matrix(a, prec)
        assert rel(R.ops.matmul_panel(k, v), a @ v) <= tol
        assert rel(R.ops.matvec(k, v[:, 0]), orc.matvec(a, v[:, 0])) <= tol
    w = orc.fill_gaussian(41, 16, 1)[:, 0]
    w /= np.linalg.norm(w)
    k = R.NormalizedKernel.from_matrix(np.outer(w, w), "fp32")  # entries far above 1/n
    assert rel(R.ops.matvec(k, w), w) <= 2e-6


def test_block_product_deterministic(R, orc):
    x = f32(orc.fill_gaussian(3, 3000, 16))
    v = orc.fill_gaussian(4, 3000, 40)
    k = R.build_kernel(x, R.GaussianKernel(4.0), "fp32")
    assert np.array_equal(R.ops.matmul_panel(k, v), R.ops.matmul_panel(k, v))


# ------------------------------------------------------------------ recurrences (K7) + fused traces (K11)
SPECS = [("int", 2, 0, 0.0, 1.0), ("int", 3, 0, 0.0, 1.0), ("taylor", 0.5, 15, 0.0, 1.0),
         ("taylor", 1.5, 30, 0.0, 0.45), ("chebyshev", 1.5, 40, 0.0, 1.0), ("chebyshev", 1.01, 60, 0.0, 1.0),
         ("chebyshev", 2.5, 20, 0.05, 0.6)]


@pytest.mark.parametrize("spec", SPECS)
def test_apply_panel_and_traces_parity(R, orc, spec):
    kind, alpha, m, u, v = spec
    n, s = 900, 11
    x = orc.fill_gaussian(17, n, 5)
    p = orc.fill_gaussian(18, n, s)
    ospec = orc.Spec(kind, alpha, m, u, v)
    rspec = {"int": lambda: R.MatrixFunctionSpec.int_power(int(alpha)),
             "taylor": lambda: R.MatrixFunctionSpec.taylor(alpha, m, v),
             "chebyshev": lambda: R.MatrixFunctionSpec.chebyshev(alpha, m, u, v)}[kind]()
    for prec in ("fp64", "fp32"):
        xx = x if prec == "fp64" else f32(x)
        a = orc.build_kernel(xx, 1.7)
        ref = orc.apply_panel(ospec, a, p)
        k = R.build_kernel(xx, R.GaussianKernel(1.7), prec)
        y = R.apply_panel(rspec, k, p)
        assert rel(y, ref) <= (1e-11 if prec == "fp64" else 5e-5)
        tr = R.matfun_traces(rspec, k, p)
        ref_tr = np.einsum("ij,ij->j", p, ref)
        assert np.max(np.abs(tr - ref_tr) / np.abs(ref_tr)) <= (1e-11 if prec == "fp64" else TOL["fp32"])


# ------------------------------------------------------------------ spectrum (a6)
def test_power_bounds_parity(R, orc):
    for key, n in ((21, 400), (22, 1200)):
        x = orc.fill_gaussian(key, n, 4)
        a = orc.build_kernel(x, 1.0)
        ref = orc.estimate_bounds(a, seed=5)
        got = R.estimate_bounds(R.build_kernel(x, R.GaussianKernel(1.0), "fp64"), R.PowerOptions(seed=5))
        assert got.iterations_used == ref["iterations_used"]
        assert abs(got.v - ref["v"]) <= 1e-9 * ref["v"]
        assert abs(got.u - ref["u"]) <= 1e-9 * max(ref["v"], 1e-300)
        assert got.rank_deficient == ref["rank_deficient"]
    b = R.estimate_bounds(R.NormalizedKernel.from_matrix(np.eye(8) / 8), R.PowerOptions())
    assert b.v == pytest.approx(1 / 8, rel=1e-5) and b.u == pytest.approx(1 / 8, rel=1e-5)
    d = R.NormalizedKernel.from_matrix(np.diag([0.5, 0.3, 0.2]))
    b = R.estimate_bounds(d, R.PowerOptions(max_iters=200, tol=1e-8, seed=7))
    assert abs(b.v - 0.5) <= 1e-6 and abs(b.u - 0.2) <= 1e-6


def test_duplicates_force_u0_on_device(R, orc):  # test_spectrum.cpp:45-61
    dd = orc.fill_gaussian(42, 5, 2)
    k = R.build_kernel(np.vstack([dd, dd]), R.GaussianKernel(1.0), "fp64")
    b = R.estimate_bounds(k, R.PowerOptions(max_iters=2000, tol=1e-13, seed=5))
    assert b.u == 0.0 and b.rank_deficient and math.isinf(b.kappa)


# ------------------------------------------------------------------ Hutch++ (a10, a11)
def _rspec(R, kind, alpha, m=0, u=0.0, v=1.0):
    if kind == "int":
        return R.MatrixFunctionSpec.int_power(int(alpha))
    if kind == "taylor":
        return R.MatrixFunctionSpec.taylor(alpha, m, v)
    return R.MatrixFunctionSpec.chebyshev(alpha, m, u, v)


@pytest.mark.parametrize("kind,alpha,m,u,v", [("int", 2, 0, 0, 1), ("taylor", 0.5, 30, 0, 0.5),
                                              ("chebyshev", 1.5, 40, 0, 1), ("chebyshev", 1.01, 60, 0, 1)])
@pytest.mark.parametrize("probe", ["gaussian", "rademacher"])
def test_hutchpp_injected_and_seeded(R, orc, kind, alpha, m, u, v, probe):
    n = 1500
    x = orc.fill_gaussian(31, n, 8)
    ospec = orc.Spec(kind, alpha, m, u, v)
    for prec in ("fp64", "fp32"):
        xx = x if prec == "fp64" else f32(x)
        a = orc.build_kernel(xx, math.sqrt(8))
        k = R.build_kernel(xx, R.GaussianKernel(math.sqrt(8)), prec)
        f = _rspec(R, kind, alpha, m, u, v)
        # seeded: the device draws the reference streams itself
        ref = orc.hutchpp(ospec, a, 5, 12, 9, probe)
        got = R.hutchpp(f, k, R.SketchConfig(s_q=5, s_g=12, seed=9, probe_kind=probe))
        assert abs(got.value - ref["value"]) <= TOL[prec] * abs(ref["value"])
        assert got.sketch_rank == ref["sketch_rank"] and got.queries_used == ref["queries_used"]
        # injected probes
        S, G = orc.fill_gaussian(1, n, 5), orc.fill_gaussian(2, n, 12)
        ref = orc.hutchpp(ospec, a, 5, 12, sketch=S, probes=G)
        got = R.hutchpp(f, k, R.SketchConfig(s_q=5, s_g=12, sketch=S, probes=G))
        assert abs(got.value - ref["value"]) <= TOL[prec] * abs(ref["value"])
        assert abs(got.low_rank_part - ref["low_rank_part"]) <= TOL[prec] * abs(ref["value"])


def test_plain_hutchinson(R, orc):  # survey §0: Q-empty residual_probe_trace
    x = orc.fill_gaussian(8, 1000, 10)
    a = orc.build_kernel(x, math.sqrt(10))
    ref = orc.hutchpp(orc.Spec("int", 2), a, 0, 30, 3, "rademacher")
    got = R.hutchpp(R.MatrixFunctionSpec.int_power(2), R.build_kernel(x, R.GaussianKernel(math.sqrt(10)), "fp64"),
                    R.SketchConfig(s_q=0, s_g=30, seed=3, probe_kind="rademacher"))
    assert abs(got.value - ref["value"]) <= 1e-9 * ref["value"] and got.sketch_rank == 0


def test_hutchpp_structural_cases(R, orc):  # test_hutchpp.cpp:12-51,120-136
    x = np.array([[0.0 if i % 2 == 0 else 1.0] for i in range(40)])
    k = R.build_kernel(x, R.GaussianKernel(1.0), "fp64")
    for seed in range(5):
        z = R.hutchpp(R.MatrixFunctionSpec.int_power(1), k, R.SketchConfig(8, seed))
        assert abs(z.value - 1.0) <= 1e-8
    a = random_low_rank_psd(60, 2, 52, orc)
    exact = oracle_trace_power(a, 2.0)
    k = R.NormalizedKernel.from_matrix(a, "fp64")
    for seed in range(5):
        z = R.hutchpp(R.MatrixFunctionSpec.int_power(2), k, R.SketchConfig(8, seed))
        assert abs(z.value - exact) <= 1e-10 * exact and z.sketch_rank == 2 and abs(z.residual_part) <= 1e-12
    a = random_unit_trace_spd(12, 54, orc)
    exact = oracle_trace_power(a, 2.0)
    k = R.NormalizedKernel.from_matrix(a, "fp64")
    z1 = R.hutchpp(R.MatrixFunctionSpec.int_power(2), k, R.SketchConfig(48, 1))
    z2 = R.hutchpp(R.MatrixFunctionSpec.int_power(2), k, R.SketchConfig(40, 2))
    assert z1.exact and z2.exact
    assert abs(z1.value - exact) <= 1e-12 * exact and abs(z2.value - exact) <= 1e-12 * exact
    with pytest.raises(R.RenyiError) as e:
        R.hutchpp(R.MatrixFunctionSpec.int_power(2), R.NormalizedKernel.from_matrix(np.zeros((10, 10))),
                  R.SketchConfig(8, 0))
    assert e.value.kind == "rank_collapse"


# ------------------------------------------------------------------ estimators (a12, a13)
def test_config1_shape_parity_and_exact(R, orc):
    """Config 1: n=2000, d=10, fp64, alpha=2, Hutchinson s=30 Rademacher; vs oracle and eigendecomposition."""
    n, d = 2000, 10
    x = orc.fill_gaussian(orc.derive_key(2024, orc.hash_name("X")), n, d)
    sigma = math.sqrt(d)
    a = orc.build_kernel(x, sigma)
    ref = orc.estimate(a, alpha=2.0, method="int", s=30, seed=7, probe_kind="rademacher", s_q=0, s_g=30)
    p = R.EstimatorParams(alpha=2.0, method="int", s=30, seed=7, probe_kind="rademacher", s_q=0, s_g=30)
    got = R.entropy(x, sigma, p, precision="fp64")
    assert abs(got.entropy - ref["entropy"]) <= 1e-9 * abs(ref["entropy"])
    assert abs(got.trace_estimate - ref["trace"]) <= 1e-9 * ref["trace"]
    # vs the eigendecomposition: only Hutchinson noise remains; Rademacher variance of x^T B x
    # is 2(||B||_F^2 - sum_i B_ii^2), so allow four standard deviations of the s=30 mean
    b = a @ a
    exact_tr = oracle_trace_power(a, 2.0)
    sd = math.sqrt(2.0 * (np.sum(b * b) - np.sum(np.diag(b) ** 2)) / 30)
    assert abs(got.trace_estimate - exact_tr) <= 4 * sd


def test_estimate_routing_parity(R, orc):  # test_entropy.cpp:236-260
    a = mixture_kernel(400, 6, 1.0, 77, orc)
    k = R.NormalizedKernel.from_matrix(a, "fp64")
    ref = orc.estimate(a, alpha=2.0, s=16, seed=5)
    got = R.estimate(k, R.EstimatorParams(alpha=2.0, s=16, seed=5))
    assert got.method_used == "int" and abs(got.entropy - ref["entropy"]) <= 1e-9 * abs(ref["entropy"])
    ref = orc.estimate(a, alpha=1.5, s=64, m=30, seed=5)
    got = R.estimate(k, R.EstimatorParams(alpha=1.5, s=64, m=30, seed=5))
    assert got.method_used == {2: "taylor", 3: "chebyshev"}[ref["method"]]
    assert abs(got.bounds_used.v - ref["v"]) <= 1e-9 * ref["v"]
    assert abs(got.entropy - ref["entropy"]) <= 1e-9 * abs(ref["entropy"])
    got = R.estimate(k, R.EstimatorParams(alpha=2.0, epsilon=0.1, delta=0.1, seed=1))
    assert got.s_used == 20


def test_entropy_paths_flat_spectrum(R):  # test_entropy.cpp:142-155
    n = 64
    k = R.NormalizedKernel.from_matrix(np.eye(n) / n, "fp64")
    s = 4 * n
    assert R.entropy_int(k, 2, s, 9).entropy == pytest.approx(math.log(n), rel=1e-12)
    assert R.entropy_taylor(k, 2.5, s, 4, 1 / n, 9).entropy == pytest.approx(math.log(n), rel=1e-12)
    assert R.entropy_chebyshev(k, 2.5, s, 20, 1 / n, 1 / n, 9).entropy == pytest.approx(math.log(n), rel=1e-2)
    assert R.entropy_exact(k, 2.0).entropy == pytest.approx(math.log(n), rel=1e-10)


def test_entropy_errors(R):
    k = R.NormalizedKernel.from_matrix(np.eye(4) / 4, "fp64")
    with pytest.raises(R.RenyiError) as e:
        R.estimate(k, R.EstimatorParams(alpha=1.0 + 1e-12, s=8))
    assert e.value.kind == "alpha_is_one" and e.value.is_usage()
    with pytest.raises(R.RenyiError) as e:
        R.entropy_taylor(k, 2.0, 8, 4, 0.5, 0)
    assert e.value.kind == "invalid_argument"


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_config2_shape_parity(R, orc, prec):
    """Config 2 reduced to n=3000: alpha=1.5 Chebyshev [0,1] m=40, Hutch++ 20+40 Rademacher."""
    n, d = 3000, 32
    x = f32(orc.fill_gaussian(orc.derive_key(7, orc.hash_name("X")), n, d))
    sigma = math.sqrt(d)
    a = orc.build_kernel(x, sigma)
    kw = dict(alpha=1.5, method="chebyshev", s=60, m=40, seed=3, bounds=(0.0, 1.0), probe_kind="rademacher",
              s_q=20, s_g=40)
    ref = orc.estimate(a, **kw)
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=60, m=40, seed=3, bounds=R.SpectrumBounds(u=0.0, v=1.0),
                          probe_kind="rademacher", s_q=20, s_g=40)
    got = R.entropy(x, sigma, p, precision=prec)
    assert abs(got.trace_estimate - ref["trace"]) <= TOL[prec] * ref["trace"]
    assert abs(got.entropy - ref["entropy"]) <= TOL[prec] * abs(ref["entropy"])


def test_config3_shape_parity(R, orc):
    """Config 3 reduced to n=2500: 10-component mixture, alpha=0.5 Taylor m=30, Hutchinson s=100 Gaussian."""
    from workloads import mixture10

    n, d = 2500, 64
    x = f32(mixture10(n, d, 11))
    sigma = math.sqrt(d)
    a = orc.build_kernel(x, sigma)
    b = orc.estimate_bounds(a, seed=orc.derive_key(5, orc.hash_name("bounds")))
    ref = orc.estimate(a, alpha=0.5, method="taylor", s=100, m=30, seed=5, bounds=(b["u"], b["v"]), s_q=0, s_g=100)
    p = R.EstimatorParams(alpha=0.5, method="taylor", s=100, m=30, seed=5, bounds=R.SpectrumBounds(u=b["u"], v=b["v"]),
                          s_q=0, s_g=100)
    got = R.entropy(x, sigma, p, precision="fp32")
    assert abs(got.entropy - ref["entropy"]) <= 1e-4 * abs(ref["entropy"])
    # and with the bounds from the device power iteration (fp64 storage: same iteration count)
    k = R.build_kernel(x, R.GaussianKernel(sigma), "fp64")
    gb = R.estimate_bounds(k, R.PowerOptions(seed=orc.derive_key(5, orc.hash_name("bounds"))))
    assert abs(gb.v - b["v"]) <= 1e-9 * b["v"]


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_mutual_information_parity(R, orc, prec):
    """Config 4 reduced to n=1200: X (d=16), Y = XW + 0.5 noise (d=8), alpha=1.01 Chebyshev m=60, s=90."""
    from workloads import mi_inputs

    n = 1200
    x, y = mi_inputs(n, 4)
    x, y = f32(x), f32(y)
    sx, sy = 4.0, math.sqrt(8)
    ax, ay = orc.build_kernel(x, sx), orc.build_kernel(y, sy)
    kw = dict(alpha=1.01, method="chebyshev", s=90, m=60, bounds=(0.0, 1.0))
    ref = orc.mutual_information(ax, ay, seed=13, **kw)
    p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=90, m=60, seed=13, bounds=R.SpectrumBounds(u=0, v=1))
    got = R.mutual_information_samples(x, R.GaussianKernel(sx), y, R.GaussianKernel(sy), p, precision=prec)
    for key in ("vars_entropy", "target_entropy", "joint_entropy"):
        assert abs(getattr(got, key) - ref[key]) <= TOL[prec] * abs(ref[key]), key
    assert got.value == pytest.approx(got.vars_entropy + got.target_entropy - got.joint_entropy, rel=1e-14)
    kx = R.build_kernel(x, R.GaussianKernel(sx), prec)
    ky = R.build_kernel(y, R.GaussianKernel(sy), prec)
    got2 = R.mutual_information([kx], ky, p)
    assert abs(got2.joint_entropy - ref["joint_entropy"]) <= TOL[prec] * abs(ref["joint_entropy"])


def test_mi_exact_identities(R, orc):  # test_measures.cpp:77-92
    a = R.build_kernel(orc.fill_gaussian(77, 30, 2), R.GaussianKernel(1.0), "fp64")
    ex = R.EstimatorParams(alpha=2.0, method="exact")
    mi = R.mutual_information([a], a, ex)
    s_a = R.joint_entropy([a], ex).entropy
    s_aa = R.joint_entropy([a, a], ex).entropy
    assert mi.value == pytest.approx(2 * s_a - s_aa, rel=1e-12)
    j = R.NormalizedKernel.from_matrix(np.full((30, 30), 1 / 30), "fp64")
    mi = R.mutual_information([a], j, ex)
    assert abs(mi.value) <= 1e-10


def test_estimates_deterministic(R, orc):
    x = f32(orc.fill_gaussian(5, 2500, 16))
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=60, m=40, seed=3, bounds=R.SpectrumBounds(u=0, v=1))
    e1 = R.entropy(x, 4.0, p, "fp32")
    e2 = R.entropy(x, 4.0, p, "fp32")
    assert e1.entropy == e2.entropy and e1.trace_estimate == e2.trace_estimate


def test_out_of_memory_is_reported_and_recoverable(R):
    """A materialised fp32 A at n = 250k needs 250 GB (> 180 GB of HBM): the build fails with the
    out_of_memory kind, and the context keeps working afterwards."""
    import torch

    n, d = 250_000, 2
    ctx = R.Context(0)
    xd = torch.zeros(d, n, dtype=torch.float64, device="cuda")
    xd[0] = torch.arange(n, dtype=torch.float64, device="cuda") * 1e-3
    with pytest.raises(R.RenyiError) as e:
        R.build_kernel_dev(xd.data_ptr(), n, d, n, R.GaussianKernel(1.0), "fp32", ctx=ctx)
    assert e.value.kind == "out_of_memory"
    # the matrix-free path handles the same samples without storing A
    k = R.build_kernel_dev(xd.data_ptr(), n, d, n, R.GaussianKernel(1.0), "mf", ctx=ctx)
    y = R.ops.matvec(k, np.ones(n))
    # interior rows: (1/n) * sum_j exp(-(1e-3 (i-j))^2 / 2) = sqrt(2 pi) / 1e-3 / n (edges: half)
    assert np.all(np.isfinite(y))
    assert abs(y[n // 2] - math.sqrt(2 * math.pi) / 1e-3 / n) <= 1e-3 * y[n // 2]
    assert abs(y[0] - 0.5 * math.sqrt(2 * math.pi) / 1e-3 / n) <= 2e-3 * y[0]


@pytest.mark.parametrize("spec", [("int", 1, 0, 0.0, 1.0), ("int", 5, 0, 0.0, 1.0), ("taylor", 0.7, 2, 0.0, 1.0),
                                  ("taylor", 2.5, 7, 0.0, 0.6), ("chebyshev", 1.5, 1, 0.0, 1.0),
                                  ("chebyshev", 1.5, 2, 0.0, 1.0), ("chebyshev", 1.2, 7, 0.0, 1.0),
                                  ("chebyshev", 2.0, 31, 0.02, 0.9)])
def test_trace_moment_doubling_edge_degrees(R, orc, spec):
    """Traces take ceil(m/2) passes by moment doubling: odd and even degrees,
    m = 1 and 2, integer powers 1 and 5, narrow Chebyshev intervals — against the oracle's
    sequential apply_panel (poly.cpp:97-134) and x.f(A)x."""
    kind, alpha, m, u, v = spec
    n, s = 700, 9
    x = orc.fill_gaussian(41, n, 4)
    p = orc.fill_gaussian(42, n, s)
    ospec = orc.Spec(kind, alpha, m, u, v)
    rspec = {"int": lambda: R.MatrixFunctionSpec.int_power(int(alpha)),
             "taylor": lambda: R.MatrixFunctionSpec.taylor(alpha, m, v),
             "chebyshev": lambda: R.MatrixFunctionSpec.chebyshev(alpha, m, u, v)}[kind]()
    for prec in ("fp64", "fp32"):
        xx = x if prec == "fp64" else f32(x)
        a = orc.build_kernel(xx, 1.3)
        ref_tr = np.einsum("ij,ij->j", p, orc.apply_panel(ospec, a, p))
        tr = R.matfun_traces(rspec, R.build_kernel(xx, R.GaussianKernel(1.3), prec), p)
        assert np.max(np.abs(tr - ref_tr) / np.abs(ref_tr)) <= (1e-10 if prec == "fp64" else TOL["fp32"]), prec
