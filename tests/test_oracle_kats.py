"""Pins the CPU oracle (oracle/renyi_oracle.cpp) to the reference's own
known-answer tests (proj/tests/test_*.cpp). The reference has no stored golden
vectors; every expectation there is analytic or comes from an eigenvalue
oracle, and each case below cites the reference test it restates."""
import math

import numpy as np
import pytest

from fixtures import (cheb_bound, chebyshev_closed_form_u0, mixture_kernel, oracle_trace_power,
                      random_low_rank_psd, random_unit_trace_spd, spd_from_spectrum)


# ------------------------------------------------------------------ rng (rng.cpp)
def test_rng_known_values(orc):
    # splitmix64 finalizer of the golden-gamma step, FNV-1a test vectors
    assert orc.mix64(0) == 0xE220A8397B1DCDAF
    assert orc.hash_name("") == 0xCBF29CE484222325
    assert orc.hash_name("a") == 0xAF63DC4C8601EC8C
    assert orc.hash_name("foobar") == 0x85944171F73967E8


def test_rng_panel_prefix_stable_and_gaussian(orc):
    a = orc.probe_panel(1000, 3, 5, "hutchpp-probe")
    b = orc.probe_panel(1000, 5, 5, "hutchpp-probe")
    assert np.array_equal(a, b[:, :3])  # column count changes never reshuffle (hutchpp.hpp:29-31)
    g = orc.probe_panel(20000, 4, 9, "x")
    assert abs(g.mean()) < 0.02 and abs(g.var() - 1.0) < 0.03
    r = orc.probe_panel(20000, 2, 9, "x", kind="rademacher")
    assert set(np.unique(r)) == {-1.0, 1.0} and abs(r.mean()) < 0.02


# ------------------------------------------------------------------ ops (test_ops.cpp)
def test_gram_matches_naive_formula(orc):  # test_ops.cpp:39-50
    x = orc.fill_gaussian(12, 23, 3)
    g = orc.gaussian_gram(x, 1.3)
    d2 = ((x[:, None, :] - x[None, :, :]) ** 2).sum(-1)
    np.testing.assert_allclose(g, np.exp(-d2 / (2 * 1.3 * 1.3)), rtol=1e-12, atol=0)


def test_matvec_and_panel_match_naive(orc):  # test_ops.cpp:52-67 and 10-37
    a = random_unit_trace_spd(31, 12, orc)
    x = orc.fill_gaussian(7, 31, 1)[:, 0]
    np.testing.assert_allclose(orc.matvec(a, x), a @ x, rtol=1e-12, atol=1e-15)
    p = orc.fill_gaussian(8, 31, 29)
    np.testing.assert_allclose(orc.matmul_panel(a, p), a @ p, rtol=1e-12, atol=1e-15)


def test_gram_exactly_symmetric_unit_diagonal(orc):  # test_ops.cpp:69-76
    x = orc.fill_gaussian(13, 64, 5)
    g = orc.gaussian_gram(x, 1.0)
    assert np.array_equal(g, g.T)
    assert np.all(np.diag(g) == 1.0)


# ------------------------------------------------------------------ kernel (test_kernel.cpp)
def _invariants(a):
    n = a.shape[0]
    assert np.max(np.abs(a - a.T)) <= 1e-12
    np.testing.assert_allclose(np.diag(a), 1.0 / n, rtol=1e-12)
    assert abs(np.trace(a) - 1.0) <= 1e-10


def test_two_identical_samples_give_half(orc):  # test_kernel.cpp:25-32
    x = np.array([[0.3, -1.2, 0.7], [0.3, -1.2, 0.7]])
    np.testing.assert_allclose(orc.build_kernel(x, 1.0), 0.5, rtol=1e-15)


def test_far_samples_give_identity_over_n(orc):  # test_kernel.cpp:34-39
    x = np.array([[0.0], [1e6], [2e6], [3e6]])
    assert np.max(np.abs(orc.build_kernel(x, 1.0) - np.eye(4) / 4)) <= 1e-15


def test_three_point_line(orc):  # test_kernel.cpp:41-50
    a = orc.build_kernel(np.array([[0.0], [1.0], [2.0]]), 1.0)
    assert a[0, 1] == pytest.approx(math.exp(-0.5) / 3, rel=1e-15)
    assert a[0, 2] == pytest.approx(math.exp(-2.0) / 3, rel=1e-15)
    assert a[1, 2] == pytest.approx(math.exp(-0.5) / 3, rel=1e-15)
    _invariants(a)


def test_kernel_invariants_and_psd(orc):  # test_kernel.cpp:52-63 (Gaussian reps)
    for rep in (0, 2):
        x = orc.fill_gaussian(21 + rep, 40 + 3 * rep, 4)
        a = orc.build_kernel(x, 0.7 + 0.3 * rep)
        _invariants(a)
        assert np.linalg.eigvalsh(a).min() >= -1e-10


def test_polynomial_gram_matches_naive_formula(orc):  # test_ops.cpp:51-56
    x = orc.fill_gaussian(12, 23, 3)
    p = orc.polynomial_gram(x, 3, 0.5)
    np.testing.assert_allclose(p, (x @ x.T + 0.5) ** 3, rtol=1e-12, atol=0)
    assert np.array_equal(p, p.T)


def test_polynomial_kernel_invariants_and_psd(orc):  # test_kernel.cpp:52-63 (polynomial reps)
    for rep in (1, 3):
        x = orc.fill_gaussian(21 + rep, 40 + 3 * rep, 4)
        a = orc.build_kernel_polynomial(x, 2, 1.0)
        _invariants(a)
        assert np.linalg.eigvalsh(a).min() >= -1e-10
        k = (x @ x.T + 1.0) ** 2
        isd = 1.0 / np.sqrt(np.diag(k))
        ref = (k / x.shape[0]) * isd[:, None] * isd[None, :]
        np.fill_diagonal(ref, 1.0 / x.shape[0])
        np.testing.assert_allclose(a, ref, rtol=1e-12, atol=1e-16)


def test_polynomial_kernel_errors(orc):  # test_kernel.cpp:65-77
    x = np.zeros((3, 2))
    x[1] = [1.0, 0.0]
    x[2] = [0.0, 1.0]
    with pytest.raises(orc.OracleError) as e:  # zero diagonal: sample 0 with offset 0
        orc.build_kernel_polynomial(x, 2, 0.0)
    assert e.value.code == 2 and "not positive" in str(e.value)
    with pytest.raises(orc.OracleError) as e:  # non-finite kernel values
        orc.build_kernel_polynomial(np.array([[1e200], [-1e200]]), 2, 1.0)
    assert e.value.code == 3
    for deg, off in ((0, 1.0), (2, -0.5)):
        with pytest.raises(orc.OracleError) as e:
            orc.build_kernel_polynomial(orc.fill_gaussian(3, 4, 2), deg, off)
        assert e.value.code == 1


def test_chebyshev_rank_deficient_polynomial_kernel(orc):  # test_entropy.cpp:121-131
    x = orc.fill_gaussian(65, 120, 4)
    x[90:] = x[:30]  # duplicates force u = 0
    a = orc.build_kernel_polynomial(x, 2, 1.0)
    exact = orc.entropy_exact(a, 2.5)
    b = orc.estimate_bounds(a)
    est = orc.estimate(a, alpha=2.5, method="chebyshev", s=64, m=30, seed=3, bounds=(0.0, b["v"]))
    assert abs(est["entropy"] - exact) <= 1e-2 * abs(exact)


def test_acceptance_rank_deficient_polynomial(orc):  # acceptance.cpp:230-254 (criterion 6)
    x = orc.fill_gaussian(888, 400, 8)
    x[300:] = x[:100]
    a = orc.build_kernel_polynomial(x, 2, 1.0)
    exact = orc.entropy_exact(a, 2.5)
    b = orc.estimate_bounds(a, seed=5)
    assert b["rank_deficient"]
    worst = max(abs(orc.estimate(a, alpha=2.5, method="chebyshev", s=64, m=30, seed=sd,
                                 bounds=(0.0, b["v"]))["entropy"] - exact) / abs(exact) for sd in range(20))
    assert worst <= 1e-2


def test_kernel_errors(orc):  # test_kernel.cpp:65-83
    with pytest.raises(orc.OracleError) as e:
        orc.build_kernel(np.array([[1.0, 2.0]]), 1.0)
    assert e.value.code == 1
    with pytest.raises(orc.OracleError) as e:
        orc.build_kernel(np.array([[np.nan], [1.0]]), 1.0)
    assert e.value.code == 3
    with pytest.raises(orc.OracleError):
        orc.build_kernel(np.array([[0.0], [1.0]]), 0.0)


def test_hadamard_kats(orc):  # test_kernel.cpp:85-127
    eye = np.eye(5) / 5
    assert np.max(np.abs(orc.hadamard_joint(eye, eye) - eye)) <= 1e-15
    a = orc.build_kernel(orc.fill_gaussian(22, 12, 3), 1.0)
    j = np.full((12, 12), 1.0 / 12)
    assert np.max(np.abs(orc.hadamard_joint(a, j) - a)) <= 1e-15
    a = orc.build_kernel(orc.fill_gaussian(23, 4, 2), 1.0)
    b = orc.build_kernel(orc.fill_gaussian(24, 4, 2), 0.5)
    assert abs(np.trace(orc.hadamard_joint(a, b)) - 1.0) <= 1e-12
    # bitwise permutation invariance (canonical content order)
    assert np.array_equal(orc.hadamard_joint(a, b), orc.hadamard_joint(b, a))
    with pytest.raises(orc.OracleError) as e:
        orc.hadamard_joint(np.eye(4) / 4, np.eye(5) / 5)
    assert e.value.code == 4


# ------------------------------------------------------------------ spectrum (test_spectrum.cpp)
def test_flat_spectrum_bounds(orc):  # test_spectrum.cpp:12-19
    b = orc.estimate_bounds(np.eye(8) / 8)
    assert b["v"] == pytest.approx(1 / 8, rel=1e-5) and b["u"] == pytest.approx(1 / 8, rel=1e-5)
    assert b["v"] >= 1 / 8 and b["u"] <= 1 / 8


def test_rank1_projector_gives_v1(orc):  # test_spectrum.cpp:21-30
    w = orc.fill_gaussian(41, 16, 1)[:, 0]
    w /= np.linalg.norm(w)
    r, _, _ = orc.power_method(np.outer(w, w), seed=3)
    assert min(max(r * (1 + 1e-6), 1 / 16), 1.0) == 1.0


def test_diag_example(orc):  # test_spectrum.cpp:32-43
    a = np.diag([0.5, 0.3, 0.2])
    b = orc.estimate_bounds(a, max_iters=200, tol=1e-8, seed=7)
    assert abs(b["v"] - 0.5) <= 1e-6 and abs(b["u"] - 0.2) <= 1e-6


def test_duplicates_force_u0(orc):  # test_spectrum.cpp:45-61
    d = orc.fill_gaussian(42, 5, 2)
    x = np.vstack([d, d])
    b = orc.estimate_bounds(orc.build_kernel(x, 1.0), max_iters=2000, tol=1e-13, seed=5)
    assert b["u"] == 0.0 and b["rank_deficient"] and math.isinf(b["kappa"])


def test_sandwich(orc):  # test_spectrum.cpp:63-80
    for rep in range(4):
        n = 40 + 32 * rep
        a = random_unit_trace_spd(n, 43 + rep, orc, 0.1)
        e = np.linalg.eigvalsh(a)
        b = orc.estimate_bounds(a, max_iters=5000, tol=1e-12, seed=100 + rep)
        assert b["u"] <= e.min() + 1e-6 and b["v"] >= e.max() - 1e-6 and b["u"] <= b["v"]


def test_nonconvergence_is_diagnostic(orc):  # test_spectrum.cpp:97-108
    a = random_unit_trace_spd(50, 46, orc)
    b = orc.estimate_bounds(a, max_iters=1, tol=1e-14)
    assert not b["v_converged"] and 1 / 50 <= b["v"] <= 1 and b["u"] <= b["v"]


# ------------------------------------------------------------------ poly (test_poly.cpp)
def test_binomials(orc):  # test_poly.cpp:38-56
    assert list(orc.binomial_coeffs(1.5, 2)) == [1.0, 1.5, 0.375]
    assert list(orc.binomial_coeffs(2.0, 4)) == [1.0, 2.0, 1.0, 0.0, 0.0]
    assert list(orc.binomial_coeffs(0.5, 3)) == [1.0, 0.5, -0.125, 0.0625]


def test_chebyshev_identity_function(orc):  # test_poly.cpp:58-64 (f = lambda on [0,1]: c0 = 1, c1 = 1/2)
    c = orc.chebyshev_coeffs(1.0, 8, 0.0, 1.0)
    assert c[0] == pytest.approx(1.0, abs=1e-13) and c[1] == pytest.approx(0.5, abs=1e-13)
    assert np.max(np.abs(c[2:])) <= 1e-12


def test_chebyshev_rejects_bad_intervals(orc):  # test_poly.cpp:66-70
    for u, v in [(-0.1, 0.9), (0.5, 0.5), (0.5, 0.2)]:
        with pytest.raises(orc.OracleError):
            orc.chebyshev_coeffs(0.5, 10, u, v)


def test_closed_form_u0(orc):  # test_poly.cpp:72-85: node sum converges to the series
    for alpha in (0.5, 1.5, 2.5):
        for v in (0.7, 1.0):
            closed = chebyshev_closed_form_u0(alpha, 30, v)
            node = orc.chebyshev_coeffs(alpha, 4095, 0.0, v)[:31]
            tol = 1e-6 if alpha == 0.5 else 1e-8  # aliasing of the 4096-node rule at the u=0 branch point
            assert np.max(np.abs(node - closed)) <= tol


def test_ellipse_bound(orc):  # test_poly.cpp:87-101
    alpha, u, v, m = 0.5, 0.1, 0.9, 15
    c = orc.chebyshev_coeffs(alpha, m, u, v)
    lam = np.linspace(u, v, 100000)
    x = (2 * lam - (v + u)) / (v - u)
    val = np.polynomial.chebyshev.chebval(x, np.concatenate([[0.5 * c[0]], c[1:]]))
    assert np.max(np.abs(val - lam ** alpha)) <= cheb_bound(alpha, u, v, m)


def test_taylor_tail_bound(orc):  # test_poly.cpp:103-122
    alpha, u, v = 1.5, 0.2, 0.5
    c = orc.taylor_tail_constant(alpha)
    for m in (5, 10, 20, 40):
        spec = orc.Spec("taylor", alpha, m, 0.0, v)
        worst = 0.0
        for lam in np.linspace(u, v, 400):
            err = abs(orc.scalar_value(spec, lam) - lam ** alpha)
            bound = c * abs(u / v - 1.0) ** (m + 1) * lam ** alpha
            worst = max(worst, err / (bound + 1e-15))
        assert worst <= 1.0


def test_apply_diag_matrices(orc):  # test_poly.cpp:138-177
    a = np.eye(6) / 6
    e1 = np.zeros(6)
    e1[0] = 1
    y = orc.apply_panel(orc.Spec("int", 2), a, e1)[:, 0]
    assert np.max(np.abs(y - e1 / 36)) <= 1e-15
    d = np.diag([0.5, 0.3, 0.2])
    y = orc.apply_panel(orc.Spec("taylor", 0.5, 40, 0.0, 0.5), d, np.ones(3))[:, 0]
    c = orc.taylor_tail_constant(0.5)
    for i, lam in enumerate([0.5, 0.3, 0.2]):
        assert abs(y[i] - lam ** 0.5) <= c * abs(0.2 / 0.5 - 1) ** 41 * lam ** 0.5 + 1e-14
    spec = orc.Spec("chebyshev", 1.5, 15, 0.2, 0.5)
    _, sv = orc.spec_coeffs(spec)
    e2 = np.array([0.0, 1.0, 0.0])
    y = orc.apply_panel(spec, d, e2)[:, 0]
    assert sv > 0.5
    assert abs(y[1] - 0.3 ** 1.5) <= cheb_bound(1.5, 0.2, sv, 15) + 1e-14
    assert abs(y[0]) <= 1e-12 and abs(y[2]) <= 1e-12


def test_scalar_consistency_linearity_panel(orc):  # test_poly.cpp:179-220
    rng = np.random.default_rng(31)
    for spec in (orc.Spec("int", 3), orc.Spec("taylor", 1.3, 12, 0, 0.8), orc.Spec("chebyshev", 2.2, 9, 0.1, 0.8)):
        for lam in 0.1 + 0.7 * rng.random(10):
            y = orc.apply_panel(spec, np.array([[lam]]), np.ones(1))[0, 0]
            assert y == pytest.approx(orc.scalar_value(spec, lam), rel=1e-13)
    a = random_unit_trace_spd(24, 32, orc)
    x, y = orc.fill_gaussian(5, 24, 1)[:, 0], orc.fill_gaussian(6, 24, 1)[:, 0]
    for spec in (orc.Spec("int", 2), orc.Spec("taylor", 0.5, 15, 0, 1.0), orc.Spec("chebyshev", 1.5, 15, 0, 1.0)):
        lhs = orc.apply_panel(spec, a, 0.7 * x - 1.9 * y)[:, 0]
        rhs = 0.7 * orc.apply_panel(spec, a, x)[:, 0] - 1.9 * orc.apply_panel(spec, a, y)[:, 0]
        assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(rhs)
    a = random_unit_trace_spd(20, 33, orc)
    p = orc.fill_gaussian(34, 20, 5)
    spec = orc.Spec("chebyshev", 0.8, 10, 0.0, 1.0)
    out = orc.apply_panel(spec, a, p)
    for j in range(5):
        assert np.max(np.abs(out[:, j] - orc.apply_panel(spec, a, p[:, j])[:, 0])) <= 1e-13


def test_safeguard_and_tail_constant(orc):  # test_poly.cpp:222-242
    assert orc.safeguard(0.0, 0.6) == 0.6
    u = 0.1
    assert orc.safeguard(u, 0.11) == pytest.approx(u + 2 * math.sqrt(2 * u - u * u))
    assert orc.safeguard(u, 0.99) == 0.99
    for alpha in (0.5, 1.5, 2.5):
        c = orc.taylor_tail_constant(alpha)
        assert 0 < c <= 1 + 1e-12


# ------------------------------------------------------------------ hutchpp (test_hutchpp.cpp)
def test_rank2_kernel_trace_is_one(orc):  # test_hutchpp.cpp:12-21
    x = np.array([[0.0 if i % 2 == 0 else 1.0] for i in range(40)])
    a = orc.build_kernel(x, 1.0)
    for seed in range(20):
        z = orc.hutchpp(orc.Spec("int", 1), a, 2, 4, seed)
        assert abs(z["value"] - 1.0) <= 1e-8


def test_low_rank_exact(orc):  # test_hutchpp.cpp:40-51
    a = random_low_rank_psd(60, 2, 52, orc)
    exact = oracle_trace_power(a, 2.0)
    for seed in range(25):
        z = orc.hutchpp(orc.Spec("int", 2), a, 2, 4, seed)
        assert abs(z["value"] - exact) <= 1e-10 * exact
        assert z["sketch_rank"] == 2 and abs(z["residual_part"]) <= 1e-12


def test_decomposition_and_queries(orc):  # test_hutchpp.cpp:53-58,74-78
    a = mixture_kernel(64, 4, 1.0, 7, orc)
    z = orc.hutchpp(orc.Spec("int", 2), a, 4, 8, 3)
    assert z["value"] == z["low_rank_part"] + z["residual_part"] and z["queries_used"] > 0
    assert orc.expected_queries(orc.Spec("int", 2), 8) == 22
    assert orc.expected_queries(orc.Spec("taylor", 0.5, 15, 0, 1.0), 8) == 100
    assert orc.expected_queries(orc.Spec("chebyshev", 1.5, 15, 0.1, 0.9), 16) == 200


def test_mixture_one_percent(orc):  # test_hutchpp.cpp:60-72
    a = mixture_kernel(1000, 10, 1.0, 2024, orc)
    exact = math.log(oracle_trace_power(a, 2.0)) / (1 - 2.0)
    hits = 0
    for seed in range(100):
        z = orc.hutchpp(orc.Spec("int", 2), a, 2, 6, seed)
        hits += abs(math.log(z["value"]) / (1 - 2.0) - exact) <= 0.01 * exact
    assert hits >= 95


def test_determinism_and_exact_degeneration(orc):  # test_hutchpp.cpp:108-136
    a = mixture_kernel(80, 4, 1.0, 5, orc)
    f = orc.Spec("taylor", 1.5, 10, 0, 1.0)
    z1, z2, z3 = (orc.hutchpp(f, a, 3, 6, s) for s in (42, 42, 43))
    assert z1 == z2 and z3["value"] != z1["value"]
    a = random_unit_trace_spd(12, 54, orc)
    exact = oracle_trace_power(a, 2.0)
    z1 = orc.hutchpp(orc.Spec("int", 2), a, 12, 24, 1)   # s=48: s/4 = n
    z2 = orc.hutchpp(orc.Spec("int", 2), a, 10, 20, 2)   # s=40: s_g >= n - rank
    assert z1["exact"] and z2["exact"]
    assert abs(z1["value"] - exact) <= 1e-12 * exact and abs(z2["value"] - exact) <= 1e-12 * exact
    with pytest.raises(orc.OracleError) as e:
        orc.hutchpp(orc.Spec("int", 2), np.zeros((10, 10)), 2, 4, 0)
    assert e.value.code == 6


# ------------------------------------------------------------------ entropy (test_entropy.cpp)
def test_exact_entropy_kats(orc):  # test_entropy.cpp:25-43
    eye3 = np.eye(3) / 3
    assert orc.entropy_exact(eye3, 2.0) == pytest.approx(math.log(3), rel=1e-12)
    assert orc.entropy_exact(eye3, 0.5) == pytest.approx(math.log(3), rel=1e-12)
    w = orc.fill_gaussian(61, 12, 1)[:, 0]
    w /= np.linalg.norm(w)
    assert abs(orc.entropy_exact(np.outer(w, w), 2.0)) <= 1e-10
    assert orc.entropy_exact(np.diag([0.5, 0.3, 0.2]), 2.0) == pytest.approx(-math.log(0.38), rel=1e-12)


def test_alpha_validation(orc):  # test_entropy.cpp:45-55
    with pytest.raises(orc.OracleError) as e:
        orc.entropy_from_trace(1.0, 1.0)
    assert e.value.code == 8
    for t in (0.0, -0.1):
        with pytest.raises(orc.OracleError) as e:
            orc.entropy_from_trace(t, 2.0)
        assert e.value.code == 7


def test_entropy_int_low_rank_exact(orc):  # test_entropy.cpp:66-74
    a = random_low_rank_psd(60, 3, 62, orc)
    exact = orc.entropy_exact(a, 3.0)
    for seed in range(10):
        est = orc.estimate(a, alpha=3.0, method="int", s=16, seed=seed)
        assert abs(est["entropy"] - exact) <= 1e-10 * abs(exact)


def test_taylor_chebyshev_rotated(orc):  # test_entropy.cpp:76-105
    a = spd_from_spectrum([0.5, 0.3, 0.2], 63, orc)
    exact = orc.entropy_exact(a, 1.5)
    est = orc.estimate(a, alpha=1.5, method="taylor", s=64, m=40, seed=1, bounds=(0.0, 0.5 * (1 + 1e-9)))
    assert abs(est["entropy"] - exact) <= 1e-3 * abs(exact)
    a = spd_from_spectrum([0.5, 0.3, 0.2], 64, orc)
    exact = orc.entropy_exact(a, 1.5)
    est = orc.estimate(a, alpha=1.5, method="chebyshev", s=64, m=15, seed=2,
                       bounds=(0.2 * (1 - 1e-6), 0.5 * (1 + 1e-6)))
    assert abs(est["entropy"] - exact) <= 1e-3 * abs(exact)


def test_all_paths_agree_on_flat_spectrum(orc):  # test_entropy.cpp:142-155
    n = 64
    a = np.eye(n) / n
    s = 4 * n
    exp_ = math.log(n)
    assert orc.entropy_exact(a, 2.0) == pytest.approx(exp_, rel=1e-10)
    assert orc.estimate(a, alpha=2.0, method="int", s=s, seed=9)["entropy"] == pytest.approx(exp_, rel=1e-12)
    assert orc.estimate(a, alpha=2.5, method="taylor", s=s, m=4, seed=9, bounds=(0.0, 1 / n))["entropy"] == \
        pytest.approx(exp_, rel=1e-12)
    assert orc.estimate(a, alpha=2.5, method="chebyshev", s=s, m=20, seed=9, bounds=(1 / n, 1 / n))["entropy"] == \
        pytest.approx(exp_, rel=1e-2)


def test_select_params(orc):  # test_entropy.cpp:157-177
    assert orc.select_params(2.0, 0.1, 0.1, 0.0, 1.0, math.inf, 100, "int") == (20, 0)
    assert orc.select_params(1.5, 0.01, 0.1, 0.001, 0.1, 100.0, 100, "chebyshev")[1] == 100
    assert orc.select_params(2.0, 0.01, 0.1, 0.0, 0.5, math.inf, 1000, "chebyshev")[1] == 71


def test_mu_bound(orc):  # test_entropy.cpp:198-234
    assert orc.mu_bound(0.0, 0.5, 2.0, 10)[0] == pytest.approx(0.5, rel=1e-14)
    assert orc.mu_bound(0.1, 0.1, 2.0, 10)[0] == pytest.approx(0.1, rel=1e-14)
    with pytest.raises(orc.OracleError):
        orc.mu_bound(0.05, 0.04, 2.0, 10)
    rng = np.random.default_rng(66)
    for rep in range(40):
        n = 5 + int(rng.integers(60))
        e = 0.05 + 0.95 * rng.random(n)
        e /= e.sum()
        alpha = 0.5 + 0.4 * rng.random() if rep % 2 == 0 else 1.5 + 3 * rng.random()
        tr = float(np.sum(e ** alpha))
        _, lo, hi = orc.mu_bound(e.min(), e.max(), alpha, n)
        assert lo - 1e-12 <= tr <= hi + 1e-12


def test_estimate_routes_and_oracle_agreement(orc):  # test_entropy.cpp:236-260
    a = mixture_kernel(200, 6, 1.0, 77, orc)
    ei = orc.estimate(a, alpha=2.0, s=16, seed=5)
    assert ei["method"] == 1 and ei["s"] == 16
    ec = orc.estimate(a, alpha=1.5, s=256, m=60, seed=5)
    assert ec["method"] in (2, 3) and ec["has_bounds"] and ec["trace"] > 0
    assert ec["entropy"] == pytest.approx(math.log(ec["trace"]) / (1 - 1.5))
    ex = orc.entropy_exact(a, 1.5)
    assert abs(ec["entropy"] - ex) / abs(ex) <= 2e-2
    assert orc.estimate(mixture_kernel(100, 4, 1.0, 78, orc), alpha=2.0, epsilon=0.1, delta=0.1, seed=1)["s"] == 20


def test_eigvals_match_numpy(orc):
    a = random_unit_trace_spd(50, 90, orc)
    np.testing.assert_allclose(orc.eigvals(a), np.linalg.eigvalsh(a), atol=1e-14)


def test_colpiv_rank_rule(orc):  # hutchpp.cpp:91-95: 1e-12 relative threshold
    w = orc.fill_gaussian(3, 50, 3)
    y = np.hstack([w, w[:, :1] + w[:, 1:2]])  # rank 3 with 4 columns
    r, q = orc.colpiv_rank(y, 1e-12, want_q=True)
    assert r == 3
    np.testing.assert_allclose(q.T @ q, np.eye(3), atol=1e-13)


# ------------------------------------------------------------------ measures (test_measures.cpp)
def test_mi_identities(orc):  # test_measures.cpp:77-92,132-146
    a = orc.build_kernel(orc.fill_gaussian(77, 30, 2), 1.0)
    ex = dict(alpha=2.0, method="exact")
    s_a = orc.entropy_exact(a, 2.0)
    s_aa = orc.entropy_exact(orc.hadamard_joint(a, a), 2.0)
    assert orc.mutual_information(a, a, **ex)["value"] == pytest.approx(2 * s_a - s_aa, rel=1e-12)
    j = np.full((30, 30), 1 / 30)
    mi = orc.mutual_information(a, j, **ex)
    assert abs(mi["value"]) <= 1e-10 and abs(mi["target_entropy"]) <= 1e-10
    a = orc.build_kernel(orc.fill_gaussian(83, 60, 2), 1.0)
    b = orc.build_kernel(orc.fill_gaussian(84, 60, 2), 1.0)
    mi = orc.mutual_information(a, b, alpha=2.0, method="int", s=16, seed=11)
    assert mi["value"] == pytest.approx(mi["vars_entropy"] + mi["target_entropy"] - mi["joint_entropy"], rel=1e-14)
    assert mi == orc.mutual_information(a, b, alpha=2.0, method="int", s=16, seed=11)


def test_hadamard_joint_n_permutation_invariant(orc):  # test_kernel.cpp:113-127
    ks = [orc.build_kernel(orc.fill_gaussian(24 + v, 10, 2), 1.0) for v in range(3)]
    ref = orc.hadamard_joint_n(ks)
    assert np.array_equal(ref, orc.hadamard_joint_n([ks[2], ks[0], ks[1]]))
    assert abs(np.trace(ref) - 1.0) <= 1e-12
    # L = 2 equals the pairwise entry bitwise
    assert np.array_equal(orc.hadamard_joint_n(ks[:2]), orc.hadamard_joint(ks[0], ks[1]))
