"""The reference's acceptance criteria (proj/tests/acceptance.cpp:86-271) run through the device path:
the same fixtures (mixture kernels from the reference stream, support.hpp:123-126), seeds, trial
schedules (measure_cell, simulate.cpp:19-72) and thresholds (criterion 1's fixtures use numpy rotations,
the reference's Eigen QR being unavailable). Criterion 6 (rank-deficient polynomial
kernel) lives in tests/test_gpu_polynomial.py; 8, 9 and 12 are host arithmetic pinned on the oracle
(tests/test_oracle_kats.py); 11 is tests/test_gpu_features.py."""
import math
import time

import numpy as np
import pytest

from fixtures import oracle_trace_power, random_low_rank_psd, random_unit_trace_spd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mixture(R):
    ctx = R.Context(0)
    k = R.build_kernel(R.mixture_samples(1000, 10, 555), R.GaussianKernel(1.0), "fp64", ctx=ctx)
    lam = np.clip(np.linalg.eigvalsh(k.matrix()), 0.0, 1.0)
    return k, lam


def exact_entropy(lam, alpha):  # entropy_exact (entropy.cpp:71-90) from the eigenvalues
    return math.log(float(np.sum(lam[lam > 0] ** alpha))) / (1.0 - alpha)


def test_criterion1_oracle_equivalence(R, orc):  # acceptance.cpp:86-131
    """50 unit-trace SPD fixtures (n log-spaced in [50, 500], spectra in [0.2, 1] before
    normalisation; rotations from numpy QR instead of Eigen's), select_params(1e-3, 1e-2) budgets,
    1000 seeded trials each: >= 990 within 1 % of the eigendecomposition entropy. The budgets put
    every fixture on Hutch++'s exact branch (s/4 >= n), so -- as in the reference's trial_agreement --
    deterministic estimates are verified on spot seeds and counted for all 1000 trials."""
    ctx = R.Context(0)
    alphas = (0.5, 1.5, 2.0, 2.5, 3.0, 5.0)
    worst, worst_desc = 1001, ""
    for f in range(50):
        n = int(round(50.0 * 10.0 ** (f / 49.0)))
        alpha = alphas[f % 6]
        a = random_unit_trace_spd(n, 20240001 + f, orc)
        lam = np.clip(np.linalg.eigvalsh(a), 0.0, 1.0)
        exact = exact_entropy(lam, alpha)
        k = R.NormalizedKernel.from_matrix(a, "fp64", ctx=ctx)
        bounds = R.estimate_bounds(k, R.PowerOptions(max_iters=3000, tol=1e-10, seed=7))
        methods = ("int",) if abs(alpha - round(alpha)) < 1e-9 else ("taylor", "chebyshev")
        for method in methods:
            sel = R.select_params(alpha, 1e-3, 1e-2, bounds, n, method)
            base = R.EstimatorParams(alpha=alpha, method=method, s=sel.s, m=sel.m, seed=1000 + f, bounds=bounds)

            def run(t):
                p = R.EstimatorParams(**{**base.__dict__, "seed": R.derive_key(base.seed, t)})
                return R.estimate(k, p)

            first = run(0)
            tol = 1e-2 * abs(exact)
            if first.deterministic:
                stable = all(abs(run(t).entropy - first.entropy) <= 1e-9 * abs(exact) for t in (1, 250, 500, 999))
                hits = 1000 if (stable and abs(first.entropy - exact) <= tol) else 0
            else:
                ents = [e.entropy for e in R.estimate_trials(k, base, 1000)]
                hits = sum(abs(e - exact) <= tol for e in ents)
            if hits < worst:
                worst, worst_desc = hits, f"n={n} alpha={alpha} method={method} s={sel.s} m={sel.m}"
    print(f"ACCEPTANCE 1: worst fixture {worst_desc}: {worst}/1000 within 1%")
    assert worst >= 990


def test_criterion2_budget_curve(R, mixture):  # acceptance.cpp:133-156
    k, lam = mixture
    exact = exact_entropy(lam, 2.0)
    cells = [R.measure_cell(k, exact, R.EstimatorParams(alpha=2.0, method="int", s=s, seed=99), 100)
             for s in (10, 50, 100, 150)]
    print("ACCEPTANCE 2: MRE(s) " + " ".join(f"{c.s}->{c.mre:.3e}" for c in cells))
    assert cells[0].mre <= 0.01
    for a, b in zip(cells, cells[1:]):
        assert b.mre <= a.mre + 2.0 * a.sd


def test_criterion3_recommended_combo(R, mixture):  # acceptance.cpp:158-175
    k, lam = mixture
    out = []
    for alpha in (0.5, 1.5, 2.5):
        cell = R.measure_cell(k, exact_entropy(lam, alpha),
                              R.EstimatorParams(alpha=alpha, method="chebyshev", s=50, m=15, seed=77), 100)
        out.append(cell.mre)
    print("ACCEPTANCE 3: MRE at s=50, m=15: " + " ".join(f"{v:.3e}" for v in out))
    assert max(out) <= 1e-2


def test_criterion4_alpha_sensitivity(R, mixture):  # acceptance.cpp:177-193
    k, lam = mixture

    def mre_at(alpha):
        p = R.EstimatorParams(alpha=alpha, method="chebyshev", s=100, m=20, seed=13)
        return R.measure_cell(k, exact_entropy(lam, alpha), p, 100).mre

    m04, m08, m12, m25 = (mre_at(a) for a in (0.4, 0.8, 1.2, 2.5))
    print(f"ACCEPTANCE 4: MRE 0.4:{m04:.3e} 0.8:{m08:.3e} 1.2:{m12:.3e} 2.5:{m25:.3e}")
    assert m08 > m04 and m12 > m25


def test_criterion5_taylor_vs_chebyshev(R):  # acceptance.cpp:195-229
    ctx = R.Context(0)
    kernel = lam = None
    for sigma in (1.5, 2.0, 3.0):
        kernel = R.build_kernel(R.mixture_samples(400, 10, 321), R.GaussianKernel(sigma), "fp64", ctx=ctx)
        lam = np.linalg.eigvalsh(kernel.matrix())
        kappa = lam.max() / max(lam.min(), 1e-300)
        if kappa >= 1e3:
            break
    assert kappa >= 1e3

    def cell(k, ev, method, m):
        exact = exact_entropy(np.clip(ev, 0.0, 1.0), 1.5)
        return R.measure_cell(k, exact, R.EstimatorParams(alpha=1.5, method=method, s=100, m=m, seed=31), 50)

    cheb, taylor = cell(kernel, lam, "chebyshev", 20), cell(kernel, lam, "taylor", 40)
    flat = R.build_kernel(R.mixture_samples(400, 10, 321), R.GaussianKernel(0.2), "fp64", ctx=ctx)
    flam = np.linalg.eigvalsh(flat.matrix())
    cf, tf = cell(flat, flam, "chebyshev", 20), cell(flat, flam, "taylor", 40)
    gap, allow = abs(cf.mre - tf.mre), 2.0 * max(cf.sd, tf.sd) + 1e-12
    print(f"ACCEPTANCE 5: sigma={sigma} kappa={kappa:.3e} cheb={cheb.mre:.3e} taylor={taylor.mre:.3e} "
          f"flat gap={gap:.3e} allow={allow:.3e}")
    assert cheb.mre <= taylor.mre and gap <= allow


def test_criterion7_structural_exactness(R, orc):  # acceptance.cpp:256-271 (fixtures: support.hpp:53-58)
    ctx = R.Context(0)
    worst = 0.0
    for r in (1, 2, 5):
        s = 8 if r <= 2 else 20
        a = random_low_rank_psd(60, r, 999 + r, orc)
        exact = oracle_trace_power(a, 2.0)
        k = R.NormalizedKernel.from_matrix(a, "fp64", ctx=ctx)
        for seed in range(100):
            z = R.hutchpp(R.MatrixFunctionSpec.int_power(2), k, R.SketchConfig(s=s, seed=seed))
            worst = max(worst, abs(z.value - exact) / exact)
    print(f"ACCEPTANCE 7: worst relative error {worst:.3e}")
    assert worst <= 1e-10


def test_criterion10_randomized_faster_than_exact(R):  # acceptance.cpp:344-366
    ctx = R.Context(0)
    k = R.build_kernel(R.mixture_samples(2000, 10, 4242), R.GaussianKernel(1.0), "fp64", ctx=ctx)
    t0 = time.perf_counter()
    exact = R.entropy_exact(k, 2.0).entropy
    t_exact = time.perf_counter() - t0
    best, est = 1e300, None
    for _ in range(3):
        t1 = time.perf_counter()
        est = R.entropy_int(k, 2, 50, 7)
        best = min(best, time.perf_counter() - t1)
    rel = abs(est.entropy - exact) / abs(exact)
    print(f"ACCEPTANCE 10: exact {t_exact * 1e3:.1f} ms vs randomized {best * 1e3:.3f} ms "
          f"({t_exact / best:.0f}x, rel err {rel:.2e})")
    assert t_exact >= 3.0 * best


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_wide_sketch_hutchpp_matches_oracle(R, orc, prec, tol):
    """select_params budgets can exceed one 128-column panel on the sketch side (s = 1080: s_q = 270,
    s_g = 540): CholeskyQR2 and the projections then work on row blocks of the Grams."""
    n = 800
    x = orc.fill_gaussian(909, n, 6)
    a = orc.build_kernel(x, math.sqrt(6.0))
    ref = orc.estimate(a, alpha=3.0, method="int", s=1080, seed=17)
    ctx = R.Context(0)
    ctx.set_probe_source("host")
    k = R.build_kernel(x, R.GaussianKernel(math.sqrt(6.0)), prec, ctx=ctx)
    est = R.estimate(k, R.EstimatorParams(alpha=3.0, method="int", s=1080, seed=17))
    assert est.trace.sketch_rank == ref["sketch_rank"]
    assert est.entropy == pytest.approx(ref["entropy"], rel=tol)


def test_generous_parameters_track_the_oracle(R, orc):  # test_entropy.cpp:273-293
    """Auto routing with select_params(1e-3, 1e-2) budgets: 50 seeds x alpha in {0.5, 2, 2.5} x n in
    {100, 220}, every estimate within 1 % of the eigendecomposition entropy."""
    ctx = R.Context(0)
    for n in (100, 220):
        a = random_unit_trace_spd(n, 68 + n, orc, floor=0.25)
        lam = np.clip(np.linalg.eigvalsh(a), 0.0, 1.0)
        k = R.NormalizedKernel.from_matrix(a, "fp64", ctx=ctx)
        for alpha in (0.5, 2.0, 2.5):
            exact = exact_entropy(lam, alpha)
            hits = sum(abs(R.estimate(k, R.EstimatorParams(alpha=alpha, epsilon=1e-3, delta=1e-2, seed=t)).entropy
                           - exact) <= 1e-2 * abs(exact) for t in range(50))
            assert hits == 50, (n, alpha, hits)
