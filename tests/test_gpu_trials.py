"""Batched trials: measure_cell's K trials of estimate()
(proj/src/simulate.cpp:19-72) run with all trials' probes as extra columns of the same
passes over A. Each trial must equal the single estimate with seed derive_key(seed, t)
and the bounds resolved once, and the oracle run trial by trial."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


CASES = [
    ("int", 2.0, 30, 0, None),
    ("int", 3.0, 24, 0, None),
    ("chebyshev", 1.5, 40, 30, (0.0, 1.0)),
    ("taylor", 0.5, 32, 20, None),  # bounds from the power iteration, resolved once
]


@pytest.mark.parametrize("prec,tol", [("fp64", 1e-12), ("fp32", 1e-12)])
@pytest.mark.parametrize("method,alpha,s,m,bounds", CASES)
def test_trials_equal_sequential_estimates(R, orc, prec, tol, method, alpha, s, m, bounds):
    n, trials, seed = 900, 6, 77
    x = orc.fill_gaussian(40, n, 6)
    xx = x if prec == "fp64" else f32(x)
    k = R.build_kernel(xx, R.GaussianKernel(math.sqrt(6)), prec)
    kw = dict(alpha=alpha, method=method, s=s, m=m, seed=seed)
    if bounds:
        kw["bounds"] = R.SpectrumBounds(u=bounds[0], v=bounds[1])
    batch = R.estimate_trials(k, R.EstimatorParams(**kw), trials)
    assert len(batch) == trials
    for t, e in enumerate(batch):
        p = dict(kw, seed=R.derive_key(seed, t))
        if e.bounds_used is not None:
            p["bounds"] = e.bounds_used  # measure_cell resolves the bounds once, from the base seed
        one = R.estimate(k, R.EstimatorParams(**p))
        assert abs(e.entropy - one.entropy) <= tol * abs(one.entropy), (t, e.entropy, one.entropy)
        assert e.trace.sketch_rank == one.trace.sketch_rank
    # trials differ from each other (independent probes)
    assert len({round(e.entropy, 12) for e in batch}) == trials


def test_trials_match_oracle(R, orc):
    n, trials, seed = 700, 5, 9
    x = orc.fill_gaussian(41, n, 5)
    a = orc.build_kernel(x, math.sqrt(5))
    k = R.build_kernel(x, R.GaussianKernel(math.sqrt(5)), "fp64")
    batch = R.estimate_trials(k, R.EstimatorParams(alpha=1.5, method="chebyshev", s=32, m=30, seed=seed,
                                                   bounds=R.SpectrumBounds(u=0, v=1)), trials)
    for t, e in enumerate(batch):
        ref = orc.estimate(a, alpha=1.5, method="chebyshev", s=32, m=30, seed=orc.derive_key(seed, t),
                           bounds=(0.0, 1.0))
        assert abs(e.entropy - ref["entropy"]) <= 1e-9 * abs(ref["entropy"])


def test_measure_cell_statistics(R, orc):
    n, trials = 600, 12
    x = orc.fill_gaussian(42, n, 4)
    k = R.build_kernel(x, R.GaussianKernel(2.0), "fp64")
    exact = R.entropy_exact(k, 2.0).entropy
    p = R.EstimatorParams(alpha=2.0, method="int", s=40, seed=3)
    cell = R.measure_cell(k, exact, p, trials)
    ents = np.array([e.entropy for e in R.estimate_trials(k, p, trials)])
    rel = np.abs(ents - exact) / abs(exact)
    assert cell.trials == trials and cell.alpha == 2.0 and cell.s == 40
    assert cell.mre == pytest.approx(rel.mean(), rel=1e-12)
    assert cell.sd == pytest.approx(rel.std(ddof=1), rel=1e-10)
    assert cell.mre < 0.05
    with pytest.raises(R.RenyiError):
        R.measure_cell(k, exact, p, 0)


def test_run_simulation_grid(R):
    spec = R.SimulationSpec(n=256, d=4, sigma=2.0, alphas=(2.0, 1.5), s_list=(16, 32), m_list=(20,), trials=8,
                            seed=5, method="auto")
    cells = R.run_simulation(spec)
    assert len(cells) == 4
    for c in cells:
        assert c.trials == 8 and 0.0 <= c.mre < 0.2 and c.oracle_elapsed >= 0.0
    with pytest.raises(R.RenyiError):
        R.run_simulation(R.SimulationSpec(n=8))
