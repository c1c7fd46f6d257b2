"""Restatements of the reference's test fixtures (proj/tests/support.hpp) in numpy,
drawing randomness from the reference RNG through the oracle. Rotations use numpy's
Householder QR instead of Eigen's; every KAT that uses them depends only on the
spectrum, so the basis convention does not matter."""
import numpy as np


def random_rotation(n, key, orc):  # support.hpp:22-27
    g = orc.fill_gaussian(key, n, n)
    q, _ = np.linalg.qr(g)
    return q


def spd_from_spectrum(eigs, key, orc):  # support.hpp:30-33
    q = random_rotation(len(eigs), key, orc)
    return (q * np.asarray(eigs)) @ q.T


def unit_trace_spectrum(n, rng, floor=0.2):  # support.hpp:37-44
    e = floor + (1.0 - floor) * rng.random(n)
    return e / e.sum()


def random_unit_trace_spd(n, key, orc, floor=0.2):  # support.hpp:46-50
    rng = np.random.default_rng(key)
    return spd_from_spectrum(unit_trace_spectrum(n, rng, floor), key + 1, orc)


def random_low_rank_psd(n, r, key, orc):  # support.hpp:53-58
    w = orc.fill_gaussian(key, n, r)
    a = w @ w.T
    return a / np.trace(a)


def oracle_trace_power(a, alpha):  # support.hpp:66-74
    lam = np.clip(np.linalg.eigvalsh(a), 0.0, 1.0)
    lam = lam[lam > 0]
    return float(np.sum(lam ** alpha))


def chebyshev_closed_form_u0(alpha, m, v):  # support.hpp:79-85
    from math import gamma, pi, sqrt

    c = np.empty(m + 1)
    c[0] = 2.0 * v ** alpha * gamma(alpha + 0.5) / (sqrt(pi) * gamma(alpha + 1.0))
    for k in range(m):
        c[k + 1] = c[k] * (alpha - k) / (alpha + k + 1.0)
    return c


def mixture_kernel(n, d, sigma, seed, orc):  # support.hpp:123-126
    return orc.build_kernel(orc.mixture_samples(n, d, seed), sigma)


def cheb_bound(alpha, u, v, m):  # test_poly.cpp:145-155
    beta = 2.0 * u / (v - u)
    k = 1.0 + beta + np.sqrt(beta * beta + 2.0 * beta)
    return 4.0 * (1.0 + beta) ** alpha / ((k - 1.0) * k ** m)
