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


class Stream:
    """RandomStream (proj/src/rng.cpp:8-54): counter-based splitmix64 + Box-Muller with spare."""
    M = (1 << 64) - 1

    def __init__(self, key):
        self.key, self.counter, self.spare = key & self.M, 0, None

    @classmethod
    def mix64(cls, x):
        x = (x + 0x9E3779B97F4A7C15) & cls.M
        x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & cls.M
        x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & cls.M
        return x ^ (x >> 31)

    def next_u64(self):
        v = self.mix64(self.key ^ self.mix64(self.counter))
        self.counter += 1
        return v

    def next_uniform(self):
        return (self.next_u64() >> 11) * 2.0 ** -53

    def next_gaussian(self):
        import math

        if self.spare is not None:
            v, self.spare = self.spare, None
            return v
        u1 = self.next_uniform()
        while u1 <= 0.0:
            u1 = self.next_uniform()
        u2 = self.next_uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        theta = 2.0 * math.pi * u2
        self.spare = r * math.sin(theta)
        return r * math.cos(theta)


def correlated_dataset(n, seed, weights):  # test_features.cpp:21-36
    st = Stream(seed)
    x = np.empty((n, len(weights)))
    labels = []
    for i in range(n):
        y = st.next_u64() % 2
        labels.append("pos" if y else "neg")
        for j, w in enumerate(weights):
            x[i, j] = w * y + (1.0 - w) * st.next_gaussian()
    return x, labels, [f"f{j}" for j in range(len(weights))]


def label_leak_dataset(n, seed):  # test_features.cpp:38-55
    st = Stream(seed)
    x = np.empty((n, 5))
    labels = []
    for i in range(n):
        y = st.next_u64() % 3
        labels.append(str(y))
        x[i, 0] = st.next_gaussian()
        x[i, 1] = float(y)
        x[i, 2] = st.next_gaussian()
        x[i, 3] = st.next_gaussian()
        x[i, 4] = st.next_gaussian()
    return x, labels, ["noise0", "leak", "noise1", "noise2", "noise3"]


def duplicate_dataset(n, seed):  # test_features.cpp:78-99
    st = Stream(seed)
    x = np.empty((n, 3))
    labels = []
    for i in range(n):
        y = st.next_u64() % 2
        labels.append("1" if y else "0")
        v = 0.8 * y + 0.2 * st.next_gaussian()
        x[i, 0] = v
        x[i, 1] = v
        x[i, 2] = st.next_gaussian()
    return x, labels, ["a", "b", "c"]


def parity_dataset(n, seed):  # test_features.cpp:116-131
    st = Stream(seed)
    x = np.empty((n, 4))
    labels = []
    for i in range(n):
        p1 = st.next_u64() & 1
        p2 = st.next_u64() & 1
        x[i] = (p1, p2, 1.0, -2.5)
        labels.append("odd" if p1 ^ p2 else "even")
    return x, labels, ["p1", "p2", "c1", "c2"]
