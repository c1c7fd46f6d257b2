"""Seeded synthetic inputs for the five BASELINE.json configurations.

All randomness comes from the reference's counter-based RNG
(proj/src/rng.cpp) through per-column substreams, so the GPU path, the oracle
and the CPU baseline see identical arrays. The reference measures no public
dataset for this path; these stand in with the shapes and distributions
BASELINE.json names.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def mix64_np(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finalizer (rng.cpp:8-14), bitwise identical."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def stream_u64(key: int, count: int) -> np.ndarray:
    """RandomStream(key).next_u64() for counters 0..count-1."""
    k = np.uint64(key & 0xFFFFFFFFFFFFFFFF)
    return mix64_np(k ^ mix64_np(np.arange(count, dtype=np.uint64)))


def _gen(gen: str):
    """The reference RNG from the product library (gen="product", the GPU arm) or from the CPU
    oracle (gen="oracle": bench.py --impl reference and the fixture generator, so that those
    never map librenyi_b200.so). Both are bitwise equal (tests/test_abi_host.py)."""
    if gen == "oracle":
        from oracle import oracle as O

        return O.gaussian_panel, O.derive_key, O.hash_name
    import paper_2205_07426_b200 as R

    return R.gaussian_panel, R.derive_key, R.hash_name


def gaussian(n: int, d: int, seed: int, label: str, gen: str = "product") -> np.ndarray:
    """n x d, column j from RandomStream(derive_key(derive_key(seed, hash(label)), j)) (gaussian_panel)."""
    return _gen(gen)[0](n, d, seed, label)


def iid(n: int, d: int, seed: int, gen: str = "product") -> np.ndarray:
    return gaussian(n, d, seed, "X", gen)


def mixture10(n: int, d: int, seed: int, gen: str = "product") -> np.ndarray:
    """Config 3: 10 isotropic unit-variance Gaussians, means ~ N(0, 4I), component = next_u64() % 10."""
    panel, derive_key, hash_name = _gen(gen)
    means = 2.0 * panel(d, 10, seed, "means")
    comp = (stream_u64(derive_key(seed, hash_name("component")), n) % np.uint64(10)).astype(np.int64)
    return means[:, comp].T + panel(n, d, seed, "noise")


def mi_inputs(n: int, seed: int, dx: int = 16, dy: int = 8, gen: str = "product"):
    """Config 4: X ~ N(0, I_16); Y = X W + 0.5 noise with W ~ N(0,1)^{16x8}. The product X W is
    summed feature by feature in fixed order (elementwise IEEE arithmetic, no BLAS), so Y is
    bitwise the same on every host CPU."""
    x = gaussian(n, dx, seed, "X", gen)
    w = gaussian(dx, dy, seed, "W", gen)
    y = np.zeros((n, dy))
    for k in range(dx):
        y += x[:, k:k + 1] * w[k:k + 1, :]
    y = y + 0.5 * gaussian(n, dy, seed, "noise", gen)
    return x, y


def f32(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def bf16(x: np.ndarray) -> np.ndarray:
    """Round to bf16 (round-to-nearest-even) and widen back to fp64."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).double().numpy()


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    d: int
    precision: str
    alpha: float
    method: str
    s: int
    m: int
    s_q: int
    s_g: int
    probe_kind: str
    note: str


CONFIGS = {
    "c1": Config("c1", 2000, 10, "fp64", 2.0, "int", 30, 0, 0, 30, "rademacher",
                 "n=2000 d=10 fp64, alpha=2 Hutchinson s=30 Rademacher"),
    "c2": Config("c2", 20000, 32, "fp32", 1.5, "chebyshev", 60, 40, 20, 40, "rademacher",
                 "n=20000 d=32 fp32, alpha=1.5 Chebyshev[0,1] m=40, Hutch++ 20+40 Rademacher"),
    "c3": Config("c3", 50000, 64, "fp32", 0.5, "taylor", 100, 30, 0, 100, "gaussian",
                 "n=50000 d=64 fp32 10-mixture, alpha=0.5 Taylor m=30, Hutchinson s=100 Gaussian"),
    "c4": Config("c4", 100000, 16, "fp32", 1.01, "chebyshev", 90, 60, 22, 46, "gaussian",
                 "MI n=100000 d=16/8 fp32, alpha=1.01 Chebyshev[0,1] m=60, Hutch++ s=90 (reference split 22+46)"),
    "c5": Config("c5", 400000, 128, "mf", 3.0, "int", 120, 0, 30, 60, "gaussian",
                 "n=400000 d=128 bf16 matrix-free, alpha=3 integer power, Hutch++ s=120 (reference split 30+60)"),
}


def sigma_for(d: int) -> float:
    return math.sqrt(d)
