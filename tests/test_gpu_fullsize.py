"""Full-size checks at BASELINE.json's configurations — config 4 (n = 100k, fp32) and config 5
(n = 400k, d = 128, matrix-free) — where the fp64 oracle cannot hold A (80 GB / 1.3 TB).

Size-independent evidence instead: exact fp64 columns of A recomputed on the host for sampled
indices (A_ij = K_ij / n, K_ij = exp(−|x_i − x_j|² / 2σ²), K_jj = 1 — proj/src/ops.cpp:9-20,
proj/src/kernel.cpp:51-70) against the device's A·e_j through the C ABI, row sums against the
exact sums of those columns, and symmetry / linearity of the block product. Tolerances follow the
storage: fp32 configuration 2e-6 of max A (3xTF32 Gram + 22-bit hi/lo storage);
matrix-free 1e-3 (fp16 kernel values, one fp16 iterate plane)."""
import math

import numpy as np
import pytest

from workloads import bf16, gaussian, mi_inputs

pytestmark = pytest.mark.gpu


def exact_column(x, j, sigma):
    d2 = np.einsum("ij,ij->i", x - x[j], x - x[j])
    k = np.exp(-d2 / (2.0 * sigma * sigma))
    k[j] = 1.0
    return k / x.shape[0]


def unit_panel(n, idx):
    e = np.zeros((n, len(idx)), order="F")
    e[idx, np.arange(len(idx))] = 1.0
    return e


def check_properties(R, k, n, tol, seed):
    rng = np.random.default_rng(seed)
    u = rng.standard_normal((n, 2))
    v = rng.standard_normal((n, 2))
    au = R.ops.matmul_panel(k, u)
    av = R.ops.matmul_panel(k, v)
    # symmetry: u^T (A v) = v^T (A u), measured against the Cauchy-Schwarz scale |u| |A v|
    lhs, rhs = u.T @ av, (v.T @ au).T
    scale = np.outer(np.linalg.norm(u, axis=0), np.linalg.norm(av, axis=0))
    assert np.max(np.abs(lhs - rhs) / scale) <= tol
    # linearity: A (2u + 3v) = 2 A u + 3 A v; the three operands are rounded to the iterate planes
    # separately, so the error is measured against |A| |x| (|A| ~ |A 1| / |1|, the top eigenvalue of
    # a Gaussian kernel matrix), not against |A x|, which cancels for random-sign x
    x = 2.0 * u + 3.0 * v
    w = R.ops.matmul_panel(k, x)
    diff = w - (2.0 * au + 3.0 * av)
    a_norm = np.linalg.norm(R.ops.matmul_panel(k, np.ones((n, 1)))) / math.sqrt(n)
    assert np.max(np.linalg.norm(diff, axis=0) / (a_norm * np.linalg.norm(x, axis=0))) <= tol


def test_config4_full_size(R):
    n = 100_000
    x, _ = mi_inputs(n, 11)
    x = x.astype(np.float32).astype(np.float64)
    sigma = 4.0
    k = R.build_kernel(x, R.GaussianKernel(sigma), "fp32")
    idx = [0, 1, 4095, 4096, 50_001, n - 1]
    cols = R.ops.matmul_panel(k, unit_panel(n, idx))
    ones = R.ops.matmul_panel(k, np.ones((n, 1)))[:, 0]
    for c, j in enumerate(idx):
        ref = exact_column(x, j, sigma)
        assert np.max(np.abs(cols[:, c] - ref)) <= 2e-6 * ref.max(), j
        assert abs(cols[j, c] - 1.0 / n) <= 1e-7 / n  # A_jj = 1/n: trace one
        assert abs(ones[j] - ref.sum()) <= 2e-6 * ref.sum()  # row sum j = column sum j (symmetry)
    check_properties(R, k, n, 1e-6, 5)


def test_config5_full_size_matrix_free(R):
    n, d = 400_000, 128
    x = bf16(gaussian(n, d, 7, "X"))
    sigma = math.sqrt(d)
    k = R.build_kernel(x, R.GaussianKernel(sigma), "mf")
    idx = [0, 127, 128, 200_003, n - 1]
    cols = R.ops.matmul_panel(k, unit_panel(n, idx))
    for c, j in enumerate(idx):
        ref = exact_column(x, j, sigma)
        assert np.max(np.abs(cols[:, c] - ref)) <= 1e-3 * ref.max(), j
        assert abs(cols[j, c] - 1.0 / n) <= 1e-3 / n
    check_properties(R, k, n, 1e-3, 9)


def test_config4_mi_sharded_matches_single_rank_at_full_size(R):
    """The whole config-4 MI estimate (three Chebyshev m = 60 Hutch++ 22 + 46 estimates at
    n = 100k) row-sharded over two ranks (the NCCL rank code over the LocalGroup transport)
    equals the single-rank result: the sharded protocol at the benchmark's size."""
    from test_gpu_sharded import run_ranks

    n = 100_000
    x, y = mi_inputs(n, 1)
    x, y = x.astype(np.float32).astype(np.float64), y.astype(np.float32).astype(np.float64)
    sx, sy = R.GaussianKernel(4.0), R.GaussianKernel(math.sqrt(8.0))
    p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=90, m=60, seed=1, s_q=22, s_g=46,
                          bounds=R.SpectrumBounds(u=0, v=1))
    ref = R.mutual_information_samples(x, sx, y, sy, p, precision="fp32", ctx=R.Context(0))
    res = run_ranks(R, 2, lambda ctx, rank: R.mutual_information_samples(x, sx, y, sy, p, "fp32", ctx))
    for r in res:
        assert r.value == res[0].value
        for key in ("vars_entropy", "target_entropy", "joint_entropy"):
            a, b = getattr(r, key), getattr(ref, key)
            assert abs(a - b) <= 1e-5 * abs(b), (key, a, b)
