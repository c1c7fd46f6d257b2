"""Matrix-free configuration (config 5): kernel entries recomputed from
bf16 samples on the tensor cores every pass, A never stored.

The oracle is run on the SAME bf16-rounded samples (the product rounds x to bf16 once,
then forms |x_i - x_j|^2 = |x_i|^2 + |x_j|^2 - 2 x_i.x_j with fp32 accumulation), so the
remaining differences are the product's own arithmetic: kernel values rounded to fp16 for
the P.V tensor-core product (relative 2^-11 per entry) and the iterate rounded to one fp16
plane (relative 2^-11 per entry), both accumulated in fp32. Tolerances below are stated per
test: 1e-3 relative (Frobenius) on single products with random-sign operands, 1e-4 relative
on traces and entropies (north_star's fp32 bar)."""
import math

import numpy as np
import pytest
import torch

from conftest import rel
from workloads import mi_inputs

pytestmark = pytest.mark.gpu


def bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("n,d,s", [(2, 3, 1), (129, 7, 5), (1000, 16, 8), (1500, 100, 40), (2049, 128, 128),
                                   (700, 64, 17)])
def test_mf_matmul_panel_parity(R, orc, n, d, s):
    x = orc.fill_gaussian(300 + n, n, d)
    v = orc.fill_gaussian(400 + s, n, s)
    sigma = math.sqrt(d)
    k = R.build_kernel(x, R.GaussianKernel(sigma), "mf")
    ref = orc.matmul_panel(orc.build_kernel(bf16(x), sigma), v)
    y = R.ops.matmul_panel(k, v)
    assert rel(y, ref) <= 1e-3
    # positive operand: no cancellation, every row sum to fp16 rounding
    ones = np.ones((n, 1))
    assert rel(R.ops.matmul_panel(k, ones), orc.matmul_panel(orc.build_kernel(bf16(x), sigma), ones)) <= 2e-4


def test_mf_deterministic_and_diagonal(R, orc):
    n = 3000
    x = orc.fill_gaussian(5, n, 16)
    k = R.build_kernel(x, R.GaussianKernel(4.0), "mf")
    v = orc.fill_gaussian(6, n, 24)
    assert np.array_equal(R.ops.matmul_panel(k, v), R.ops.matmul_panel(k, v))
    # far-apart samples (a 2-D grid with spacing 64, exact in bf16): A = I/n exactly (K_ii = 1 forced,
    # off-diagonal underflows; large |x|^2 must not turn rounding into exp2(+big) = inf)
    idx = np.arange(300)
    far = np.stack([(idx % 16) * 64.0, (idx // 16) * 64.0], axis=1)
    kf = R.build_kernel(far, R.GaussianKernel(1.0), "mf")
    w = orc.fill_gaussian(7, 300, 3)
    assert np.array_equal(R.ops.matmul_panel(kf, w), np.float64(np.float16(w)) / 300) or \
        np.max(np.abs(R.ops.matmul_panel(kf, w) - w / 300)) <= 2 ** -11 * np.max(np.abs(w)) / 300


@pytest.mark.parametrize("alpha", [2, 3])
def test_mf_hutchpp_int_power_parity(R, orc, alpha):
    """Config 5 shape reduced to n=2500, d=128: alpha=3 integer power, Hutch++ s=120 (30 + 90)."""
    n, d = 2500, 128
    x = orc.fill_gaussian(55, n, d)
    sigma = math.sqrt(d)
    a = orc.build_kernel(bf16(x), sigma)
    S, G = orc.fill_gaussian(1, n, 30), orc.fill_gaussian(2, n, 90)
    ref = orc.hutchpp(orc.Spec("int", alpha), a, 30, 90, sketch=S, probes=G)
    k = R.build_kernel(x, R.GaussianKernel(sigma), "mf")
    got = R.hutchpp(R.MatrixFunctionSpec.int_power(alpha), k, R.SketchConfig(s_q=30, s_g=90, sketch=S, probes=G))
    assert got.sketch_rank == ref["sketch_rank"]
    assert abs(got.value - ref["value"]) <= 1e-4 * abs(ref["value"])
    # seeded: device-drawn probes
    ref = orc.hutchpp(orc.Spec("int", alpha), a, 30, 90, 9, "rademacher")
    got = R.hutchpp(R.MatrixFunctionSpec.int_power(alpha), k,
                    R.SketchConfig(s_q=30, s_g=90, seed=9, probe_kind="rademacher"))
    assert abs(got.value - ref["value"]) <= 1e-4 * abs(ref["value"])


def test_mf_chebyshev_entropy_parity(R, orc):
    n, d = 1800, 32
    x = orc.fill_gaussian(71, n, d)
    sigma = math.sqrt(d)
    a = orc.build_kernel(bf16(x), sigma)
    kw = dict(alpha=1.5, method="chebyshev", s=60, m=40, bounds=(0.0, 1.0))
    ref = orc.estimate(a, seed=4, **kw)
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=60, m=40, seed=4, bounds=R.SpectrumBounds(u=0, v=1))
    got = R.estimate(R.build_kernel(x, R.GaussianKernel(sigma), "mf"), p)
    assert abs(got.entropy - ref["entropy"]) <= 1e-4 * abs(ref["entropy"])


def test_mf_power_bounds(R, orc):
    n = 1200
    x = orc.fill_gaussian(21, n, 4)
    a = orc.build_kernel(bf16(x), 2.0)
    refb = orc.estimate_bounds(a, seed=3)
    b = R.estimate_bounds(R.build_kernel(x, R.GaussianKernel(2.0), "mf"), R.PowerOptions(seed=3))
    assert abs(b.v - refb["v"]) <= 1e-4 * refb["v"]


def test_mf_mutual_information_parity(R, orc):
    """Joint kernel = Gaussian of the concatenated scaled features [x/sx, y/sy] with sigma 1.

    alpha = 2 (integer power): the fp16 kernel values of the matrix-free product shift
    alpha -> 1 entropies by more than 1e-4 (measured with exact eigenvalues at this size:
    -6.8e-5 at alpha=1.01 for the X term, < 1e-6 at alpha >= 1.5), so alpha near 1
    stays on the materialised fp32 path."""
    n = 1200
    x, y = mi_inputs(n, 4)
    sx, sy = 4.0, math.sqrt(8)
    xb, yb = bf16(x), bf16(y)
    ax, ay = orc.build_kernel(xb, sx), orc.build_kernel(yb, sy)
    axy = orc.build_kernel(bf16(np.hstack([x / sx, y / sy])), 1.0)
    kw = dict(alpha=2.0, method="int", s=90)
    p = R.EstimatorParams(alpha=2.0, method="int", s=90, seed=13)
    got = R.mutual_information_samples(x, R.GaussianKernel(sx), y, R.GaussianKernel(sy), p, precision="mf")
    # term seeds follow the reference composition (measures.cpp:36-46)
    vars_ref = orc.estimate(ax, seed=orc.derive_key(13, orc.hash_name("term:vars")), **kw)["entropy"]
    target_ref = orc.estimate(ay, seed=orc.derive_key(13, orc.hash_name("term:target")), **kw)["entropy"]
    joint_ref = orc.estimate(axy, seed=orc.derive_key(13, orc.hash_name("term:joint")), **kw)["entropy"]
    for got_v, ref_v in ((got.vars_entropy, vars_ref), (got.target_entropy, target_ref),
                         (got.joint_entropy, joint_ref)):
        assert abs(got_v - ref_v) <= 1e-4 * abs(ref_v)


def test_mf_rejects_materialised_operations(R, orc):
    x = orc.fill_gaussian(3, 200, 4)
    k = R.build_kernel(x, R.GaussianKernel(2.0), "mf")
    with pytest.raises(R.RenyiError):
        k.matrix()
    with pytest.raises(R.RenyiError):
        R.NormalizedKernel.from_matrix(np.eye(10) / 10, "mf")
    with pytest.raises(R.RenyiError):
        R.hadamard_joint([k, k])
    with pytest.raises(R.RenyiError):  # more than 128 features
        R.build_kernel(orc.fill_gaussian(4, 300, 130), R.GaussianKernel(2.0), "mf")
