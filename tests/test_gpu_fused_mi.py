"""The fused mutual-information pass (launch_block_av_tri): the three terms of
I(X;Y) = S(A) + S(B) - S(n·A∘B) (proj/src/measures.cpp:36-46) estimated in lockstep, each pass
reading A and B once and forming the joint kernel (proj/src/kernel.cpp:74-108) tile by tile.

Checked against (a) the pinned oracle (fp32 tolerance 1e-4, north_star) and (b) the unfused
device path on the same inputs (three separate estimates over a materialised joint), whose
products differ only in fp32 accumulation order and the fp32 rounding of the joint entries."""
import math

import numpy as np
import pytest

from workloads import mi_inputs

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def _inputs(n, seed):
    x, y = mi_inputs(n, seed)
    return f32(x), f32(y)


def _both(R, x, sx, y, sy, p, operand="split"):
    out = []
    for fused in (True, False):
        ctx = R.Context(0)
        ctx.set_operand_mode(operand)
        ctx.set_fused_mi(fused)
        out.append(R.mutual_information_samples(x, R.GaussianKernel(sx), y, R.GaussianKernel(sy), p,
                                                precision="fp32", ctx=ctx))
    return out


TERMS = ("vars_entropy", "target_entropy", "joint_entropy")


@pytest.mark.parametrize("n", [1200, 2999])
def test_fused_mi_matches_oracle_and_unfused(R, orc, n):
    """Config 4 reduced: alpha = 1.01 Chebyshev m = 60 on [0,1], Hutch++ s = 90 (22 + 46)."""
    x, y = _inputs(n, 4)
    sx, sy = 4.0, math.sqrt(8)
    ax, ay = orc.build_kernel(x, sx), orc.build_kernel(y, sy)
    kw = dict(alpha=1.01, method="chebyshev", s=90, m=60, bounds=(0.0, 1.0))
    ref = orc.mutual_information(ax, ay, seed=13, **kw)
    p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=90, m=60, seed=13, bounds=R.SpectrumBounds(u=0, v=1))
    fused, plain = _both(R, x, sx, y, sy, p)
    for key in TERMS:
        r = ref[key]
        assert abs(getattr(fused, key) - r) <= 1e-4 * abs(r), key
        assert abs(getattr(fused, key) - getattr(plain, key)) <= 2e-5 * abs(r), key
    assert fused.value == pytest.approx(fused.vars_entropy + fused.target_entropy - fused.joint_entropy, rel=1e-14)


def test_fused_mi_integer_alpha_and_wide_panels(R, orc):
    """Integer alpha (power recurrence, no bounds needed) and s = 200: a 50-column sketch and
    150 Q|W columns, i.e. two lockstep panel groups of <= 80 columns."""
    n = 2100
    x, y = _inputs(n, 7)
    sx, sy = 4.0, math.sqrt(8)
    ax, ay = orc.build_kernel(x, sx), orc.build_kernel(y, sy)
    ref = orc.mutual_information(ax, ay, seed=3, alpha=2.0, method="int", s=200)
    p = R.EstimatorParams(alpha=2.0, method="int", s=200, seed=3)
    fused, plain = _both(R, x, sx, y, sy, p)
    for key in TERMS:
        r = ref[key]
        assert abs(getattr(fused, key) - r) <= 1e-4 * abs(r), key
        assert abs(getattr(fused, key) - getattr(plain, key)) <= 2e-5 * abs(r), key


@pytest.mark.parametrize("operand", ["fast", "auto"])
def test_fused_mi_single_plane_operands(R, operand):
    """The fast operand mode (one fp16 V plane) through the fused kernel agrees with the unfused
    kernel in the same mode."""
    n = 1500
    x, y = _inputs(n, 9)
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=60, m=40, seed=5, bounds=R.SpectrumBounds(u=0, v=1))
    fused, plain = _both(R, x, 4.0, y, math.sqrt(8), p, operand)
    for key in TERMS:
        b = getattr(plain, key)
        assert abs(getattr(fused, key) - b) <= 2e-5 * abs(b), key


def test_fused_mi_kernel_level_entry(R, orc):
    """mutual_information over prebuilt kernels takes the fused path too (no joint is built)."""
    n = 1400
    x, y = _inputs(n, 11)
    sx, sy = 4.0, math.sqrt(8)
    ref = orc.mutual_information(orc.build_kernel(x, sx), orc.build_kernel(y, sy), seed=2, alpha=1.5,
                                 method="chebyshev", s=60, m=40, bounds=(0.0, 1.0))
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=60, m=40, seed=2, bounds=R.SpectrumBounds(u=0, v=1))
    kx = R.build_kernel(x, R.GaussianKernel(sx), "fp32")
    ky = R.build_kernel(y, R.GaussianKernel(sy), "fp32")
    got = R.mutual_information([kx], ky, p)
    for key in TERMS:
        assert abs(getattr(got, key) - ref[key]) <= 1e-4 * abs(ref[key]), key


def test_fused_mi_bitwise_reproducible(R):
    """Three runs of the fused pass at n = 20000 (157 row blocks, waves plus a stream-K tail) give
    bitwise identical terms: the partial slots are summed in a fixed order and no ring phase may
    alias (an A/B ring variant whose consumers could read a stale stage failed exactly this)."""
    n = 20000
    x, y = _inputs(n, 1)
    p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=90, m=60, seed=1, s_q=22, s_g=46,
                          bounds=R.SpectrumBounds(u=0, v=1))
    ctx = R.Context(0)
    runs = [R.mutual_information_samples(x, R.GaussianKernel(4.0), y, R.GaussianKernel(math.sqrt(8)), p,
                                         precision="fp32", ctx=ctx) for _ in range(3)]
    for r in runs[1:]:
        for key in TERMS:
            assert getattr(r, key) == getattr(runs[0], key), key
