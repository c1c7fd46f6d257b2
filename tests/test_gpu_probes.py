"""Probe sources (renyi_ctx_set_probe_source): seeded Gaussian probes drawn on the host with the
reference's own stream arithmetic (detail::gaussian_panel, proj/src/hutchpp.cpp:13-22; rng.cpp:41-64)
are the reference's probes bit for bit, so an estimate over host-drawn probes equals the same
estimate over the oracle's probes injected explicitly -- bitwise, not just within tolerance. The
device draws (CUDA log/sin/cos) agree to a few ulp per draw, and their estimates to the fp32 bar."""
import math

import numpy as np
import pytest

from workloads import mi_inputs

pytestmark = pytest.mark.gpu


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


@pytest.mark.parametrize("prec", ["fp32", "fp64"])
def test_host_probes_equal_injected_reference_probes(R, orc, prec):
    n, d, seed, s_q, s_g = 2600, 12, 97, 10, 21
    x = f32(orc.fill_gaussian(4242, n, d))
    spec = R.MatrixFunctionSpec.chebyshev(1.5, 30, 0.0, 1.0)
    ctx = R.Context(0)
    k = R.build_kernel(x, R.GaussianKernel(math.sqrt(d)), prec, ctx=ctx)
    sk = orc.probe_panel(n, s_q, seed, "hutchpp-sketch")
    pr = orc.probe_panel(n, s_g, seed, "hutchpp-probe")
    injected = R.hutchpp(spec, k, R.SketchConfig(s_q=s_q, s_g=s_g, seed=seed, sketch=sk, probes=pr))
    ctx.set_probe_source("host")
    host = R.hutchpp(spec, k, R.SketchConfig(s_q=s_q, s_g=s_g, seed=seed))
    ctx.set_probe_source("device")
    dev = R.hutchpp(spec, k, R.SketchConfig(s_q=s_q, s_g=s_g, seed=seed))
    assert host.value == injected.value and host.low_rank_part == injected.low_rank_part
    assert host.residual_part == injected.residual_part and host.sketch_rank == injected.sketch_rank
    assert dev.value == pytest.approx(injected.value, rel=1e-9 if prec == "fp64" else 1e-5)


def test_host_probes_mutual_information(R, orc):
    """The fused MI path prefetches its six panels on the host while A and B are built: the result
    equals the one over device draws to the fp32 bar, and is reproducible bitwise."""
    n = 3000
    x, y = mi_inputs(n, 31)
    x, y = f32(x), f32(y)
    p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=40, m=30, seed=5, bounds=R.SpectrumBounds(u=0.0, v=1.0))
    out = {}
    for src in ("host", "device", "host"):
        ctx = R.Context(0)
        ctx.set_probe_source(src)
        mi = R.mutual_information_samples(x, R.GaussianKernel(4.0), y, R.GaussianKernel(math.sqrt(8.0)), p,
                                          precision="fp32", ctx=ctx)
        if src in out:
            assert mi.value == out[src].value and mi.joint_entropy == out[src].joint_entropy
        out[src] = mi
    for key in ("vars_entropy", "target_entropy", "joint_entropy"):
        assert getattr(out["host"], key) == pytest.approx(getattr(out["device"], key), rel=1e-4)


def test_probe_source_rejects_unknown(R):
    ctx = R.Context(0)
    with pytest.raises(ValueError):
        ctx.set_probe_source("gpu")


def test_host_power_start_matches_oracle(R, orc):
    """seeded_start (spectrum.cpp:13-21) drawn on the host: the fp64 power iteration then follows the
    oracle's to rounding and stops at the same iteration."""
    n = 1800
    x = orc.fill_gaussian(77, n, 5)
    a = orc.build_kernel(x, math.sqrt(5.0))
    ref = orc.estimate_bounds(a, seed=4)
    ctx = R.Context(0)
    ctx.set_probe_source("host")
    k = R.build_kernel(x, R.GaussianKernel(math.sqrt(5.0)), "fp64", ctx=ctx)
    b = R.estimate_bounds(k, R.PowerOptions(seed=4))
    assert b.iterations_used == ref["iterations_used"]
    assert b.v == pytest.approx(ref["v"], rel=1e-12) and b.u == pytest.approx(ref["u"], rel=1e-9, abs=1e-15)
