"""Row-sharded (multi-rank) path on one GPU: ranks are host threads of this process,
each with its own context, joined in a LocalGroup (host-driven collectives: every
rank synchronises its stream and the threads copy at a barrier, so no kernel waits
on another). The per-rank engine code is the one NCCL ranks run; only the
transport differs. Results must match the single-rank path."""
import math
import threading

import numpy as np
import pytest

from workloads import f32, mi_inputs

pytestmark = pytest.mark.gpu


def run_ranks(R, world, fn):
    """fn(ctx, rank) on `world` threads; returns the per-rank results."""
    group = R.LocalGroup(world)
    out, errs = [None] * world, []

    def body(rank):
        try:
            ctx = R.Context(0)
            ctx.join_local_group(group, rank)
            assert ctx.rank_world() == (rank, world)
            out[rank] = fn(ctx, rank)
        except Exception as exc:  # surface the first failure
            errs.append(exc)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_mutual_information_matches_single_rank(R, orc, world, fused):
    """Both MI paths (fused pass over A and B, or three estimates over a materialised joint)
    row-sharded: every rank agrees bitwise, each term is within the fp32 contract (1e-4) of the
    oracle, and within 2e-5 (fused: 5e-5) of the single-rank run. alpha = 1.01 turns trace
    differences into x100 entropy differences; the fused pass accumulates all three split
    products in one TMEM accumulator, so its fp32 accumulation order differs most between
    shardings (measured: 2.0e-5 from the oracle at world 1, 1.9e-5 at world 2, unfused 1.4e-5 / 4e-6)."""
    n = 2600  # not a multiple of 256: the last shard is short
    x, y = mi_inputs(n, 21)
    x, y = f32(x), f32(y)
    sx, sy = R.GaussianKernel(4.0), R.GaussianKernel(math.sqrt(8.0))
    p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=60, m=40, seed=5, bounds=R.SpectrumBounds(u=0, v=1))
    oref = orc.mutual_information(orc.build_kernel(x, 4.0), orc.build_kernel(y, math.sqrt(8.0)), seed=5,
                                  alpha=1.01, method="chebyshev", s=60, m=40, bounds=(0.0, 1.0))
    ctx0 = R.Context(0)
    ctx0.set_fused_mi(fused)
    ref = R.mutual_information_samples(x, sx, y, sy, p, precision="fp32", ctx=ctx0)

    def fn(ctx, rank):
        ctx.set_fused_mi(fused)
        return R.mutual_information_samples(x, sx, y, sy, p, "fp32", ctx)

    res = run_ranks(R, world, fn)
    tol = 5e-5 if fused else 2e-5
    for r in res:
        assert r.value == res[0].value  # identical on every rank
        for key in ("vars_entropy", "target_entropy", "joint_entropy"):
            a, b = getattr(r, key), getattr(ref, key)
            assert abs(a - b) <= tol * abs(b), (key, a, b)
            assert abs(a - oref[key]) <= 1e-4 * abs(oref[key]), (key, a, oref[key])


def test_sharded_hutchpp_and_bounds(R, orc):
    n = 1800
    x = f32(orc.fill_gaussian(9, n, 8))
    sigma = math.sqrt(8)
    a = orc.build_kernel(x, sigma)
    S, G = orc.fill_gaussian(1, n, 6), orc.fill_gaussian(2, n, 14)
    ospec = orc.Spec("chebyshev", 1.5, 30, 0.0, 1.0)
    ref = orc.hutchpp(ospec, a, 6, 14, sketch=S, probes=G)
    refb = orc.estimate_bounds(a, seed=3)

    def fn(ctx, rank):
        k = R.build_kernel(x, R.GaussianKernel(sigma), "fp32", ctx=ctx)
        t = R.hutchpp(R.MatrixFunctionSpec.chebyshev(1.5, 30, 0.0, 1.0), k,
                      R.SketchConfig(s_q=6, s_g=14, sketch=S, probes=G))
        ts = R.hutchpp(R.MatrixFunctionSpec.int_power(2), k,
                       R.SketchConfig(s_q=4, s_g=10, seed=11, probe_kind="rademacher"))
        b = R.estimate_bounds(k, R.PowerOptions(seed=3))
        return t, ts, b

    res = run_ranks(R, 2, fn)
    single = R.build_kernel(x, R.GaussianKernel(sigma), "fp32", ctx=R.Context(0))
    ts_ref = R.hutchpp(R.MatrixFunctionSpec.int_power(2), single,
                       R.SketchConfig(s_q=4, s_g=10, seed=11, probe_kind="rademacher"))
    for t, ts, b in res:
        assert abs(t.value - ref["value"]) <= 1e-4 * abs(ref["value"])
        assert t.sketch_rank == ref["sketch_rank"]
        assert abs(ts.value - ts_ref.value) <= 1e-6 * abs(ts_ref.value)  # device-drawn probes, sharded counters
        assert abs(b.v - refb["v"]) <= 1e-4 * refb["v"]


def test_sharded_rejects_single_rank_seams(R):
    def fn(ctx, rank):
        k = R.NormalizedKernel.from_matrix(np.eye(300) / 300, "fp32", ctx=ctx)
        with pytest.raises(R.RenyiError):
            R.ops.matmul_panel(k, np.ones((300, 2)))
        return True

    assert all(run_ranks(R, 2, fn))


def test_sharded_matrix_free_matches_single_rank(R, orc):
    """Matrix-free path row-sharded over 2 ranks: each rank recomputes its rows of K from the full
    bf16 sample set; the fp16 operand planes are all-gathered per pass as in the materialised path."""
    n, d = 2300, 32
    x = orc.fill_gaussian(19, n, d)
    sigma = math.sqrt(d)
    S, G = orc.fill_gaussian(1, n, 10), orc.fill_gaussian(2, n, 30)
    spec = R.MatrixFunctionSpec.int_power(3)
    ref = R.hutchpp(spec, R.build_kernel(x, R.GaussianKernel(sigma), "mf", ctx=R.Context(0)),
                    R.SketchConfig(s_q=10, s_g=30, sketch=S, probes=G))

    def fn(ctx, rank):
        k = R.build_kernel(x, R.GaussianKernel(sigma), "mf", ctx=ctx)
        return R.hutchpp(spec, k, R.SketchConfig(s_q=10, s_g=30, sketch=S, probes=G))

    for t in run_ranks(R, 2, fn):
        assert t.sketch_rank == ref.sketch_rank
        # different stream-K splits change the fp32 TMEM chunk boundaries: agreement to ~1e-6
        assert abs(t.value - ref.value) <= 1e-5 * abs(ref.value)


def test_nccl_transport_single_rank(R):
    """The NCCL transport end to end with a 1-rank communicator (no cross-rank waits on one GPU):
    dlopen, comm init, in-place all-gather and the f64-sum / u32-max all-reduces on the estimator
    path; results must equal the transport-free run bit for bit."""
    n = 1500
    x, y = mi_inputs(n, 23)
    x, y = f32(x), f32(y)
    sx, sy = R.GaussianKernel(4.0), R.GaussianKernel(math.sqrt(8))
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=40, m=30, seed=2, bounds=R.SpectrumBounds(u=0, v=1))
    ref = R.mutual_information_samples(x, sx, y, sy, p, "fp32", R.Context(0))
    try:
        uid = R.nccl_unique_id()
    except R.RenyiError as e:
        pytest.skip(f"no NCCL: {e}")
    ctx = R.Context(0)
    ctx.init_nccl(0, 1, uid)
    assert ctx.rank_world() == (0, 1)
    got = R.mutual_information_samples(x, sx, y, sy, p, "fp32", ctx)
    assert got.value == ref.value and got.joint_entropy == ref.joint_entropy


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_polynomial_kernel_estimate(R, orc, world):
    """The polynomial kernel (kernel.cpp:35-72, ops.cpp:22-28) built row-sharded: each rank computes the
    whole diagonal (normalisation) and its own rows; the Hutch++ estimate over the shards equals the
    single-rank one to the fp32 sharding tolerance and the oracle to the fp32 contract."""
    n = 2600
    x = orc.fill_gaussian(44, n, 5)
    p = R.EstimatorParams(alpha=2.5, method="chebyshev", s=40, m=30, seed=3, bounds=R.SpectrumBounds(u=0, v=1))
    ref = orc.estimate(orc.build_kernel_polynomial(x, 2, 1.0), alpha=2.5, method="chebyshev", s=40, m=30, seed=3,
                       bounds=(0.0, 1.0))
    one = R.estimate(R.build_kernel(x, R.PolynomialKernel(2, 1.0), "fp32", ctx=R.Context(0)), p).entropy

    def fn(ctx, rank):
        return R.estimate(R.build_kernel(x, R.PolynomialKernel(2, 1.0), "fp32", ctx=ctx), p).entropy

    got = run_ranks(R, world, fn)
    assert all(g == got[0] for g in got)
    assert got[0] == pytest.approx(one, rel=2e-5)
    assert got[0] == pytest.approx(ref["entropy"], rel=1e-4)
