"""Small-n invocations of every device kernel family, for compute-sanitizer runs on the GPU box:

    compute-sanitizer --tool memcheck  python tests/sanitize_cases.py
    compute-sanitizer --tool racecheck python tests/sanitize_cases.py

(one tool per run; logs under profiles/r2_sanitizer_*.log). Covers the tcgen05 Gram (gram_tc),
the single-matrix product (block_av_tc), the fused MI pass (block_av_tri), the matrix-free
product (block_av_mf), the fp64 path (gram_kernel, block_av_f64), the pass epilogues, CholeskyQR2
and the device RNG, each at sizes with ragged edges (n not a multiple of the tiles). Each result is
checked against the oracle so a silent corruption also fails the run.
"""
from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2205_07426_b200 as R  # noqa: E402
from oracle import oracle as O  # noqa: E402


def check(name, got, ref, tol):
    err = abs(got - ref) / abs(ref)
    print(f"{name}: {got:.12e} vs oracle {ref:.12e} (rel {err:.1e})", flush=True)
    assert err <= tol, name


def main():
    ctx = R.Context(0)
    n, d = 777, 6
    x = O.fill_gaussian(101, n, d).astype(np.float32).astype(np.float64)
    y = O.fill_gaussian(102, n, 3).astype(np.float32).astype(np.float64)
    sx, sy = math.sqrt(d), math.sqrt(3)
    a, b = O.build_kernel(x, sx), O.build_kernel(y, sy)
    sk = O.probe_panel(n, 6, 7, "hutchpp-sketch")
    pr = O.probe_panel(n, 13, 7, "hutchpp-probe")
    spec = O.Spec("chebyshev", 1.5, 12, 0.0, 1.0)
    ref = O.hutchpp(spec, a, 6, 13, sketch=sk, probes=pr)["value"]
    for prec, tol in (("fp32", 1e-4), ("fp64", 1e-9)):
        k = R.build_kernel(x, R.GaussianKernel(sx), prec, ctx=ctx)
        got = R.hutchpp(R.MatrixFunctionSpec.chebyshev(1.5, 12, 0.0, 1.0), k,
                        R.SketchConfig(s_q=6, s_g=13, sketch=sk, probes=pr)).value
        check(f"hutchpp {prec}", got, ref, tol)
        v = O.probe_panel(n, 37, 3, "v")
        yv = R.ops.matmul_panel(k, v)
        ry = O.matmul_panel(a, v)
        check(f"matmul_panel {prec}", float(np.abs(yv).sum()), float(np.abs(ry).sum()), tol)
    p = R.EstimatorParams(alpha=1.5, method="chebyshev", s=40, m=10, seed=11, bounds=R.SpectrumBounds(u=0, v=1))
    ctx.set_fused_mi(True)
    mi = R.mutual_information_samples(x, R.GaussianKernel(sx), y, R.GaussianKernel(sy), p, precision="fp32", ctx=ctx)
    ref_mi = O.mutual_information(a, b, seed=11, alpha=1.5, method="chebyshev", s=40, m=10, bounds=(0.0, 1.0))
    check("fused MI joint entropy", mi.joint_entropy, ref_mi["joint_entropy"], 1e-4)
    import torch

    xb = torch.from_numpy(x).to(torch.bfloat16).double().numpy()
    ref_mf = O.hutchpp(O.Spec("int", 3), O.build_kernel(xb, sx), 6, 13, sketch=sk, probes=pr)["value"]
    k = R.build_kernel(x, R.GaussianKernel(sx), "mf", ctx=ctx)
    got = R.hutchpp(R.MatrixFunctionSpec.int_power(3), k, R.SketchConfig(s_q=6, s_g=13, sketch=sk, probes=pr)).value
    check("matrix-free hutchpp", got, ref_mf, 1e-4)
    e = R.estimate(R.build_kernel(x, R.GaussianKernel(sx), "fp32", ctx=ctx),
                   R.EstimatorParams(alpha=0.5, method="taylor", s=24, m=8, seed=5))
    ref_e = O.estimate(a, alpha=0.5, method="taylor", s=24, m=8, seed=5)
    check("taylor estimate (device power iteration, seeded device probes)", e.entropy, ref_e["entropy"], 1e-4)
    print(f"sanitize cases ok; launches {ctx.launch_count()}")


if __name__ == "__main__":
    main()
