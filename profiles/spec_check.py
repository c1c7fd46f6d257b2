import os, time
import numpy as np
import sys; sys.path.insert(0, ".")
import paper_2205_07426_b200 as R

def run(flag, prec, n, shift_only=False):
    os.environ["RB_SPECULATE"] = flag
    ctx = R.Context(0)
    k = R.build_kernel(R.mixture_samples(n, 10, 555), R.GaussianKernel(1.0), prec, ctx=ctx)
    out = []
    for rep in range(3):
        t = time.perf_counter()
        b = R.estimate_bounds(k, R.PowerOptions(max_iters=300, tol=1e-7, seed=5 + rep))
        dt = time.perf_counter() - t
        out.append((b.u, b.v, b.u_converged, b.v_converged, dt))
    r = R.power_method(k, R.PowerOptions(max_iters=1, tol=1e-16, seed=3))
    out.append((r.rayleigh, r.iterations))
    r = R.power_method(k, R.PowerOptions(max_iters=40, tol=1e-16, seed=3))
    out.append((r.rayleigh, r.iterations))
    return out

for prec, n in (("fp32", 20000), ("fp64", 2000), ("fp32", 300), ("fp32", 50000)):
    a = run("0", prec, n); b = run("1", prec, n)
    same = all(x[:4] == y[:4] for x, y in zip(a[:3], b[:3])) and a[3:] == b[3:]
    print(prec, n, "identical" if same else "DIFFER", [round(x[4]*1e3, 2) for x in a[:3]], [round(x[4]*1e3, 2) for x in b[:3]])
    if not same: print(a, b)
