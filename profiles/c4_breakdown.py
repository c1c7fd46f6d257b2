"""Where the config-4 MI step's time goes beyond the fused pass (developer probe, not a bench)."""
import math, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2205_07426_b200 as R
from bench import c4_inputs
n = 100000
x, y = c4_inputs(n, 2205, "product")
ctx = R.Context(0)
ctx.set_fused_mi(True)
sx, sy = R.GaussianKernel(4.0), R.GaussianKernel(math.sqrt(8.0))
params = R.EstimatorParams(alpha=1.01, method="chebyshev", s=90, m=60, seed=2205, bounds=R.SpectrumBounds(u=0.0, v=1.0))
d_x = torch.from_numpy(np.ascontiguousarray(x.T)).cuda(); d_y = torch.from_numpy(np.ascontiguousarray(y.T)).cuda()
torch.cuda.synchronize()
def step():
    return R.mutual_information_samples_dev(d_x.data_ptr(), n, 16, n, sx, d_y.data_ptr(), 8, n, sy, params, "fp32", ctx)
for _ in range(2): step()
ctx.sync()
for rep in range(3):
    ctx.timer_begin(); step(); full = ctx.timer_end()
    ctx.timer_begin(); ka = R.build_kernel_dev(d_x.data_ptr(), n, 16, n, sx, "fp32", ctx); kb = R.build_kernel_dev(d_y.data_ptr(), n, 8, n, sy, "fp32", ctx); gram = ctx.timer_end()
    ctx.profile(True); l0 = ctx.launch_count(); t0 = time.perf_counter()
    ctx.timer_begin(); mi = R.mutual_information([ka], kb, params); est = ctx.timer_end()
    wall = time.perf_counter() - t0
    launches = ctx.launch_count() - l0
    nprof, pms, pb, pf = ctx.profile_read(); ctx.profile(False)
    print(f"step {full:.1f} ms | grams {gram:.1f} | MI from kernels {est:.1f} (host wall {wall*1e3:.1f}) | products {nprof} launches {pms:.1f} ms | rest {est-pms:.1f} ms over {launches} launches")
    del ka, kb
