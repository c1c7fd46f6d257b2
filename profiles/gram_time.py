import math, os, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2205_07426_b200 as R
from bench import c4_inputs
n = 100000
x, y = c4_inputs(n, 2205, "product")
ctx = R.Context(0)
sx = R.GaussianKernel(4.0)
d_x = torch.from_numpy(np.ascontiguousarray(x.T)).cuda()
torch.cuda.synchronize()
ts = []
for rep in range(6):
    ctx.timer_begin(); ka = R.build_kernel_dev(d_x.data_ptr(), n, 16, n, sx, "fp32", ctx); ts.append(ctx.timer_end()); del ka
print(os.environ.get("RB_LIB_VARIANT", "main"), " ".join(f"{t:.2f}" for t in ts))
