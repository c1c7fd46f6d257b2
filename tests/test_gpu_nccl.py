"""NCCL world 2 (one process per GPU, torchrun) on the row-sharded path, when the box has >= 2 GPUs.

Every rank must return the same MI terms, and they must equal, bit for bit, the same estimate run
as a LocalGroup world 2 on one GPU (same engine code and partition; only the transport differs:
NCCL moves the operand planes byte for byte and a two-rank fp64 sum is order-free). The 1-GPU
boxes of this pool skip it; tests/test_gpu_sharded.py covers the sharded protocol there.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]

WORKER = r'''
import json, math, os, sys
sys.path.insert(0, os.environ["RB_ROOT"])
import torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
import paper_2205_07426_b200 as R
from workloads import f32, mi_inputs
x, y = mi_inputs(3000, 21)
x, y = f32(x), f32(y)
ctx = R.Context(rank)
uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
if rank == 0:
    uid.copy_(torch.frombuffer(bytearray(R.nccl_unique_id()), dtype=torch.uint8))
dist.broadcast(uid, src=0)
ctx.init_nccl(rank, world, bytes(uid.cpu().numpy().tobytes()))
out = {}
for fused in (True, False):
    ctx.set_fused_mi(fused)
    p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=60, m=40, seed=5, bounds=R.SpectrumBounds(u=0, v=1))
    mi = R.mutual_information_samples(x, R.GaussianKernel(4.0), y, R.GaussianKernel(math.sqrt(8.0)), p, "fp32", ctx)
    out[str(fused)] = [mi.value, mi.vars_entropy, mi.target_entropy, mi.joint_entropy]
open(os.environ["RB_OUT"].format(rank=rank), "w").write(json.dumps(out))
dist.destroy_process_group()
'''


def test_nccl_world2_matches_local_group_bitwise(R):
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (this pool's boxes have 1; tests/test_gpu_sharded.py covers LocalGroup ranks)")
    import math
    import threading

    from workloads import f32, mi_inputs

    with tempfile.TemporaryDirectory() as td:
        script = Path(td) / "w.py"
        script.write_text(WORKER)
        env = dict(os.environ, RB_ROOT=str(ROOT), RB_OUT=str(Path(td) / "r{rank}.json"))
        r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                            "--master-addr", "127.0.0.1", "--master-port", str(29700 + os.getpid() % 200),
                            str(script)], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        res = [json.loads((Path(td) / f"r{k}.json").read_text()) for k in range(2)]
    assert res[0] == res[1]
    # the same world-2 estimate over the host-driven LocalGroup transport on GPU 0
    x, y = mi_inputs(3000, 21)
    x, y = f32(x), f32(y)
    group = R.LocalGroup(2)
    local = [None, None]

    def body(rank):
        ctx = R.Context(0)
        ctx.join_local_group(group, rank)
        out = {}
        for fused in (True, False):
            ctx.set_fused_mi(fused)
            p = R.EstimatorParams(alpha=1.01, method="chebyshev", s=60, m=40, seed=5,
                                  bounds=R.SpectrumBounds(u=0, v=1))
            mi = R.mutual_information_samples(x, R.GaussianKernel(4.0), y, R.GaussianKernel(math.sqrt(8.0)), p,
                                              "fp32", ctx)
            out[str(fused)] = [mi.value, mi.vars_entropy, mi.target_entropy, mi.joint_entropy]
        local[rank] = out

    ts = [threading.Thread(target=body, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    assert local[0] == res[0], (local[0], res[0])
