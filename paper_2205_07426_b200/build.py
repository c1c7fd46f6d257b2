"""Builds librenyi_b200.so in-tree (nvcc, sm_100a) — the only product artefact.

Usage: python -m paper_2205_07426_b200.build [--force]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# RB_LIB_VARIANT=<name>: developer A/B builds into _build_<name>/ and librenyi_b200_<name>.so
_VARIANT = os.environ.get("RB_LIB_VARIANT", "")
OBJ = PKG / (f"_build_{_VARIANT}" if _VARIANT else "_build")
LIB = PKG / (f"librenyi_b200_{_VARIANT}.so" if _VARIANT else "librenyi_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]
# developer builds only (e.g. -DRB_MF_TRACE for the matrix-free kernel's clock64 timeline)
COMMON += os.environ.get("RB_EXTRA_NVCC_FLAGS", "").split()

SOURCES = sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))
HEADERS = sorted(list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + [PKG.parent / "include" / "renyi_b200.h"])


def _stale(target: Path, deps) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps)


def _compile(src: Path) -> Path:
    obj = OBJ / (src.name + ".o")
    if _stale(obj, [src, *HEADERS]):
        cmd = [NVCC, *ARCH, *COMMON, "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cu":
            cmd[1:1] = ["-Xptxas", "-warn-spills"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src.name}:\n{r.stdout}\n{r.stderr}")
    return obj


def build(force: bool = False) -> Path:
    OBJ.mkdir(exist_ok=True)
    if force:
        for o in OBJ.glob("*.o"):
            o.unlink()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static", "-ldl", "-lrt",
               "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
