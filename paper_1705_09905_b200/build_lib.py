"""Compile libfcoo.so in-tree for sm_100a (nvcc; no torch extension machinery).

python -m paper_1705_09905_b200.build_lib   (also called by __graft_entry__.build())
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# FCOO_BUILD_TAG / FCOO_NVCC_EXTRA: experiment builds (e.g. -DFCOO_L1POL_INNER=1) go to
# libfcoo_<tag>.so with their own object dir; the binding loads them when FCOO_LIB points there.
TAG = os.environ.get("FCOO_BUILD_TAG", "")
EXTRA = os.environ.get("FCOO_NVCC_EXTRA", "").split()
LIB = os.path.join(PKG, f"libfcoo_{TAG}.so" if TAG else "libfcoo.so")
OBJ = os.path.join(PKG, f"build_{TAG}" if TAG else "build")
SOURCES = ["fcoo_api.cu", "fcoo_build.cu", "fcoo_engine.cu", "fcoo_cp.cu", "fcoo_comm.cu", "fcoo_ttmc.cu", "fcoo_ttm.cu", "fcoo_dist.cu", "fcoo_tns.cpp"] + [
    f"fcoo_engine_np{k}.cu" for k in range(1, 8)] + [f"fcoo_blocked_np{k}_{a}.cu" for k in range(1, 5) for a in ("f32", "f64")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dirs():
    import nvidia.nccl  # the wheel torch itself loads (same libnccl.so.2 at run time)
    base = list(nvidia.nccl.__path__)[0]
    return os.path.join(base, "include"), os.path.join(base, "lib")


def _flags():
    inc, _ = nccl_dirs()
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-I", os.path.join(ROOT, "include"),
                   "-I", inc, "--expt-relaxed-constexpr", "-Xptxas", "-v" if os.environ.get("FCOO_PTXAS_V") else "-O3"
                   ] + EXTRA


def _deps(path: str, seen=None) -> set:
    """The source and every in-tree header it includes, transitively (#include "...")."""
    import re
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return seen
    seen.add(path)
    with open(path) as f:
        for m in re.finditer(r'^\s*#\s*include\s+"([^"]+)"', f.read(), re.M):
            for d in (os.path.dirname(path), CSRC, os.path.join(ROOT, "include")):
                h = os.path.join(d, m.group(1))
                if os.path.exists(h):
                    _deps(h, seen)
                    break
    return seen


def _compile(src: str) -> str:
    obj = os.path.join(OBJ, os.path.splitext(src)[0] + ".o")
    path = os.path.join(CSRC, src)
    deps = sorted(_deps(path))
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [NVCC] + _flags() + ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if os.environ.get("FCOO_PTXAS_V"):
        sys.stderr.write(r.stderr)
    return obj


def build(force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    if force:
        for f in os.listdir(OBJ):
            os.remove(os.path.join(OBJ, f))
    with cf.ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        _, libdir = nccl_dirs()
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + [
            "-L", libdir, "-l:libnccl.so.2", "-Xlinker", f"-rpath={libdir}", "--cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
