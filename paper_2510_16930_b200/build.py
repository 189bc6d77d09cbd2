"""Builds the native libraries in-tree (sm_100a only).

  lib/libhoqri_b200.so  — the CUDA engine + C-ABI (include/hoqri_b200.h)
  lib/libtucker_b200.so — the C++ `tucker::` drop-in shim over the C-ABI
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
ENGINE = os.path.join(LIB, "libhoqri_b200.so")
SHIM = os.path.join(LIB, "libtucker_b200.so")


def _newer(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_engine(force=False, verbose=False):
    """One object per .cu (compiled in parallel, rebuilt when the file or any
    header / .inc changed), then one shared-library link."""
    os.makedirs(LIB, exist_ok=True)
    obj_dir = os.path.join(ROOT, "build", "obj")
    os.makedirs(obj_dir, exist_ok=True)
    cus = sorted(glob.glob(os.path.join(CSRC, "hq_*.cu")))
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.inc")) + [os.path.join(ROOT, "include", "hoqri_b200.h")]
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills",
             "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]
    objs, jobs = [], []
    for cu in cus:
        o = os.path.join(obj_dir, os.path.basename(cu)[:-3] + ".o")
        objs.append(o)
        if force or _newer(o, [cu] + hdrs):
            jobs.append([NVCC, *flags, "-c", cu, "-o", o])
    if jobs:
        from concurrent.futures import ThreadPoolExecutor
        def run(cmd):
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            list(ex.map(run, jobs))
    if not force and not jobs and not _newer(ENGINE, objs):
        return ENGINE
    cmd = [NVCC, *ARCH, "-shared", *objs, "-lcublas", "-lcusolver", "-o", ENGINE]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return ENGINE


def build_shim(force=False, verbose=False):
    src = os.path.join(CSRC, "tucker_shim.cpp")
    if not os.path.exists(src):
        return None
    deps = [src] + glob.glob(os.path.join(ROOT, "include", "tucker", "*.hpp")) + [ENGINE]
    if not force and not _newer(SHIM, deps):
        return SHIM
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"), src,
           "-L", LIB, "-lhoqri_b200", "-Wl,-rpath,$ORIGIN", "-o", SHIM]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return SHIM


def build(force=False, verbose=False):
    build_engine(force, verbose)
    build_shim(force, verbose)


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
