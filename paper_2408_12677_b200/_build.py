"""Build libgsr.so (and the GSR_EXACT_EXP debug build libgsr_exact.so) for sm_100a.

Plain nvcc, in-tree, no torch extension machinery: the library has a C ABI
(include/gsr.h) and is loaded with ctypes, so it never links against torch.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
SOURCES = ["api.cu", "project.cu", "project_bwd.cu", "binning.cu", "render.cu", "optim.cu", "naive.cu", "schedule.cpp", "tsdf.cu", "seed.cu", "frame.cu", "exchange.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
LIBS = {"libgsr.so": [], "libgsr_exact.so": ["-DGSR_EXACT_EXP"], "libgsr_check.so": ["-DGSR_BOUNDS_CHECK"]}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libgsr.so")


def _stale(target: str) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "gsr.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, obj: str, defines: list) -> None:
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE,
           "-Xptxas", "-warn-spills", *defines, "-c", os.path.join(CSRC, src), "-o", obj]
    subprocess.check_call(cmd)


def build(force: bool = False, verbose: bool = False) -> list:
    built = []
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    jobs = []
    for lib, defines in LIBS.items():
        target = os.path.join(PKG, lib)
        if not (force or _stale(target)):
            continue
        tag = lib.replace(".so", "")
        objs = [os.path.join(objdir, f"{tag}_{os.path.splitext(s)[0]}.o") for s in SOURCES]
        jobs.append((target, objs, defines))
    with cf.ThreadPoolExecutor(max_workers=min(10, os.cpu_count() or 4)) as ex:
        futs = [ex.submit(_compile, s, o, d) for (_, objs, d) in jobs for s, o in zip(SOURCES, objs)]
        for f in futs:
            f.result()
    for target, objs, _ in jobs:
        tmp = target + ".tmp"
        subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs])
        os.replace(tmp, target)
        built.append(target)
        if verbose:
            print("built", target)
    return built


if __name__ == "__main__":
    build(force=True, verbose=True)
