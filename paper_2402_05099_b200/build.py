"""Build libhydra.so in-tree: nvcc for sm_100a (cross-compiles without a GPU).

    python -m paper_2402_05099_b200.build [--force] [--debug]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "hydra")
LIB = os.path.join(PKG, "libhydra.so")
# Testing build (-DHYDRA_TESTING): diagnostics, timing experiments and the parity suite's
# sabotage switches, which the release library does not contain (include/hydra.h).
TEST_LIB = os.path.join(PKG, "libhydra_test.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "hydra.h")]


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(p) > t for p in _deps())


def _build_one(lib: str, objdir: str, defines, force: bool, verbose: bool, extra) -> str:
    if not force and not needs_build(lib):
        return lib
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *defines, *extra, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr.strip():
            print(r.stderr, file=sys.stderr)
        return obj

    with ThreadPoolExecutor(max(1, min(8, os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-ldl", "-lpthread", "-lrt"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


def build(force: bool = False, verbose: bool = False, extra=(), testing: bool = True) -> str:
    """Builds the release library (libhydra.so) and, unless testing=False, the testing
    build (libhydra_test.so, -DHYDRA_TESTING) used by the parity suite's sabotage tests
    and by tools/.  Returns the release library's path."""
    with ThreadPoolExecutor(2) as ex:
        jobs = [ex.submit(_build_one, LIB, BUILD, [], force, verbose, extra)]
        if testing:
            jobs.append(ex.submit(_build_one, TEST_LIB, BUILD + "_test", ["-DHYDRA_TESTING"], force, verbose, extra))
        for j in jobs:
            j.result()
    return LIB


if __name__ == "__main__":
    extra = ["-Xptxas", "-v"] if "--ptxas-v" in sys.argv else []
    print(build(force="--force" in sys.argv, verbose=True, extra=extra))
