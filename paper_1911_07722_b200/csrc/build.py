"""Build libsyscd_b200.so in-tree for sm_100a with nvcc (no JIT cache).

Usage: python -m paper_1911_07722_b200.csrc.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
ROOT = os.path.dirname(PKG)
TRACE = bool(os.environ.get("SYSCD_TRACE"))
LIB = os.path.join(PKG, "libsyscd_b200_trace.so" if TRACE else
                   os.environ.get("SYSCD_LIB_NAME", "libsyscd_b200.so"))
SOURCES = ["capi.cu", "plan.cu", "epoch_dense.cu", "epoch_grid.cu", "epoch_small.cu", "epoch_mid.cu", "epoch_sparse.cu", "exact_logistic.cu", "vecops.cu", "libsvm_io.cu", "epoch_wild.cu"]
HEADERS = ["common.cuh", "rng.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
] + (["-DSYSCD_TRACE"] if TRACE else []) + os.environ.get("SYSCD_NVCC_DEFS", "").split()


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(HERE, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "syscd_b200.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    objdir = os.path.join(HERE, "_obj_trace" if TRACE else "_obj")
    if os.environ.get("SYSCD_NVCC_DEFS"):  # experiment variants build in their own tree
        objdir = os.path.join(HERE, "_obj_" + os.path.basename(LIB).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)
    hdr_t = max(os.path.getmtime(p) for p in
                [os.path.join(HERE, h) for h in HEADERS]
                + [os.path.join(ROOT, "include", "syscd_b200.h"), os.path.abspath(__file__)])

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        srcp = os.path.join(HERE, src)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(srcp), hdr_t)):
            return obj, ""
        cmd = [NVCC, *FLAGS, "-c", srcp, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return obj, r.stderr

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", tmp,
           "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
