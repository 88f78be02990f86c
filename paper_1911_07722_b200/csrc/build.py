"""Build libsyscd_b200.so in-tree for sm_100a with nvcc (no JIT cache).

Usage: python -m paper_1911_07722_b200.csrc.build [--force]
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
ROOT = os.path.dirname(PKG)
TRACE = bool(os.environ.get("SYSCD_TRACE"))
LIB = os.path.join(PKG, "libsyscd_b200_trace.so" if TRACE else
                   os.environ.get("SYSCD_LIB_NAME", "libsyscd_b200.so"))
SOURCES = ["capi.cu", "plan.cu", "epoch_dense.cu", "epoch_grid.cu", "epoch_small.cu", "epoch_mid.cu", "epoch_sparse.cu", "exact_logistic.cu", "vecops.cu", "libsvm_io.cu", "epoch_wild.cu", "datagen.cu"]
HEADERS = ["common.cuh", "rng.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
    "--expt-relaxed-constexpr", "-Xptxas", "-v",
] + (["-DSYSCD_TRACE"] if TRACE else []) + os.environ.get("SYSCD_NVCC_DEFS", "").split()


def _read(path):
    with open(path, "rb") as f:
        return f.read()


def _hdr_digest():
    h = hashlib.sha256()
    for p in [os.path.join(HERE, x) for x in HEADERS] + [os.path.join(ROOT, "include",
                                                                       "syscd_b200.h")]:
        h.update(_read(p))
    h.update(" ".join([NVCC] + FLAGS).encode())
    return h.hexdigest()


def _digest(src, hdr):
    return hashlib.sha256(_read(os.path.join(HERE, src)) + hdr.encode()).hexdigest()


def _stamp_ok(path, digest):
    return (os.path.exists(path) and os.path.exists(path + ".sha256")
            and _read(path + ".sha256").decode().strip() == digest)


def _write_stamp(path, digest):
    with open(path + ".sha256", "w") as f:
        f.write(digest)


def build(force=False, verbose=False):
    """Compile every source whose content (or a header / the flags) changed
    since its object was built -- content hashes, not mtimes, so a binary
    that does not match the tree is never reused -- and link the library."""
    hdr = _hdr_digest()
    digests = {src: _digest(src, hdr) for src in SOURCES}
    lib_digest = hashlib.sha256("".join(digests[s] for s in SOURCES).encode()).hexdigest()
    if not force and _stamp_ok(LIB, lib_digest):
        return LIB
    objdir = os.path.join(HERE, "_obj_trace" if TRACE else "_obj")
    if os.environ.get("SYSCD_NVCC_DEFS"):  # experiment variants build in their own tree
        objdir = os.path.join(HERE, "_obj_" + os.path.basename(LIB).replace(".so", ""))
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, src.replace(".cu", ".o"))
        if not force and _stamp_ok(obj, digests[src]):
            return obj, ""
        cmd = [NVCC, *FLAGS, "-c", os.path.join(HERE, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        _write_stamp(obj, digests[src])
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
    _write_stamp(LIB, lib_digest)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
