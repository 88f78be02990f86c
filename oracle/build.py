"""Build the C++/OpenMP oracle restatement (oracle/syscd_cpu.cpp) in-tree.

TEST INFRASTRUCTURE ONLY: the checker's library, never linked by the product.
Output: oracle/_build/libsyscd_oracle.so (git-ignored; it travels to the GPU
box with the snapshot like the product library).  The build is keyed by a
hash of the source and the flags, so a stale binary is never reused.
"""

from __future__ import annotations

import hashlib
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "syscd_cpu.cpp")
OUT_DIR = os.path.join(HERE, "_build")
LIB = os.path.join(OUT_DIR, "libsyscd_oracle.so")
# the system g++ (its libgomp); $CXX in this image points at a toolchain without OpenMP
CXX = os.environ.get("SYSCD_ORACLE_CXX", "/usr/bin/g++")
# x86-64-v3 (AVX2/FMA) runs on this container and on the GPU box's host;
# no contraction so every a*b+c rounds like the Python restatement
FLAGS = ["-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
         "-std=c++17", "-Wall"]


def _digest():
    h = hashlib.sha256()
    with open(SRC, "rb") as f:
        h.update(f.read())
    h.update(" ".join([CXX] + FLAGS).encode())
    return h.hexdigest()


def build(force=False):
    os.makedirs(OUT_DIR, exist_ok=True)
    stamp = LIB + ".sha256"
    digest = _digest()
    if not force and os.path.exists(LIB) and os.path.exists(stamp):
        with open(stamp) as f:
            if f.read().strip() == digest:
                return LIB
    tmp = LIB + ".tmp"
    r = subprocess.run([CXX, *FLAGS, SRC, "-o", tmp], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(digest)
    return LIB


if __name__ == "__main__":
    print(build(force=True))
