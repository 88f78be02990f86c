"""CPU baseline: the oracle restatement timed on the host cores.

TEST / MEASUREMENT INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg and its
--impl reference arm).  It runs the reference's per-partition chain
(solvers.py:303-313: two column dots, the step, one axpy on a private replica,
float64 numpy/BLAS with OPENBLAS_NUM_THREADS=1 as SURVEY finding 7 requires)
on a bounded sample of the workload: every host core runs one partition's
chain over its own block of columns with the workload's shape and value
distribution, for a fixed wall-clock budget.  Partitions are independent
within a round, so this is the reference's own
parallelism with the GIL removed by using processes.
"""

from __future__ import annotations

import os
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

from . import objectives as obj  # noqa: E402


def _worker(args):
    kind, d, ncols, lam, a, n_coords, budget_s, seed, sparse_nnz = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from scipy.linalg.blas import daxpy
    g = np.random.default_rng(seed)
    if sparse_nnz:
        idx = [np.sort(g.choice(d, size=sparse_nnz, replace=False)) for _ in range(ncols)]
        vals = [np.where(g.random(sparse_nnz) < 0.25, 1.0, -1.0) for _ in range(ncols)]
        sq = np.array([float(np.dot(v, v)) for v in vals])
    else:
        A = np.asfortranarray(g.standard_normal((d, ncols)))
        if kind == obj.LASSO:
            A /= np.linalg.norm(A, axis=0)
        sq = np.einsum("ij,ij->j", A, A)
    u = g.standard_normal(d) * 0.01
    alpha = np.zeros(ncols)
    dv = np.zeros(d)
    upd = 0
    t0 = time.perf_counter()
    while True:
        for j in range(ncols):
            if sparse_nnz:
                ix, vx = idx[j], vals[j]
                lin = float(np.dot(vx, u[ix])) + a * float(np.dot(vx, dv[ix]))
            else:
                col = A[:, j]
                lin = float(np.dot(col, u)) + a * float(np.dot(col, dv))
            delta = obj.surrogate_step(kind, lin, a, sq[j], lam, alpha[j], n_coords)
            alpha[j] += delta
            if sparse_nnz:
                dv[ix] += delta * vx
            else:
                daxpy(col, dv, a=delta)
            upd += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return upd, time.perf_counter() - t0


def measure(kind, d, lam, a, n_coords, budget_s=8.0, cores=None, ncols=16, sparse_nnz=0,
            seed=0):
    """Updates/s of the oracle chain on `cores` processes (default: all)."""
    import multiprocessing as mp
    cores = cores or len(os.sched_getaffinity(0))
    args = [(kind, d, ncols, lam, a, n_coords, budget_s, seed + i, sparse_nnz)
            for i in range(cores)]
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        t0 = time.perf_counter()
        res = pool.map(_worker, args)
        wall = time.perf_counter() - t0
    updates = sum(r[0] for r in res)
    busy = max(r[1] for r in res)
    return {
        "updates": updates,
        "seconds": busy,
        "wall": wall,
        "updates_per_s": updates / busy,
        "cores": cores,
        "sample": (f"{cores} partitions x {ncols} cols of d={d} ({'sparse ' + str(sparse_nnz) + ' nnz' if sparse_nnz else 'dense'}), "
                   f"{kind} chain, fp64 numpy/BLAS 1 thread per process, {budget_s:.0f} s budget"),
    }
