"""High-accuracy optimum F* on the GPU (mirror of compute_reference_optimum,
pkg/src/syscd/cli.py:74-111).

Ridge: conjugate gradients on the normal equations (A^T A + lam I) alpha =
A^T y with the metrics kernels (fp32 A, fp64 accumulation and vectors; the
iterate is rounded to fp32 only for the A alpha product, which bounds the
attainable relative residual near 1e-7 -- enough for F*, which is quadratic
around the optimum).  Other objectives: a K=P=1 run (exact updates) to the
model-change tolerance, as the reference's "run" mode does.
"""

from __future__ import annotations

import numpy as np

from .device import DeviceProblem, Dist, _matvec_raw, _rmatvec_raw, _torch
from .objective import RIDGE


def _ridge_cg(problem, rtol=1e-10, max_iter=500):
    """(x over this rank's store columns, iterations, relative residual)."""
    torch = _torch()
    dp = problem.device()
    d, n = dp.d, dp.n_store
    md = dp.mdev
    work = dp._mv_work
    v = torch.empty(d, dtype=torch.float64, device="cuda")

    def normal_op(x64):
        _matvec_raw(md, d, x64.float(), v, work)
        dp.dist.allreduce_(v)  # a sharded problem: A x sums every rank's columns
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        _rmatvec_raw(md, d, v, out)
        return out + dp.lam * x64

    def dot(a, b):  # over every rank's coordinates (a sharded problem)
        return float(dp.dist.allreduce_(torch.dot(a, b).reshape(1)))

    b = torch.empty(n, dtype=torch.float64, device="cuda")
    _rmatvec_raw(md, d, dp.y, b)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = b.clone()
    p = r.clone()
    rs = dot(r, r)
    bnorm = max(np.sqrt(dot(b, b)), 1e-300)
    rs_new = rs
    it = 0
    for it in range(max_iter):
        Ap = normal_op(p)
        alpha = rs / dot(p, Ap)
        x += alpha * p
        r -= alpha * Ap
        rs_new = dot(r, r)
        if np.sqrt(rs_new) <= rtol * bnorm:
            break
        p = r + (rs_new / rs) * p
        rs = rs_new
    return x, it + 1, float(np.sqrt(rs_new) / bnorm)


def compute_reference_optimum(problem, mode="closed-form", max_epochs=2000):
    """(alpha_star as fp64 numpy, F*) like cli.py:74-111."""
    if problem.kind == RIDGE and mode != "run":
        x, _, _ = _ridge_cg(problem)
        alpha = x.cpu().numpy()
        return alpha, problem.device().objective_host(alpha)
    from .solvers import SolverConfig, run_syscd
    cfg = SolverConfig(algorithm="syscd", K=1, P=1, bucket_size=8, seed=problem.n_coordinates,
                       max_epochs=max_epochs, tolerance=1e-9, metrics_every=10 ** 9)
    res = run_syscd(problem, cfg, dist=Dist.single())  # the full problem, this process
    return res.alpha, res.metrics[-1].objective
