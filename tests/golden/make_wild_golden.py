"""Golden trajectories of the REFERENCE's run_wild_parallel_scd (P = 1, the
deterministic schedule) and run_sequential_scd (solvers.py:180-286).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_wild_golden.py
"""

from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

import syscd  # noqa: E402  (the reference)

CASES = [
    # (solver, loss, n_rows, n_cols, lam, data_seed, cfg kwargs)
    ("wild", "squared_error", 300, 37, 1.0, 4, dict(P=1, seed=4, T1=5)),
    ("wild", "squared_error", 250, 20, 0.2, 6, dict(P=1, seed=11, T1=4)),
    ("wild", "logistic", 200, 24, 0.5, 3, dict(P=1, seed=3, T1=4)),
    ("sequential", "squared_error", 300, 37, 1.0, 2, dict(bucket_size=8, seed=2, T1=4)),
    # the reference ignores K / P for the sequential solver
    ("sequential", "squared_error", 300, 37, 1.0, 2, dict(K=2, P=3, bucket_size=8, seed=2, T1=4)),
    ("sequential", "logistic", 200, 24, 0.5, 1, dict(bucket_size=4, seed=1, T1=3)),
]


def main():
    out = []
    for solver, loss, nr, nc, lam, dseed, kw in CASES:
        ds = syscd.generate_synthetic_dense(nr, nc, dseed)
        sl = syscd.SmoothLoss.squared_error() if loss == "squared_error" else syscd.SmoothLoss.logistic()
        pb = syscd.GlmProblem.build(ds, sl, lam)
        cfg = syscd.SolverConfig(algorithm=solver, **kw)
        res = syscd.run_solver(pb, cfg)
        out.append({"solver": solver, "loss": loss, "n_rows": nr, "n_cols": nc, "lam": lam,
                    "data_seed": dseed, "cfg": kw,
                    "objective": [float(m.objective) for m in res.metrics],
                    "updates": [int(m.updates) for m in res.metrics],
                    "alpha": [float(a) for a in res.alpha],
                    "converged": bool(res.converged), "diverged": bool(res.diverged)})
    with open(os.path.join(HERE, "wild_runs.json"), "w") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out)} runs")


if __name__ == "__main__":
    main()
