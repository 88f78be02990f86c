"""Generate the golden fixtures from the REFERENCE implementation.

Run in a container where /root/reference exists (read-only; imported with
bytecode writing disabled):

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

Writes tests/golden/*.json.  The fixtures pin
  * the RNG contract: RngStream(seed, key).generator().permutation(n) and
    .integers(lo, hi) draws (partitioning.py:30-38, solvers.py:159-166);
  * static_node_partition / dynamic_repartition / permute_within_bucket
    outputs (partitioning.py:89-117);
  * run_syscd trajectories (per-epoch objective, final alpha, update counts)
    of the reference on small ridge / logistic problems (solvers.py:337-453);
  * run_syscd trajectories for lasso / svm-dual / logistic-dual obtained by
    running the reference driver with only the per-coordinate step and f/g
    swapped (the SURVEY 8(c) monkeypatch mechanism), which pins the
    orchestration of the extended objectives to the reference's own code.
"""

from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import syscd  # noqa: E402  (the reference)
import syscd.solvers as ref_solvers  # noqa: E402
from oracle import objectives as oobj  # noqa: E402


def rng_fixture():
    g = np.random.default_rng(20261019)
    perms, ints = [], []
    for t in range(120):
        seed = int(g.integers(0, 2**62)) if t % 3 else int(g.integers(0, 50))
        kl = int(g.integers(0, 4))
        key = [int(g.integers(0, 2**34 if t % 9 == 0 else 2000)) for _ in range(kl)]
        n = int(g.integers(1, 700))
        p = syscd.RngStream(seed, tuple(key)).generator().permutation(n)
        perms.append({"seed": seed, "key": key, "n": n, "perm": [int(x) for x in p]})
        lo = int(g.integers(0, 40))
        hi = lo + int(g.integers(1, 10**6 if t % 2 else 33))
        gen = syscd.RngStream(seed, tuple(key)).generator()
        draws = [int(gen.integers(lo, hi)) for _ in range(12)]
        ints.append({"seed": seed, "key": key, "lo": lo, "hi": hi, "draws": draws})
    return {"permutations": perms, "integers": ints}


def partition_fixture():
    out = {"static": [], "dynamic": [], "within": []}
    g = np.random.default_rng(7)
    for _ in range(40):
        n = int(g.integers(8, 500))
        B = int(g.integers(1, 17))
        lay = syscd.build_buckets(n, B)
        K = int(g.integers(1, min(5, lay.n_buckets) + 1))
        seed = int(g.integers(0, 1 << 30))
        part = syscd.static_node_partition(lay, K, syscd.RngStream(seed, (0,)))
        out["static"].append({"n": n, "B": B, "K": K, "seed": seed,
                              "assignment": [list(a) for a in part.assignment]})
        k = int(g.integers(0, K))
        P = int(g.integers(1, len(part.assignment[k]) + 1))
        rid = int(g.integers(0, 100))
        asg = syscd.dynamic_repartition(part.assignment[k], P,
                                        syscd.RngStream(seed, (1, k, rid)))
        out["dynamic"].append({"buckets": list(part.assignment[k]), "P": P, "seed": seed, "k": k,
                               "rid": rid, "assignment": [list(a) for a in asg.assignment]})
        b = int(g.integers(0, lay.n_buckets))
        lo, hi = lay.range_of(b)
        perm = syscd.permute_within_bucket((lo, hi), syscd.RngStream(seed, (2, rid, b)))
        out["within"].append({"lo": lo, "hi": hi, "seed": seed, "rid": rid, "b": b,
                              "coords": [int(x) for x in perm]})
    return out


def _traj(result):
    return {"objective": [float(m.objective) for m in result.metrics],
            "updates": [int(m.updates) for m in result.metrics],
            "alpha": [float(a) for a in result.alpha]}


def _data(n_rows, n_cols, seed):
    ds = syscd.generate_synthetic_dense(n_rows, n_cols, seed)
    return ds


RUN_CASES = [
    # (loss, n_rows, n_cols, lam, data_seed, cfg kwargs)
    ("squared_error", 300, 32, 1.0, 8, dict(K=2, P=2, bucket_size=8, seed=8, T1=5)),
    ("squared_error", 300, 37, 1.0, 0, dict(K=1, P=4, bucket_size=4, seed=0, T1=5)),
    ("squared_error", 300, 37, 1.0, 5, dict(K=2, P=2, bucket_size=8, T2=2, repartition="static",
                                            seed=5, T1=4)),
    ("squared_error", 300, 37, 1.0, 12, dict(K=1, P=2, bucket_size=8, T2=2, sampling="iid",
                                             T3=2, T4=5, seed=12, T1=4)),
    ("squared_error", 300, 37, 1.0, 9, dict(K=3, P=1, bucket_size=4, seed=9, T1=4)),
    ("squared_error", 300, 37, 1.0, 6, dict(K=1, P=1, bucket_size=37, T3=1, T4=37, seed=7, T1=4)),
    ("squared_error", 400, 40, 0.5, 3, dict(K=1, P=3, bucket_size=5, T3=2, T4=3, seed=3, T1=4)),
    ("logistic", 200, 24, 0.5, 3, dict(K=2, P=2, bucket_size=4, seed=3, T1=4)),
]


def reference_runs():
    out = []
    for loss, nr, nc, lam, dseed, kw in RUN_CASES:
        ds = _data(nr, nc, dseed)
        sl = syscd.SmoothLoss.squared_error() if loss == "squared_error" else syscd.SmoothLoss.logistic()
        pb = syscd.GlmProblem.build(ds, sl, lam)
        res = syscd.run_syscd(pb, syscd.SolverConfig(algorithm="syscd", **kw))
        out.append({"loss": loss, "n_rows": nr, "n_cols": nc, "lam": lam, "data_seed": dseed,
                    "cfg": kw, **_traj(res)})
    return out


def extended_runs():
    """Reference driver with the step/f/g swapped for the Appendix-A rows."""
    out = []
    cases = [
        ("lasso", 400, 30, 0.3, dict(K=1, P=3, bucket_size=4, seed=2, T1=5)),
        ("lasso", 400, 30, 0.3, dict(K=2, P=2, bucket_size=4, seed=4, T1=5)),
        ("svm_dual", 12, 300, None, dict(K=1, P=4, bucket_size=8, seed=1, T1=5)),
        ("logistic_dual", 12, 300, 1e-2, dict(K=1, P=4, bucket_size=8, seed=5, T1=5)),
    ]
    saved = (ref_solvers.surrogate_delta, ref_solvers.grad_f, ref_solvers.full_objective)
    try:
        for kind, d, n, lam, kw in cases:
            g = np.random.default_rng(100 + len(out))
            A = g.standard_normal((d, n))
            if kind == "lasso":
                A /= np.linalg.norm(A, axis=0)
                w = np.zeros(n)
                w[: n // 5] = g.standard_normal(n // 5)
                y = A @ w + 0.05 * g.standard_normal(d)
            else:
                lab = np.where(g.random(n) < 0.5, -1.0, 1.0)
                A = A / np.linalg.norm(A, axis=0) * lab  # columns y_i x_i
                y = np.zeros(d)
                if lam is None:
                    lam = 1.0 / n
            gamma = oobj.gamma_of(kind, lam, n)
            sq = np.einsum("ij,ij->j", A, A)
            ds = syscd.LabeledDataset(syscd.ColumnMatrix(d, n, dense=A), y)
            stats = syscd.DatasetStats(sq, float("nan"), float(sq.max()))
            # gamma enters the reference only through problem.loss.gamma (solvers.py:358)
            pb = syscd.GlmProblem(ds, syscd.SmoothLoss("squared_error", gamma),
                                  syscd.Regularizer("l2", lam), stats)

            def step(lin, a, q, lam_, alpha_j, _k=kind, _n=n):
                return oobj.surrogate_step(_k, lin, a, q, lam_, alpha_j, _n)

            def gradf(problem, v, _k=kind, _n=n, _lam=lam, _y=y):
                return oobj.f_grad(_k, np.asarray(v, dtype=np.float64), _y, _lam, _n)

            def fobj(problem, alpha, _k=kind, _n=n, _lam=lam, _y=y):
                alpha = np.asarray(alpha, dtype=np.float64)
                v = problem.data.matrix.matvec(alpha)
                return oobj.f_value(_k, v, _y, _lam, _n) + oobj.g_value(_k, alpha, _lam, _n)

            ref_solvers.surrogate_delta = step
            ref_solvers.grad_f = gradf
            ref_solvers.full_objective = fobj
            res = syscd.run_syscd(pb, syscd.SolverConfig(algorithm="syscd", **kw))
            out.append({"kind": kind, "A": A.tolist(), "y": y.tolist(), "lam": lam, "cfg": kw,
                        **_traj(res)})
    finally:
        ref_solvers.surrogate_delta, ref_solvers.grad_f, ref_solvers.full_objective = saved
    return out


def main():
    fixtures = {
        "rng_kat.json": rng_fixture(),
        "partition_kat.json": partition_fixture(),
        "reference_runs.json": reference_runs(),
        "extended_runs.json": extended_runs(),
    }
    for name, obj in fixtures.items():
        with open(os.path.join(HERE, name), "w") as f:
            json.dump(obj, f)
        print("wrote", name)


if __name__ == "__main__":
    main()
