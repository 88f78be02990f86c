"""The CPU oracle is pinned to the reference: bitwise on the reference's own
objectives (golden runs produced by the reference), tightly on the extended
objectives run through the reference driver; plus step KATs."""
import math
import os
import sys

import numpy as np
import pytest

from oracle import objectives as obj
from oracle import syscd_oracle as O


def _ref_dense(n_rows, n_cols, seed):
    """generate_synthetic_dense (dataset.py:266-273) streams."""
    g = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(100,)))
    A = np.asfortranarray(g.random((n_rows, n_cols)))
    gl = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(102,)))
    y = gl.integers(0, 2, size=n_rows).astype(np.float64) * 2.0 - 1.0
    return A, y


def test_oracle_reproduces_reference_runs_bitwise(golden):
    for case in golden("reference_runs.json"):
        A, y = _ref_dense(case["n_rows"], case["n_cols"], case["data_seed"])
        kind = "ridge" if case["loss"] == "squared_error" else "logistic"
        pb = O.OracleProblem(O.OracleMatrix(dense=A), y, kind, case["lam"])
        res = O.run_syscd(pb, O.OracleConfig(**case["cfg"]))
        assert [r.objective for r in res.rows] == case["objective"], case["cfg"]
        assert [r.updates for r in res.rows] == case["updates"]
        assert res.alpha.tolist() == case["alpha"]


def test_oracle_reproduces_reference_wild_and_sequential_bitwise(golden):
    """run_wild_parallel_scd (P = 1) and run_sequential_scd (which ignores K
    and P) of the reference, tests/golden/wild_runs.json."""
    import dataclasses
    for case in golden("wild_runs.json"):
        A, y = _ref_dense(case["n_rows"], case["n_cols"], case["data_seed"])
        kind = "ridge" if case["loss"] == "squared_error" else "logistic"
        pb = O.OracleProblem(O.OracleMatrix(dense=A), y, kind, case["lam"])
        cfg = O.OracleConfig(**case["cfg"])
        if case["solver"] == "wild":
            res = O.run_wild(pb, cfg)
        else:
            res = O.run_syscd(pb, dataclasses.replace(cfg, K=1, P=1))
        assert [r.objective for r in res.rows] == case["objective"], case["cfg"]
        assert [r.updates for r in res.rows] == case["updates"]
        assert res.alpha.tolist() == case["alpha"]


def test_oracle_matches_reference_driver_on_extended_objectives(golden):
    for case in golden("extended_runs.json"):
        A = np.asfortranarray(np.array(case["A"]))
        pb = O.OracleProblem(O.OracleMatrix(dense=A), np.array(case["y"]), case["kind"],
                             case["lam"])
        res = O.run_syscd(pb, O.OracleConfig(**case["cfg"]))
        np.testing.assert_allclose([r.objective for r in res.rows], case["objective"],
                                   rtol=1e-12, atol=1e-14)
        np.testing.assert_allclose(res.alpha, case["alpha"], rtol=1e-10, atol=1e-13)


def _golden_section(f, lo, hi, iters=200):
    gr = (math.sqrt(5) - 1) / 2
    a, b = lo, hi
    for _ in range(iters):
        c, d = b - gr * (b - a), a + gr * (b - a)
        if f(c) < f(d):
            b = d
        else:
            a = c
    return 0.5 * (a + b)


@pytest.mark.parametrize("kind", ["ridge", "lasso", "svm_dual", "logistic_dual"])
def test_step_minimises_the_surrogate(kind):
    """Each step is the exact 1-D minimiser of lin*d + aq/2 d^2 + g(alpha+d)
    (pattern of test_objective.py:106-135)."""
    g = np.random.default_rng(5)
    n = 50
    for _ in range(40):
        lin = float(g.normal())
        a, q, lam = float(g.uniform(0.5, 3)), float(g.uniform(0.2, 2)), float(g.uniform(0.01, 1))
        alpha = float(g.uniform(0.05, 0.95)) if kind in ("svm_dual", "logistic_dual") else float(g.normal())

        def model(dl):
            t = alpha + dl
            return lin * dl + 0.5 * a * q * dl * dl + float(
                obj.g_value(kind, np.array([t]), lam, n))

        if kind in ("svm_dual", "logistic_dual"):
            lo, hi = -alpha + 1e-15, 1 - alpha - 1e-15
        else:
            lo, hi = -50.0, 50.0
        ref = _golden_section(model, lo, hi)
        got = obj.surrogate_step(kind, lin, a, q, lam, alpha, n)
        assert model(got) <= model(ref) + 1e-10
        assert abs(got - ref) < 1e-5 * max(1.0, abs(ref))


def test_duality_gaps_nonnegative_and_vanish_at_optimum():
    g = np.random.default_rng(3)
    A = g.standard_normal((60, 8))
    y = g.standard_normal(60)
    M = O.OracleMatrix(dense=A)
    for kind, lam in [("ridge", 0.5), ("lasso", 2.0)]:
        pb = O.OracleProblem(M, y, kind, lam)
        res = O.run_syscd(pb, O.OracleConfig(K=1, P=1, bucket_size=8, T1=400, seed=1))
        assert pb.gap(np.zeros(8)) > 0
        scale = max(1.0, abs(pb.objective(res.alpha)))
        assert -1e-12 * scale <= pb.gap(res.alpha) < 1e-8 * scale
    lab = np.where(g.random(40) < 0.5, -1.0, 1.0)
    Ad = g.standard_normal((6, 40)) * lab
    for kind in ("svm_dual", "logistic_dual"):
        pb = O.OracleProblem(O.OracleMatrix(dense=Ad), np.zeros(6), kind, 0.05)
        res = O.run_syscd(pb, O.OracleConfig(K=1, P=1, bucket_size=8, T1=300, seed=2))
        assert pb.gap(res.alpha) >= -1e-12
        assert pb.gap(res.alpha) < 1e-4
        assert np.all((res.alpha >= 0) & (res.alpha <= 1))


REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")
def test_oracle_vs_live_reference():
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    try:
        import syscd
    finally:
        sys.path.remove(REF)
    for K, P, B, T2, samp, rep, seed in [(1, 4, 4, 1, "perm", "dynamic", 0),
                                           (2, 2, 8, 2, "perm", "static", 5),
                                           (1, 2, 8, 1, "iid", "dynamic", 12)]:
        ds = syscd.generate_synthetic_dense(300, 37, seed)
        pr = syscd.GlmProblem.build(ds, syscd.SmoothLoss.squared_error(), 1.0)
        kw = dict(K=K, P=P, bucket_size=B, T1=4, T2=T2, sampling=samp, repartition=rep, seed=seed,
                  T3=2 if samp == "iid" else None, T4=5 if samp == "iid" else None)
        r = syscd.run_syscd(pr, syscd.SolverConfig(algorithm="syscd", **kw))
        o = O.run_syscd(O.OracleProblem(O.OracleMatrix(dense=ds.matrix.to_dense()), ds.labels,
                                        "ridge", 1.0), O.OracleConfig(**kw))
        assert np.array_equal(r.alpha, o.alpha)


def test_oracle_errors():
    A = np.ones((4, 4))
    pb = O.OracleProblem(O.OracleMatrix(dense=A), np.ones(4), "ridge", 1.0)
    with pytest.raises(ValueError, match="bucket count"):
        O.run_syscd(pb, O.OracleConfig(K=2, P=2, bucket_size=2))
    with pytest.raises(ValueError):
        O.OracleProblem(O.OracleMatrix(dense=A), np.ones(4), "hinge", 1.0)
