"""The C++/OpenMP oracle (oracle/syscd_cpu.cpp) is pinned like the Python
restatement: the RNG on the reference-generated KAT, the solver on the
reference's own golden runs and the extended-objective runs of the reference
driver, and against oracle/syscd_oracle.py on every BASELINE config geometry
and solver option at small sizes (1e-12 relative: same arithmetic, different
dot-product association).  Results do not depend on the thread count."""
import numpy as np
import pytest

from gpu_helpers import oracle_problem
from oracle import cpu as C
from oracle import syscd_oracle as O

REL = 1e-11


def _spec_from_oracle(ob):
    m = ob.A
    if m.dense is not None:
        return C.CppProblem(ob.kind, ob.d, ob.n, ob.lam, dense=m.dense,
                            y=None if ob.kind in ("svm_dual", "logistic_dual") else ob.y)
    cp = np.zeros(m.n_cols + 1, dtype=np.int64)
    np.cumsum([len(c[0]) for c in m.cols], out=cp[1:])
    ri = np.concatenate([c[0] for c in m.cols]).astype(np.int32)
    va = np.concatenate([c[1] for c in m.cols])
    return C.CppProblem(ob.kind, ob.d, ob.n, ob.lam, csc=(cp, ri, va),
                        y=None if ob.kind in ("svm_dual", "logistic_dual") else ob.y)


def _close(res, ores, rel=REL):
    a = np.array([r.objective for r in res.rows])
    b = np.array([r.objective for r in ores.rows])
    assert a.shape == b.shape
    scale = max(abs(b[0]), 1e-300)
    err = np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-9 * scale))
    assert err < rel, f"objective rel err {err:.3e}"
    assert [r.updates for r in res.rows] == [r.updates for r in ores.rows]
    na = max(np.linalg.norm(ores.alpha), 1e-300)
    e = np.linalg.norm(res.alpha - ores.alpha) / na
    assert e < 100 * rel, f"alpha rel L2 {e:.3e}"
    if ores.rows[-1].gap is not None:
        for r, q in zip(res.rows, ores.rows):
            assert abs(r.gap - q.gap) <= rel * (abs(q.objective) + abs(q.gap)) + 1e-12


def test_rng_kat(golden):
    kat = golden("rng_kat.json")
    for c in kat["permutations"]:
        assert C.rng_permutation(c["seed"], c["key"], c["n"]).tolist() == c["perm"]
    for c in kat["integers"]:
        got = C.rng_integers(c["seed"], c["key"], c["lo"], c["hi"], len(c["draws"]))
        assert got.tolist() == c["draws"]


def _ref_dense(n_rows, n_cols, seed):
    g = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(100,)))
    A = np.asfortranarray(g.random((n_rows, n_cols)))
    gl = np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(102,)))
    y = gl.integers(0, 2, size=n_rows).astype(np.float64) * 2.0 - 1.0
    return A, y


def test_reference_golden_runs(golden):
    """The reference's own run_syscd trajectories (ridge / primal logistic,
    K>1, T2>1, static, iid, T3/T4, K=P=1 exact)."""
    for case in golden("reference_runs.json"):
        A, y = _ref_dense(case["n_rows"], case["n_cols"], case["data_seed"])
        kind = "ridge" if case["loss"] == "squared_error" else "logistic"
        spec = C.CppProblem(kind, A.shape[0], A.shape[1], case["lam"], dense=A, y=y)
        res = C.run_syscd(spec, O.OracleConfig(**case["cfg"]), threads=3)
        got = np.array([r.objective for r in res.rows])
        ref = np.array(case["objective"])
        assert np.max(np.abs(got - ref) / np.abs(ref)) < REL, case["cfg"]
        assert [r.updates for r in res.rows] == case["updates"]
        a = np.array(case["alpha"])
        assert np.linalg.norm(res.alpha - a) / np.linalg.norm(a) < 100 * REL


def test_extended_golden_runs(golden):
    """Lasso / SVM-dual / logistic-dual through the reference driver."""
    for case in golden("extended_runs.json"):
        A = np.asfortranarray(np.array(case["A"]))
        y = np.array(case["y"])
        dual = case["kind"] in ("svm_dual", "logistic_dual")
        spec = C.CppProblem(case["kind"], A.shape[0], A.shape[1], case["lam"], dense=A,
                            y=None if dual else y)
        res = C.run_syscd(spec, O.OracleConfig(**case["cfg"]), threads=2)
        ref = np.array(case["objective"])
        got = np.array([r.objective for r in res.rows])
        floor = 1e-9 * np.max(np.abs(ref))
        assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), floor)) < 1e-10, case["kind"]
        a = np.array(case["alpha"])
        assert np.linalg.norm(res.alpha - a) / max(np.linalg.norm(a), 1e-300) < 1e-9


CASES = [
    (0, 0.05, dict(K=1, P=4, bucket_size=4, T1=4)),
    (0, 0.05, dict(K=2, P=2, bucket_size=4, T2=3, T1=3)),
    (0, 0.05, dict(K=2, P=2, bucket_size=4, T2=2, repartition="static", T1=3)),
    (0, 0.05, dict(K=1, P=3, bucket_size=5, T3=2, T4=3, T1=3)),
    (0, 0.05, dict(K=1, P=2, bucket_size=4, sampling="iid", T3=2, T4=3, T1=3)),
    (0, 0.05, dict(K=1, P=1, bucket_size=8, T1=3)),
    (1, 0.0005, dict(K=1, P=8, bucket_size=4, T1=3)),
    (1, 0.0005, dict(K=1, P=1, bucket_size=16, T1=3)),
    (2, 0.01, dict(K=1, P=4, bucket_size=2, T1=3)),
    (2, 0.01, dict(K=1, P=1, bucket_size=8, T1=3)),
    (3, 0.002, dict(K=2, P=2, bucket_size=4, T1=3)),
    (3, 0.002, dict(K=1, P=1, bucket_size=8, sampling="iid", T3=4, T4=8, T1=2)),
    (4, 0.0002, dict(K=1, P=4, bucket_size=8, T1=3)),
    (4, 0.0002, dict(K=2, P=3, bucket_size=16, sampling="iid", T3=3, T4=4, T1=2)),
    (4, 0.0002, dict(K=1, P=1, bucket_size=8, T1=2)),
    # d >= 4096: every chain of a T2 = 1 round at once, each by a team of
    # threads (round_teams / team_chain in oracle/syscd_cpu.cpp)
    (2, 0.02, dict(K=1, P=4, bucket_size=2, T1=3)),
    (2, 0.02, dict(K=2, P=3, bucket_size=2, T1=3)),
    (0, 0.25, dict(K=2, P=2, bucket_size=4, T1=3)),
    (3, 0.005, dict(K=3, P=1, bucket_size=8, T1=2)),
]


@pytest.mark.parametrize("cfg_id,scale,kw", CASES)
def test_matches_python_oracle(cfg_id, scale, kw):
    ob = oracle_problem(cfg_id, scale)
    cfg = O.OracleConfig(with_gap=True, **kw)
    ores = O.run_syscd(ob, cfg)
    res = C.run_syscd(_spec_from_oracle(ob), cfg, threads=4)
    _close(res, ores)


def test_thread_count_independent():
    for cfg_id, scale, kw in [(0, 0.05, dict(K=1, P=4, bucket_size=4, T1=3)),
                              (4, 0.0002, dict(K=1, P=4, bucket_size=8, T1=2)),
                              (3, 0.002, dict(K=1, P=1, bucket_size=8, T1=2)),
                              (2, 0.02, dict(K=2, P=3, bucket_size=2, T1=2))]:
        spec = _spec_from_oracle(oracle_problem(cfg_id, scale))
        cfg = O.OracleConfig(**kw)
        r1 = C.run_syscd(spec, cfg, threads=1)
        r5 = C.run_syscd(spec, cfg, threads=5)
        assert [r.objective for r in r1.rows] == [r.objective for r in r5.rows]
        assert r1.alpha.tolist() == r5.alpha.tolist()


def test_float32_store_layouts_agree():
    """An (n, lda) float32 store (the GPU layout) and a Fortran (d, n) float32
    array give the same run; float32 widened to float64 equals the float64
    copy the reference makes (dataset.py:38)."""
    from paper_1911_07722_b200.configs import host_arrays
    kind, A, y, lam = host_arrays(2, 0.01)
    d, n = A.shape
    lda = (d + 3) // 4 * 4
    store = np.zeros((n, lda), dtype=np.float32)
    store[:, :d] = A.T
    cfg = O.OracleConfig(K=1, P=4, bucket_size=2, T1=2)
    r1 = C.run_syscd(C.CppProblem(kind, d, n, lam, dense=A, y=y), cfg)
    r2 = C.run_syscd(C.CppProblem(kind, d, n, lam, dense=store, y=y), cfg)
    r3 = C.run_syscd(C.CppProblem(kind, d, n, lam, dense=A.astype(np.float64), y=y), cfg)
    assert [r.objective for r in r1.rows] == [r.objective for r in r2.rows]
    assert [r.objective for r in r1.rows] == [r.objective for r in r3.rows]


def test_configuration_errors():
    spec = C.CppProblem("ridge", 10, 8, 0.1, dense=np.ones((10, 8)), y=np.zeros(10))
    with pytest.raises(ValueError):
        C.CppOracle(spec, O.OracleConfig(K=3, P=3, bucket_size=1))
    with pytest.raises(ValueError):
        C.CppOracle(spec, O.OracleConfig(K=1, P=2, bucket_size=8))
