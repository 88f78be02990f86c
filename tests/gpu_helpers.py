"""Shared helpers for the -m gpu tests: identical seeded data on both sides."""
import numpy as np

from oracle import syscd_oracle as O
from paper_1911_07722_b200.configs import _dims, host_arrays, host_problem

OBJ_RTOL = 1e-4     # per-epoch objective, relative (north_star)
ALPHA_RTOL = 1e-3   # final alpha, relative L2 (north_star)


def oracle_problem(cfg_id, scale, seed=0):
    kind, A, y, lam = host_arrays(cfg_id, scale, seed)
    if kind == "logistic_dual":
        cp, ri, va = A
        d, n = _dims(cfg_id, scale)
        vals = va.astype(np.float64) * np.repeat(y, np.diff(cp))
        return O.OracleProblem(O.OracleMatrix(csc=(cp, ri, vals), shape=(d, n)), np.zeros(d), kind,
                               lam)
    A64 = A.astype(np.float64)
    if kind == "svm_dual":
        return O.OracleProblem(O.OracleMatrix(dense=A64 * y[None, :]), np.zeros(A.shape[0]), kind,
                               lam)
    return O.OracleProblem(O.OracleMatrix(dense=A64), y, kind, lam)


def both(cfg_id, scale, seed=0):
    return host_problem(cfg_id, scale, seed), oracle_problem(cfg_id, scale, seed)


def rel_err(a, b, floor=1e-30):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return np.max(np.abs(a - b) / np.maximum(np.abs(b), floor))


def assert_parity(res, ores, obj_rtol=OBJ_RTOL, alpha_rtol=ALPHA_RTOL):
    got = [m.objective for m in res.metrics]
    ref = [r.objective for r in ores.rows]
    assert len(got) == len(ref)
    assert [m.updates for m in res.metrics] == [r.updates for r in ores.rows]
    scale = max(abs(ref[0]), 1e-12)
    err = np.max(np.abs(np.array(got) - np.array(ref)) / np.maximum(np.abs(ref), 1e-6 * scale))
    assert err < obj_rtol, f"objective trajectory rel err {err:.3e}"
    na = np.linalg.norm(ores.alpha)
    if na > 0:
        e = np.linalg.norm(res.alpha - ores.alpha) / na
        assert e < alpha_rtol, f"alpha rel L2 {e:.3e}"
