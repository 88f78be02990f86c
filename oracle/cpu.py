"""ctypes wrapper of the C++/OpenMP oracle (oracle/syscd_cpu.cpp).

TEST / MEASUREMENT INFRASTRUCTURE ONLY.  Used by tests/ (full-size parity),
__graft_entry__.smoke() and bench.py's cpu_baseline leg and --impl reference
arm.  The product package never imports it.

`run_syscd(spec, cfg)` has the result shape of oracle.syscd_oracle.run_syscd
(OracleResult with OracleRow per epoch) so the parity helpers compare either
restatement against the GPU.  The data is borrowed, not copied: dense
float32 stores (n, lda) row-major (= column-major A, the GPU store layout) or
Fortran (d, n); CSC arrays as they are.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import objectives as obj
from .syscd_oracle import NonFiniteUpdate, OracleConfig, OracleResult, OracleRow

KIND_ID = {obj.RIDGE: 0, obj.LOGISTIC: 1, obj.LASSO: 2, obj.SVM_DUAL: 3, obj.LOGISTIC_DUAL: 4}


class _Desc(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("d", ctypes.c_int64), ("n", ctypes.c_int64),
        ("A32", ctypes.c_void_p), ("A64", ctypes.c_void_p), ("lda", ctypes.c_int64),
        ("col_ptr", ctypes.c_void_p), ("row_idx", ctypes.c_void_p),
        ("val32", ctypes.c_void_p), ("val64", ctypes.c_void_p),
        ("col_scale", ctypes.c_void_p), ("y", ctypes.c_void_p), ("sq", ctypes.c_void_p),
        ("lam", ctypes.c_double),
        ("K", ctypes.c_int32), ("P", ctypes.c_int32), ("B", ctypes.c_int32),
        ("T2", ctypes.c_int32), ("T3", ctypes.c_int32), ("T4", ctypes.c_int32),
        ("sampling", ctypes.c_int32), ("repartition", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("threads", ctypes.c_int32),
    ]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        from .build import build
        L = ctypes.CDLL(build())
        L.oracle_create.restype = ctypes.c_void_p
        L.oracle_create.argtypes = [ctypes.POINTER(_Desc), ctypes.POINTER(ctypes.c_int)]
        L.oracle_destroy.argtypes = [ctypes.c_void_p]
        L.oracle_round.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)]
        L.oracle_metrics.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(ctypes.c_double)]
        L.oracle_get_state.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_threads.argtypes = [ctypes.c_void_p]
        L.oracle_rng_permutation.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                                             ctypes.c_int64, ctypes.c_void_p]
        L.oracle_rng_integers.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int,
                                          ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_void_p]
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


@dataclass
class CppProblem:
    """The data of one problem, borrowed by the oracle.

    dense: float32/float64 array, either (d, n) Fortran order or an (n, lda)
    C-order store (column j is row j, first d entries).  csc: (col_ptr int64,
    row_idx int32, values float32/float64).  col_scale: per-column factor
    (dual labels, so column j is y_j x_j).  y: length-d targets (primal)."""

    kind: str
    d: int
    n: int
    lam: float
    dense: np.ndarray | None = None
    csc: tuple | None = None
    col_scale: np.ndarray | None = None
    y: np.ndarray | None = None
    sq: np.ndarray | None = None


class CppOracle:
    """One solver state (alpha, v) driven round by round."""

    def __init__(self, spec: CppProblem, cfg: OracleConfig, threads=0):
        L = lib()
        self.spec, self.cfg = spec, cfg
        D = _Desc()
        D.kind = KIND_ID[spec.kind]
        D.d, D.n = int(spec.d), int(spec.n)
        keep = []
        if spec.dense is not None:
            A = spec.dense
            if A.ndim != 2:
                raise ValueError("dense store must be 2-D")
            if A.flags.f_contiguous and A.shape == (spec.d, spec.n):
                lda = spec.d
            elif A.flags.c_contiguous and A.shape[0] == spec.n and A.shape[1] >= spec.d:
                lda = A.shape[1]
            else:
                A = np.asfortranarray(A)
                lda = spec.d
            if A.dtype == np.float32:
                D.A32 = A.ctypes.data
            else:
                A = A.astype(np.float64, copy=False)
                D.A64 = A.ctypes.data
            D.lda = lda
            keep.append(A)
        else:
            cp, ri, va = spec.csc
            cp = np.ascontiguousarray(cp, dtype=np.int64)
            ri = np.ascontiguousarray(ri, dtype=np.int32)
            va = np.ascontiguousarray(va)
            if va.dtype != np.float32:
                va = va.astype(np.float64, copy=False)
                D.val64 = va.ctypes.data
            else:
                D.val32 = va.ctypes.data
            D.col_ptr, D.row_idx = cp.ctypes.data, ri.ctypes.data
            keep += [cp, ri, va]
        for name in ("col_scale", "y", "sq"):
            arr = getattr(spec, name)
            if arr is not None:
                arr = np.ascontiguousarray(arr, dtype=np.float64)
                setattr(D, name, arr.ctypes.data)
                keep.append(arr)
        if spec.kind in (obj.RIDGE, obj.LASSO, obj.LOGISTIC) and spec.y is None:
            raise ValueError("primal objectives need y")
        D.lam = float(spec.lam)
        D.K, D.P, D.B = int(cfg.K), int(cfg.P), int(cfg.bucket_size)
        D.T2 = int(cfg.T2)
        D.T3 = -1 if cfg.T3 is None else int(cfg.T3)
        D.T4 = -1 if cfg.T4 is None else int(cfg.T4)
        D.sampling = 0 if cfg.sampling == "perm" else 1
        D.repartition = 0 if cfg.repartition == "dynamic" else 1
        D.seed = int(cfg.seed)
        D.threads = int(threads)
        self._keep = keep
        self._desc = D
        st = ctypes.c_int(0)
        h = L.oracle_create(ctypes.byref(D), ctypes.byref(st))
        if not h:
            raise ValueError("invalid oracle configuration (K*P, buckets per node, lambda)")
        self.h = ctypes.c_void_p(h)
        self.threads = int(L.oracle_threads(self.h))

    def close(self):
        if getattr(self, "h", None):
            lib().oracle_destroy(self.h)
            self.h = None

    __del__ = close

    def round(self, t1):
        upd = ctypes.c_int64(0)
        secs = ctypes.c_double(0.0)
        st = lib().oracle_round(self.h, int(t1), ctypes.byref(upd), ctypes.byref(secs))
        if st == 2:
            raise NonFiniteUpdate("non-finite coordinate update")
        return int(upd.value), float(secs.value)

    def metrics(self, gap=False):
        F = ctypes.c_double(0.0)
        G = ctypes.c_double(np.nan)
        lib().oracle_metrics(self.h, ctypes.byref(F), ctypes.byref(G) if gap else None)
        return float(F.value), (float(G.value) if gap else None)

    def alpha(self):
        out = np.empty(int(self.spec.n))
        lib().oracle_get_state(self.h, _p(out), None)
        return out

    def v(self):
        out = np.empty(int(self.spec.d))
        lib().oracle_get_state(self.h, None, _p(out))
        return out


def run_syscd(spec: CppProblem, cfg: OracleConfig, threads=0, metrics_every=1):
    """oracle.syscd_oracle.run_syscd's loop over the C++ rounds."""
    o = CppOracle(spec, cfg, threads)
    try:
        F, g = o.metrics(cfg.with_gap)
        rows = [OracleRow(0, F, 0.0, 0, np.inf, g)]
        prev = o.alpha()
        total = 0
        converged = diverged = False
        snaps = []
        for t1 in range(cfg.n_rounds):
            upd, secs = o.round(t1)
            total += upd
            alpha = o.alpha()
            if not np.all(np.isfinite(alpha)):
                rows.append(OracleRow(t1 + 1, np.inf, secs, upd, np.inf))
                diverged = True
                break
            rel = float(np.max(np.abs(alpha - prev)) / max(1.0, float(np.max(np.abs(alpha)))))
            prev = alpha
            last = t1 == cfg.n_rounds - 1
            if (t1 + 1) % metrics_every == 0 or last:
                F, g = o.metrics(cfg.with_gap)
                rows.append(OracleRow(t1 + 1, F, secs, upd, rel, g))
            if cfg.record_alpha:
                snaps.append(alpha.copy())
            if cfg.T1 is None and rel < cfg.tolerance:
                converged = True
                break
        return OracleResult(prev, rows, converged, total, diverged, snaps, o.v())
    finally:
        o.close()


def rng_permutation(seed, key, m):
    out = np.empty(max(m, 1), dtype=np.int64)
    k = np.asarray(key, dtype=np.uint64)
    lib().oracle_rng_permutation(int(seed), _p(k), len(key), int(m), _p(out))
    return out[:m]


def rng_integers(seed, key, lo, hi, count):
    out = np.empty(count, dtype=np.int64)
    k = np.asarray(key, dtype=np.uint64)
    lib().oracle_rng_integers(int(seed), _p(k), len(key), int(lo), int(hi), int(count), _p(out))
    return out
