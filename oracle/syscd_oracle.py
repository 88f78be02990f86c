"""CPU oracle for the SySCD training epoch (float64, numpy/scipy).

TEST INFRASTRUCTURE ONLY — the checker, never the product.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it.  The product path (paper_1911_07722_b200) never calls into
oracle/ and fails loudly when its CUDA library is missing.

It restates the reference's hot path (pkg/src/syscd/solvers.py:289-453) with
the same arithmetic order so that, on ridge, it reproduces the reference
bitwise (pinned in tests/test_oracle.py against the reference-generated
tests/golden/reference_runs.json, and live when /root/reference is mounted):

  * buckets            partitioning.py:77-82 (consecutive ranges, last partial)
  * node partition     partitioning.py:89-96  key (0,)
  * repartition        partitioning.py:99-109 key (1, k, rid) (static: rid=0,
                       solvers.py:174-178)
  * within-bucket perm partitioning.py:112-117 key (2, rid, b)
  * iid draws          solvers.py:159-170,326-333 key (3, k, p, rid)
  * thread round       solvers.py:289-334: lin = x.u + a x.dv ; step ; axpy on dv
  * node reduction     solvers.py:393 / reduce_replicas solvers.py:112-125
  * global reduction   solvers.py:423
  * K=P=1 exact path   solvers.py:403-410 / _exact_worker_pass :140-171
  * metrics            solvers.py:128-137,425-443 (epoch time excludes metrics)

Partitions within a round are independent (each starts from dv = 0 and reads
only the round-constant u and its own alpha entries), so the
oracle runs them one after another instead of on a thread pool; the
reduction order is the reference's ascending-index order.

Extended objectives (lasso, svm_dual, logistic_dual) swap
only the per-coordinate step and f/g, exactly as the survey's monkeypatch
probe did on the reference driver.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg.blas import daxpy

from . import objectives as obj

NODE_PARTITION, REPARTITION, COORD_PERM, IID_DRAW = 0, 1, 2, 3


def stream(seed, key):
    """partitioning.py:30-38 — np.random.default_rng(SeedSequence(seed, key))."""
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=tuple(key)))


# ----------------------------------------------------------------------------
# data
# ----------------------------------------------------------------------------
class OracleMatrix:
    """Column access over dense (Fortran f64) or per-column sparse storage.

    Mirrors ColumnMatrix.col_dot / col_axpy / matvec / rmatvec
    (dataset.py:73-116) with the same BLAS calls.
    """

    def __init__(self, dense=None, csc=None, shape=None):
        if dense is not None:
            self.dense = np.asfortranarray(dense, dtype=np.float64)
            self.n_rows, self.n_cols = self.dense.shape
            self.cols = None
        else:
            indptr, indices, values = csc
            self.dense = None
            self.n_rows, self.n_cols = shape
            indptr = np.asarray(indptr, dtype=np.int64)
            self.cols = [
                (np.asarray(indices[indptr[j]:indptr[j + 1]], dtype=np.intp),
                 np.ascontiguousarray(values[indptr[j]:indptr[j + 1]], dtype=np.float64))
                for j in range(self.n_cols)
            ]

    def col_dot(self, j, vec):
        if self.dense is not None:
            return float(np.dot(self.dense[:, j], vec))
        idx, vals = self.cols[j]
        return float(np.dot(vals, vec[idx]))

    def col_axpy(self, out, j, s):
        if self.dense is not None:
            daxpy(self.dense[:, j], out, a=s)
        else:
            idx, vals = self.cols[j]
            out[idx] += s * vals

    def col_sq_norm(self, j):
        if self.dense is not None:
            c = self.dense[:, j]
            return float(np.dot(c, c))
        return float(np.dot(self.cols[j][1], self.cols[j][1]))

    def matvec(self, x):
        if self.dense is not None:
            return self.dense @ np.asarray(x, dtype=np.float64)
        out = np.zeros(self.n_rows)
        for j in range(self.n_cols):
            if x[j] != 0.0:
                idx, vals = self.cols[j]
                out[idx] += x[j] * vals
        return out

    def rmatvec(self, y):
        if self.dense is not None:
            return self.dense.T @ np.asarray(y, dtype=np.float64)
        return np.array([self.col_dot(j, y) for j in range(self.n_cols)])


@dataclass
class OracleProblem:
    """kind in objectives.KINDS.  For dual kinds the columns are y_i x_i and y
    is ignored by f (pass zeros of length n_rows)."""

    A: OracleMatrix
    y: np.ndarray
    kind: str
    lam: float
    sq: np.ndarray = None

    def __post_init__(self):
        if self.kind not in obj.KINDS:
            raise ValueError(f"unknown objective {self.kind}")
        if self.lam <= 0.0:
            raise ValueError("lambda must be > 0")
        self.y = np.asarray(self.y, dtype=np.float64)
        if self.sq is None:
            self.sq = np.array([self.A.col_sq_norm(j) for j in range(self.A.n_cols)])

    @property
    def n(self):
        return self.A.n_cols

    @property
    def d(self):
        return self.A.n_rows

    @property
    def gamma(self):
        return obj.gamma_of(self.kind, self.lam, self.n)

    def objective(self, alpha):
        """full_objective (objective.py:95-102): fresh v = A alpha."""
        v = self.A.matvec(alpha)
        return obj.f_value(self.kind, v, self.y, self.lam, self.n) + obj.g_value(
            self.kind, alpha, self.lam, self.n)

    def gap(self, alpha):
        v = self.A.matvec(alpha)
        return obj.duality_gap(self.kind, alpha, v, self.A.rmatvec, self.y, self.lam, self.n)[0]

    def grad(self, v):
        return obj.f_grad(self.kind, v, self.y, self.lam, self.n)

    def step(self, lin, a, j, alpha_j):
        return obj.surrogate_step(self.kind, lin, a, self.sq[j], self.lam, alpha_j, self.n)

    def exact_delta(self, j, alpha_j, v):
        """exact_coordinate_update (objective.py:113-125) on the live v."""
        if self.kind == RIDGE_KIND:
            t = self.A.col_dot(j, self.y - v)
            return (t - self.lam * alpha_j) / (self.sq[j] + self.lam)
        if self.kind == obj.LOGISTIC:
            return _logistic_newton(self, j, alpha_j, v)
        # every other f is quadratic: the surrogate with a = gamma is exact
        u = self.grad(v)
        return self.step(self.A.col_dot(j, u), self.gamma, j, alpha_j)


RIDGE_KIND = obj.RIDGE


def _logistic_newton(pb, j, alpha_j, v, max_iter=20, step_tol=1e-12):
    """Restates objective.py:128-184 (bracket widening + safeguarded Newton)."""
    from scipy.special import expit
    m = pb.A
    lam = pb.lam
    if m.dense is not None:
        xs, vs, ys = m.dense[:, j], v, pb.y
    else:
        idx, xs = m.cols[j]
        vs, ys = v[idx], pb.y[idx]

    def dphi(dd):
        s = expit(-ys * (vs + dd * xs))
        return (-float(np.dot(xs, ys * s)) + lam * (alpha_j + dd),
                float(np.dot(xs * xs, s * (1.0 - s))) + lam)

    rad = 10.0 / max(np.sqrt(pb.sq[j]), 1e-30) + abs(alpha_j)
    lo, hi = -rad, rad
    glo, _ = dphi(lo)
    ghi, _ = dphi(hi)
    widen = 0
    while glo > 0.0 and widen < 60:
        lo *= 2.0
        glo, _ = dphi(lo)
        widen += 1
    while ghi < 0.0 and widen < 120:
        hi *= 2.0
        ghi, _ = dphi(hi)
        widen += 1
    dd = 0.0
    for _ in range(max_iter):
        g, h = dphi(dd)
        if g > 0.0:
            hi = dd
        elif g < 0.0:
            lo = dd
        else:
            break
        st = -g / h
        nd = dd + st
        if not (lo < nd < hi) or not np.isfinite(nd):
            nd = 0.5 * (lo + hi)
            st = nd - dd
        dd = nd
        if abs(st) < step_tol:
            break
    return dd


# ----------------------------------------------------------------------------
# scheduling (pure functions of seed and configuration)
# ----------------------------------------------------------------------------
def n_buckets(n, B):
    return -(-n // B)


def bucket_range(b, B, n):
    lo = b * B
    return lo, min(lo + B, n)


def node_partition(n, B, K, seed):
    nb = n_buckets(n, B)
    if K < 1 or K > nb:
        raise ValueError("bad node-group count")
    order = stream(seed, (NODE_PARTITION,)).permutation(nb)
    order = [int(b) for b in order]
    return [order[k::K] for k in range(K)]


def repartition(node_buckets, P, seed, k, rid):
    if P < 1 or not node_buckets or P > len(node_buckets):
        raise ValueError("bad thread count for this node")
    order = stream(seed, (REPARTITION, k, rid)).permutation(len(node_buckets))
    shuffled = [node_buckets[i] for i in order]
    return [shuffled[p::P] for p in range(P)]


def bucket_coords(b, B, n, seed, rid):
    lo, hi = bucket_range(b, B, n)
    return lo + stream(seed, (COORD_PERM, rid, b)).permutation(hi - lo)


@dataclass
class OracleConfig:
    """SolverConfig's fields (solvers.py:44-88) that the epoch path reads."""

    K: int = 1
    P: int = 1
    bucket_size: int = 8
    T1: int | None = None
    T2: int = 1
    T3: int | None = None
    T4: int | None = None
    sampling: str = "perm"
    repartition: str = "dynamic"
    seed: int = 0
    max_epochs: int = 100
    tolerance: float = 1e-5
    verify: bool = False
    record_alpha: bool = False
    with_gap: bool = False

    @property
    def n_rounds(self):
        return self.T1 if self.T1 is not None else self.max_epochs


def thread_sequence(cfg, n, buckets, k, p, rid):
    """Coordinates one worker visits in one round, in order.

    perm: solvers.py:315-324 ; iid: solvers.py:325-333.
    """
    B = cfg.bucket_size
    seq = []
    if cfg.sampling == "perm":
        t3 = len(buckets) if cfg.T3 is None else min(cfg.T3, len(buckets))
        for b in buckets[:t3]:
            lo, hi = bucket_range(b, B, n)
            coords = bucket_coords(b, B, n, cfg.seed, rid)
            t4 = (hi - lo) if cfg.T4 is None else min(cfg.T4, hi - lo)
            seq.extend(int(j) for j in coords[:t4])
    else:
        g = stream(cfg.seed, (IID_DRAW, k, p, rid))
        t3 = len(buckets) if cfg.T3 is None else cfg.T3
        t4 = cfg.T4 if cfg.T4 is not None else B
        for _ in range(t3):
            b = buckets[int(g.integers(len(buckets)))]
            lo, hi = bucket_range(b, B, n)
            for _ in range(t4):
                seq.append(int(g.integers(lo, hi)))
    return seq


def round_schedule(cfg, n, node_part, rid):
    """[(k, p, coords)] for one node-local round id."""
    out = []
    order_round = rid if cfg.repartition == "dynamic" else 0
    for k, nbk in enumerate(node_part):
        assign = repartition(nbk, cfg.P, cfg.seed, k, order_round)
        for p in range(cfg.P):
            out.append((k, p, thread_sequence(cfg, n, assign[p], k, p, rid)))
    return out


# ----------------------------------------------------------------------------
# solver
# ----------------------------------------------------------------------------
@dataclass
class OracleRow:
    epoch: int
    objective: float
    seconds: float
    updates: int
    rel_change: float
    gap: float | None = None


@dataclass
class OracleResult:
    alpha: np.ndarray
    rows: list
    converged: bool
    total_updates: int
    diverged: bool = False
    snapshots: list = field(default_factory=list)
    v: np.ndarray | None = None


def reduce_replicas(base, replicas):
    """solvers.py:112-125: base + sum_r (r - base), ascending r."""
    if len(replicas) == 1:
        return np.array(replicas[0], dtype=np.float64)
    acc = np.zeros_like(base)
    for r in replicas:
        acc += r - base
    return base + acc


def _rel_change(alpha, prev):
    return float(np.max(np.abs(alpha - prev)) / max(1.0, np.max(np.abs(alpha))))


def _row(pb, cfg, alpha, epoch, secs, upd, rel):
    if cfg.with_gap:
        g, F = obj.duality_gap(pb.kind, alpha, pb.A.matvec(alpha), pb.A.rmatvec, pb.y,
                               pb.lam, pb.n)
        return OracleRow(epoch, F, secs, upd, rel, g)
    return OracleRow(epoch, pb.objective(alpha), secs, upd, rel)


class NonFiniteUpdate(ValueError):
    pass


def _thread_round(pb, seq, lin_vec, v_node, alpha, a):
    """solvers.py:289-334 on a private replica dv (zero at start, :300)."""
    m = pb.A
    dv = np.zeros(v_node.shape[0])
    for j in seq:
        lin = m.col_dot(j, lin_vec) + a * m.col_dot(j, dv)
        delta = pb.step(lin, a, j, alpha[j])
        if not np.isfinite(delta):
            raise NonFiniteUpdate(f"coordinate {j}: non-finite update")
        alpha[j] += delta
        m.col_axpy(dv, j, delta)
    return v_node + dv


def run_syscd(pb: OracleProblem, cfg: OracleConfig, init_alpha=None):
    n = pb.n
    B = cfg.bucket_size
    if cfg.K * cfg.P > n_buckets(n, B):
        raise ValueError(f"K*P={cfg.K * cfg.P} exceeds the bucket count {n_buckets(n, B)}")
    node_part = node_partition(n, B, cfg.K, cfg.seed)
    gamma = pb.gamma
    a = gamma * cfg.P * cfg.K
    alpha = np.zeros(n) if init_alpha is None else np.array(init_alpha, dtype=np.float64)
    v = pb.A.matvec(alpha) if init_alpha is not None else np.zeros(pb.d)
    single = cfg.K == 1 and cfg.P == 1
    rows = [_row(pb, cfg, alpha, 0, 0.0, 0, np.inf)]
    snaps = []
    prev = alpha.copy()
    total = 0
    converged = diverged = False
    for t1 in range(cfg.n_rounds):
        t0 = time.perf_counter()
        upd = 0
        if single and pb.kind == obj.LOGISTIC:
            # solvers.py:403-410: exact updates on the live v
            for t2 in range(cfg.T2):
                rid = t1 * cfg.T2 + t2
                for (_, _, seq) in round_schedule(cfg, n, node_part, rid):
                    for j in seq:
                        delta = pb.exact_delta(j, alpha[j], v)
                        if not np.isfinite(delta):
                            raise NonFiniteUpdate(f"coordinate {j}: non-finite update")
                        alpha[j] += delta
                        pb.A.col_axpy(v, j, delta)
                        upd += 1
        elif single:
            # the exact ridge update (objective.py:118-120) equals the
            # surrogate with a = gamma = 1 on the live v; for the other
            # quadratic f it is the same statement.  Use the reference's
            # exact form for ridge to stay bitwise.
            for t2 in range(cfg.T2):
                rid = t1 * cfg.T2 + t2
                for (_, _, seq) in round_schedule(cfg, n, node_part, rid):
                    for j in seq:
                        delta = pb.exact_delta(j, alpha[j], v)
                        if not np.isfinite(delta):
                            raise NonFiniteUpdate(f"coordinate {j}: non-finite update")
                        alpha[j] += delta
                        pb.A.col_axpy(v, j, delta)
                        upd += 1
        else:
            grad = pb.grad(v)
            node_vs = []
            for k in range(cfg.K):
                v_node = v.copy()
                for t2 in range(cfg.T2):
                    rid = t1 * cfg.T2 + t2
                    order_round = rid if cfg.repartition == "dynamic" else 0
                    assign = repartition(node_part[k], cfg.P, cfg.seed, k, order_round)
                    lin_vec = grad if t2 == 0 else grad + (cfg.K * gamma) * (v_node - v)
                    reps = []
                    census = []
                    for p in range(cfg.P):
                        seq = thread_sequence(cfg, n, assign[p], k, p, rid)
                        census.extend(seq)
                        reps.append(_thread_round(pb, seq, lin_vec, v_node, alpha, a))
                        upd += len(seq)
                    v_node = reduce_replicas(v_node, reps)
                    if cfg.verify and cfg.sampling == "perm" and len(census) != len(set(census)):
                        raise AssertionError("write census: coordinate updated twice in one round")
                node_vs.append(v_node)
            v = reduce_replicas(v, node_vs)
        secs = time.perf_counter() - t0
        total += upd
        if cfg.verify:
            vv = pb.A.matvec(alpha)
            scale = max(1.0, float(np.max(np.abs(vv))))
            if float(np.max(np.abs(vv - v))) > 1e-8 * scale:
                raise AssertionError("replica consistency: v != A @ alpha after reduction")
        if not np.all(np.isfinite(alpha)):
            rows.append(OracleRow(t1 + 1, np.inf, secs, upd, np.inf))
            diverged = True
            break
        rel = _rel_change(alpha, prev)
        prev = alpha.copy()
        rows.append(_row(pb, cfg, alpha, t1 + 1, secs, upd, rel))
        if cfg.record_alpha:
            snaps.append(alpha.copy())
        if cfg.T1 is None and rel < cfg.tolerance:
            converged = True
            break
    return OracleResult(alpha, rows, converged, total, diverged, snaps, v)


def run_wild(pb: OracleProblem, cfg: OracleConfig):
    """run_wild_parallel_scd (solvers.py:214-286) with the P chunks of
    np.array_split(perm, P) run back to back: for P = 1 this is the
    reference's (deterministic) schedule; for P > 1 it is the zero-staleness
    interleaving of the asynchronous workers.  Exact updates on the live v
    (exact_coordinate_update, objective.py:113-125)."""
    n = pb.n
    alpha = np.zeros(n)
    v = np.zeros(pb.d)
    init = pb.objective(alpha)
    rows = [OracleRow(0, init, 0.0, 0, np.inf)]
    prev = alpha.copy()
    total = 0
    converged = diverged = False
    for epoch in range(cfg.n_rounds):
        perm = stream(cfg.seed, (COORD_PERM, epoch, 0)).permutation(n)
        failed = False
        upd = 0
        for chunk in np.array_split(perm, cfg.P):
            for j in chunk:
                j = int(j)
                delta = pb.exact_delta(j, alpha[j], v)
                if not np.isfinite(delta):
                    failed = True
                    break
                alpha[j] += delta
                pb.A.col_axpy(v, j, delta)
                upd += 1
        total += upd
        obj = pb.objective(alpha) if np.all(np.isfinite(alpha)) else np.inf
        if failed or not np.isfinite(obj) or obj > 1e6 * max(init, 1e-300):
            rows.append(OracleRow(epoch + 1, obj, 0.0, upd, np.inf))
            diverged = True
            break
        rel = _rel_change(alpha, prev)
        prev = alpha.copy()
        rows.append(OracleRow(epoch + 1, obj, 0.0, upd, rel))
        if cfg.T1 is None and rel < cfg.tolerance:
            converged = True
            break
    return OracleResult(alpha, rows, converged, total, diverged, [], v)
