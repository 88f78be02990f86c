"""Single-coordinate updates of the reference API (objective.py:113-232):
exact_coordinate_update, SurrogateContext, surrogate_delta and
surrogate_coordinate_update.

These are host utilities kept for API parity -- a caller that drives its own
loop over coordinates can use them on host vectors.  The GPU solvers never
call them: the epoch kernels evaluate the same steps on the device
(csrc/common.cuh coord_step / coord_step_fr, csrc/exact_logistic.cu).  fp64
numpy on the problem's host columns (float32 values promoted).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .objective import LASSO, LOGISTIC, LOGISTIC_DUAL, RIDGE, SVM_DUAL, NonFiniteUpdateError


def _column(problem, j):
    """(row indices or None, values as float64) of coordinate j, with the
    labels folded in for the dual orientation."""
    m = problem.data.matrix
    col = m.column(j)
    if m.storage_kind == "dense":
        idx, x = None, np.asarray(col, dtype=np.float64)
    else:
        idx, x = col[0], np.asarray(col[1], dtype=np.float64)
    if problem.is_dual:
        x = x * problem.data.labels[j]
    return idx, x


def _dot(idx, x, vec):
    return float(np.dot(x, vec if idx is None else vec[idx]))


def _sigmoid(z):
    return 1.0 / (1.0 + math.exp(-z)) if z >= 0 else math.exp(z) / (1.0 + math.exp(z))


def _logistic_dual_root(lin, aq, alpha, n, max_iter=200):
    """Root of lin + aq (sigma(s) - alpha) + s/n in the log-odds s (the
    logistic-dual coordinate minimiser): bracketed Newton with bisection."""
    lo = -n * (lin + aq * (1.0 - alpha)) - 1.0
    hi = n * (aq * alpha - lin) + 1.0
    s = 0.0
    if 0.0 < alpha < 1.0:
        s = math.log(alpha) - math.log1p(-alpha)
    s = min(max(s, lo), hi)
    for _ in range(max_iter):
        t = _sigmoid(s)
        h = lin + aq * (t - alpha) + s / n
        if h > 0.0:
            hi = s
        elif h < 0.0:
            lo = s
        else:
            break
        ns = s - h / (aq * t * (1.0 - t) + 1.0 / n)
        if not (lo < ns < hi):
            ns = 0.5 * (lo + hi)
        step = ns - s
        s = ns
        if abs(step) <= 1e-13 * max(1.0, abs(s)):
            break
    return _sigmoid(s)


def _step(kind, lin, a, q, lam, alpha, n):
    """alpha_j after minimising the quadratic surrogate with curvature a*q
    (SURVEY Appendix A); for the quadratic f and a = gamma this is exact."""
    aq = a * q
    if kind in (RIDGE, LOGISTIC):
        return alpha - (lin + lam * alpha) / (aq + lam)
    if kind == LASSO:
        if aq <= 0.0:
            return 0.0
        z = alpha - lin / aq
        m = abs(z) - lam / aq
        return math.copysign(m, z) if m > 0.0 else 0.0
    if kind == SVM_DUAL:
        if aq <= 0.0:
            return 1.0
        return min(max(alpha - (lin - 1.0 / n) / aq, 0.0), 1.0)
    return _logistic_dual_root(lin, aq, alpha, n)


def _grad(problem, v):
    """grad f(v) on the host (objective.py:105-110 and Appendix A)."""
    v = np.asarray(v, dtype=np.float64)
    kind = problem.kind
    if kind in (RIDGE, LASSO):
        return v - problem.data.labels
    if kind == LOGISTIC:
        y = problem.data.labels
        z = -y * v
        return -y * np.where(z >= 0, 1.0 / (1.0 + np.exp(-np.abs(z))),
                             np.exp(-np.abs(z)) / (1.0 + np.exp(-np.abs(z))))
    return problem.gamma * v  # dual: f(v) = |v|^2 / (2 lam n^2)


def _logistic_newton(problem, j, alpha_j, v, sq, max_iter=20, step_tol=1e-12):
    """Safeguarded 1-D Newton for the primal logistic coordinate
    (objective.py:128-184): same bracket, widening, iteration cap and
    tolerance."""
    lam = problem.reg.lam
    idx, xs = _column(problem, j)
    vs = v if idx is None else v[idx]
    ys = problem.data.labels if idx is None else problem.data.labels[idx]

    def dphi(d):
        z = -ys * (vs + d * xs)
        s = np.where(z >= 0, 1.0 / (1.0 + np.exp(-np.abs(z))),
                     np.exp(-np.abs(z)) / (1.0 + np.exp(-np.abs(z))))
        return (-float(np.dot(xs, ys * s)) + lam * (alpha_j + d),
                float(np.dot(xs * xs, s * (1.0 - s))) + lam)

    rad = 10.0 / max(math.sqrt(sq), 1e-30) + abs(alpha_j)
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
    d = 0.0
    for _ in range(max_iter):
        g, h = dphi(d)
        if g > 0.0:
            hi = d
        elif g < 0.0:
            lo = d
        else:
            break
        step = -g / h
        nd = d + step
        if not (lo < nd < hi) or not math.isfinite(nd):
            nd = 0.5 * (lo + hi)
            step = nd - d
        d = nd
        if abs(step) < step_tol:
            break
    return d


def exact_coordinate_update(problem, j, alpha_j, v):
    """One-dimensional exact minimisation over coordinate j at shared state v
    (objective.py:113-125); the extended objectives use their closed-form (or
    Newton, logistic dual) minimiser with a = gamma."""
    v = np.asarray(v, dtype=np.float64)
    sq = float(problem.stats.column_sq_norms[j])
    kind = problem.kind
    lam = problem.reg.lam
    if kind == RIDGE:
        idx, x = _column(problem, j)
        delta = (_dot(idx, x, problem.data.labels - v) - lam * alpha_j) / (sq + lam)
    elif kind == LOGISTIC:
        delta = _logistic_newton(problem, j, alpha_j, v, sq)
    else:
        idx, x = _column(problem, j)
        lin = _dot(idx, x, _grad(problem, v))
        delta = _step(kind, lin, problem.gamma, sq, lam, alpha_j,
                      float(problem.n_coordinates)) - alpha_j
    if not math.isfinite(delta):
        raise NonFiniteUpdateError(f"coordinate {j}: non-finite update")
    return delta


@dataclass
class SurrogateContext:
    """Read-only quantities fixed at the last node synchronisation
    (objective.py:188-210): scale_a = gamma*P*K, shift_scale = K*gamma."""

    grad_at_sync: np.ndarray
    v_global: np.ndarray
    v_node: np.ndarray
    scale_a: float
    shift_scale: float
    linear: np.ndarray = field(init=False)

    def __post_init__(self):
        if self.v_node is self.v_global:
            self.linear = self.grad_at_sync
        else:
            self.linear = self.grad_at_sync + self.shift_scale * (self.v_node - self.v_global)


def surrogate_delta(lin, scale_a, sq, lam, alpha_j):
    """Closed-form l2 minimiser of the local quadratic surrogate in delta
    (objective.py:213-215)."""
    return -(lin + lam * alpha_j) / (scale_a * sq + lam)


def surrogate_coordinate_update(ctx, problem, j, alpha_j, v_thread):
    """Minimise the separable quadratic surrogate over coordinate j
    (objective.py:218-232); the extended objectives use their own step."""
    idx, x = _column(problem, j)
    lin = _dot(idx, x, ctx.linear)
    if v_thread is not ctx.v_node:
        lin += ctx.scale_a * _dot(idx, x, np.asarray(v_thread) - ctx.v_node)
    sq = float(problem.stats.column_sq_norms[j])
    if problem.kind in (RIDGE, LOGISTIC):
        delta = surrogate_delta(lin, ctx.scale_a, sq, problem.reg.lam, alpha_j)
    else:
        delta = _step(problem.kind, lin, ctx.scale_a, sq, problem.reg.lam, alpha_j,
                      float(problem.n_coordinates)) - alpha_j
    if not math.isfinite(delta):
        raise NonFiniteUpdateError(f"coordinate {j}: non-finite update")
    return delta
