"""Oracle objectives: F(alpha) = f(A alpha) + sum_j g_j(alpha_j), float64.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs use it, and only as the checker.

Reference rows (pkg/src/syscd/objective.py):
  * squared loss f = 1/2 ||v - y||^2, gamma = 1        (objective.py:26,33-35,40-41)
  * logistic loss f = sum log(1+exp(-y v)), gamma=1/4   (objective.py:30,36-37,42)
  * l2 penalty g = lam/2 alpha^2                        (objective.py:62-63)
  * surrogate step delta = -(lin + lam a_j)/(a q_j + lam) (objective.py:213-215)
  * exact ridge step (objective.py:118-120) and safeguarded logistic Newton
    (objective.py:128-184)
The reference rejects everything else (objective.py:52-56,74-77); the three
extra rows (lasso, hinge-SVM dual, logistic dual) follow SURVEY.md Appendix A
and are parity-unpinned by the reference's own tests (pinned here by 1-D
golden-section KATs and by running them through the reference driver with the
step swapped: tests/test_oracle.py, fixtures by tests/golden/make_golden.py).
"""

from __future__ import annotations

import math

import numpy as np
from scipy.special import expit

RIDGE = "ridge"
LOGISTIC = "logistic"            # primal L2-regularised logistic regression
LASSO = "lasso"
SVM_DUAL = "svm_dual"            # hinge loss, dual, columns = y_i x_i
LOGISTIC_DUAL = "logistic_dual"  # logistic loss, dual, columns = y_i x_i

KINDS = (RIDGE, LOGISTIC, LASSO, SVM_DUAL, LOGISTIC_DUAL)
DUAL_KINDS = (SVM_DUAL, LOGISTIC_DUAL)


def gamma_of(kind, lam, n_coords):
    """Smoothness of the scalar component of f (the a = gamma*K*P factor)."""
    if kind in (RIDGE, LASSO):
        return 1.0
    if kind == LOGISTIC:
        return 0.25
    return 1.0 / (lam * float(n_coords) ** 2)


def f_value(kind, v, y, lam, n_coords):
    if kind in (RIDGE, LASSO):
        r = v - y
        return 0.5 * float(np.dot(r, r))
    if kind == LOGISTIC:
        return float(np.sum(np.logaddexp(0.0, -y * v)))
    return float(np.dot(v, v)) / (2.0 * lam * float(n_coords) ** 2)


def f_grad(kind, v, y, lam, n_coords):
    if kind in (RIDGE, LASSO):
        return v - y
    if kind == LOGISTIC:
        return -y * expit(-y * v)
    return v / (lam * float(n_coords) ** 2)


def _xlogx(t):
    t = np.asarray(t, dtype=np.float64)
    out = np.zeros_like(t)
    m = t > 0.0
    out[m] = t[m] * np.log(t[m])
    return out


def g_value(kind, alpha, lam, n_coords):
    if kind in (RIDGE, LOGISTIC):
        return 0.5 * lam * float(np.dot(alpha, alpha))
    if kind == LASSO:
        return lam * float(np.sum(np.abs(alpha)))
    if kind == SVM_DUAL:
        return -float(np.sum(alpha)) / n_coords
    return float(np.sum(_xlogx(alpha) + _xlogx(1.0 - alpha))) / n_coords


def surrogate_step(kind, lin, a, q, lam, alpha_j, n_coords):
    """argmin_delta lin*delta + (a q / 2) delta^2 + g_j(alpha_j + delta)."""
    if kind in (RIDGE, LOGISTIC):
        return -(lin + lam * alpha_j) / (a * q + lam)
    aq = a * q
    if kind == LASSO:
        if aq <= 0.0:
            return -alpha_j
        z = alpha_j - lin / aq
        thr = lam / aq
        new = math.copysign(max(abs(z) - thr, 0.0), z)
        return new - alpha_j
    if kind == SVM_DUAL:
        if aq <= 0.0:
            return 1.0 - alpha_j
        new = min(max(alpha_j - (lin - 1.0 / n_coords) / aq, 0.0), 1.0)
        return new - alpha_j
    return logistic_dual_newton(lin, aq, alpha_j, n_coords) - alpha_j


def _sigmoid(s):
    return 1.0 / (1.0 + math.exp(-s)) if s >= 0 else math.exp(s) / (1.0 + math.exp(s))


def logistic_dual_newton(lin, aq, alpha_j, n_coords, max_iter=200):
    """Root of h(s) = lin + aq (sigma(s) - alpha_j) + s/n over s = logit(t).

    h is strictly increasing (h' = aq s(1-s) + 1/n) with h(lo) < 0 < h(hi)
    on the bracket below, so a bracketed Newton converges; working in
    log-odds keeps t = sigma(s) strictly inside (0, 1).  Safeguards (the
    bracket-and-bisect pattern of objective.py:146-184, tightened): bisect
    whenever the Newton iterate would leave the bracket or the step is not
    at least halving (the log-odds Newton oscillates between the sigmoid's
    flat tails otherwise); stop on a relative step below 1e-13 or when no
    representable progress is left.
    """
    inv_n = 1.0 / n_coords
    lo = -n_coords * (lin + aq * (1.0 - alpha_j)) - 1.0
    hi = n_coords * (aq * alpha_j - lin) + 1.0
    if 0.0 < alpha_j < 1.0:
        s = math.log(alpha_j) - math.log1p(-alpha_j)
        s = min(max(s, lo), hi)
    else:
        s = min(max(0.0, lo), hi)
    dx_old = dx = hi - lo
    for _ in range(max_iter):
        t = _sigmoid(s)
        h = lin + aq * (t - alpha_j) + s * inv_n
        if h > 0.0:
            hi = s
        elif h < 0.0:
            lo = s
        else:
            break
        dh = aq * t * (1.0 - t) + inv_n
        if ((s - hi) * dh - h) * ((s - lo) * dh - h) > 0.0 or abs(2.0 * h) > abs(dx_old * dh):
            dx_old, dx = dx, 0.5 * (hi - lo)
            ns = lo + dx
        else:
            dx_old, dx = dx, h / dh
            ns = s - dx
        if ns == s:
            break
        s = ns
        if abs(dx) <= 1e-13 * max(1.0, abs(s)):
            break
    return _sigmoid(s)


def duality_gap(kind, alpha, v, atw_fn, y, lam, n_coords):
    """Fenchel duality gap at (alpha, v = A alpha).  atw_fn(w) returns A^T w.

    Primal kinds: dual point w = grad f(v) (lasso: scaled
    into the dual-feasible box).  Dual kinds: primal point w = v / (lam n).
    """
    F = f_value(kind, v, y, lam, n_coords) + g_value(kind, alpha, lam, n_coords)
    if kind in (RIDGE, LASSO):
        w = v - y
        atw = atw_fn(w)
        if kind == RIDGE:
            D = -0.5 * float(np.dot(w, w)) - float(np.dot(w, y)) - float(np.dot(atw, atw)) / (2 * lam)
        else:
            m = float(np.max(np.abs(atw))) if atw.size else 0.0
            s = 1.0 if m <= lam else lam / m
            w = w * s
            D = -0.5 * float(np.dot(w, w)) - float(np.dot(w, y))
        return F - D, F
    if kind == LOGISTIC:
        w = -y * expit(-y * v)
        s = np.clip(-y * w, 0.0, 1.0)
        atw = atw_fn(w)
        D = -float(np.sum(_xlogx(s) + _xlogx(1.0 - s))) - float(np.dot(atw, atw)) / (2 * lam)
        return F - D, F
    w = v / (lam * n_coords)
    margins = atw_fn(w)
    if kind == SVM_DUAL:
        loss = float(np.sum(np.maximum(0.0, 1.0 - margins))) / n_coords
    else:
        loss = float(np.sum(np.logaddexp(0.0, -margins))) / n_coords
    P = 0.5 * lam * float(np.dot(w, w)) + loss
    return P + F, F
