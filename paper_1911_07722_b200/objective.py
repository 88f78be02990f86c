"""GLM objective F(alpha) = f(A alpha) + sum_j g_j(alpha_j): the problem API.

Mirrors pkg/src/syscd/objective.py (SmoothLoss :17-42, Regularizer :45-63,
GlmProblem :66-92, full_objective :95-102, grad_f :105-110) and extends it
as SURVEY section 8(b) asks:

  * Regularizer accepts "l1" as well as "l2" (the reference rejects it,
    objective.py:52-54);
  * GlmProblem accepts the COORDINATES_ARE_EXAMPLES orientation, which selects
    the dual formulation (the reference rejects it, objective.py:74-77):
      - SmoothLoss.hinge()    + l2 -> hinge-SVM dual
      - SmoothLoss.logistic() + l2 -> logistic-regression dual
    labels are then one per column and are folded into the columns (y_i x_i)
    when the data is placed on the device.

Objective values and gradients are computed on the GPU (metrics.py); the
small numpy helpers on SmoothLoss/Regularizer exist only for API parity.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .dataset import (
    COORDINATES_ARE_EXAMPLES,
    COORDINATES_ARE_FEATURES,
    DatasetStats,
    LabeledDataset,
    compute_stats,
)

# objective kinds (must match include/syscd_b200.h)
RIDGE, LOGISTIC, LASSO, SVM_DUAL, LOGISTIC_DUAL = 0, 1, 2, 3, 4
KIND_NAMES = {RIDGE: "ridge", LOGISTIC: "logistic", LASSO: "lasso", SVM_DUAL: "svm_dual",
              LOGISTIC_DUAL: "logistic_dual"}


class NonFiniteUpdateError(ValueError):
    """A coordinate update produced a non-finite value (objective.py:13-14)."""


@dataclass(frozen=True)
class SmoothLoss:
    """Data-fit term; gamma is the smoothness of its scalar component."""

    kind: str
    gamma: float

    @staticmethod
    def squared_error():
        return SmoothLoss("squared_error", 1.0)

    @staticmethod
    def logistic():
        return SmoothLoss("logistic", 0.25)

    @staticmethod
    def hinge():
        """Hinge loss; only usable in the dual (example-as-coordinate) form,
        where the smooth part is ||A alpha||^2 / (2 lam n^2)."""
        return SmoothLoss("hinge", float("nan"))

    def value(self, v, y):
        if self.kind == "squared_error":
            r = v - y
            return 0.5 * float(np.dot(r, r))
        if self.kind == "logistic":
            return float(np.sum(np.logaddexp(0.0, -y * v)))
        raise ValueError("hinge has no primal smooth value")

    def grad(self, v, y):
        if self.kind == "squared_error":
            return v - y
        if self.kind == "logistic":
            z = -y * v
            return -y * np.where(z >= 0, 1.0 / (1.0 + np.exp(-np.abs(z))),
                                 np.exp(-np.abs(z)) / (1.0 + np.exp(-np.abs(z))))
        raise ValueError("hinge has no primal gradient")


@dataclass(frozen=True)
class Regularizer:
    """Separable penalty: "l2" (lam/2 a^2, objective.py:62-63) or "l1" (lam |a|)."""

    kind: str = "l2"
    lam: float = 1.0

    def __post_init__(self):
        if self.kind not in ("l2", "l1"):
            raise ValueError(f"unsupported regularizer: {self.kind}")
        if self.lam <= 0.0:
            raise ValueError("lambda must be > 0")

    @property
    def mu(self):
        return self.lam if self.kind == "l2" else 0.0

    def value(self, alpha):
        alpha = np.asarray(alpha, dtype=np.float64)
        if self.kind == "l2":
            return 0.5 * self.lam * float(np.dot(alpha, alpha))
        return self.lam * float(np.sum(np.abs(alpha)))


@dataclass
class GlmProblem:
    data: LabeledDataset
    loss: SmoothLoss
    reg: Regularizer
    stats: DatasetStats
    _device: object = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        dual = self.data.orientation == COORDINATES_ARE_EXAMPLES
        labels = self.data.labels
        if self.loss.kind not in ("squared_error", "logistic", "hinge"):
            raise ValueError(f"unknown loss: {self.loss.kind}")
        if dual:
            if self.loss.kind == "squared_error":
                raise ValueError("the dual orientation supports hinge and logistic losses")
            if self.reg.kind != "l2":
                raise ValueError("dual problems need the l2 regularizer")
            if not np.all(np.abs(labels) == 1.0):
                raise ValueError(f"{self.loss.kind} loss requires labels in {{-1, +1}}")
        else:
            if self.loss.kind == "hinge":
                raise ValueError("hinge loss needs the coordinates_are_examples orientation")
            if self.loss.kind == "logistic":
                if self.reg.kind != "l2":
                    raise ValueError("primal logistic regression needs the l2 regularizer")
                if not np.all(np.abs(labels) == 1.0):
                    raise ValueError("logistic loss requires labels in {-1, +1}")

    @staticmethod
    def build(data, loss, lam, reg="l2", with_spectral=False):
        """Attach a loss and penalty to a dataset, computing column norms on
        the GPU (the spectral constant c_A is theory-only and skipped unless
        requested)."""
        return GlmProblem(data, loss, Regularizer(reg, lam),
                          compute_stats(data.matrix, with_spectral=with_spectral))

    @property
    def kind(self):
        if self.data.orientation == COORDINATES_ARE_EXAMPLES:
            return SVM_DUAL if self.loss.kind == "hinge" else LOGISTIC_DUAL
        if self.loss.kind == "logistic":
            return LOGISTIC
        return LASSO if self.reg.kind == "l1" else RIDGE

    @property
    def is_dual(self):
        return self.kind in (SVM_DUAL, LOGISTIC_DUAL)

    @property
    def gamma(self):
        """Smoothness of f's scalar component: the a = gamma*K*P factor."""
        if self.is_dual:
            return 1.0 / (self.reg.lam * float(self.n_coordinates) ** 2)
        return self.loss.gamma

    @property
    def n_coordinates(self):
        m = self.data.matrix
        return m.n_cols_global if m.global_cols is not None else m.n_cols

    @property
    def n_shared(self):
        return self.data.matrix.n_rows

    def device(self):
        """The GPU-resident mirror (created once, cached)."""
        if self._device is None:
            from .device import DeviceProblem, Dist
            m = self.data.matrix
            if m.global_cols is not None:  # a shard: metrics reduce over the ranks
                self._device = DeviceProblem(self, store_cols=m.global_cols, dist=Dist())
            else:
                self._device = DeviceProblem(self)
        return self._device


def full_objective(problem, alpha):
    """F(alpha) with the shared vector materialised fresh (GPU, fp64 sums)."""
    alpha = np.asarray(alpha, dtype=np.float64)
    if alpha.shape != (problem.n_coordinates,):
        raise ValueError("alpha length does not match coordinate count")
    return problem.device().objective_host(alpha)


def duality_gap(problem, alpha):
    """Fenchel duality gap at alpha, GPU, fp64 sums."""
    alpha = np.asarray(alpha, dtype=np.float64)
    if alpha.shape != (problem.n_coordinates,):
        raise ValueError("alpha length does not match coordinate count")
    return problem.device().gap_host(alpha)[0]


def grad_f(problem, v):
    """Componentwise derivative of the smooth term at v (GPU)."""
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (problem.n_shared,):
        raise ValueError("v length does not match shared dimension")
    return problem.device().grad_host(v)
