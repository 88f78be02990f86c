"""Host-side API contract (no GPU): SolverConfig validation (solvers.py:63-79,
test_solvers.py:210-228), problem validation and objective-kind mapping,
reduce_replicas order (test_solvers.py:27-54), sharding."""
import numpy as np
import pytest

from paper_1911_07722_b200 import (
    COORDINATES_ARE_EXAMPLES,
    ColumnMatrix,
    DatasetStats,
    GlmProblem,
    LabeledDataset,
    Regularizer,
    SmoothLoss,
    SolverConfig,
    reduce_replicas,
)
from paper_1911_07722_b200.objective import LASSO, LOGISTIC, LOGISTIC_DUAL, RIDGE, SVM_DUAL
from paper_1911_07722_b200.sharding import shard_plan


def test_config_validation():
    for kw in (dict(K=0), dict(P=0), dict(T2=0), dict(T3=0), dict(T4=0), dict(sampling="sobol"),
               dict(repartition="greedy"), dict(tolerance=0.0), dict(max_epochs=-1),
               dict(algorithm="gradient_descent"), dict(metrics_every=0)):
        with pytest.raises(ValueError):
            SolverConfig(**kw)
    assert SolverConfig(cache_line_bytes=128).resolved_bucket_size() == 16
    assert SolverConfig().resolved_bucket_size() == 8
    assert SolverConfig(T1=7).n_rounds == 7 and SolverConfig(max_epochs=9).n_rounds == 9


def _stats(n):
    return DatasetStats(np.ones(n), float("nan"), 1.0)


def test_problem_kinds_and_validation():
    m = ColumnMatrix(4, 3, dense=np.ones((4, 3)))
    feat = LabeledDataset(m, np.array([1.0, -1, 1, -1]))
    ex = LabeledDataset(m, np.array([1.0, -1, 1]), COORDINATES_ARE_EXAMPLES)
    assert GlmProblem(feat, SmoothLoss.squared_error(), Regularizer("l2", 1.0), _stats(3)).kind == RIDGE
    assert GlmProblem(feat, SmoothLoss.squared_error(), Regularizer("l1", 1.0), _stats(3)).kind == LASSO
    assert GlmProblem(feat, SmoothLoss.logistic(), Regularizer("l2", 1.0), _stats(3)).kind == LOGISTIC
    svm = GlmProblem(ex, SmoothLoss.hinge(), Regularizer("l2", 0.5), _stats(3))
    assert svm.kind == SVM_DUAL and svm.gamma == pytest.approx(1 / (0.5 * 9))
    assert GlmProblem(ex, SmoothLoss.logistic(), Regularizer("l2", 1.0), _stats(3)).kind == LOGISTIC_DUAL
    with pytest.raises(ValueError):
        Regularizer("elastic", 1.0)
    with pytest.raises(ValueError):
        Regularizer("l2", 0.0)
    with pytest.raises(ValueError):  # hinge needs the dual orientation
        GlmProblem(feat, SmoothLoss.hinge(), Regularizer("l2", 1.0), _stats(3))
    with pytest.raises(ValueError):  # squared loss has no dual row here
        GlmProblem(ex, SmoothLoss.squared_error(), Regularizer("l2", 1.0), _stats(3))
    with pytest.raises(ValueError):  # labels must be +-1 for logistic
        GlmProblem(LabeledDataset(m, np.array([0.5, 1, 1, 1])), SmoothLoss.logistic(),
                   Regularizer("l2", 1.0), _stats(3))
    with pytest.raises(ValueError):
        LabeledDataset(m, np.ones(5))


def test_column_matrix_validation():
    with pytest.raises(ValueError):
        ColumnMatrix(2, 2, dense=np.array([[1.0, np.nan], [0, 1]]))
    with pytest.raises(ValueError):
        ColumnMatrix(3, 1, sparse_cols=[([2, 1], [1.0, 1.0])])
    with pytest.raises(ValueError):
        ColumnMatrix(3, 1, sparse_cols=[([0, 5], [1.0, 1.0])])
    m = ColumnMatrix(3, 2, sparse_cols=[([0, 2], [1.0, 2.0]), ([1], [3.0])])
    assert m.nnz() == 3
    np.testing.assert_array_equal(m.to_dense(), [[1, 0], [0, 3], [2, 0]])


def test_reduce_replicas_order_and_copy():
    g = np.random.default_rng(0)
    base = g.standard_normal(40)
    reps = [base + g.standard_normal(40) * 0.1 for _ in range(5)]
    got = reduce_replicas(base, reps)
    exp = np.empty(40)
    for i in range(40):
        acc = 0.0
        for r in reps:
            acc += r[i] - base[i]
        exp[i] = base[i] + acc
    assert np.array_equal(got, exp)
    one = np.array([1.0, -2.0, 3.0])
    out = reduce_replicas(np.zeros(3), [one])
    assert np.array_equal(out, one) and out is not one
    with pytest.raises(ValueError):
        reduce_replicas(np.zeros(3), [])
    with pytest.raises(ValueError):
        reduce_replicas(np.zeros(3), [np.zeros(4)])


def test_shard_plan_single_and_errors(built_lib):
    sp = shard_plan(100, 8, 1, 4, seed=3)
    assert sp.store_cols is None and sorted(sp.buckets.tolist()) == list(range(13))
    assert (sp.bucket_store_col == sp.buckets * 8).all()
    with pytest.raises(ValueError, match="bucket count"):
        shard_plan(16, 8, 2, 2, seed=0)
    with pytest.raises(ValueError):
        shard_plan(100, 8, 3, 1, seed=0, world=2, rank=0)


def test_spec_validation_and_thread_split():
    from paper_1911_07722_b200 import SolverConfig
    from paper_1911_07722_b200.experiment import ExperimentSpec, node_thread_split
    base = SolverConfig()
    with pytest.raises(ValueError, match="exactly one dataset source"):
        ExperimentSpec("syscd", None, None, None, "squared", 1.0, 1, [1], [8], base, "a", "b")
    with pytest.raises(ValueError, match="nonempty"):
        ExperimentSpec("syscd", None, (10, 2), None, "squared", 1.0, 1, [], [8], base, "a", "b")
    assert node_thread_split("syscd", 8, 2) == (2, 4)
    assert node_thread_split("wild", 8, 1) == (1, 8)
    with pytest.raises(ValueError):
        node_thread_split("syscd", 6, 4)
    with pytest.raises(ValueError):
        node_thread_split("sequential", 2, 1)


# ---------------------------------------------------------------------------
# single-coordinate API (host utilities, objective.py:113-232): no device
# ---------------------------------------------------------------------------
def _host_pair(kind, d, n, seed):
    """A tiny problem with host-computed column norms (no GPU) and the same
    problem for the oracle."""
    from oracle import syscd_oracle as O
    from paper_1911_07722_b200 import (COORDINATES_ARE_EXAMPLES, COORDINATES_ARE_FEATURES,
                                       ColumnMatrix, GlmProblem, LabeledDataset, Regularizer,
                                       SmoothLoss)
    from paper_1911_07722_b200.dataset import DatasetStats
    g = np.random.default_rng(seed)
    A = g.standard_normal((d, n)).astype(np.float32)
    sq = (A.astype(np.float64) ** 2).sum(axis=0)
    stats = DatasetStats(sq, float("nan"), float(sq.max()))
    if kind in ("ridge", "lasso", "logistic"):
        y = (g.standard_normal(d) if kind != "logistic"
             else np.where(g.random(d) < 0.5, -1.0, 1.0))
        lam = 0.5 if kind != "lasso" else 0.05 * float(np.abs(A.T @ y).max())
        ds = LabeledDataset(ColumnMatrix(d, n, dense=A), y, COORDINATES_ARE_FEATURES)
        loss = SmoothLoss.logistic() if kind == "logistic" else SmoothLoss.squared_error()
        pb = GlmProblem(ds, loss, Regularizer("l1" if kind == "lasso" else "l2", lam), stats)
        ob = O.OracleProblem(O.OracleMatrix(dense=A.astype(np.float64)), y, kind, lam)
    else:
        y = np.where(g.random(n) < 0.5, -1.0, 1.0)
        lam = 1.0 / n
        ds = LabeledDataset(ColumnMatrix(d, n, dense=A), y, COORDINATES_ARE_EXAMPLES)
        loss = SmoothLoss.hinge() if kind == "svm_dual" else SmoothLoss.logistic()
        pb = GlmProblem(ds, loss, Regularizer("l2", lam), stats)
        ob = O.OracleProblem(O.OracleMatrix(dense=A.astype(np.float64) * y[None, :]),
                             np.zeros(d), kind, lam)
    return pb, ob


@pytest.mark.parametrize("kind", ["ridge", "lasso", "svm_dual", "logistic_dual", "logistic"])
def test_single_coordinate_api_matches_oracle(kind):
    """exact_coordinate_update / surrogate_coordinate_update against the
    oracle's per-coordinate steps."""
    from paper_1911_07722_b200 import (SurrogateContext, exact_coordinate_update,
                                       surrogate_coordinate_update)
    pb, ob = _host_pair(kind, 40, 12, seed=21)
    g = np.random.default_rng(3)
    alpha = g.uniform(0.05, 0.9, 12) if kind.endswith("dual") else g.standard_normal(12)
    v = ob.A.matvec(alpha)
    for j in range(12):
        got = exact_coordinate_update(pb, j, alpha[j], v)
        ref = ob.exact_delta(j, alpha[j], v)
        assert abs(got - ref) <= 1e-5 * max(1.0, abs(ref)), (j, got, ref)
    if kind == "logistic":
        return
    grad = ob.grad(v)
    a = 4.0 * ob.gamma
    ctx = SurrogateContext(grad, v, v, a, ob.gamma)
    v_thread = v + 0.01 * g.standard_normal(v.shape)
    for j in range(12):
        got = surrogate_coordinate_update(ctx, pb, j, alpha[j], v_thread)
        lin = ob.A.col_dot(j, grad) + a * ob.A.col_dot(j, v_thread - v)
        ref = ob.step(lin, a, j, alpha[j])
        assert abs(got - ref) <= 1e-5 * max(1.0, abs(ref)), (j, got, ref)
