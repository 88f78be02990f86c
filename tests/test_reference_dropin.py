"""The boundary proven from the reference's side: the reference package
`syscd` (installed read-only into baseline/_ref from /root/reference/pkg,
git-ignored; it travels to the GPU box with the snapshot) gets the
INTEGRATION.md dispatch stub (paper_1911_07722_b200.dropin.install), and the
behaviours its own solver tests pin (pkg/tests/test_solvers.py:57-151) are
re-checked through its public API -- syscd.run_syscd / run_sequential_scd /
run_solver -- with every solve running on the GPU.  The cases are restated
here, not copied; float tolerances are fp32-level where the reference
compares fp64 values to 1e-12."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def syscd(cuda):
    if not os.path.isdir(os.path.join(REF, "syscd")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, REF)
    try:
        import syscd as ref
    finally:
        sys.path.remove(REF)
    assert os.path.realpath(ref.__file__).startswith(os.path.realpath(REF))
    from paper_1911_07722_b200 import dropin
    ref._b200_undo = dropin.install(ref)
    yield ref
    ref._b200_undo()


def _ridge(syscd, n_rows=300, n_cols=32, lam=1.0, seed=0):
    ds = syscd.generate_synthetic_dense(n_rows, n_cols, seed)
    return syscd.GlmProblem.build(ds, syscd.SmoothLoss.squared_error(), lam)


def test_stub_routes_to_the_gpu(syscd):
    assert syscd.run_syscd.__module__ == "paper_1911_07722_b200.dropin"
    assert syscd.solvers.run_sequential_scd is syscd.run_sequential_scd
    res = syscd.run_solver(_ridge(syscd), syscd.SolverConfig(algorithm="syscd", K=2, P=2,
                                                             bucket_size=8, T1=2))
    assert isinstance(res, syscd.TrainResult)
    assert all(isinstance(m, syscd.EpochMetrics) for m in res.metrics)


def test_one_coordinate_ridge_lands_on_half(syscd):
    """A = [[1]], y = [1], lam = 1: the exact step gives alpha = 1/2."""
    ds = syscd.LabeledDataset(syscd.ColumnMatrix(1, 1, dense=np.array([[1.0]])), np.array([1.0]))
    pb = syscd.GlmProblem.build(ds, syscd.SmoothLoss.squared_error(), 1.0)
    res = syscd.run_sequential_scd(pb, syscd.SolverConfig(algorithm="sequential",
                                                         bucket_size=1, seed=0))
    assert res.converged
    assert abs(res.alpha[0] - 0.5) < 1e-6


def test_zero_epochs(syscd):
    res = syscd.run_sequential_scd(_ridge(syscd), syscd.SolverConfig(
        algorithm="sequential", max_epochs=0, seed=0))
    assert len(res.metrics) == 1 and res.metrics[0].epoch == 0
    assert res.total_updates == 0 and not res.converged
    assert np.all(res.alpha == 0.0)


def test_sequential_epoch_accounting(syscd):
    res = syscd.run_sequential_scd(_ridge(syscd), syscd.SolverConfig(
        algorithm="sequential", bucket_size=8, seed=1, T1=3))
    assert [m.updates for m in res.metrics[1:]] == [32, 32, 32]
    assert res.total_updates == 96


def test_degenerate_syscd_equals_sequential_bitwise(syscd):
    """K=P=1, one bucket, T3=1, T4=n is the sequential solver, bit for bit."""
    pb = _ridge(syscd, seed=6)
    n = pb.n_coordinates
    seq = syscd.run_sequential_scd(pb, syscd.SolverConfig(
        algorithm="sequential", bucket_size=n, seed=7, T1=4, record_alpha=True))
    deg = syscd.run_syscd(pb, syscd.SolverConfig(
        algorithm="syscd", K=1, P=1, bucket_size=n, T2=1, T3=1, T4=n, seed=7, T1=4,
        record_alpha=True))
    assert len(seq.alpha_snapshots) == len(deg.alpha_snapshots) == 4
    for a, b in zip(seq.alpha_snapshots, deg.alpha_snapshots):
        assert np.array_equal(a, b)


def test_parallel_accounting_with_verify(syscd):
    res = syscd.run_syscd(_ridge(syscd, seed=8), syscd.SolverConfig(
        algorithm="syscd", K=2, P=2, bucket_size=8, seed=8, T1=5, verify=True))
    assert all(m.updates == 32 for m in res.metrics[1:])
    assert not res.diverged


def test_parallel_descent_and_determinism(syscd):
    pb = _ridge(syscd, seed=9)
    cfg = syscd.SolverConfig(algorithm="syscd", K=2, P=2, bucket_size=8, seed=9, T1=15)
    a = syscd.run_syscd(pb, cfg)
    objs = [m.objective for m in a.metrics]
    assert all(y <= x + 1e-6 * abs(x) for x, y in zip(objs, objs[1:]))
    b = syscd.run_syscd(pb, cfg)
    assert np.array_equal(a.alpha, b.alpha)
    assert [m.objective for m in a.metrics] == [m.objective for m in b.metrics]


def test_matches_the_reference_cpu_path(syscd):
    """The same call with the stub (GPU) and without it (the reference's own
    fp64 CPU path): per-epoch objective within 1e-4 relative, alpha within
    1e-3 relative L2 (north_star), identical update counts."""
    from paper_1911_07722_b200 import dropin
    pb = _ridge(syscd, seed=3)
    cfg = syscd.SolverConfig(algorithm="syscd", K=2, P=2, bucket_size=4, seed=3, T1=6)
    gpu = syscd.run_syscd(pb, cfg)
    syscd._b200_undo()
    try:
        assert syscd.run_syscd.__module__ == "syscd.solvers"
        ref = syscd.run_syscd(pb, cfg)
    finally:
        syscd._b200_undo = dropin.install(syscd)
    g = np.array([m.objective for m in gpu.metrics])
    r = np.array([m.objective for m in ref.metrics])
    assert np.max(np.abs(g - r) / np.abs(r)) < 1e-4
    assert [m.updates for m in gpu.metrics] == [m.updates for m in ref.metrics]
    assert np.linalg.norm(gpu.alpha - ref.alpha) / np.linalg.norm(ref.alpha) < 1e-3
