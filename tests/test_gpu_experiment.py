"""Experiment sweeps (cli.py:128-205) against CSVs written by the reference's
own run_experiment (tests/golden/experiment_runs.json): same columns, rows and
flags; objectives within the trajectory tolerance; timings not compared."""
import csv

import pytest

pytestmark = pytest.mark.gpu


def _f(x):
    return float(x) if x != "" else None


def test_sweeps_match_reference_csvs(cuda, golden, tmp_path):
    from paper_1911_07722_b200 import SolverConfig
    from paper_1911_07722_b200.experiment import ExperimentSpec, exit_code, run_experiment
    for k, case in enumerate(golden("experiment_runs.json")):
        s = case["spec"]
        spec = ExperimentSpec(
            solver=s["solver"], libsvm_path=None, synthetic_shape=tuple(s["synthetic_shape"]),
            density=s["density"], loss=s["loss"], lam=s["lam"], nodes=s["nodes"],
            thread_counts=s["thread_counts"], bucket_sizes=s["bucket_sizes"],
            base=SolverConfig(algorithm=s["solver"], **s["base"]),
            out_path=str(tmp_path / f"m{k}.csv"), summary_path=str(tmp_path / f"s{k}.csv"),
            reference=s["reference"])
        _, summaries = run_experiment(spec)
        assert exit_code(summaries) == 0
        got_m = list(csv.reader(open(spec.out_path)))
        got_s = list(csv.reader(open(spec.summary_path)))
        ref_m, ref_s = case["metrics_csv"], case["summary_csv"]
        assert got_m[0] == ref_m[0] and got_s[0] == ref_s[0]
        assert len(got_s) == len(ref_s)
        h = ref_s[0]
        for g, r in zip(got_s[1:], ref_s[1:]):
            for col in ("experiment_id", "algorithm", "threads", "bucket_size", "converged",
                        "reason"):
                assert g[h.index(col)] == r[h.index(col)], (col, g, r)
            # a tolerance stop may land one epoch apart at fp32
            assert abs(int(g[h.index("epochs")]) - int(r[h.index("epochs")])) <= 1
            assert float(g[h.index("total_time")]) > 0
        hm = ref_m[0]
        by_exp = {}
        for row in ref_m[1:]:
            by_exp.setdefault((row[0], row[hm.index("epoch")]), row)
        n_cmp = 0
        for g in got_m[1:]:
            r = by_exp.get((g[0], g[hm.index("epoch")]))
            if r is None:
                continue
            for col in ("algorithm", "threads", "converged", "reason"):
                assert g[hm.index(col)] == r[hm.index(col)]
            go, ro = float(g[hm.index("objective")]), float(r[hm.index("objective")])
            assert abs(go - ro) <= 1e-4 * abs(ro), (k, g, r)
            gs, rs = _f(g[hm.index("suboptimality")]), _f(r[hm.index("suboptimality")])
            assert (gs is None) == (rs is None)
            if rs is not None:
                assert abs(gs - rs) <= 1e-4 * abs(ro) + 1e-6 * abs(rs)
            n_cmp += 1
        assert n_cmp >= len(ref_m) - 1 - len(ref_s) + 1



def test_libsvm_file_through_the_solver(cuda, tmp_path):
    """LIBSVM text -> native parser -> CSC on the GPU -> run_syscd gives the
    same trajectory as the in-memory sparse dataset it was written from."""
    from paper_1911_07722_b200 import (GlmProblem, SmoothLoss, SolverConfig,
                                       generate_synthetic_sparse, run_syscd)
    from paper_1911_07722_b200.dataset import load_libsvm, save_libsvm
    ds = generate_synthetic_sparse(400, 48, 0.2, 7)
    path = str(tmp_path / "d.svm")
    save_libsvm(ds, path)
    ds2 = load_libsvm(path, n_features=48)
    cfg = SolverConfig(K=1, P=4, bucket_size=4, seed=2, T1=4)
    r1 = run_syscd(GlmProblem.build(ds, SmoothLoss.squared_error(), 0.5), cfg)
    r2 = run_syscd(GlmProblem.build(ds2, SmoothLoss.squared_error(), 0.5), cfg)
    # the sparse node sum uses fp32 atomics: equal up to summation order
    import numpy as np
    o1 = np.array([m.objective for m in r1.metrics])
    o2 = np.array([m.objective for m in r2.metrics])
    assert np.max(np.abs(o1 - o2) / np.abs(o1)) < 1e-6
    assert np.linalg.norm(r1.alpha - r2.alpha) / np.linalg.norm(r1.alpha) < 1e-5


def test_libsvm_examples_orientation_dual(cuda, tmp_path):
    """A LIBSVM file in the example orientation drives the SVM dual: same
    trajectory as the dataset it was written from, alpha in its box."""
    import numpy as np
    from paper_1911_07722_b200 import (COORDINATES_ARE_EXAMPLES, GlmProblem, LabeledDataset,
                                       SmoothLoss, SolverConfig, generate_synthetic_sparse,
                                       run_syscd)
    from paper_1911_07722_b200.dataset import ColumnMatrix, load_libsvm, save_libsvm
    ds = generate_synthetic_sparse(300, 24, 0.3, 3)
    path = str(tmp_path / "d.svm")
    save_libsvm(ds, path)
    ex = load_libsvm(path, n_features=24, orientation=COORDINATES_ARE_EXAMPLES)
    assert (ex.matrix.n_rows, ex.matrix.n_cols) == (24, 300)
    # the same data built in memory: columns = examples
    dense_t = ds.matrix.to_dense().T.copy()
    mem = LabeledDataset(ColumnMatrix(24, 300, dense=dense_t), ds.labels,
                         COORDINATES_ARE_EXAMPLES)
    cfg = SolverConfig(K=1, P=4, bucket_size=8, seed=1, T1=4, compute_gap=True)
    r1 = run_syscd(GlmProblem.build(ex, SmoothLoss.hinge(), 1.0 / 300), cfg)
    r2 = run_syscd(GlmProblem.build(mem, SmoothLoss.hinge(), 1.0 / 300), cfg)
    o1 = np.array([m.objective for m in r1.metrics])
    o2 = np.array([m.objective for m in r2.metrics])
    assert np.max(np.abs(o1 - o2) / np.maximum(np.abs(o2), 1e-12)) < 1e-5
    assert np.all(r1.alpha >= 0) and np.all(r1.alpha <= 1)
    assert all(m.gap >= -1e-9 for m in r1.metrics)
