"""Experiment sweeps with the reference's CSV schema (mirror of
pkg/src/syscd/cli.py:26-205, the library half of the `syscd train` command).

run_experiment(spec) loads or generates the dataset, computes F* when asked,
sweeps thread counts x bucket sizes through run_solver on the GPU and writes
the per-epoch metrics CSV and the summary CSV with the reference's columns,
row order and formatting (non-finite floats and None as empty cells).  The
argparse front end itself is out of scope; a spec is built in
Python.  Extension: `loss` also accepts "hinge" (dual problems) and `reg`
selects "l1" (Lasso) -- the reference's names keep their meaning.
"""

from __future__ import annotations

import csv
import dataclasses
import math
from dataclasses import dataclass

from .dataset import generate_synthetic_dense, generate_synthetic_sparse, load_libsvm
from .objective import GlmProblem, SmoothLoss
from .optimum import compute_reference_optimum
from .solvers import SolverConfig, run_solver

EXIT_OK = 0
EXIT_USAGE = 2
EXIT_DIVERGED = 3

METRIC_FIELDS = ["experiment_id", "algorithm", "threads", "epoch", "seconds", "objective",
                 "suboptimality", "rel_change", "converged", "reason"]
SUMMARY_FIELDS = ["experiment_id", "algorithm", "threads", "bucket_size", "epochs",
                  "time_per_epoch", "epochs_to_tolerance", "total_time", "converged", "reason"]


@dataclass
class ExperimentSpec:
    """cli.py:26-49."""

    solver: str
    libsvm_path: str | None
    synthetic_shape: tuple | None  # (n_examples, n_features)
    density: float | None
    loss: str
    lam: float
    nodes: int
    thread_counts: list
    bucket_sizes: list
    base: SolverConfig
    out_path: str
    summary_path: str
    verify: bool = False
    reference: str = "closed-form"  # closed-form | run | none
    reg: str = "l2"

    def __post_init__(self):
        if (self.libsvm_path is None) == (self.synthetic_shape is None):
            raise ValueError("exactly one dataset source must be given")
        if not self.thread_counts or not self.bucket_sizes:
            raise ValueError("sweep lists must be nonempty")


def loss_from_name(name):
    if name == "squared":
        return SmoothLoss.squared_error()
    if name == "logistic":
        return SmoothLoss.logistic()
    if name == "hinge":
        return SmoothLoss.hinge()
    raise ValueError(f"unknown loss: {name}")


def load_spec_dataset(spec):
    """cli.py:65-71."""
    if spec.libsvm_path is not None:
        return load_libsvm(spec.libsvm_path)
    n_ex, n_feat = spec.synthetic_shape
    if spec.density is not None:
        return generate_synthetic_sparse(n_ex, n_feat, spec.density, spec.base.seed)
    return generate_synthetic_dense(n_ex, n_feat, spec.base.seed)


def split_threads(solver, total, nodes):
    """(K, P) for a total thread count (cli.py:114-125)."""
    if solver == "sequential":
        if total != 1:
            raise ValueError("sequential solver runs on one thread")
        return 1, 1
    if solver == "wild":
        if nodes != 1:
            raise ValueError("wild solver is flat (K must be 1)")
        return 1, total
    if total % nodes != 0 or total < nodes:
        raise ValueError(f"thread count {total} is not divisible by {nodes} nodes")
    return nodes, total // nodes


def run_experiment(spec):
    """Execute the sweep and write the two CSVs (cli.py:128-187).

    Returns (metric_rows, summary_rows).  Divergence is a row with
    converged=False and reason="diverged", never an exception.
    """
    dataset = load_spec_dataset(spec)
    problem = GlmProblem.build(dataset, loss_from_name(spec.loss), spec.lam, reg=spec.reg)
    f_star = None
    if spec.reference != "none":
        _, f_star = compute_reference_optimum(problem, spec.reference)
    rows, summaries = [], []
    exp_id = 0
    for threads in spec.thread_counts:
        for bucket in spec.bucket_sizes:
            K, P = split_threads(spec.solver, threads, spec.nodes)
            cfg = dataclasses.replace(spec.base, algorithm=spec.solver, K=K, P=P,
                                      bucket_size=bucket, verify=spec.verify)
            result = run_solver(problem, cfg, f_star=f_star)
            epochs = result.metrics[1:]  # row 0 is the initial state
            for em in epochs:
                rows.append({
                    "experiment_id": exp_id, "algorithm": spec.solver, "threads": K * P,
                    "epoch": em.epoch, "seconds": em.seconds, "objective": em.objective,
                    "suboptimality": em.suboptimality, "rel_change": em.rel_change,
                    "converged": result.converged, "reason": result.reason or "",
                })
            total_time = sum(em.seconds for em in epochs)
            summaries.append({
                "experiment_id": exp_id, "algorithm": spec.solver, "threads": K * P,
                "bucket_size": cfg.resolved_bucket_size(), "epochs": len(epochs),
                "time_per_epoch": total_time / len(epochs) if epochs else "",
                "epochs_to_tolerance": len(epochs) if result.converged else "",
                "total_time": total_time, "converged": result.converged,
                "reason": result.reason or "",
            })
            exp_id += 1
    write_csv(spec.out_path, rows, METRIC_FIELDS)
    write_csv(spec.summary_path, summaries, SUMMARY_FIELDS)
    return rows, summaries


def write_csv(path, rows, fields):
    """cli.py:190-205: non-finite floats and None become empty cells."""
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=fields)
        w.writeheader()
        for row in rows:
            out = {}
            for key in fields:
                val = row[key]
                if isinstance(val, float) and not math.isfinite(val):
                    val = ""
                if val is None:
                    val = ""
                out[key] = val
            w.writerow(out)


def exit_code(summaries):
    """The `train` command's exit status (cli.py:335-342): 3 when every run
    of the sweep diverged, else 0."""
    if summaries and all(s["reason"] == "diverged" for s in summaries):
        return EXIT_DIVERGED
    return EXIT_OK
