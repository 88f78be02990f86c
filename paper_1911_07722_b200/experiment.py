"""Parameter sweeps on the GPU solver, reported in the reference's CSV schema.

The reference's `syscd train` command (pkg/src/syscd/cli.py:128-205) runs a
grid of (thread count, bucket size) through run_solver and writes two CSVs:
one row per epoch and one summary row per run.  This module keeps that
schema -- column names and order, row order, empty cells for missing or
non-finite values, the exit status -- so downstream tooling reads either
implementation's files (tests/test_gpu_experiment.py compares against CSVs
the reference itself wrote).  The argparse front end is out of scope
(DESIGN.md): a sweep is described by an ExperimentSpec built in Python.

Extensions: `loss="hinge"` (dual problems, with the example orientation of
the dataset) and `reg="l1"` (Lasso).
"""

from __future__ import annotations

import csv
import dataclasses
import itertools
import math
from dataclasses import dataclass

from .dataset import generate_synthetic_dense, generate_synthetic_sparse, load_libsvm
from .objective import GlmProblem, SmoothLoss
from .optimum import compute_reference_optimum
from .solvers import SolverConfig, run_solver

EXIT_OK, EXIT_USAGE, EXIT_DIVERGED = 0, 2, 3

# the reference's column layouts (cli.py:190-205)
METRIC_FIELDS = ("experiment_id", "algorithm", "threads", "epoch", "seconds", "objective",
                 "suboptimality", "rel_change", "converged", "reason")
SUMMARY_FIELDS = ("experiment_id", "algorithm", "threads", "bucket_size", "epochs",
                  "time_per_epoch", "epochs_to_tolerance", "total_time", "converged", "reason")

_LOSSES = {"squared": SmoothLoss.squared_error, "logistic": SmoothLoss.logistic,
           "hinge": SmoothLoss.hinge}


@dataclass
class ExperimentSpec:
    """One sweep: a dataset source (LIBSVM file or synthetic shape), the
    objective, the grid of thread counts x bucket sizes, the base solver
    settings and the two output paths (fields of cli.py's spec)."""

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

    def dataset(self):
        if self.libsvm_path is not None:
            return load_libsvm(self.libsvm_path)
        rows, cols = self.synthetic_shape
        if self.density is None:
            return generate_synthetic_dense(rows, cols, self.base.seed)
        return generate_synthetic_sparse(rows, cols, self.density, self.base.seed)

    def problem(self):
        if self.loss not in _LOSSES:
            raise ValueError(f"unknown loss: {self.loss}")
        return GlmProblem.build(self.dataset(), _LOSSES[self.loss](), self.lam, reg=self.reg)


def loss_from_name(name):
    if name not in _LOSSES:
        raise ValueError(f"unknown loss: {name}")
    return _LOSSES[name]()


def node_thread_split(algorithm, threads, nodes):
    """(K, P) realising `threads` workers: the flat solvers take no node
    groups; SySCD spreads them evenly over `nodes` groups."""
    if algorithm == "sequential":
        if threads != 1:
            raise ValueError("sequential solver runs on one thread")
        return 1, 1
    if algorithm == "wild":
        if nodes != 1:
            raise ValueError("wild solver is flat (K must be 1)")
        return 1, threads
    if threads < nodes or threads % nodes:
        raise ValueError(f"thread count {threads} is not divisible by {nodes} nodes")
    return nodes, threads // nodes


class _Report:
    """Accumulates the per-epoch and per-run records of a sweep."""

    def __init__(self, algorithm):
        self.algorithm = algorithm
        self.epochs = []
        self.runs = []

    def add(self, run_id, cfg, result):
        threads = cfg.K * cfg.P
        tail = result.metrics[1:]  # metrics[0] is the state before the first epoch
        status = dict(converged=result.converged, reason=result.reason or "")
        self.epochs.extend(
            dict(experiment_id=run_id, algorithm=self.algorithm, threads=threads, epoch=m.epoch,
                 seconds=m.seconds, objective=m.objective, suboptimality=m.suboptimality,
                 rel_change=m.rel_change, **status)
            for m in tail)
        elapsed = math.fsum(m.seconds for m in tail)
        self.runs.append(dict(
            experiment_id=run_id, algorithm=self.algorithm, threads=threads,
            bucket_size=cfg.resolved_bucket_size(), epochs=len(tail),
            time_per_epoch=elapsed / len(tail) if tail else "",
            epochs_to_tolerance=len(tail) if result.converged else "",
            total_time=elapsed, **status))


def _cell(value):
    """CSV cell text: None and non-finite floats become empty cells."""
    if value is None or (isinstance(value, float) and not math.isfinite(value)):
        return ""
    return value


def write_csv(path, rows, fields):
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(fields)
        out.writerows([_cell(r[f]) for f in fields] for r in rows)


def run_experiment(spec):
    """Run every (threads, bucket size) point of the sweep on the GPU and
    write both CSVs; returns (epoch rows, run rows).  A diverged run is a
    row with reason "diverged", never an exception."""
    problem = spec.problem()
    f_star = None if spec.reference == "none" else \
        compute_reference_optimum(problem, spec.reference)[1]
    report = _Report(spec.solver)
    grid = itertools.product(spec.thread_counts, spec.bucket_sizes)
    for run_id, (threads, bucket) in enumerate(grid):
        K, P = node_thread_split(spec.solver, threads, spec.nodes)
        cfg = dataclasses.replace(spec.base, algorithm=spec.solver, K=K, P=P,
                                  bucket_size=bucket, verify=spec.verify)
        report.add(run_id, cfg, run_solver(problem, cfg, f_star=f_star))
    write_csv(spec.out_path, report.epochs, METRIC_FIELDS)
    write_csv(spec.summary_path, report.runs, SUMMARY_FIELDS)
    return report.epochs, report.runs


def exit_code(summaries):
    """The train command's status (cli.py:335-342): EXIT_DIVERGED when every
    run of the sweep diverged, else EXIT_OK."""
    if summaries and all(s["reason"] == "diverged" for s in summaries):
        return EXIT_DIVERGED
    return EXIT_OK
