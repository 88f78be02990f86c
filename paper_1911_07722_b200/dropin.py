"""The drop-in stub of INTEGRATION.md as code: route the reference package's
solver entry points to this GPU implementation.

    import syscd                              # the reference (pkg/src/syscd)
    from paper_1911_07722_b200 import dropin
    undo = dropin.install(syscd)              # syscd.run_syscd etc. now run on the B200
    ...
    undo()

install() replaces run_syscd (solvers.py:337), run_sequential_scd (:181),
run_wild_parallel_scd (:214) -- and with them run_solver (:456-462), which
dispatches through the module globals -- by wrappers that convert the
reference's GlmProblem / SolverConfig to this package's, solve on the GPU
and hand back the reference's own TrainResult / EpochMetrics.  Everything
else in the reference (data loading, objectives, CLI) is untouched.
"""

from __future__ import annotations

import dataclasses

_ENTRY = ("run_syscd", "run_sequential_scd", "run_wild_parallel_scd")


def _problem(syscd, problem):
    """The reference problem as a paper_1911_07722_b200 problem (float32
    data on the GPU; labels, loss, regulariser and orientation unchanged)."""
    from . import (ColumnMatrix, GlmProblem, LabeledDataset, Regularizer, SmoothLoss)
    from .dataset import compute_stats
    m = problem.data.matrix
    if m.storage_kind == "dense":
        mat = ColumnMatrix(m.n_rows, m.n_cols, dense=m.to_dense())
    else:
        mat = ColumnMatrix(m.n_rows, m.n_cols, sparse_cols=[m.column(j) for j in range(m.n_cols)])
    ds = LabeledDataset(mat, problem.data.labels, problem.data.orientation)
    loss = SmoothLoss(problem.loss.kind, problem.loss.gamma)
    return GlmProblem(ds, loss, Regularizer(problem.reg.kind, problem.reg.lam),
                      compute_stats(mat))


def _config(cfg):
    from . import SolverConfig
    names = {f.name for f in dataclasses.fields(SolverConfig)}
    return SolverConfig(**{k: v for k, v in dataclasses.asdict(cfg).items() if k in names})


def _result(syscd, res):
    rows = [syscd.EpochMetrics(m.epoch, m.objective, m.suboptimality, m.seconds, m.updates,
                               m.rel_change) for m in res.metrics]
    return syscd.TrainResult(res.alpha, rows, res.converged, res.total_updates, res.diverged,
                             res.reason, res.alpha_snapshots)


def install(syscd):
    """Patch the reference package `syscd` (an imported module); returns a
    function that restores the original entry points.  Idempotent: a second
    call returns the first call's undo()."""
    if getattr(syscd, "_b200_dropin", None) is not None:
        return syscd._b200_dropin
    from . import solvers as ours
    saved = [(mod, name, getattr(mod, name)) for mod in (syscd, syscd.solvers) for name in _ENTRY]
    cache = {}

    def wrap(name):
        gpu_fn = getattr(ours, name)

        def entry(problem, cfg, f_star=None):
            key = id(problem)
            if key not in cache or cache[key][0] is not problem:
                cache[key] = (problem, _problem(syscd, problem))
            return _result(syscd, gpu_fn(cache[key][1], _config(cfg), f_star=f_star))

        entry.__name__ = name
        entry.__doc__ = f"{name} of the reference, solved by paper_1911_07722_b200 on the GPU"
        return entry

    for name in _ENTRY:
        fn = wrap(name)
        setattr(syscd.solvers, name, fn)
        setattr(syscd, name, fn)

    def undo():
        for mod, name, fn in saved:
            setattr(mod, name, fn)
        cache.clear()
        syscd._b200_dropin = None

    syscd._b200_dropin = undo
    return undo
