"""Golden CSVs of the REFERENCE's run_experiment (cli.py:128-205) on small
sweeps (timings are not compared; every other cell is).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_experiment_golden.py
"""

from __future__ import annotations

import csv
import json
import os
import sys
import tempfile

sys.dont_write_bytecode = True
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from syscd import cli  # noqa: E402
from syscd.solvers import SolverConfig  # noqa: E402

SPECS = [
    dict(solver="syscd", synthetic_shape=(300, 24), density=None, loss="squared", lam=1.0,
         nodes=1, thread_counts=[1, 2, 4], bucket_sizes=[4, 6], base=dict(seed=3, max_epochs=6),
         reference="closed-form"),
    dict(solver="syscd", synthetic_shape=(200, 16), density=None, loss="logistic", lam=0.5,
         nodes=2, thread_counts=[2, 4], bucket_sizes=[4], base=dict(seed=1, max_epochs=4, tolerance=1e-3),
         reference="none"),
    dict(solver="sequential", synthetic_shape=(250, 20), density=None, loss="squared", lam=0.7,
         nodes=1, thread_counts=[1], bucket_sizes=[5], base=dict(seed=2, max_epochs=200,
                                                                 tolerance=1e-4),
         reference="closed-form"),
    dict(solver="wild", synthetic_shape=(250, 20), density=None, loss="squared", lam=0.7,
         nodes=1, thread_counts=[1], bucket_sizes=[8], base=dict(seed=2, T1=3),
         reference="none"),
]


def main():
    out = []
    with tempfile.TemporaryDirectory() as td:
        for k, s in enumerate(SPECS):
            base = SolverConfig(algorithm=s["solver"], **s["base"])
            spec = cli.ExperimentSpec(
                solver=s["solver"], libsvm_path=None, synthetic_shape=s["synthetic_shape"],
                density=s["density"], loss=s["loss"], lam=s["lam"], nodes=s["nodes"],
                thread_counts=s["thread_counts"], bucket_sizes=s["bucket_sizes"], base=base,
                out_path=os.path.join(td, f"m{k}.csv"), summary_path=os.path.join(td, f"s{k}.csv"),
                reference=s["reference"])
            cli.run_experiment(spec)
            rows = list(csv.reader(open(spec.out_path)))
            summ = list(csv.reader(open(spec.summary_path)))
            out.append({"spec": s, "metrics_csv": rows, "summary_csv": summ})
    with open(os.path.join(HERE, "experiment_runs.json"), "w") as fh:
        json.dump(out, fh)
    print(f"wrote {len(out)} sweeps")


if __name__ == "__main__":
    main()
