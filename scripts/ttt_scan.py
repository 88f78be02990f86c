"""Relative duality gap against summed epoch time for several partition
counts P (the surrogate scale a = gamma K P slows convergence per epoch as P
grows; fewer partitions mean longer chains per epoch).  Used to choose
config 4's P by wall-clock to a target (BASELINE leaves it open).
Usage: python scripts/ttt_scan.py <config> <seconds budget per P> P1 P2 ..."""
import dataclasses
import json
import sys
import time

sys.path.insert(0, ".")
from paper_1911_07722_b200 import run_syscd  # noqa: E402
from paper_1911_07722_b200.configs import workload  # noqa: E402

cfg_id = int(sys.argv[1])
budget = float(sys.argv[2])
Ps = [int(x) for x in sys.argv[3:]]
wl = workload(cfg_id)
pb = wl.problem
out = {}
for P in Ps:
    # epochs per metrics row chosen so the rows are ~1/20 of the budget
    cfg = dataclasses.replace(wl.solver, P=P, T1=2, metrics_every=1, compute_gap=False)
    t0 = time.perf_counter()
    r = run_syscd(pb, cfg)
    ep = max(1e-4, sum(m.seconds for m in r.metrics[1:]) / 2)
    epochs = max(2, int(budget / ep))
    every = max(1, epochs // 20)
    cfg = dataclasses.replace(wl.solver, P=P, T1=epochs, metrics_every=every, compute_gap=True)
    r = run_syscd(pb, cfg)
    rows, t = [], 0.0
    for m in r.metrics[1:]:
        t += m.seconds * every
        primal = m.gap - m.objective
        rows.append((m.epoch, round(t, 4), m.gap / abs(primal)))
    out[P] = rows
    print(f"P={P}: epoch {ep * 1e3:.2f} ms; " + " ".join(f"[{e} {s:.3f}s {g:.2e}]" for e, s, g in rows[::max(1, len(rows) // 8)]) + f" last {rows[-1]}", flush=True)
json.dump(out, open(f"gpurun_out/ttt_scan_cfg{cfg_id}.json", "w"))
