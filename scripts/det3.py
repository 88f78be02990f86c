"""Config-3 determinism and replica-consistency probe (2 epochs, verify off)."""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_07722_b200 import run_syscd
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = workload(cfg_id)
outs = []
for rep in range(int(os.environ.get("REPS", "3"))):
    cfg = dataclasses.replace(wl.solver, T1=2)
    eng = _Engine(wl.problem, cfg, Dist())
    for t in range(2):
        eng.global_round(t)
    torch.cuda.synchronize()
    vv = eng.dp.matvec(eng.alpha)
    err = float((vv - eng.v).abs().max()); scale = float(vv.abs().max())
    outs.append(eng.alpha.clone())
    print(f"rep {rep}: max|Aa - v| {err:.3e}  scale {scale:.3e}  rel {err/scale:.2e}  "
          f"alpha==rep0 {bool(torch.equal(outs[0], outs[-1]))}  "
          f"max|da| {float((outs[0]-outs[-1]).abs().max()):.3e}", flush=True)
