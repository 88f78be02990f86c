"""Nonzero fraction of the config-2 Lasso optimum against lambda / ||A^T y||_inf
(K=P=1 solves certified by the duality gap): the calibration behind
configs.LASSO_RATIO (BASELINE config 2: about 10% nonzero)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1911_07722_b200 import SolverConfig, run_syscd  # noqa: E402
from paper_1911_07722_b200 import configs  # noqa: E402
from paper_1911_07722_b200.objective import Regularizer  # noqa: E402

wl = configs.workload(2)
pb = wl.problem
lam_max = pb.reg.lam / configs.LASSO_RATIO
for ratio in [float(r) for r in sys.argv[1:]] or [0.02, 0.03, 0.04, 0.05, 0.06, 0.08]:
    pb.reg = Regularizer("l1", ratio * lam_max)
    pb._device = None
    cfg = SolverConfig(K=1, P=1, bucket_size=8, T1=400, metrics_every=400, compute_gap=True)
    res = run_syscd(pb, cfg)
    m = res.metrics[-1]
    print(f"ratio {ratio:.4f}: nnz {np.mean(res.alpha != 0):.4f}  F {m.objective:.6e}  "
          f"rel gap {m.gap / abs(m.objective):.2e}", flush=True)
