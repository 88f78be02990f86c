"""Ad-hoc GPU parity check across configs (small scale) vs the oracle."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import syscd_oracle as O
from paper_1911_07722_b200 import SolverConfig, run_syscd
from paper_1911_07722_b200.configs import host_arrays, host_problem

def oracle_for(cfg_id, scale):
    kind, A, y, lam = host_arrays(cfg_id, scale, 0)
    if kind == 'logistic_dual':
        cp, ri, va = A
        ylab = y
        vals = va.astype(np.float64) * np.repeat(ylab, np.diff(cp))
        d = int(ri.max()) + 1
        from paper_1911_07722_b200.configs import _dims
        d, n = _dims(cfg_id, scale)
        M = O.OracleMatrix(csc=(cp, ri, vals), shape=(d, n))
        return O.OracleProblem(M, np.zeros(d), kind, lam)
    A64 = A.astype(np.float64)
    if kind == 'svm_dual':
        A64 = A64 * y[None, :]
        return O.OracleProblem(O.OracleMatrix(dense=A64), np.zeros(A.shape[0]), kind, lam)
    return O.OracleProblem(O.OracleMatrix(dense=A64), y, kind, lam)

cases = [(0, 0.05, dict(K=1,P=4,bucket_size=4,T1=6)), (0, 0.05, dict(K=2,P=2,bucket_size=4,T1=6)),
         (0, 1.0, dict(K=1,P=4,bucket_size=16,T1=4)),
         (1, 0.0005, dict(K=1,P=8,bucket_size=4,T1=4)), (2, 0.01, dict(K=1,P=4,bucket_size=2,T1=5)),
         (0, 0.05, dict(K=1,P=1,bucket_size=8,T1=4)), (0, 0.05, dict(K=1,P=2,bucket_size=4,T1=4,T2=2)),
         (0, 0.05, dict(K=1,P=2,bucket_size=4,T1=4,sampling='iid',T3=2,T4=3)),
         (4, 0.0002, dict(K=1,P=4,bucket_size=8,T1=4))]
if len(sys.argv) > 1:
    cases = [cases[int(i)] for i in sys.argv[1:]]
for cfg_id, scale, kw in cases:
    pb = host_problem(cfg_id, scale, 0)
    cfg = SolverConfig(seed=0, compute_gap=True, **kw)
    t0 = time.time(); res = run_syscd(pb, cfg); t1 = time.time()
    ob = oracle_for(cfg_id, scale)
    okw = {k: v for k, v in kw.items()}
    ores = O.run_syscd(ob, O.OracleConfig(seed=0, with_gap=True, **okw))
    got = np.array([m.objective for m in res.metrics]); ref = np.array([r.objective for r in ores.rows])
    gg = np.array([m.gap for m in res.metrics]); gr = np.array([r.gap for r in ores.rows])
    rel = np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30))
    arel = np.linalg.norm(res.alpha - ores.alpha) / max(np.linalg.norm(ores.alpha), 1e-30)
    print(f"cfg{cfg_id} s={scale} {kw}: obj rel {rel:.2e}  alpha rel {arel:.2e}  gpu {t1-t0:.2f}s  upd {[m.updates for m in res.metrics]} vs {[r.updates for r in ores.rows]}")
    print("   obj gpu", np.array2string(got[:4], precision=8), " ref", np.array2string(ref[:4], precision=8))
    print("   gap gpu", np.array2string(gg[:4], precision=5), " ref", np.array2string(gr[:4], precision=5))
    print("   epoch secs", [round(m.seconds*1e3,3) for m in res.metrics[1:4]], "ms")
