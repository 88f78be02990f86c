"""Timing of the metrics kernels (column norms, A x, A^T w) on a config."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import column_sq_norms

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workload(cfg_id)
pb = wl.problem
dp = pb.device()
alpha = torch.randn(dp.n_store, device="cuda", dtype=torch.float32)
alpha[torch.rand(dp.n_store, device="cuda") < 0.9] = 0  # Lasso-like sparsity

def timeit(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

gb = wl.a_bytes / 1e9
t = timeit(lambda: column_sq_norms(pb.data.matrix)); print(f"col_sq_norms {t:.3f} ms ({gb / t * 1e3:.0f} GB/s)")
t = timeit(lambda: dp.matvec(alpha)); print(f"matvec (10% nnz alpha) {t:.3f} ms")
a2 = torch.randn(dp.n_store, device="cuda", dtype=torch.float32)
t = timeit(lambda: dp.matvec(a2)); print(f"matvec (dense alpha) {t:.3f} ms ({gb / t * 1e3:.0f} GB/s)")
t = timeit(lambda: dp.objective(a2)); print(f"objective {t:.3f} ms")
t = timeit(lambda: dp.gap(a2)); print(f"gap {t:.3f} ms")
