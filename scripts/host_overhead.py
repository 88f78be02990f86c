"""Host (Python) time per enqueued round vs GPU time per round."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 0
wl = workload(cfg_id)
cfg = wl.solver
cfg.T1 = 400
eng = _Engine(wl.problem, cfg, Dist())
for t in range(10):
    eng.global_round(t)
torch.cuda.synchronize()
n = 200
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
s.record()
for t in range(10, 10 + n):
    eng.global_round(t)
e.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"config {cfg_id}: host enqueue {1e6 * (t1 - t0) / n:.1f} us/round, "
      f"GPU {1e3 * s.elapsed_time(e) / n:.1f} us/round")

if os.environ.get("HOST_PROFILE"):
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for t in range(10 + n, 10 + 2 * n):
        eng.global_round(t)
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
