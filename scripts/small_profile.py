"""Chain-warp phase breakdown of k_small_epoch on config 1 (debug hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine

wl = workload(1)
eng = _Engine(wl.problem, wl.solver, Dist())
for t in range(2):
    eng.global_round(t)
W = eng.n_workers
buf = torch.zeros(W * 4, dtype=torch.int64, device="cuda")
L = lib()
L.syscd_debug_set_small_profile.argtypes = [ctypes.c_void_p]
L.syscd_debug_set_small_profile(buf.data_ptr())
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
eng.global_round(2)
e.record()
torch.cuda.synchronize()
L.syscd_debug_set_small_profile(None)
ph = buf.view(W, 4).double().mean(0) / 1.965e6
print(f"round {s.elapsed_time(e):.3f} ms, workers {W}; chain-warp ms:",
      " ".join(f"{n}={v:.3f}" for n, v in zip(["wait_full", "c+G", "chain", "w_update"], ph.tolist())))
