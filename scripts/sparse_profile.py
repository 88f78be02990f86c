"""Per-phase cycle breakdown of k_sparse_epoch on config 4 (debug hook)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_07722_b200 import SolverConfig, run_syscd
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import device_problem
from paper_1911_07722_b200.objective import GlmProblem, SmoothLoss

scale = float(os.environ.get("SCALE", "1.0"))
P = int(os.environ.get("P", "512"))
pb = device_problem(4, scale, 0)
names = ["C.wait_full", "C.chain", "C.wait_next", "C.patch", "P.wait_empty", "P.writeback",
         "P.produce", "-"]
L = lib()
L.syscd_debug_set_sparse_profile.argtypes = [ctypes.c_void_p]
for name, prob in (("logistic", pb), ("hinge", GlmProblem.build(pb.data, SmoothLoss.hinge(), 1e-6))):
    buf = torch.zeros(P * 8, dtype=torch.int64, device="cuda")
    run_syscd(prob, SolverConfig(K=1, P=P, bucket_size=64, T1=1, seed=0))  # warm
    L.syscd_debug_set_sparse_profile(buf.data_ptr())
    res = run_syscd(prob, SolverConfig(K=1, P=P, bucket_size=64, T1=1, seed=0))
    L.syscd_debug_set_sparse_profile(None)
    torch.cuda.synchronize()
    ph = buf.view(P, 8).double().mean(0) / 1.965e6  # ms at 1965 MHz
    print(f"{name}: epoch {res.metrics[-1].seconds*1e3:.2f} ms; per-worker phase ms:",
          " ".join(f"{n}={v:.2f}" for n, v in zip(names, ph.tolist())), flush=True)
