"""Iteration histogram of the logistic-dual fast path on config 4 (experiment
build with -DSYSCD_NEWTON_HIST; SYSCD_LIB_NAME=libsyscd_b200_nh.so)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
torch.cuda.set_device(0)
wl = workload(4)
eng = _Engine(wl.problem, wl.solver, Dist())
L = lib()
L.syscd_debug_newton_hist.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 24)()
for t in range(12):
    eng.global_round(t)
    torch.cuda.synchronize()
    L.syscd_debug_newton_hist(buf)
    h = np.array(buf[:], dtype=np.int64).reshape(2, 12)
    if t in (0, 1, 2, 5, 11):
        tot = h.sum()
        print(f"epoch {t}: body its 1..8 {h[0][1:9].tolist()} noconv {h[0][9]} fallback {h[0][10]} | "
              f"tail its 1..8 {h[1][1:9].tolist()} noconv {h[1][9]} fallback {h[1][10]} | total {tot}")
