"""Per-partition timeline of the partition-Gram epoch (config 2): the trace
build (-DSYSCD_PG_TRACE) stamps, per partition and CTA, P1 start (0), P1
published (1), stage-A total published (2), stage-B totals gathered (3),
deltas handed over (4) and P2 start (5).
Usage (GPU box): SYSCD_LIB_NAME=libsyscd_b200_pgt.so python scripts/pg_timeline.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
torch.cuda.set_device(0)
wl = workload(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
eng = _Engine(wl.problem, wl.solver, Dist())
eng.global_round(0)
P, G = eng.n_parts_local, 148
buf = torch.zeros(P * G * 8, dtype=torch.int64, device="cuda")
L = lib(); L.syscd_debug_set_pgram_timeline.argtypes = [ctypes.c_void_p]
L.syscd_debug_set_pgram_timeline(buf.data_ptr())
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); eng.global_round(1); e.record()
torch.cuda.synchronize()
L.syscd_debug_set_pgram_timeline(None)
print(f"round {s.elapsed_time(e):.3f} ms (trace build)")
t = buf.cpu().numpy().reshape(P, G, 8).astype(np.float64)
t0 = t[:, :, 0][t[:, :, 0] > 0].min()
t = np.where(t > 0, t - t0, np.nan) / 1e3  # us
med = lambda a, ax: np.nanmedian(a, axis=ax)
p1s, p1e = t[:, :, 0], t[:, :, 1]
print("P1 duration (publish - start), median over CTAs, per partition (us):", np.round(med(p1e - p1s, 1)[:12], 2))
last_pub = np.nanmax(p1e, axis=1)
first_pub = np.nanmin(p1e, axis=1)
print("publish skew (last - first) median us:", round(float(np.nanmedian(last_pub - first_pub)), 2))
sa_last = np.nanmax(t[:, :, 2], axis=1)
print("last publish -> last stage-A total (us): median", round(float(np.nanmedian(sa_last - last_pub)), 2))
print("last stage-A -> stage-B done (median CTA) us:", round(float(np.nanmedian(med(t[:, :, 3], 1) - sa_last)), 2))
print("stage-B -> deltas (chain) us:", round(float(np.nanmedian(med(t[:, :, 4] - t[:, :, 3], 1))), 2))
print("deltas -> P2 start us:", round(float(np.nanmedian(med(t[:, :, 5] - t[:, :, 4], 1))), 2))
print("P1 start interval between partitions (median CTA) us:", np.round(np.diff(med(p1s, 1))[:16], 2))
print("partition P1 start (us) every 10:", np.round(med(p1s, 1)[::10], 1))
print("deltas ready (us) every 10:", np.round(med(t[:, :, 4], 1)[::10], 1))
