"""Publication skew of the grid-wide epoch kernel without CTA-0 stamps:
the light trace build (-DSYSCD_TRACE -DSYSCD_TRACE_LIGHT) records, for every
CTA, only when it publishes each event's partials and when its reducer hands
over each event's totals (two stores per CTA per event).
Usage (GPU box): SYSCD_LIB_NAME=libsyscd_b200_tl.so python scripts/grid_skew.py"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
torch.cuda.set_device(0)
wl = workload(3)
eng = _Engine(wl.problem, wl.solver, Dist())
eng.global_round(0)
buf = torch.zeros(8192 + 2 * 1024 * 160 + 1024 * 160 * 8, dtype=torch.int64, device="cuda")
L = lib(); L.syscd_debug_set_grid_timeline.argtypes = [ctypes.c_void_p]
L.syscd_debug_set_grid_timeline(buf.data_ptr())
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); eng.global_round(1); e.record()
torch.cuda.synchronize()
L.syscd_debug_set_grid_timeline(None)
print(f"epoch {s.elapsed_time(e):.3f} ms (light trace)")
allb = buf.cpu().numpy().astype(np.float64)
pubt = allb[8192:8192 + 1024 * 160].reshape(1024, 160)
tott = allb[8192 + 1024 * 160:8192 + 2 * 1024 * 160].reshape(1024, 160)
G = int((pubt[200] > 0).sum())
P = pubt[100:1000, :G]; T = tott[100:1000, :G]
first, last = P.min(axis=1), P.max(axis=1)
ev = np.diff(np.median(P, axis=1))
print(f"CTAs {G}; event interval median {np.median(ev):.0f} ns mean {ev.mean():.0f}")
print(f"publish skew (last - first) median {np.median(last - first):.0f} p90 {np.percentile(last - first, 90):.0f} ns")
print(f"last publish -> totals handed over (median over CTAs): {np.median(np.median(T, axis=1) - last):.0f} ns")
lag = P - np.median(P, axis=1)[:, None]
ml = np.median(lag, axis=0)
order = np.argsort(ml)[::-1]
print("slowest CTAs (median lag vs median CTA, ns):", [(int(c), int(ml[c])) for c in order[:10]])
print("fastest CTAs:", [(int(c), int(ml[c])) for c in order[-5:]])
lastc = np.argmax(P, axis=1)
vals, cnts = np.unique(lastc, return_counts=True)
top = np.argsort(cnts)[::-1][:10]
print("CTA most often last:", [(int(vals[i]), int(cnts[i])) for i in top])
np.savez_compressed("gpurun_out/grid_skew.npz", pubt=pubt, tott=tott)
smid = allb[8192 + 2 * 1024 * 160:8192 + 2 * 1024 * 160 + G].astype(int)
print("CTA -> SM:", smid.tolist())
print("slowest CTAs' SMs:", [(int(c), int(smid[c]), int(ml[c])) for c in order[:16]])
print("lag by SM id (sorted by SM):", [(int(smid[c]), int(ml[c])) for c in np.argsort(smid)])
np.savez_compressed("gpurun_out/grid_skew_sm.npz", smid=smid, lag=ml)
