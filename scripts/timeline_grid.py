"""Per-event timeline of the grid-wide epoch kernel (CTA 0, first partition)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SYSCD_TRACE"] = "1"  # instrumented build (per-event stamps)
import numpy as np, torch
from paper_1911_07722_b200.csrc.build import build
build()
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 3
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
torch.cuda.set_device(0)
wl = workload(cfg_id, scale=scale)
eng = _Engine(wl.problem, wl.solver, Dist())
eng.global_round(0)
buf = torch.zeros(8192 + 2 * 1024 * 160 + 1024 * 160 * 8, dtype=torch.int64, device="cuda")
L = lib(); L.syscd_debug_set_grid_timeline.argtypes = [ctypes.c_void_p]
L.syscd_debug_set_grid_timeline(buf.data_ptr())
eng.global_round(1)
torch.cuda.synchronize()
L.syscd_debug_set_grid_timeline(None)
allb = buf.cpu().numpy().astype(np.float64)
t = allb[:8192].reshape(1024, 8)
pubt = allb[8192:8192 + 1024 * 160].reshape(1024, 160)
tott = allb[8192 + 1024 * 160:8192 + 2 * 1024 * 160].reshape(1024, 160)
allc = allb[8192 + 2 * 1024 * 160:].reshape(1024, 160, 8)
t = t[100:900]
ev = np.diff(t[:, 0])
print(f"mean event {ev.mean():.0f} ns, median {np.median(ev):.0f}")
print(f"  wait x staged   {np.mean(t[:,1]-t[:,0]):7.0f}")
print(f"  partials+publish{np.mean(t[:,2]-t[:,1]):7.0f}")
print(f"  wait totals     {np.mean(t[:,3]-t[:,2]):7.0f}")
print(f"  resolve+axpy    {np.mean(t[:,4]-t[:,3]):7.0f}")
print(f"  loop overhead   {np.mean(t[1:,0]-t[:-1,4]):7.0f}")
# reducer: totals for pub r ready at t[r,5]; needed at event r+L (stamp 2)
Lk = 3
ready = t[:, 5]
need = np.roll(t[:, 2], -Lk)
print(f"  reducer interval {np.mean(np.diff(ready)):7.0f} ns; slack (need - ready) median {np.median((need-ready)[:-Lk]):7.0f}")
print(f"  publish(r) -> totals(r) latency median {np.median(ready - t[:,2]):7.0f}")

G = int((pubt[200] > 0).sum())
P = pubt[100:900, :G]; T = tott[100:900, :G]
first, last = P.min(axis=1), P.max(axis=1)
print(f"CTAs {G}: publish skew (last - first) median {np.median(last - first):.0f} ns, p90 {np.percentile(last-first, 90):.0f}")
print(f"  last publish -> totals (median over CTAs) {np.median(np.median(T, axis=1) - last):.0f} ns")
print(f"  totals spread across CTAs median {np.median(T.max(axis=1) - T.min(axis=1)):.0f} ns")
print(f"  CTA0 publish -> last publish {np.median(last - P[:, 0]):.0f} ns")
lag = P - first[:, None]
ml = np.median(lag, axis=0)
order = np.argsort(ml)[::-1]
print("  slowest CTAs (median lag ns):", [(int(c), int(ml[c])) for c in order[:8]])
print("  fastest CTAs (median lag ns):", [(int(c), int(ml[c])) for c in order[-4:]])
lastc = np.argmax(P, axis=1)
vals, cnts = np.unique(lastc, return_counts=True)
top = np.argsort(cnts)[::-1][:8]
print("  CTA most often last:", [(int(vals[i]), int(cnts[i])) for i in top])
# per-CTA event interval (publish-to-publish)
iv = np.diff(P, axis=0)
print(f"  publish interval median over CTAs {np.median(iv):.0f} ns")

# per-CTA phase breakdown over events 100..900
C = allc[100:900, :G, :]
ph = {"wait x": C[:, :, 1] - C[:, :, 0], "partials": C[:, :, 2] - C[:, :, 1],
      "wait tot": C[:, :, 3] - C[:, :, 2], "resolve": C[:, :, 4] - C[:, :, 3]}
print("per-CTA mean phases (ns): CTA  " + "  ".join(ph))
for c in list(order[:6]) + list(order[-3:]):
    print(f"  {int(c):4d} " + "  ".join(f"{np.mean(v[:, c]):8.0f}" for v in ph.values()))
print("  all  " + "  ".join(f"{np.mean(v):8.0f}" for v in ph.values()))
print("  p90 wait x over CTAs/events", np.percentile(ph["wait x"], 90), "max", ph["wait x"].max())
if os.environ.get("TL_SAVE"):
    np.savez_compressed(os.environ["TL_SAVE"], t=allb[:8192].reshape(1024, 8), pubt=pubt, tott=tott, allc=allc)
