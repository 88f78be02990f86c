"""Per-chunk phase timeline of the medium-height epoch kernel (CTA 0)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SYSCD_TRACE"] = "1"  # the stamps exist only in the instrumented build
import numpy as np, torch
from paper_1911_07722_b200.csrc.build import build
build()
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 0
wl = workload(cfg_id)
eng = _Engine(wl.problem, wl.solver, Dist())
for t in range(3):
    eng.global_round(t)
buf = torch.zeros(256 * 8, dtype=torch.int64, device="cuda")
L = lib(); L.syscd_debug_set_mid_timeline.argtypes = [ctypes.c_void_p]
L.syscd_debug_set_mid_timeline(buf.data_ptr())
eng.global_round(3)
torch.cuda.synchronize()
L.syscd_debug_set_mid_timeline(None)
allb = buf.view(256, 8).cpu().numpy().astype(np.float64)
enter, started, ended = allb[255, 0], allb[255, 1], allb[255, 2]
t = allb[:128, :7]
gt = allb[128:192, :2]
gt = gt[gt[:, 0] > 0]
if len(gt):
    t0g = gt[:, 0].min()
    print("clusters (start, end) us:", [(round((a - t0g) / 1e3, 1), round((b - t0g) / 1e3, 1)) for a, b in gt])
t = t[t[:, 0] > 0] / 1.965
d = np.diff(t, axis=1)
names = ["wait staged", "Gram", "push", "totals wait", "chain", "w update"]
print(f"chunks {len(t)}; mean chunk {np.mean(t[:, 6] - t[:, 0]):.0f} ns; "
      f"setup {(started - enter) / 1.965:.0f} ns, first chunk at {(t[0, 0] * 1.965 - started) / 1.965:.0f} ns, "
      f"last chunk end -> exit {(ended - t[-1, 6] * 1.965) / 1.965:.0f} ns, total {(ended - enter) / 1.965:.0f} ns")
for i, nm in enumerate(names):
    print(f"  {nm:12s} mean {d[:, i].mean():7.0f} ns  median {np.median(d[:, i]):7.0f}")
