"""Per-step phase timeline of the dense epoch kernel (CTA 0)."""
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
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
torch.cuda.set_device(0)
wl = workload(cfg_id)
eng = _Engine(wl.problem, wl.solver, Dist())
for t in range(3):
    eng.global_round(t)
buf = torch.zeros(16384, dtype=torch.int64, device="cuda")
L = lib(); L.syscd_debug_set_timeline.argtypes = [ctypes.c_void_p]
L.syscd_debug_set_timeline(buf.data_ptr())
eng.global_round(3)
torch.cuda.synchronize()
L.syscd_debug_set_timeline(None)
raw = buf.cpu().numpy().astype(np.float64)
t = raw[:3072].reshape(512, 6)
fl = raw[3072:7168].reshape(512, 8)
pu = raw[7168:7168 + 4096].reshape(512, 8)
t = t[t[:, 0] > 0] / 1.965  # SM cycles -> ns at the 1965 MHz boost clock
d = np.diff(t, axis=1)
step = np.diff(t[:, 0])
names = ["dot(wait+pass)", "cta_reduce+push", "exchange_wait", "step", "axpy(+release)"]
print(f"steps recorded {len(t)}; mean step {step.mean():.0f} ns (median {np.median(step):.0f})")
for i, nm in enumerate(names):
    print(f"  {nm:18s} mean {d[:, i].mean():7.0f} ns  median {np.median(d[:, i]):7.0f}  p90 {np.percentile(d[:, i], 90):7.0f}")
tail = t[1:, 0] - t[:-1, 5]
print(f"  {'flush/loop':18s} mean {tail.mean():7.0f} ns  median {np.median(tail):7.0f}  max {tail.max():7.0f}")
fi = np.nonzero(fl[:len(t), 0] > 0)[0]
if len(fi):
    base = t[fi, 5] * 1.965
    for c in range(6):
        print(f"  flush chunk {c} ready at +{((fl[fi, c] - base) / 1.965).mean():.0f} ns")
    print(f"  flush done at +{((fl[fi, 7] - base) / 1.965).mean():.0f} ns ({len(fi)} flushes)")
    for c in range(6):
        print(f"  u chunk {c} wait begins at +{((pu[fi, c] - base) / 1.965).mean():.0f} ns")

# per-CTA kernel spans (trace build): entry, work done, after the final cluster sync, columns
sp = buf.cpu().numpy()[12288:12288 + 4 * 160].reshape(160, 4).astype(np.float64)
sp = sp[sp[:, 0] > 0]
t0 = sp[:, 0].min()
print(f"CTAs {len(sp)}: entry spread {sp[:,0].max()-t0:.0f} ns; work end min/median/max "
      f"{sp[:,1].min()-t0:.0f}/{np.median(sp[:,1])-t0:.0f}/{sp[:,1].max()-t0:.0f} ns; exit max {sp[:,2].max()-t0:.0f}")
cols = sp[:, 3].astype(np.int64) & 0xffffffff
smid = sp[:, 3].astype(np.int64) >> 32
C = 16
for g in range(len(sp) // C):
    blk = slice(g * C, (g + 1) * C)
    print(f"  cluster {g}: {int(cols[g * C])} columns, work end {sp[blk, 1].max() - t0:.0f} ns "
          f"({(sp[blk, 1].max() - t0) / cols[g * C]:.0f} ns/column), SMs {sorted(int(x) for x in smid[blk])[:3]}..{int(smid[blk].max())}")
