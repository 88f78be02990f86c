"""Which CTAs disagree, and from which event (trace build: per-CTA delta and totals)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if not os.environ.get("SYSCD_LIB_NAME"):
    os.environ["SYSCD_TRACE"] = "1"
import numpy as np, torch, ctypes
from paper_1911_07722_b200.csrc.build import build
if not os.environ.get("SYSCD_LIB_NAME"):
    build()
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
wl = workload(3)
eng = _Engine(wl.problem, wl.solver, Dist())
OFF = 8192 + 2 * 1024 * 160 + 1024 * 160 * 8
buf = torch.zeros(OFF + 8192 * 160, dtype=torch.int64, device="cuda")
L = lib(); L.syscd_debug_set_grid_timeline.argtypes = [ctypes.c_void_p]
for rnd in range(int(os.environ.get('ROUNDS', '3'))):
    buf.zero_()
    L.syscd_debug_set_grid_timeline(buf.data_ptr())
    eng.global_round(rnd)
    torch.cuda.synchronize()
    L.syscd_debug_set_grid_timeline(None)
    hb = buf.cpu().numpy()
    allc = hb[8192 + 2 * 1024 * 160:OFF].reshape(1024, 160, 8)[:, :142, :]
    dl = hb[OFF:].reshape(8192, 160)[:8000, :142]
    badall = np.where((dl != dl[:, :1]).any(axis=1))[0]
    print(f"round {rnd}: all events: {len(badall)} with CTA disagreement (delta|t0); first {badall[:8]}")
    if len(badall):
        e = badall[0]
        vals, cnt = np.unique(dl[e], return_counts=True)
        maj = vals[np.argmax(cnt)]
        print("   minority CTAs", [int(c) for c in np.where(dl[e] != maj)[0][:12]],
              "t0 maj", np.uint32(maj & 0xffffffff).view(np.float32),
              "t0 min", [np.uint32(v & 0xffffffff).view(np.float32) for v in dl[e][dl[e] != maj][:3]])
    for k, name in ((5, "delta|t0"), (6, "t1|t2"), (7, "w0|t3")):
        col = allc[:, :, k]
        bad = np.where((col != col[:, :1]).any(axis=1))[0]
        bad = bad[bad >= 3]
        if k == 7:  # w0 differs per CTA by design: compare the t3 half only
            lo = col & 0xffffffff
            bad = np.where((lo != lo[:, :1]).any(axis=1))[0]; bad = bad[bad >= 3]
        print(f"round {rnd} {name}: {len(bad)} events with CTA disagreement; first {bad[:5]}")
        if len(bad) and k in (5, 6):
            e = bad[0]
            vals, cnt = np.unique(col[e], return_counts=True)
            print("   distinct values", len(vals), "counts", cnt[:6], "CTAs with minority:",
                  [int(c) for c in np.where(col[e] != vals[np.argmax(cnt)])[0][:10]])
