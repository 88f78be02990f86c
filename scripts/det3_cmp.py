"""Run round 0 of config 3 on fresh engines and compare per-event (delta, S total)
of CTA 0 across repetitions (DCHK build: SYSCD_LIB_NAME=libsyscd_b200_dchk.so)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes
from paper_1911_07722_b200._lib import lib
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist
from paper_1911_07722_b200.solvers import _Engine
wl = workload(3)
OFF = 8192 + 2 * 1024 * 160 + 1024 * 160 * 8
buf = torch.zeros(OFF + 8192 * 160 + 8192 * 160 * 4 + 8192 * 160 * 2, dtype=torch.int64, device="cuda")
L = lib(); L.syscd_debug_set_grid_timeline.argtypes = [ctypes.c_void_p]
ref = None
for rep in range(int(os.environ.get("REPS", "6"))):
    eng = _Engine(wl.problem, wl.solver, Dist())
    buf.zero_()
    L.syscd_debug_set_grid_timeline(buf.data_ptr())
    eng.global_round(0)
    torch.cuda.synchronize()
    L.syscd_debug_set_grid_timeline(None)
    hb = buf.cpu().numpy()
    dl = hb[OFF:OFF + 8192 * 160].reshape(8192, 160)[:8000, :142]
    pp = hb[OFF + 8192 * 160:OFF + 8192 * 160 * 5].reshape(8192, 160, 4)[:8000, :142, :]
    ck = hb[OFF + 8192 * 160 * 5:].reshape(8192, 160, 2)[:8000, :142, :]
    dis = np.where((dl != dl[:, :1]).any(axis=1))[0]
    if ref is None:
        ref = dl[:, 0].copy(); pref = pp.copy(); ref_dl = dl.copy(); cref = ck.copy()
        print(f"rep 0: CTA disagreement events {len(dis)}", flush=True)
        continue
    diff = np.where(dl[:, 0] != ref)[0]
    msg = f"rep {rep}: CTA disagreement events {len(dis)}; events differing from rep 0: {len(diff)}"
    if len(diff):
        e = diff[0]
        f = lambda v: (np.uint32(v >> 32).view(np.float32), np.uint32(v & 0xffffffff).view(np.float32))
        msg += f"; first {e}: (delta, S) rep0 {f(ref[e])} now {f(dl[e, 0])}; prev event same: {dl[e-1,0]==ref[e-1]}"
    pd = np.argwhere(pp != pref)
    if len(pd):
        # expected partial (fp64 on the device) of the first differing (event, CTA)
        e, c = int(pd[0][0]), int(pd[0][1])
        seq, _ = eng.round_tables(0)
        js = seq[:e + 1].long()
        At = wl.problem.data.matrix._dev_dense
        y = torch.as_tensor(wl.problem.data.labels, device="cuda")
        rows = slice(c * 7072, min((c + 1) * 7072, At.shape[1]))
        for name, dd in (("rep0", ref_dl), ("now", dl)):
            dlt = torch.tensor([np.uint32(v >> 32).view(np.float32) for v in dd[:e + 1, 0]],
                               dtype=torch.float64, device="cuda")
            w = -y[rows].double()
            for cc in range(0, e - 3):
                w += dlt[cc] * At[js[cc], rows].double()
            print(f"   expected partial {name}-deltas: {float(At[js[e], rows].double() @ w):.4f}")
    if len(pd):
        e, c, k = pd[0]
        same_e = pd[pd[:, 0] == e]
        fv = lambda v: np.uint32(v).view(np.float32)
        msg += (f"\n   x checksum same {ck[e, c, 0] == cref[e, c, 0]}, w checksum same {ck[e, c, 1] == cref[e, c, 1]}"
                f"; first x-checksum diff anywhere: {np.argwhere(ck[:, :, 0] != cref[:, :, 0])[:2].tolist()}"
                f"; first w-checksum diff: {np.argwhere(ck[:, :, 1] != cref[:, :, 1])[:2].tolist()}")
        msg += (f"\n   first partial diff: event {e} CTA {c} comp {k}: {fv(pref[e,c,k])} vs {fv(pp[e,c,k])}; "
                f"{len(same_e)} (cta,comp) differ at that event: {same_e[:6, 1:].tolist()}")
    print(msg, flush=True)
