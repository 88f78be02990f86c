"""Replay the GPU logistic-dual Newton (common.cuh) in numpy on config-4 data."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_07722_b200.configs import workload
from paper_1911_07722_b200.device import Dist, _rmatvec_raw
from paper_1911_07722_b200.solvers import _Engine
torch.cuda.set_device(0)
wl = workload(4, scale=float(sys.argv[1]) if len(sys.argv) > 1 else 0.1)
eng = _Engine(wl.problem, wl.solver, Dist())
for t in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    eng.global_round(t)
torch.cuda.synchronize()
dp = eng.dp
lin = torch.empty(dp.n_store, dtype=torch.float64, device="cuda")
_rmatvec_raw(dp.mdev, dp.d, eng.u.double(), lin)
lin = lin.cpu().numpy(); alpha = eng.alpha.double().cpu().numpy(); q = dp.sq.double().cpu().numpy()
n = dp.n_coords; aq = eng.a * q
def sig(s):
    e = np.exp(-np.abs(s)); r = 1 / (1 + e); return np.where(s >= 0, r, e * r)
def run(start_kind, clamp):
    lo = -n * (lin + aq * (1 - alpha)) - 1; hi = n * (aq * alpha - lin) + 1
    if start_kind == "logit_alpha":
        s = np.where((alpha > 0) & (alpha < 1), np.log(np.clip(alpha, 1e-300, 1)) - np.log1p(-np.clip(alpha, 0, 1 - 1e-16)), 0.0)
        h0 = lin + aq * (0.5 - alpha)
        st0 = -n * (lin - aq * alpha); st1 = -n * (lin + aq * (1 - alpha))
        s = np.where((h0 > 0) & (st0 < -30), st0, s); s = np.where((h0 < 0) & (st1 > 30), st1, s)
    else:
        r0 = alpha - lin / aq
        ok = (r0 > 1e-30) & (r0 < 1 - 1e-16)
        s = np.where(ok, np.log(np.clip(r0, 1e-300, 1)) - np.log1p(-np.clip(r0, 0, 1 - 1e-16)), 0.0)
        r1 = r0 - s / n / aq
        ok1 = ok & (r1 > 1e-30) & (r1 < 1 - 1e-16)
        s = np.where(ok1, np.log(np.clip(r1, 1e-300, 1)) - np.log1p(-np.clip(r1, 0, 1 - 1e-16)), s)
        s = np.where(~ok & (r0 <= 1e-30), -n * (lin - aq * alpha), s)
        s = np.where(~ok & (r0 > 1e-30), -n * (lin + aq * (1 - alpha)), s)
    s = np.clip(s, lo, hi)
    active = np.ones_like(s, dtype=bool); its = np.zeros(s.size, int); bis = np.zeros(s.size, int)
    for it in range(100):
        t = sig(s); h = lin + aq * (t - alpha) + s / n
        hi = np.where(active & (h > 0), s, hi); lo = np.where(active & (h < 0), s, lo)
        done0 = h == 0
        dh = aq * t * (1 - t) + 1 / n
        step = -h / dh
        if clamp: step = np.where(np.abs(s) < 60, np.clip(step, -8, 8), step)
        ns = s + step
        bad = ~((lo < ns) & (ns < hi)); ns = np.where(bad, 0.5 * (lo + hi), ns)
        bis += (active & bad)
        step = ns - s; s = np.where(active, ns, s); its += active
        active &= ~done0 & ~(np.abs(step) <= 1e-9 * np.maximum(1, np.abs(s)))
        if not active.any(): break
    return its, bis, s
print("n", n, "a", eng.a, "lin pct", np.percentile(lin, [1, 25, 50, 75, 99]))
print("aq pct", np.percentile(aq, [1, 50, 99]), "alpha pct", np.percentile(alpha, [1, 25, 50, 75, 99]))
for kind in ("logit_alpha", "fixed_point"):
    for clamp in (False, True):
        its, bis, sroot = run(kind, clamp)
        print(f"{kind:12s} clamp={clamp}: iterations mean {its.mean():.2f} p50/p90/p99 {np.percentile(its, [50, 90, 99])} bisections {bis.mean():.2f}")
print("root s pct", np.percentile(sroot, [1, 25, 50, 75, 99]))
