"""Kernel-level GPU checks: device round plans are bit-identical to the
oracle's schedule (the reference's numpy streams), and the metrics kernels
(fresh A alpha, A^T w, objective and gap terms, column norms) match numpy."""
import ctypes

import numpy as np
import pytest

from gpu_helpers import both
from oracle import syscd_oracle as O

pytestmark = pytest.mark.gpu

PLAN_CASES = [
    dict(n=203, B=8, K=1, P=4, seed=3),
    dict(n=203, B=8, K=3, P=2, seed=5),
    dict(n=500, B=16, K=1, P=4, seed=0),
    dict(n=203, B=8, K=2, P=3, seed=7, T3=2, T4=5),
    dict(n=203, B=8, K=2, P=2, seed=9, repartition="static"),
    dict(n=203, B=8, K=2, P=2, seed=9, sampling="iid", T3=3, T4=4),
    dict(n=203, B=8, K=1, P=2, seed=9, sampling="iid"),
    dict(n=10_000, B=100, K=1, P=7, seed=1),          # B > 64: scratch permutation path
    dict(n=200_000, B=2, K=1, P=64, seed=2),          # 100k buckets: global-memory shuffle
]


@pytest.mark.parametrize("case", PLAN_CASES)
def test_device_plan_matches_oracle_schedule(cuda, case):
    torch = cuda
    from paper_1911_07722_b200._lib import PlanDesc, call, lib
    from paper_1911_07722_b200.device import _ptr, _stream
    from paper_1911_07722_b200.sharding import shard_plan
    c = dict(T3=None, T4=None, sampling="perm", repartition="dynamic")
    c.update(case)
    sp = shard_plan(c["n"], c["B"], c["K"], c["P"], c["seed"])
    d = PlanDesc()
    d.seed, d.n_global, d.bucket_size = c["seed"], c["n"], c["B"]
    d.n_nodes_local, d.node0, d.P = c["K"], 0, c["P"]
    d.T3 = -1 if c["T3"] is None else c["T3"]
    d.T4 = -1 if c["T4"] is None else c["T4"]
    d.sampling = 0 if c["sampling"] == "perm" else 1
    d.repartition = 0 if c["repartition"] == "dynamic" else 1
    ptr = (ctypes.c_int32 * (c["K"] + 1))(*sp.node_ptr.tolist())
    d.node_bucket_ptr = ptr
    bk = torch.from_numpy(sp.buckets.astype(np.int32)).cuda()
    sc = torch.from_numpy(sp.bucket_store_col).cuda()
    d.node_buckets, d.bucket_store_col = bk.data_ptr(), sc.data_ptr()
    L = lib()
    R = 3
    stride = L.syscd_plan_max_updates(ctypes.byref(d))
    ws = torch.empty(L.syscd_plan_workspace_bytes(ctypes.byref(d), R), dtype=torch.uint8,
                     device="cuda")
    seq = torch.empty(R * stride, dtype=torch.int32, device="cuda")
    wp = torch.empty(R * (c["K"] * c["P"] + 1), dtype=torch.int64, device="cuda")
    rid0 = 4
    call("syscd_plan", ctypes.byref(d), rid0, R, _ptr(seq), stride, _ptr(wp), _ptr(ws),
         ws.numel(), _stream())
    torch.cuda.synchronize()
    oc = O.OracleConfig(K=c["K"], P=c["P"], bucket_size=c["B"], T3=c["T3"], T4=c["T4"],
                        sampling=c["sampling"], repartition=c["repartition"], seed=c["seed"])
    node_part = O.node_partition(c["n"], c["B"], c["K"], c["seed"])
    seq_h = seq.cpu().numpy().reshape(R, stride)
    wp_h = wp.cpu().numpy().reshape(R, -1)
    for r in range(R):
        sched = O.round_schedule(oc, c["n"], node_part, rid0 + r)
        for part, (_, _, coords) in enumerate(sched):
            got = seq_h[r, wp_h[r, part]:wp_h[r, part + 1]]
            assert got.tolist() == coords, (r, part)


def _np_objective(kind, A, y, alpha, lam):
    v = A @ alpha
    n = A.shape[1]
    if kind in ("ridge", "lasso"):
        f = 0.5 * np.sum((v - y) ** 2)
    else:
        f = np.dot(v, v) / (2 * lam * n * n)
    g = {"ridge": 0.5 * lam * alpha @ alpha, "lasso": lam * np.abs(alpha).sum(),
         "svm_dual": -alpha.sum() / n}[kind]
    return f + g


@pytest.mark.parametrize("cfg_id,scale", [(0, 0.05), (2, 0.01), (1, 0.0005), (4, 0.0002)])
def test_metrics_kernels_match_numpy(cuda, cfg_id, scale):
    pb, ob = both(cfg_id, scale)
    dp = pb.device()
    g = np.random.default_rng(1)
    alpha = g.uniform(0.01, 0.99, size=pb.n_coordinates).astype(np.float32).astype(np.float64)
    F = dp.objective_host(alpha)
    assert F == pytest.approx(ob.objective(alpha), rel=1e-9, abs=1e-12)
    gap, F2 = dp.gap_host(alpha)
    assert gap == pytest.approx(ob.gap(alpha), rel=1e-7, abs=1e-9 * abs(F))
    sq = pb.stats.column_sq_norms
    np.testing.assert_allclose(sq, ob.sq, rtol=1e-6)


def test_reference_optimum_ridge_cg(cuda):
    """GPU CG optimum vs the dense normal-equation solve (cli.py:87-90)."""
    from paper_1911_07722_b200 import compute_reference_optimum
    pb, ob = both(0, 0.05)
    a_star, f_star = compute_reference_optimum(pb)
    A = ob.A.dense
    x = np.linalg.solve(A.T @ A + ob.lam * np.eye(A.shape[1]), A.T @ ob.y)
    assert np.linalg.norm(a_star - x) / np.linalg.norm(x) < 1e-5
    assert f_star == pytest.approx(ob.objective(x), rel=1e-9)
    # the dual certificate vanishes at the optimum
    gap = pb.device().gap_host(a_star)[0]
    assert gap <= 1e-5 * abs(f_star)  # fp32 alpha, lam=1e-3 amplifies ||A^T w||^2/(2 lam)
