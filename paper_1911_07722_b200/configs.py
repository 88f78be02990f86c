"""The five BASELINE.json workloads as seeded synthetic problems.

Each config exists at any `scale` (rows and columns shrink together, the
distributions are unchanged) so parity tests run small instances through the
CPU oracle and the GPU with identical data, and bench.py runs the full size.

host=True  -> numpy generation (bit-reproducible, used by parity tests and
              the oracle; fp32 values handed to both sides)
host=False -> torch generation directly in HBM (the 3.2 GB / 32 GB configs
              never touch the host); same distributions, different streams.

Config table (BASELINE.json "configs"):
  0 ridge  20000 x 500       N(0,1), y = A w* + 0.1 e, lam 1e-3, P 4,  B 16, 20 ep
  1 svm    2M samples x 28   rows unit-norm, 10% flips, lam 1/n,  P 64, B 32, 30 ep
  2 lasso  400000 x 2000     unit columns, 5% w*, 0.01 noise, ~10% nnz, P 148, B 8, 50 ep
  3 ridge  1M x 8000         N(0,1), lam 1e-4, K = #GPUs, 40 ep
  4 logdual 10M x 1M CSC     39 distinct Zipf(1.1) features, 25% positives, lam 1e-6, 20 ep
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dataset import (
    COORDINATES_ARE_EXAMPLES,
    COORDINATES_ARE_FEATURES,
    ColumnMatrix,
    LabeledDataset,
    padded_ld,
)
from .objective import GlmProblem, SmoothLoss
from .solvers import SolverConfig

# lambda = LASSO_RATIO * ||A^T y||_inf for config 2: about 10% of the
# coordinates are nonzero at the optimum (BASELINE config 2).  Measured on the
# full-size problem (scripts/lasso_lambda_scan.py, K=P=1 solves certified by
# the duality gap): ratio 0.006 -> 15.0%, 0.007 -> 10.15%, 0.008 -> 7.5%,
# 0.05 -> 4.6% (the 5% support of w* alone); tests/test_gpu_fullsize.py pins it.
LASSO_RATIO = 0.007


@dataclass
class Workload:
    cfg_id: int
    problem: GlmProblem
    solver: SolverConfig
    name: str
    a_bytes: int          # algorithmic A bytes per epoch
    info: dict


def _rng(seed, tag):
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(7000 + tag,)))


def _dims(cfg_id, scale):
    base = {0: (20000, 500), 1: (28, 2_000_000), 2: (400_000, 2000), 3: (1_000_000, 8000),
            4: (1_000_000, 10_000_000)}[cfg_id]
    d, n = base
    if cfg_id == 1:
        return d, max(64, int(round(n * scale)))
    return max(8, int(round(d * scale))), max(8, int(round(n * scale)))


def default_solver(cfg_id, n_gpus=1, epochs=None):
    """BASELINE.json's partitioning at one GPU.  On N GPUs the node groups
    become the GPUs (K = N) and the partitions per GPU shrink so
    that K*P -- and with it the surrogate scale a = gamma K P and the
    per-epoch convergence -- stays that of one GPU: a fixed problem split N
    ways (strong scaling)."""
    if cfg_id == 0:
        return SolverConfig(K=n_gpus, P=max(1, 4 // n_gpus), bucket_size=16, T1=epochs or 20,
                            seed=0)
    if cfg_id == 1:
        return SolverConfig(K=n_gpus, P=max(1, 64 // n_gpus), bucket_size=32, T1=epochs or 30,
                            seed=0)
    if cfg_id == 2:
        return SolverConfig(K=n_gpus, P=max(1, 148 // n_gpus), bucket_size=8, T1=epochs or 50,
                            seed=0)
    if cfg_id == 3:
        return SolverConfig(K=n_gpus, P=1, bucket_size=8, T1=epochs or 40, seed=0)
    # config 4: BASELINE leaves P open; chosen by wall-clock to a duality-gap
    # target (scripts/ttt_scan.py): K*P = 128 beats 512 and 256 at
    # every budget from ~10 s on (fewer, longer chains converge faster per
    # second than more partitions with a larger surrogate scale a = gamma K P)
    return SolverConfig(K=n_gpus, P=max(1, 128 // n_gpus), bucket_size=64, T1=epochs or 20,
                        seed=0)


# ---------------------------------------------------------------------------
# host (numpy) generation
# ---------------------------------------------------------------------------
def host_arrays(cfg_id, scale=1.0, seed=0):
    """Returns (kind_tag, A (d x n fp32, F-order) or CSC tuple, labels, lam)."""
    d, n = _dims(cfg_id, scale)
    if cfg_id in (0, 3):
        g = _rng(seed, cfg_id)
        A = np.asfortranarray(g.standard_normal((d, n), dtype=np.float32))
        w = g.standard_normal(n)
        y = A.astype(np.float64) @ w + 0.1 * g.standard_normal(d)
        return "ridge", A, y, (1e-3 if cfg_id == 0 else 1e-4)
    if cfg_id == 1:
        g = _rng(seed, 1)
        X = g.standard_normal((n, d))
        X /= np.linalg.norm(X, axis=1, keepdims=True)
        w = g.standard_normal(d)
        y = np.sign(X @ w)
        y[y == 0] = 1.0
        flip = g.random(n) < 0.1
        y[flip] = -y[flip]
        A = np.asfortranarray(X.T.astype(np.float32))  # 28 x n, column = sample
        return "svm_dual", A, y, 1.0 / n
    if cfg_id == 2:
        g = _rng(seed, 2)
        A = g.standard_normal((d, n), dtype=np.float32)
        A /= np.linalg.norm(A.astype(np.float64), axis=0).astype(np.float32)
        A = np.asfortranarray(A)
        w = np.zeros(n)
        nz = g.choice(n, size=max(1, int(round(0.05 * n))), replace=False)
        w[nz] = g.standard_normal(nz.size)
        y = A.astype(np.float64) @ w + 0.01 * g.standard_normal(d)
        lam = LASSO_RATIO * float(np.max(np.abs(A.astype(np.float64).T @ y)))
        return "lasso", A, y, lam
    # config 4: logistic dual on one-hot rows
    g = _rng(seed, 4)
    nnz_row = 39 if d >= 390 else max(1, d // 10)
    ranks = np.arange(1, d + 1, dtype=np.float64)
    p = ranks ** -1.1
    p /= p.sum()
    rows = np.empty((n, nnz_row), dtype=np.int64)
    for i in range(n):
        chosen = []
        seen = set()
        while len(chosen) < nnz_row:
            for f in g.choice(d, size=4 * nnz_row, p=p):
                if f not in seen:
                    seen.add(f)
                    chosen.append(f)
                    if len(chosen) == nnz_row:
                        break
        rows[i] = np.sort(chosen)
    wfeat = np.zeros(d)
    nzf = g.choice(d, size=max(1, d // 100), replace=False)
    wfeat[nzf] = g.standard_normal(nzf.size) * 3.0
    score = wfeat[rows].sum(axis=1)
    t = _threshold_for_rate(score, 0.25)
    prob = 1.0 / (1.0 + np.exp(-(score - t)))
    y = np.where(g.random(n) < prob, 1.0, -1.0)
    col_ptr = np.arange(0, (n + 1) * nnz_row, nnz_row, dtype=np.int64)
    return "logistic_dual", (col_ptr, rows.reshape(-1).astype(np.int32),
                             np.ones(n * nnz_row, dtype=np.float32)), y, 1e-6


def _threshold_for_rate(score, rate):
    lo, hi = float(score.min()) - 20.0, float(score.max()) + 20.0
    for _ in range(100):
        mid = 0.5 * (lo + hi)
        m = float(np.mean(1.0 / (1.0 + np.exp(-(score - mid)))))
        if m > rate:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def host_problem(cfg_id, scale=1.0, seed=0):
    kind, A, y, lam = host_arrays(cfg_id, scale, seed)
    if kind == "logistic_dual":
        col_ptr, ri, va = A
        d, n = _dims(cfg_id, scale)
        m = ColumnMatrix(d, n, csc=(col_ptr, ri, va))
        ds = LabeledDataset(m, y, COORDINATES_ARE_EXAMPLES)
        return GlmProblem.build(ds, SmoothLoss.logistic(), lam)
    d, n = A.shape
    m = ColumnMatrix(d, n, dense=A)
    if kind == "svm_dual":
        ds = LabeledDataset(m, y, COORDINATES_ARE_EXAMPLES)
        return GlmProblem.build(ds, SmoothLoss.hinge(), lam)
    ds = LabeledDataset(m, y, COORDINATES_ARE_FEATURES)
    return GlmProblem.build(ds, SmoothLoss.squared_error(), lam,
                            reg="l1" if kind == "lasso" else "l2")


# ---------------------------------------------------------------------------
# device generation for full-size runs: counter-based, shard-local
# ---------------------------------------------------------------------------
# Philox stream tags (csrc/datagen.cu): every value is a function of (seed,
# tag, global column or row id), so rank r generates exactly its store
# columns and a sharded job holds the one-GPU matrix.
TAG_A, TAG_W, TAG_WMASK, TAG_NOISE, TAG_FLIP, TAG_ZIPF, TAG_WFEAT, TAG_WFEAT_MASK, TAG_LABEL = \
    range(1, 10)


class _DeviceGen:
    def __init__(self, cfg_id, seed):
        self.seed = (1_000_003 * (int(seed) + 1) + 7919 * cfg_id) & ((1 << 64) - 1)

    def _ids(self, ids):
        import torch
        if isinstance(ids, int):
            return None, ids
        t = torch.as_tensor(ids, dtype=torch.int64).cuda()
        return t, t.numel()

    def normal_cols(self, cols, d, lda):
        import torch
        from .device import _ptr, _stream
        from ._lib import call
        t, n = self._ids(cols)
        out = torch.empty((n, lda), dtype=torch.float32, device="cuda")
        call("syscd_gen_normal_cols", self.seed, TAG_A, _ptr(t), n, d, lda, _ptr(out), _stream())
        return out

    def ids(self, ids, tag, uniform=False):
        import torch
        from .device import _ptr, _stream
        from ._lib import call
        t, n = self._ids(ids)
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        call("syscd_gen_ids", self.seed, tag, _ptr(t), n, 1 if uniform else 0, _ptr(out),
             _stream())
        return out

    def onehot(self, cols, d, nnz, cdf):
        import torch
        from .device import _ptr, _stream
        from ._lib import call
        t, n = self._ids(cols)
        rows = torch.empty((n, nnz), dtype=torch.int32, device="cuda")
        failed = torch.zeros(1, dtype=torch.int32, device="cuda")
        call("syscd_gen_zipf_onehot", self.seed, TAG_ZIPF, _ptr(t), n, d, nnz, _ptr(cdf),
             _ptr(rows), _ptr(failed), _stream())
        if int(failed.item()):
            raise RuntimeError("one-hot generation: a column could not draw enough rows")
        return rows


def _chunks(n, ld):
    step = max(1, (1 << 28) // max(ld, 1))
    return [(j0, min(n, j0 + step)) for j0 in range(0, n, step)]


def shard_arrays(cfg_id, scale=1.0, seed=0, cols=None, dist=None, gen=None, device="cuda"):
    """The config's data for the global columns `cols` (store order; None =
    all), generated where it will live.  Quantities that depend on every
    column (y = A w* + noise, the Lasso lambda, the logistic label threshold)
    are reduced over `dist`, so every rank ends up with the problem a single
    GPU builds while holding only its own columns.

    Returns dict(kind, d, n, lam, and either At (n_loc, lda) float32 or csc
    (col_ptr, row_idx, vals), plus y (length d, primal) or labels (n_loc,
    dual)).  gen: the column-keyed generator (default: the CUDA kernels)."""
    import torch
    from .device import Dist
    dist = dist or Dist.single()
    d, n = _dims(cfg_id, scale)
    gen = gen or _DeviceGen(cfg_id, seed)
    sel = None if cols is None else np.asarray(cols, dtype=np.int64)
    n_loc = n if sel is None else int(sel.size)
    ids = n if sel is None else sel
    f64 = dict(dtype=torch.float64, device=device)
    if cfg_id == 4:
        nnz_row = 39 if d >= 390 else max(1, d // 10)
        ranks = torch.arange(1, d + 1, **f64)
        cdf = torch.cumsum(ranks.pow(-1.1), 0)
        cdf /= cdf[-1].clone()
        rows = gen.onehot(ids, d, nnz_row, cdf)
        wfeat = 3.0 * gen.ids(d, TAG_WFEAT) * (gen.ids(d, TAG_WFEAT_MASK, uniform=True) < 0.01)
        score = torch.empty(n_loc, **f64)
        for j0, j1 in _chunks(n_loc, nnz_row * 64):
            score[j0:j1] = wfeat[rows[j0:j1].long()].sum(dim=1)
        ext = torch.tensor([float(score.max()) if n_loc else -1e300,
                            -float(score.min()) if n_loc else -1e300], **f64)
        dist.allreduce_(ext, op="max")
        lo, hi = -float(ext[1]) - 20.0, float(ext[0]) + 20.0
        for _ in range(60):  # bias so that the expected positive rate is 25%
            mid = 0.5 * (lo + hi)
            m = torch.sigmoid(score - mid).sum().reshape(1)
            if float(dist.allreduce_(m)) / n > 0.25:
                lo = mid
            else:
                hi = mid
        prob = torch.sigmoid(score - 0.5 * (lo + hi))
        labels = torch.where(gen.ids(ids, TAG_LABEL, uniform=True) < prob, 1.0, -1.0)
        col_ptr = torch.arange(0, (n_loc + 1) * nnz_row, nnz_row, dtype=torch.int64,
                               device=device)
        vals = torch.ones(n_loc * nnz_row, dtype=torch.float32, device=device)
        return dict(kind="logistic_dual", d=d, n=n, lam=1e-6,
                    csc=(col_ptr, rows.reshape(-1), vals), labels=labels)
    ld = padded_ld(d)
    At = gen.normal_cols(ids, d, ld)
    if cfg_id == 1:
        # columns = samples: each normalised to unit norm; labels from w*
        At[:, :d] /= torch.linalg.norm(At[:, :d], dim=1, keepdim=True)
        w = gen.ids(d, TAG_W)
        labels = torch.sign(At[:, :d].double() @ w)
        labels[labels == 0] = 1.0
        flip = gen.ids(ids, TAG_FLIP, uniform=True) < 0.1
        labels[flip] = -labels[flip]
        return dict(kind="svm_dual", d=d, n=n, lam=1.0 / n, At=At, labels=labels)
    if cfg_id == 2:
        for j0, j1 in _chunks(n_loc, ld):
            nrm = torch.linalg.norm(At[j0:j1, :d].double(), dim=1, keepdim=True)
            At[j0:j1, :d] = (At[j0:j1, :d].double() / nrm).float()
        w = gen.ids(ids, TAG_W) * (gen.ids(ids, TAG_WMASK, uniform=True) < 0.05)
        noise = 0.01
    else:
        w = gen.ids(ids, TAG_W)
        noise = 0.1
    y = torch.zeros(d, **f64)
    for j0, j1 in _chunks(n_loc, ld):
        y += At[j0:j1, :d].double().T @ w[j0:j1]
    dist.allreduce_(y)
    y += noise * gen.ids(d, TAG_NOISE)
    if cfg_id == 2:
        aty = torch.zeros(1, **f64)
        for j0, j1 in _chunks(n_loc, ld):
            aty = torch.maximum(aty, (At[j0:j1, :d].double() @ y).abs().max().reshape(1))
        lam = LASSO_RATIO * float(dist.allreduce_(aty, op="max"))
        return dict(kind="lasso", d=d, n=n, lam=lam, At=At, y=y)
    return dict(kind="ridge", d=d, n=n, lam=1e-3 if cfg_id == 0 else 1e-4, At=At, y=y)


def problem_from_arrays(arr, cols=None):
    """A GlmProblem over device arrays from shard_arrays (or their uploaded
    copies); cols marks the matrix as this rank's shard."""
    d, n = arr["d"], arr["n"]
    if "csc" in arr:
        m = ColumnMatrix.from_device_csc(*arr["csc"], d)
    else:
        m = ColumnMatrix.from_device(arr["At"], d)
    if cols is not None:
        m.mark_shard(cols, n)
    kind = arr["kind"]
    if kind in ("svm_dual", "logistic_dual"):
        labels = arr["labels"]
        labels = labels.cpu().numpy() if hasattr(labels, "cpu") else np.asarray(labels)
        ds = LabeledDataset(m, labels, COORDINATES_ARE_EXAMPLES)
        loss = SmoothLoss.hinge() if kind == "svm_dual" else SmoothLoss.logistic()
        return GlmProblem.build(ds, loss, arr["lam"])
    y = arr["y"]
    y = y.cpu().numpy() if hasattr(y, "cpu") else np.asarray(y)
    ds = LabeledDataset(m, y, COORDINATES_ARE_FEATURES)
    return GlmProblem.build(ds, SmoothLoss.squared_error(), arr["lam"],
                            reg="l1" if kind == "lasso" else "l2")


def device_problem(cfg_id, scale=1.0, seed=0, cols=None, dist=None):
    """The config's problem generated in HBM (cols: a rank's shard)."""
    return problem_from_arrays(shard_arrays(cfg_id, scale, seed, cols, dist), cols)


def workload(cfg_id, scale=1.0, seed=0, host=None, n_gpus=1, epochs=None, dist=None):
    """The config's problem and solver settings.  On a multi-GPU job (dist
    with world > 1, device generation) each rank generates only its own
    store columns (the shard of its node groups, sharding.shard_plan)."""
    if host is None:
        host = cfg_id == 0 or (scale < 0.2 and cfg_id != 4) or (cfg_id == 4 and scale < 0.002)
    solver = default_solver(cfg_id, n_gpus, epochs)
    d, n = _dims(cfg_id, scale)
    world = dist.world if dist is not None else 1
    if host:
        pb = host_problem(cfg_id, scale, seed)
    elif world > 1:
        from .sharding import shard_plan
        sp = shard_plan(n, solver.resolved_bucket_size(), solver.K, solver.P, solver.seed, world,
                        dist.rank)
        pb = device_problem(cfg_id, scale, seed, cols=sp.store_cols, dist=dist)
    else:
        pb = device_problem(cfg_id, scale, seed)
    m = pb.data.matrix
    if m.storage_kind == "dense":
        a_bytes = 4 * d * n
    else:
        nnz_row = 39 if d >= 390 else max(1, d // 10)
        a_bytes = (8 * nnz_row + 8) * n if not host else 8 * m.nnz() + 8 * n
    names = {0: "ridge-20000x500", 1: "svm-dual-2Mx28", 2: "lasso-400000x2000",
             3: "ridge-1Mx8000", 4: "logreg-dual-10Mx1M-csc"}
    return Workload(cfg_id, pb, solver, names[cfg_id], a_bytes,
                    {"d": d, "n": n, "lam": pb.reg.lam, "scale": scale})
