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

# lambda = LASSO_RATIO * ||A^T y||_inf for config 2 (calibrated so that about
# 10% of the coordinates are nonzero at the optimum)
LASSO_RATIO = 0.08


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
    return SolverConfig(K=n_gpus, P=max(8, 512 // n_gpus), bucket_size=64, T1=epochs or 20,
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
# device (torch) generation for full-size runs
# ---------------------------------------------------------------------------
def _device_onehot_rows(n, d, nnz_row, gen, chunk=1 << 20):
    """n rows of nnz_row distinct features drawn from Zipf(1.1) over d
    features (inverse-CDF draws, first nnz_row distinct in draw order),
    returned sorted per row as an (n, nnz_row) int32 CUDA tensor."""
    import torch
    ranks = torch.arange(1, d + 1, dtype=torch.float64, device="cuda")
    cdf = torch.cumsum(ranks.pow(-1.1), 0)
    cdf /= cdf[-1].clone()
    out = torch.empty((n, nnz_row), dtype=torch.int32, device="cuda")
    ncand = 4 * nnz_row
    for r0 in range(0, n, chunk):
        rows = torch.arange(r0, min(n, r0 + chunk), device="cuda")
        while rows.numel():
            R = rows.numel()
            u = torch.rand((R, ncand), generator=gen, device="cuda", dtype=torch.float64)
            cand = torch.searchsorted(cdf, u).clamp_(max=d - 1)
            sv, pos = torch.sort(cand, dim=1, stable=True)
            first = torch.ones_like(sv, dtype=torch.bool)
            first[:, 1:] = sv[:, 1:] != sv[:, :-1]
            keep = torch.zeros_like(first)
            keep.scatter_(1, pos, first)                 # first occurrence, draw order
            rank = torch.cumsum(keep.to(torch.int32), 1)
            ok = rank[:, -1] >= nnz_row
            sel = keep & (rank <= nnz_row)
            good = rows[ok]
            feats = cand[ok][sel[ok]].view(-1, nnz_row)
            out[good] = torch.sort(feats, dim=1).values.to(torch.int32)
            rows = rows[~ok]
    return out


def _device_config4(d, n, seed, gen):
    import torch
    nnz_row = 39 if d >= 390 else max(1, d // 10)
    feats = _device_onehot_rows(n, d, nnz_row, gen)
    w = torch.zeros(d, dtype=torch.float64, device="cuda")
    k = max(1, d // 100)
    idx = torch.randperm(d, generator=gen, device="cuda")[:k]
    w[idx] = 3.0 * torch.randn(k, generator=gen, device="cuda", dtype=torch.float64)
    score = w[feats.long()].sum(dim=1)
    lo, hi = float(score.min()) - 20.0, float(score.max()) + 20.0
    for _ in range(60):  # bias so that the expected positive rate is 25%
        mid = 0.5 * (lo + hi)
        if float(torch.sigmoid(score - mid).mean()) > 0.25:
            lo = mid
        else:
            hi = mid
    prob = torch.sigmoid(score - 0.5 * (lo + hi))
    y = torch.where(torch.rand(n, generator=gen, device="cuda", dtype=torch.float64) < prob,
                    1.0, -1.0)
    col_ptr = torch.arange(0, (n + 1) * nnz_row, nnz_row, dtype=torch.int64, device="cuda")
    vals = torch.ones(n * nnz_row, dtype=torch.float32, device="cuda")
    m = ColumnMatrix.from_device_csc(col_ptr, feats.reshape(-1).contiguous(), vals, d)
    ds = LabeledDataset(m, y.cpu().numpy(), COORDINATES_ARE_EXAMPLES)
    return GlmProblem.build(ds, SmoothLoss.logistic(), 1e-6)


def device_problem(cfg_id, scale=1.0, seed=0):
    import torch
    d, n = _dims(cfg_id, scale)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1_000_003 * (seed + 1) + cfg_id)
    if cfg_id == 4:
        return _device_config4(d, n, seed, gen)
    ld = padded_ld(d)
    At = torch.empty((n, ld), dtype=torch.float32, device="cuda")
    chunk = max(1, (1 << 28) // ld)
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        At[j0:j1].normal_(generator=gen)
    if ld > d:
        At[:, d:] = 0
    if cfg_id == 1:
        # columns = samples: normalise each sample (column) to unit norm
        At[:, :d] /= torch.linalg.norm(At[:, :d], dim=1, keepdim=True)
        w = torch.randn(d, generator=gen, device="cuda", dtype=torch.float64)
        y = torch.sign(At[:, :d].double() @ w)
        y[y == 0] = 1.0
        flip = torch.rand(n, generator=gen, device="cuda") < 0.1
        y[flip] = -y[flip]
        m = ColumnMatrix.from_device(At, d)
        ds = LabeledDataset(m, y.cpu().numpy(), COORDINATES_ARE_EXAMPLES)
        return GlmProblem.build(ds, SmoothLoss.hinge(), 1.0 / n)
    if cfg_id == 2:
        for j0 in range(0, n, chunk):
            j1 = min(n, j0 + chunk)
            nrm = torch.linalg.norm(At[j0:j1, :d].double(), dim=1, keepdim=True)
            At[j0:j1, :d] = (At[j0:j1, :d].double() / nrm).float()
    w = torch.zeros(n, dtype=torch.float64, device="cuda")
    if cfg_id == 2:
        k = max(1, int(round(0.05 * n)))
        idx = torch.randperm(n, generator=gen, device="cuda")[:k]
        w[idx] = torch.randn(k, generator=gen, device="cuda", dtype=torch.float64)
        noise = 0.01
    else:
        w = torch.randn(n, generator=gen, device="cuda", dtype=torch.float64)
        noise = 0.1
    y = torch.zeros(d, dtype=torch.float64, device="cuda")
    for j0 in range(0, n, chunk):
        j1 = min(n, j0 + chunk)
        y += At[j0:j1, :d].double().T @ w[j0:j1]
    y += noise * torch.randn(d, generator=gen, device="cuda", dtype=torch.float64)
    m = ColumnMatrix.from_device(At, d)
    if cfg_id == 2:
        aty = torch.empty(n, dtype=torch.float64, device="cuda")
        for j0 in range(0, n, chunk):
            j1 = min(n, j0 + chunk)
            aty[j0:j1] = At[j0:j1, :d].double() @ y
        lam = LASSO_RATIO * float(aty.abs().max())
        ds = LabeledDataset(m, y.cpu().numpy(), COORDINATES_ARE_FEATURES)
        return GlmProblem.build(ds, SmoothLoss.squared_error(), lam, reg="l1")
    ds = LabeledDataset(m, y.cpu().numpy(), COORDINATES_ARE_FEATURES)
    return GlmProblem.build(ds, SmoothLoss.squared_error(), 1e-3 if cfg_id == 0 else 1e-4)


def workload(cfg_id, scale=1.0, seed=0, host=None, n_gpus=1, epochs=None):
    if host is None:
        host = cfg_id == 0 or (scale < 0.2 and cfg_id != 4) or (cfg_id == 4 and scale < 0.002)
    pb = host_problem(cfg_id, scale, seed) if host else device_problem(cfg_id, scale, seed)
    solver = default_solver(cfg_id, n_gpus, epochs)
    m = pb.data.matrix
    if m.storage_kind == "dense":
        a_bytes = 4 * m.n_rows * m.n_cols
    else:
        nnz = m.nnz()
        a_bytes = 8 * nnz + 8 * m.n_cols
    names = {0: "ridge-20000x500", 1: "svm-dual-2Mx28", 2: "lasso-400000x2000",
             3: "ridge-1Mx8000", 4: "logreg-dual-10Mx1M-csc"}
    return Workload(cfg_id, pb, solver, names[cfg_id], a_bytes,
                    {"d": m.n_rows, "n": m.n_cols, "lam": pb.reg.lam, "scale": scale})
