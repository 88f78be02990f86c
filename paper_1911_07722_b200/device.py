"""GPU-resident problem mirror and the metrics passes (all through the C ABI).

DeviceProblem places one shard of a GlmProblem in HBM (DESIGN.md "data
layout"): the store holds the shard's columns in the order the solver's
bucket tables address them, dual problems get their labels folded into the
columns (y_i x_i), and the model alpha, the shared vector v (fp64) and
lin_vec u (fp32) live next to it.  Metrics follow full_objective
(objective.py:95-102): a fresh v = A alpha in fp64, then f(v) + g(alpha), and
optionally the Fenchel duality gap.
"""

from __future__ import annotations

import ctypes

import numpy as np

from ._lib import call
from .dataset import padded_ld
from .objective import LASSO, LOGISTIC, RIDGE, SVM_DUAL


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1911_07722_b200 needs a CUDA device (there is no CPU path)")
    return torch


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream():
    """Raw handle of the current CUDA stream (the cheap accessor: this runs
    several times per round on the host-bound small configs)."""
    import torch
    return ctypes.c_void_p(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


# ---------------------------------------------------------------------------
# device copies of a ColumnMatrix (cached on the matrix object)
# ---------------------------------------------------------------------------
def device_dense(matrix):
    """(n_cols, lda) float32 CUDA tensor of A, column-major, zero padded."""
    torch = _torch()
    if matrix._dev_dense is None:
        host = matrix._dense
        ld = padded_ld(matrix.n_rows)
        At = torch.zeros((matrix.n_cols, ld), dtype=torch.float32, device="cuda")
        At[:, : matrix.n_rows].copy_(torch.from_numpy(np.ascontiguousarray(host.T)))
        matrix._dev_dense = At
    return matrix._dev_dense


def device_csc(matrix):
    torch = _torch()
    if matrix._dev_csc is None:
        cp, ri, va = matrix._csc
        matrix._dev_csc = (torch.from_numpy(cp.astype(np.int64)).cuda(),
                           torch.from_numpy(ri.astype(np.int32)).cuda(),
                           torch.from_numpy(va.astype(np.float32)).cuda())
    return matrix._dev_csc


def column_sq_norms(matrix):
    """q_j = ||x_j||^2 on the GPU (compute_stats, dataset.py:307)."""
    torch = _torch()
    out = torch.empty(matrix.n_cols, dtype=torch.float32, device="cuda")
    if matrix.storage_kind == "dense":
        At = device_dense(matrix)
        call("syscd_dense_col_sq_norms", matrix.n_rows, matrix.n_cols, At.shape[1], _ptr(At),
             _ptr(out), _stream())
    else:
        cp, ri, va = device_csc(matrix)
        call("syscd_sparse_col_sq_norms", matrix.n_cols, _ptr(cp), _ptr(va), _ptr(out), _stream())
    return out.double().cpu().numpy()


def _matvec_raw(matrix_dev, d, x, out, work):
    """out (fp64, d) = A x for a float32 x over the store columns."""
    kind, data = matrix_dev
    if kind == "dense":
        At = data
        call("syscd_dense_matvec", d, At.shape[0], At.shape[1], _ptr(At), _ptr(x), _ptr(out),
             _ptr(work), work.numel() * 8 if work is not None else 0, _stream())
    else:
        cp, ri, va = data
        call("syscd_sparse_matvec", d, cp.shape[0] - 1, _ptr(cp), _ptr(ri), _ptr(va), _ptr(x),
             _ptr(out), _stream())


def _rmatvec_raw(matrix_dev, d, w, out):
    kind, data = matrix_dev
    if kind == "dense":
        At = data
        call("syscd_dense_rmatvec", d, At.shape[0], At.shape[1], _ptr(At), _ptr(w), _ptr(out),
             _stream())
    else:
        cp, ri, va = data
        call("syscd_sparse_rmatvec", cp.shape[0] - 1, _ptr(cp), _ptr(ri), _ptr(va), _ptr(w),
             _ptr(out), _stream())


def spectral_constant(matrix, power_iters=200, tol=1e-9):
    """lambda_max(A^T A) by power iteration (dataset.py:308-321), on the GPU."""
    torch = _torch()
    md = (("dense", device_dense(matrix)) if matrix.storage_kind == "dense"
          else ("sparse", device_csc(matrix)))
    n, d = matrix.n_cols, matrix.n_rows
    x = torch.full((n,), 1.0 / np.sqrt(n), dtype=torch.float64, device="cuda")
    v = torch.empty(d, dtype=torch.float64, device="cuda")
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    work = torch.empty(2 * 148 * 8 * d if d < 65536 else 1, dtype=torch.float64, device="cuda")
    est = 0.0
    for _ in range(power_iters):
        _matvec_raw(md, d, x.float(), v, work)
        _rmatvec_raw(md, d, v, z)
        new_est = float(torch.dot(x, z))
        nz = float(torch.linalg.norm(z))
        if nz == 0.0:
            return 0.0
        x = z / nz
        if est > 0.0 and abs(new_est - est) <= tol * abs(new_est):
            return new_est
        est = new_est
    return max(est, 0.0)


class Dist:
    """Rank/world view used by the metrics (single process: identity)."""

    def __init__(self, group=None):
        import torch.distributed as tdist
        self.on = tdist.is_available() and tdist.is_initialized()
        self.rank = tdist.get_rank() if self.on else 0
        self.world = tdist.get_world_size() if self.on else 1
        self.group = group

    @classmethod
    def single(cls):
        """This process alone (no collectives), also inside a distributed job."""
        obj = cls.__new__(cls)
        obj.on, obj.rank, obj.world, obj.group = False, 0, 1, None
        return obj

    def allgather(self, t):
        """[t from rank 0, t from rank 1, ...] (equal shapes)."""
        if self.world == 1:
            return [t]
        import torch
        import torch.distributed as tdist
        out = [torch.empty_like(t) for _ in range(self.world)]
        tdist.all_gather(out, t, group=self.group)
        return out

    def allreduce_(self, t, op="sum"):
        if self.world > 1:
            import torch.distributed as tdist
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX if op == "max" else tdist.ReduceOp.SUM,
                             group=self.group)
        return t


class DeviceProblem:
    """One shard of a GlmProblem in HBM.

    store_cols: global column ids held by this process, in store order
    (None = all columns in natural order).
    """

    def __init__(self, problem, store_cols=None, dist=None):
        torch = _torch()
        self.problem = problem
        m = problem.data.matrix
        # a shard-local matrix already holds exactly this rank's store columns
        presharded = m.global_cols is not None
        if presharded and (store_cols is None or not np.array_equal(store_cols, m.global_cols)):
            raise ValueError("the problem holds a different shard than this rank's node groups")
        # a full (unsharded) problem has nothing to reduce across ranks
        self.dist = dist if (dist is not None and store_cols is not None) else Dist.single()
        self.kind = problem.kind
        self.d = m.n_rows
        self.n_global = problem.n_coordinates
        self.lam = float(problem.reg.lam)
        self.n_coords = float(self.n_global)
        self.gamma = float(problem.gamma)
        self.storage = m.storage_kind
        dual = problem.is_dual
        labels = problem.data.labels
        natural = store_cols is None or presharded
        cols = (np.arange(m.n_cols, dtype=np.int64) if store_cols is None
                else np.asarray(store_cols, np.int64))
        self.store_cols = cols
        self.n_store = cols.size
        # rows of the held arrays (labels, norms, device columns) to use
        local = np.arange(m.n_cols, dtype=np.int64) if natural else cols
        cols_t = None if natural else torch.from_numpy(cols).cuda()
        if self.storage == "dense":
            At = device_dense(m)
            if not natural:
                At = At.index_select(0, cols_t)
            if dual:
                yl = torch.from_numpy(labels[local].astype(np.float32)).cuda()
                At = At * yl[:, None]
            self.At = At.contiguous()
            self.lda = self.At.shape[1]
            self.mdev = ("dense", self.At)
        else:
            cp, ri, va = device_csc(m)
            if not natural:
                # gather the shard's columns (vectorised on the device)
                cols_d = torch.from_numpy(cols).cuda()
                starts = cp.index_select(0, cols_d)
                cnt = cp.index_select(0, cols_d + 1) - starts
                new_cp = torch.zeros(cols.size + 1, dtype=torch.int64, device="cuda")
                torch.cumsum(cnt, 0, out=new_cp[1:])
                nnz = int(new_cp[-1])
                rep = torch.repeat_interleave(torch.arange(cols.size, device="cuda"), cnt,
                                              output_size=nnz)
                src = starts.index_select(0, rep) + (torch.arange(nnz, device="cuda") -
                                                     new_cp.index_select(0, rep))
                cp, ri, va = new_cp, ri.index_select(0, src), va.index_select(0, src)
            if dual:
                # fold labels into the values: column i becomes y_i x_i
                cnt = cp[1:] - cp[:-1]
                ycol = torch.from_numpy(labels[local].astype(np.float32)).cuda()
                va = va * torch.repeat_interleave(ycol, cnt, output_size=int(cp[-1]))
            cp, ri, va = cp.contiguous(), ri.contiguous(), va.contiguous()
            self.csc = (cp, ri, va)
            self.mdev = ("sparse", self.csc)
            self.lda = None
        sq_held = np.asarray(problem.stats.column_sq_norms, dtype=np.float64)
        self.sq = torch.from_numpy(sq_held[local].astype(np.float32)).cuda()
        self.y = None if dual else torch.from_numpy(labels.astype(np.float64)).cuda()
        d = self.d
        self.v = torch.zeros(d, dtype=torch.float64, device="cuda")
        self.u = torch.empty(d, dtype=torch.float32, device="cuda")
        self.dv = torch.empty(d, dtype=torch.float32, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._terms_work = torch.empty(296 * 4, dtype=torch.float64, device="cuda")
        self._terms_out = torch.empty(4, dtype=torch.float64, device="cuda")
        nch = 0
        if self.storage == "dense":
            tiles = (d + 255) // 256 if d >= 256 else 1
            nch = min(4096, max(1, (2 * 148 * 8 + tiles - 1) // tiles), self.n_store)
        self._mv_work = torch.empty(max(1, nch * d) if nch > 1 else 1, dtype=torch.float64,
                                    device="cuda")
        self._vm = torch.empty(d, dtype=torch.float64, device="cuda")
        self._w = torch.empty(d, dtype=torch.float64, device="cuda")
        self._atw = torch.empty(self.n_store, dtype=torch.float64, device="cuda")

    # -- primitives -----------------------------------------------------------
    def matvec(self, alpha_store, out=None):
        """fp64 A alpha over this shard's columns, summed over ranks."""
        out = self._vm if out is None else out
        _matvec_raw(self.mdev, self.d, alpha_store, out, self._mv_work)
        self.dist.allreduce_(out)
        return out

    def grad_into(self, v, u, v_node=None, drift=0.0):
        call("syscd_grad", self.kind, self.d, _ptr(v), _ptr(self.y), self.lam, self.n_coords,
             _ptr(v_node), float(drift), _ptr(u), _stream())

    def _terms(self, v, alpha_store):
        call("syscd_objective_terms", self.kind, self.d, self.n_store, _ptr(v), _ptr(self.y),
             _ptr(alpha_store), self.lam, self.n_coords, _ptr(self._terms_out),
             _ptr(self._terms_work), _stream())
        t = self._terms_out.clone()
        # f-term is identical on every rank (v is global); g-term is per shard
        g = self.dist.allreduce_(t[1:2].clone())
        return float(t[0]), float(g[0])

    def objective(self, alpha_store, v=None):
        """F(alpha) with a fresh v = A alpha (or the given fp64 v)."""
        if v is None:
            v = self.matvec(alpha_store)
        fterm, gterm = self._terms(v, alpha_store)
        lam, n = self.lam, self.n_coords
        k = self.kind
        if k in (RIDGE, LASSO, LOGISTIC):
            f = fterm
        else:
            f = fterm / (2.0 * lam * n * n)
        if k in (RIDGE, LOGISTIC):
            g = 0.5 * lam * gterm
        elif k == LASSO:
            g = lam * gterm
        elif k == SVM_DUAL:
            g = -gterm / n
        else:
            g = gterm / n
        return f + g

    def gap(self, alpha_store):
        """(duality gap, F) at alpha (fresh v)."""
        v = self.matvec(alpha_store)
        F = self.objective(alpha_store, v=v)
        call("syscd_dual_point", self.kind, self.d, _ptr(v), _ptr(self.y), self.lam, self.n_coords,
             _ptr(self._w), _stream())
        _rmatvec_raw(self.mdev, self.d, self._w, self._atw)
        call("syscd_gap_terms", self.kind, self.d, self.n_store, _ptr(v), _ptr(self.y),
             _ptr(self._atw), self.lam, self.n_coords, 1.0, _ptr(self._terms_out),
             _ptr(self._terms_work), _stream())
        t = self._terms_out.clone()
        col_sum = self.dist.allreduce_(t[2:3].clone())
        col_max = self.dist.allreduce_(t[3:4].clone(), op="max")
        t0, t1, t2, t3 = float(t[0]), float(t[1]), float(col_sum[0]), float(col_max[0])
        lam, n, k = self.lam, self.n_coords, self.kind
        if k == RIDGE:
            D = -0.5 * t0 - t1 - t2 / (2.0 * lam)
            return F - D, F
        if k == LASSO:
            s = 1.0 if t3 <= lam else lam / t3
            D = -0.5 * s * s * t0 - s * t1
            return F - D, F
        if k == LOGISTIC:
            D = -t0 - t2 / (2.0 * lam)
            return F - D, F
        P = 0.5 * lam * t0 + t2 / n
        return P + F, F

    # -- host-facing helpers (API parity) --------------------------------------
    def upload_alpha(self, alpha_global):
        torch = _torch()
        a = np.asarray(alpha_global, dtype=np.float64)
        if a.shape != (self.n_global,):
            raise ValueError("alpha length does not match coordinate count")
        a = a[self.store_cols].astype(np.float32)
        return torch.from_numpy(a).cuda()

    def objective_host(self, alpha_global):
        return self.objective(self.upload_alpha(alpha_global))

    def gap_host(self, alpha_global):
        return self.gap(self.upload_alpha(alpha_global))

    def grad_host(self, v):
        torch = _torch()
        vt = torch.from_numpy(np.asarray(v, dtype=np.float64)).cuda()
        u = torch.empty(self.d, dtype=torch.float32, device="cuda")
        self.grad_into(vt, u)
        return u.double().cpu().numpy()
