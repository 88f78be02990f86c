"""Column-major training data (mirror of pkg/src/syscd/dataset.py).

ColumnMatrix keeps the reference's constructor and accessors
(dataset.py:24-130) but stores float32, the compute type of the GPU path, and
can also wrap data that already lives on the GPU (``ColumnMatrix.from_device``)
so that the 3.2 GB / 32 GB configurations never round-trip through the host.

Device layout: a dense matrix is a
(n_cols, lda) float32 torch tensor, i.e. column-major A with leading dimension
lda = d rounded up to a multiple of 4 (16-byte rows for the bulk TMA copies,
padding zero-filled).  A sparse matrix is CSC: int64 col_ptr, int32 row_idx,
float32 values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

COORDINATES_ARE_FEATURES = "coordinates_are_features"
COORDINATES_ARE_EXAMPLES = "coordinates_are_examples"


def padded_ld(d):
    return (int(d) + 3) // 4 * 4


class ColumnMatrix:
    """Training data stored column by column (dense or per-column sparse)."""

    def __init__(self, n_rows, n_cols, dense=None, sparse_cols=None, csc=None):
        given = sum(x is not None for x in (dense, sparse_cols, csc))
        if given != 1:
            raise ValueError("exactly one of dense / sparse_cols must be given")
        self.n_rows = int(n_rows)
        self.n_cols = int(n_cols)
        self._dev_dense = None
        self._dev_csc = None
        if dense is not None:
            dense = np.asfortranarray(dense, dtype=np.float32)
            if dense.shape != (self.n_rows, self.n_cols):
                raise ValueError("dense array shape does not match dims")
            if not np.all(np.isfinite(dense)):
                raise ValueError("non-finite entries in data matrix")
            self.storage_kind = "dense"
            self._dense = dense
            self._csc = None
        else:
            if sparse_cols is not None:
                if len(sparse_cols) != self.n_cols:
                    raise ValueError("sparse column count does not match n_cols")
                ptr = np.zeros(self.n_cols + 1, dtype=np.int64)
                idx_l, val_l = [], []
                for j, (idx, vals) in enumerate(sparse_cols):
                    idx = np.asarray(idx, dtype=np.int64)
                    vals = np.asarray(vals, dtype=np.float64)
                    if idx.shape != vals.shape:
                        raise ValueError(f"column {j}: index/value length mismatch")
                    idx_l.append(idx)
                    val_l.append(vals)
                    ptr[j + 1] = ptr[j] + idx.size
                indices = np.concatenate(idx_l) if idx_l else np.zeros(0, np.int64)
                values = np.concatenate(val_l) if val_l else np.zeros(0)
            else:
                ptr, indices, values = (np.asarray(csc[0], dtype=np.int64),
                                        np.asarray(csc[1], dtype=np.int64),
                                        np.asarray(csc[2], dtype=np.float64))
                if ptr.shape != (self.n_cols + 1,) or ptr[0] != 0 or ptr[-1] != indices.size:
                    raise ValueError("bad CSC column pointer")
            self._check_sparse(ptr, indices, values)
            self.storage_kind = "sparse"
            self._dense = None
            self._csc = (ptr, indices.astype(np.int32), values.astype(np.float32))

    def _check_sparse(self, ptr, indices, values):
        if indices.shape != values.shape:
            raise ValueError("index/value length mismatch")
        if np.any(np.diff(ptr) < 0):
            raise ValueError("column pointer not monotone")
        if indices.size:
            if indices.min() < 0 or indices.max() >= self.n_rows:
                raise ValueError("row index out of range")
            d = np.diff(indices)
            starts = ptr[1:-1]
            ok = np.ones(d.size, dtype=bool)
            ok[starts[(starts > 0) & (starts < indices.size)] - 1] = False
            if np.any((d <= 0) & ok):
                raise ValueError("indices not strictly increasing within a column")
        if not np.all(np.isfinite(values)):
            raise ValueError("non-finite values")

    # -- device-resident construction ---------------------------------------
    @classmethod
    def from_device(cls, At, n_rows):
        """Wrap a (n_cols, lda) float32 CUDA tensor holding A column-major."""
        import torch
        if At.dtype != torch.float32 or not At.is_cuda or At.dim() != 2 or not At.is_contiguous():
            raise ValueError("from_device expects a contiguous float32 CUDA tensor (n_cols, lda)")
        if At.shape[1] % 4 != 0 or At.shape[1] < n_rows:
            raise ValueError("lda must be >= n_rows and a multiple of 4")
        obj = cls.__new__(cls)
        obj.n_rows = int(n_rows)
        obj.n_cols = int(At.shape[0])
        obj.storage_kind = "dense"
        obj._dense = None
        obj._csc = None
        obj._dev_dense = At
        obj._dev_csc = None
        return obj

    @classmethod
    def from_device_csc(cls, col_ptr, row_idx, vals, n_rows):
        """Wrap CUDA CSC tensors (int64 col_ptr, int32 row_idx, float32 vals)."""
        obj = cls.__new__(cls)
        obj.n_rows = int(n_rows)
        obj.n_cols = int(col_ptr.shape[0] - 1)
        obj.storage_kind = "sparse"
        obj._dense = None
        obj._csc = None
        obj._dev_dense = None
        obj._dev_csc = (col_ptr, row_idx, vals)
        return obj

    # -- shards (multi-GPU) ---------------------------------------
    global_cols = None   # global column id of every held column (None: unsharded)
    n_cols_global = None

    def mark_shard(self, global_cols, n_cols_global):
        """Declare that this matrix holds only the columns `global_cols` (in
        store order) of an n_cols_global-column problem: the rank's shard of
        the static node partition (partitioning.py:89-96), generated or
        loaded shard-locally so no rank ever holds the whole matrix."""
        global_cols = np.asarray(global_cols, dtype=np.int64)
        if global_cols.shape != (self.n_cols,):
            raise ValueError("one global column id per held column expected")
        self.global_cols = global_cols
        self.n_cols_global = int(n_cols_global)
        return self

    # -- reference accessors (host) ------------------------------------------
    def _host_dense(self):
        if self._dense is None and self._dev_dense is not None:
            self._dense = np.asfortranarray(
                self._dev_dense[:, : self.n_rows].cpu().numpy().T)
        return self._dense

    def _host_csc(self):
        if self._csc is None and self._dev_csc is not None:
            cp, ri, va = (t.cpu().numpy() for t in self._dev_csc)
            self._csc = (cp.astype(np.int64), ri.astype(np.int32), va.astype(np.float32))
        return self._csc

    def column(self, j):
        if self.storage_kind == "dense":
            return self._host_dense()[:, j]
        ptr, idx, val = self._host_csc()
        return idx[ptr[j]:ptr[j + 1]].astype(np.intp), val[ptr[j]:ptr[j + 1]].astype(np.float64)

    def to_dense(self):
        if self.storage_kind == "dense":
            return self._host_dense().astype(np.float64)
        out = np.zeros((self.n_rows, self.n_cols), order="F")
        ptr, idx, val = self._host_csc()
        for j in range(self.n_cols):
            out[idx[ptr[j]:ptr[j + 1]], j] = val[ptr[j]:ptr[j + 1]]
        return out

    def csc(self):
        """(col_ptr int64, row_idx int32, values float32) host arrays."""
        if self.storage_kind != "sparse":
            raise ValueError("not a sparse matrix")
        return self._host_csc()

    def nnz(self):
        if self.storage_kind == "dense":
            if self._dense is not None:
                return int(np.count_nonzero(self._dense))
            return int((self._dev_dense[:, : self.n_rows] != 0).sum().item())
        if self._csc is not None:
            return int(self._csc[0][-1])
        return int(self._dev_csc[0][-1].item())


@dataclass
class LabeledDataset:
    """A ColumnMatrix plus labels: one per shared-vector row in the feature
    orientation, one per column in the example (dual) orientation
    (dataset.py:132-157)."""

    matrix: ColumnMatrix
    labels: np.ndarray
    orientation: str = COORDINATES_ARE_FEATURES

    def __post_init__(self):
        if self.orientation not in (COORDINATES_ARE_FEATURES, COORDINATES_ARE_EXAMPLES):
            raise ValueError(f"unknown orientation: {self.orientation}")
        self.labels = np.ascontiguousarray(self.labels, dtype=np.float64)
        expected = (self.matrix.n_rows if self.orientation == COORDINATES_ARE_FEATURES
                    else self.matrix.n_cols)
        if self.labels.shape != (expected,):
            raise ValueError("label count does not match dataset orientation")
        if not np.all(np.isfinite(self.labels)):
            raise ValueError("non-finite labels")


@dataclass
class DatasetStats:
    """Per-column squared norms plus the spectral constant (dataset.py:160-166)."""

    column_sq_norms: np.ndarray
    c_A: float
    max_col_sq_norm: float


def compute_stats(matrix, with_spectral=False, power_iters=200, tol=1e-9):
    """Column squared norms on the GPU (dataset.py:307).  c_A (the power
    iteration of dataset.py:308-321) is theory-only; it runs on the GPU when
    requested, else c_A is NaN."""
    from .device import column_sq_norms, spectral_constant
    sq = column_sq_norms(matrix)
    c_a = spectral_constant(matrix, power_iters, tol) if with_spectral else float("nan")
    return DatasetStats(column_sq_norms=sq, c_A=c_a, max_col_sq_norm=float(sq.max()))


# ---------------------------------------------------------------------------
# reference-style synthetic generators (dataset.py:262-295), same streams
# ---------------------------------------------------------------------------
_SYNTH_DENSE, _SYNTH_SPARSE, _SYNTH_LABELS = 100, 101, 102


def _rng(seed, tag):
    return np.random.default_rng(np.random.SeedSequence(seed, spawn_key=(tag,)))


def generate_synthetic_dense(n_examples, n_features, seed):
    if n_examples < 1 or n_features < 1:
        raise ValueError("n_examples and n_features must be >= 1")
    data = np.asfortranarray(_rng(seed, _SYNTH_DENSE).random((n_examples, n_features)))
    labels = _rng(seed, _SYNTH_LABELS).integers(0, 2, size=n_examples) * 2.0 - 1.0
    return LabeledDataset(ColumnMatrix(n_examples, n_features, dense=data), labels)


def generate_synthetic_sparse(n_examples, n_features, density, seed):
    if n_examples < 1 or n_features < 1:
        raise ValueError("n_examples and n_features must be >= 1")
    if not (0.0 < density <= 1.0):
        raise ValueError("density must be in (0, 1]")
    g = _rng(seed, _SYNTH_SPARSE)
    cols = []
    for _ in range(n_features):
        idx = np.nonzero(g.random(n_examples) < density)[0]
        cols.append((idx, g.random(idx.size)))
    labels = _rng(seed, _SYNTH_LABELS).integers(0, 2, size=n_examples) * 2.0 - 1.0
    return LabeledDataset(ColumnMatrix(n_examples, n_features, sparse_cols=cols), labels)


# ---------------------------------------------------------------------------
# LIBSVM text ingest / export (dataset.py:169-259)
# ---------------------------------------------------------------------------
def _nonfinite_column(ptr, vals):
    bad = np.flatnonzero(~np.isfinite(vals))
    return int(np.searchsorted(ptr, bad[0], side="right") - 1)


def load_libsvm(path, n_features=None, orientation=COORDINATES_ARE_FEATURES, n_threads=0):
    """Parse a LIBSVM text file (1-based ascending feature indices) into a
    LabeledDataset in the requested orientation (dataset.py:169-233).

    The text is parsed by the library's multi-threaded host parser
    (syscd_libsvm_scan / syscd_libsvm_fill); the errors are the reference's
    ValueErrors with the same line numbers and messages.  The feature
    orientation transposes the example-major arrays into CSC (rows of a
    column ascending).  Values are stored float32 like every ColumnMatrix;
    labels stay float64.
    """
    import ctypes
    from . import _lib
    if orientation not in (COORDINATES_ARE_FEATURES, COORDINATES_ARE_EXAMPLES):
        raise ValueError(f"unknown orientation: {orientation}")
    with open(path, "rb") as fh:
        buf = fh.read()
    cbuf = ctypes.cast(ctypes.c_char_p(buf), ctypes.c_void_p)
    info = _lib.LibsvmInfo()
    _lib.call("syscd_libsvm_scan", cbuf, len(buf), int(n_threads), ctypes.byref(info))
    if info.err:
        line = info.err_line
        tok = buf[info.err_tok_off:info.err_tok_off + info.err_tok_len].decode(errors="replace")
        msg = {
            1: f"bad label {tok!r}",
            2: f"bad entry {tok!r}",
            3: f"index {info.err_index} is not 1-based",
            4: "indices not ascending",
            5: f"index {info.err_index} exceeds the int32 row-index store",
        }[info.err]
        raise ValueError(f"line {line}: {msg}")
    nex, nnz = int(info.n_examples), int(info.nnz)
    if nex == 0:
        raise ValueError("empty dataset")
    nfeat = max(int(info.max_feature), n_features or 0)
    if nfeat == 0:
        raise ValueError("dataset has no features")
    labels = np.empty(nex, dtype=np.float64)
    ex_ptr = np.empty(nex + 1, dtype=np.int64)
    feat = np.empty(max(nnz, 1), dtype=np.int32)
    vals = np.empty(max(nnz, 1), dtype=np.float64)
    _lib.call("syscd_libsvm_fill", cbuf, len(buf), int(n_threads), labels.ctypes.data,
              ex_ptr.ctypes.data, feat.ctypes.data, vals.ctypes.data)
    feat, vals = feat[:nnz], vals[:nnz]
    if orientation == COORDINATES_ARE_EXAMPLES:
        if not np.all(np.isfinite(vals)):
            raise ValueError(f"column {_nonfinite_column(ex_ptr, vals)}: non-finite values")
        matrix = ColumnMatrix(nfeat, nex, csc=(ex_ptr, feat, vals))
        return LabeledDataset(matrix, labels, orientation)
    col_ptr = np.empty(nfeat + 1, dtype=np.int64)
    rows = np.empty(max(nnz, 1), dtype=np.int32)
    cvals = np.empty(max(nnz, 1), dtype=np.float64)
    _lib.call("syscd_csr_transpose", nex, nfeat, ex_ptr.ctypes.data, feat.ctypes.data,
              vals.ctypes.data, col_ptr.ctypes.data, rows.ctypes.data, cvals.ctypes.data)
    rows, cvals = rows[:nnz], cvals[:nnz]
    if not np.all(np.isfinite(cvals)):
        raise ValueError(f"column {_nonfinite_column(col_ptr, cvals)}: non-finite values")
    matrix = ColumnMatrix(nex, nfeat, csc=(col_ptr, rows, cvals))
    return LabeledDataset(matrix, labels, orientation)


def save_libsvm(dataset, path):
    """Write a feature-oriented LabeledDataset as LIBSVM text with 17
    significant digits (dataset.py:236-259), so a reload reproduces the
    stored values exactly."""
    from . import _lib
    if dataset.orientation != COORDINATES_ARE_FEATURES:
        raise ValueError("save_libsvm expects the feature orientation")
    m = dataset.matrix
    if m.storage_kind == "dense":
        dense = m._host_dense()
        rr, cc = np.nonzero(dense.T)  # column-major walk: (feature, example)
        order = np.lexsort((rr, cc))
        feats, exs = rr[order], cc[order]
        vals = dense[exs, feats].astype(np.float64)
        ex_ptr = np.zeros(m.n_rows + 1, dtype=np.int64)
        np.add.at(ex_ptr, exs + 1, 1)
        ex_ptr = np.cumsum(ex_ptr)
    else:
        col_ptr, rows, cvals = m.csc()
        nnz = int(col_ptr[-1])
        ex_ptr = np.empty(m.n_rows + 1, dtype=np.int64)
        feats = np.empty(max(nnz, 1), dtype=np.int32)
        vals = np.empty(max(nnz, 1), dtype=np.float64)
        cv64 = np.ascontiguousarray(cvals, dtype=np.float64)
        _lib.call("syscd_csr_transpose", m.n_cols, m.n_rows, np.ascontiguousarray(col_ptr).ctypes.data,
                  np.ascontiguousarray(rows).ctypes.data, cv64.ctypes.data, ex_ptr.ctypes.data,
                  feats.ctypes.data, vals.ctypes.data)
        feats, vals = feats[:nnz], vals[:nnz]
    with open(path, "w") as fh:
        for i in range(m.n_rows):
            a, b = ex_ptr[i], ex_ptr[i + 1]
            toks = ["%.17g" % dataset.labels[i]]
            toks += ["%d:%.17g" % (int(j) + 1, float(v)) for j, v in zip(feats[a:b], vals[a:b])]
            fh.write(" ".join(toks) + "\n")
