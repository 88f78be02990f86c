"""ctypes binding of libsyscd_b200.so (include/syscd_b200.h).

The library is built in-tree (paper_1911_07722_b200/csrc/build.py).  There is
no fallback: if the library is missing or a CUDA device is required and
absent, the call fails loudly.
"""

from __future__ import annotations

import ctypes
import os

from .objective import NonFiniteUpdateError

_HERE = os.path.dirname(os.path.abspath(__file__))
# SYSCD_TRACE=1 selects the instrumented build (per-event %globaltimer stamps,
# scripts/timeline*.py only); the product is always libsyscd_b200.so
LIB_PATH = os.path.join(_HERE, "libsyscd_b200_trace.so" if os.environ.get("SYSCD_TRACE")
                        else os.environ.get("SYSCD_LIB_NAME", "libsyscd_b200.so"))

SYSCD_OK, SYSCD_EINVAL, SYSCD_ENONFINITE, SYSCD_ECUDA = 0, 1, 2, 3
RIDGE, LOGISTIC, LASSO, SVM_DUAL, LOGISTIC_DUAL = 0, 1, 2, 3, 4

c_i32, c_i64, c_u64, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                     ctypes.c_double, ctypes.c_void_p)


class PlanDesc(ctypes.Structure):
    _fields_ = [
        ("seed", c_u64), ("n_global", c_i64), ("bucket_size", c_i32), ("n_nodes_local", c_i32),
        ("node0", c_i32), ("P", c_i32), ("T3", c_i32), ("T4", c_i32), ("sampling", c_i32),
        ("repartition", c_i32), ("node_bucket_ptr", ctypes.POINTER(c_i32)),
        ("node_buckets", c_vp), ("bucket_store_col", c_vp), ("round_updates", c_vp),
    ]


class DenseEpochArgs(ctypes.Structure):
    _fields_ = [
        ("kind", c_i32), ("d", c_i64), ("lda", c_i64), ("A", c_vp), ("sq", c_vp),
        ("alpha", c_vp), ("u", c_vp), ("seq", c_vp), ("work_prefix", c_vp), ("n_parts", c_i32),
        ("a", c_f64), ("lam", c_f64), ("n_coords", c_f64), ("iid", c_i32), ("n_store", c_i64),
        ("partials", c_vp), ("part_ld", c_i64), ("status", c_vp), ("workspace", c_vp),
        ("workspace_bytes", c_i64),
    ]


class SparseEpochArgs(ctypes.Structure):
    _fields_ = [
        ("kind", c_i32), ("d", c_i64), ("col_ptr", c_vp), ("row_idx", c_vp), ("vals", c_vp),
        ("sq", c_vp), ("alpha", c_vp), ("u", c_vp), ("seq", c_vp), ("work_prefix", c_vp),
        ("n_parts", c_i32), ("a", c_f64), ("lam", c_f64), ("n_coords", c_f64), ("iid", c_i32),
        ("dv_work", c_vp), ("n_workers", c_i32), ("delta_v", c_vp), ("status", c_vp),
        ("replica_tag", ctypes.c_uint32),
    ]


class LibsvmInfo(ctypes.Structure):
    _fields_ = [
        ("n_examples", c_i64), ("nnz", c_i64), ("max_feature", c_i64), ("err", c_i32),
        ("pad_", c_i32), ("err_line", c_i64), ("err_tok_off", c_i64), ("err_tok_len", c_i64),
        ("err_index", c_i64),
    ]


class WildEpochArgs(ctypes.Structure):
    _fields_ = [
        ("kind", c_i32), ("d", c_i64), ("lda", c_i64), ("A", c_vp), ("col_ptr", c_vp),
        ("row_idx", c_vp), ("vals", c_vp), ("sq", c_vp), ("alpha", c_vp), ("u", c_vp),
        ("dv", c_vp), ("perm", c_vp), ("n", c_i64), ("P", c_i32), ("gamma", c_f64),
        ("lam", c_f64), ("n_coords", c_f64), ("status", c_vp),
    ]


class ExactArgs(ctypes.Structure):
    _fields_ = [
        ("d", c_i64), ("lda", c_i64), ("A", c_vp), ("col_ptr", c_vp), ("row_idx", c_vp),
        ("vals", c_vp), ("sq", c_vp), ("alpha", c_vp), ("v", c_vp), ("y", c_vp), ("lam", c_f64),
        ("seq", c_vp), ("work_prefix", c_vp), ("status", c_vp),
    ]


# (name, restype, argtypes) for every symbol declared in include/syscd_b200.h
SIGNATURES = {
    "syscd_abi_version": (c_i32, []),
    "syscd_last_error": (ctypes.c_char_p, []),
    "syscd_rng_permutation": (c_i32, [c_u64, ctypes.POINTER(c_u64), c_i32, c_i64, c_vp]),
    "syscd_rng_integers": (c_i32, [c_u64, ctypes.POINTER(c_u64), c_i32, c_i64, c_i64, c_i64, c_vp]),
    "syscd_plan_workspace_bytes": (c_i64, [ctypes.POINTER(PlanDesc), c_i32]),
    "syscd_plan_max_updates": (c_i64, [ctypes.POINTER(PlanDesc)]),
    "syscd_plan": (c_i32, [ctypes.POINTER(PlanDesc), c_i64, c_i32, c_vp, c_i64, c_vp, c_vp, c_i64,
                           c_vp]),
    "syscd_dense_epoch_workers": (c_i32, [c_i64, c_i32, ctypes.POINTER(c_i32),
                                          ctypes.POINTER(c_i32)]),
    "syscd_dense_epoch_workspace_bytes": (c_i64, [c_i64, c_i32]),
    "syscd_dense_epoch": (c_i32, [ctypes.POINTER(DenseEpochArgs), c_vp]),
    "syscd_sparse_epoch_workers": (c_i32, [c_i64, c_i32, ctypes.POINTER(c_i32)]),
    "syscd_sparse_epoch": (c_i32, [ctypes.POINTER(SparseEpochArgs), c_vp]),
    "syscd_exact_logistic_round": (c_i32, [ctypes.POINTER(ExactArgs), c_vp]),
    "syscd_reduce_partials": (c_i32, [c_vp, c_i64, c_i32, c_i64, c_vp, c_vp]),
    "syscd_apply_dv": (c_i32, [c_i32, c_i64, c_vp, c_vp, c_vp, c_f64, c_f64, c_vp, c_vp]),
    "syscd_grad": (c_i32, [c_i32, c_i64, c_vp, c_vp, c_f64, c_f64, c_vp, c_f64, c_vp, c_vp]),
    "syscd_dual_point": (c_i32, [c_i32, c_i64, c_vp, c_vp, c_f64, c_f64, c_vp, c_vp]),
    "syscd_node_delta": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_i32, c_vp]),
    "syscd_vec_add": (c_i32, [c_i64, c_vp, c_vp, c_vp]),
    "syscd_dense_matvec": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "syscd_dense_rmatvec": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "syscd_dense_col_sq_norms": (c_i32, [c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "syscd_sparse_matvec": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "syscd_sparse_rmatvec": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "syscd_sparse_col_sq_norms": (c_i32, [c_i64, c_vp, c_vp, c_vp, c_vp]),
    "syscd_objective_terms": (c_i32, [c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_f64, c_f64, c_vp,
                                      c_vp, c_vp]),
    "syscd_gap_terms": (c_i32, [c_i32, c_i64, c_i64, c_vp, c_vp, c_vp, c_f64, c_f64, c_f64, c_vp,
                                c_vp, c_vp]),
    "syscd_wild_epoch": (c_i32, [ctypes.POINTER(WildEpochArgs), c_vp]),
    "syscd_libsvm_scan": (c_i32, [c_vp, c_i64, c_i32, ctypes.POINTER(LibsvmInfo)]),
    "syscd_libsvm_fill": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp, c_vp]),
    "syscd_csr_transpose": (c_i32, [c_i64, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "syscd_gen_normal_cols": (c_i32, [c_u64, ctypes.c_uint32, c_vp, c_i64, c_i64, c_i64, c_vp,
                                      c_vp]),
    "syscd_gen_ids": (c_i32, [c_u64, ctypes.c_uint32, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "syscd_gen_zipf_onehot": (c_i32, [c_u64, ctypes.c_uint32, c_vp, c_i64, c_i64, c_i32, c_vp,
                                      c_vp, c_vp, c_vp]),
}

_lib = None


def lib():
    """Load (once) and return the CDLL; raises if the library is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        dll = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(dll, name)
            fn.restype = res
            fn.argtypes = args
        if dll.syscd_abi_version() != 1:
            raise RuntimeError("libsyscd_b200.so ABI version mismatch")
        _lib = dll
    return _lib


def check(status, what=""):
    """Map a C-ABI status to the reference's exception types."""
    if status == SYSCD_OK:
        return
    msg = lib().syscd_last_error().decode(errors="replace")
    if status == SYSCD_EINVAL:
        raise ValueError(f"{what}: {msg}" if what else msg)
    if status == SYSCD_ENONFINITE:
        raise NonFiniteUpdateError(f"{what}: non-finite update {msg}".strip())
    raise RuntimeError(f"{what}: CUDA error {msg}")


def call(name, *args):
    check(getattr(lib(), name)(*args), name)
