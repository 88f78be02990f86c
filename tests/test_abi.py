"""The C-ABI library loads and exports every symbol include/syscd_b200.h declares."""
import ctypes
import os
import re

from conftest import ROOT


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "syscd_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(syscd_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(built_lib):
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(built_lib, name), f"{name} declared but not exported"


def test_binding_covers_header():
    from paper_1911_07722_b200._lib import SIGNATURES
    assert set(declared_symbols()) == set(SIGNATURES)


def test_abi_version_and_errors(built_lib):
    from paper_1911_07722_b200._lib import PlanDesc
    assert built_lib.syscd_abi_version() == 1
    d = PlanDesc()  # all zero -> invalid, rejected before any device work
    assert built_lib.syscd_plan_workspace_bytes(ctypes.byref(d), 1) == -1
    assert b"invalid" in built_lib.syscd_last_error()


def test_plan_sizes_host_only(built_lib):
    from paper_1911_07722_b200._lib import PlanDesc
    d = PlanDesc()
    d.seed, d.n_global, d.bucket_size, d.n_nodes_local, d.P = 0, 100, 8, 1, 2
    d.T3, d.T4, d.sampling, d.repartition = -1, -1, 0, 0
    ptr = (ctypes.c_int32 * 2)(0, 13)
    d.node_bucket_ptr = ptr
    assert built_lib.syscd_plan_max_updates(ctypes.byref(d)) == 13 * 8
    assert built_lib.syscd_plan_workspace_bytes(ctypes.byref(d), 4) > 0
    d.P = 14  # more threads than buckets on the node (partitioning.py:105-106)
    assert built_lib.syscd_plan_max_updates(ctypes.byref(d)) == -1
