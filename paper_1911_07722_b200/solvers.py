"""SySCD solver entry points on the GPU (mirror of pkg/src/syscd/solvers.py).

run_syscd(problem, cfg, f_star) keeps the reference's signature, parameter
contract (SolverConfig, solvers.py:44-88), result types (EpochMetrics,
TrainResult, solvers.py:91-109), error behaviour (ValueError on bad
configurations, NonFiniteUpdateError on a non-finite step, divergence as a
result flag) and per-round structure (solvers.py:400-443):

  round t1:  plan (device RNG, partitioning.py)  ->  epoch kernel (all K*P
             partitions, private replicas)  ->  replica reduction  ->
             [multi-GPU: NCCL all-reduce of dv]  ->  v += dv, u = grad f(v)
  metrics:   fresh A alpha on the GPU, fp64 (excluded from the epoch time,
             as the reference's `elapsed` is taken before _metrics_row).

Everything on the path runs in libsyscd_b200.so; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from ._lib import (DenseEpochArgs, ExactArgs, PlanDesc, SparseEpochArgs, WildEpochArgs, call,
                   check, lib)
from .device import DeviceProblem, Dist, _ptr, _stream, _torch
from .objective import LOGISTIC, NonFiniteUpdateError
from .partitioning import DEFAULT_CACHE_LINE_BYTES, default_bucket_size
from .sharding import shard_plan

DIVERGENCE_FACTOR = 1e6


@dataclass
class SolverConfig:
    algorithm: str = "syscd"
    K: int = 1                      # node groups (GPUs x logical nodes per GPU)
    P: int = 1                      # threads (partitions) per node group
    bucket_size: int | None = None  # None: cache_line_bytes / 8
    cache_line_bytes: int = DEFAULT_CACHE_LINE_BYTES
    T1: int | None = None           # fixed outer round count; None: run to tolerance
    T2: int = 1                     # node-local rounds per global round
    T3: int | None = None           # buckets per thread per round; None: all assigned
    T4: int | None = None           # updates per bucket; None: bucket length (perm) / B (iid)
    sampling: str = "perm"
    repartition: str = "dynamic"
    seed: int = 0
    max_epochs: int = 100
    tolerance: float = 1e-5
    verify: bool = False
    record_alpha: bool = False
    # extensions; defaults keep the reference's behaviour
    compute_gap: bool = False       # add the duality gap to every metrics row
    metrics_every: int = 1          # evaluate metrics every k rounds (and the last)
    plan_batch: int = 8             # rounds planned per device planning launch

    def __post_init__(self):
        if self.algorithm not in ("sequential", "wild", "syscd"):
            raise ValueError(f"unknown algorithm: {self.algorithm}")
        if self.K < 1 or self.P < 1 or self.T2 < 1:
            raise ValueError("K, P and T2 must be >= 1")
        if self.T3 is not None and self.T3 < 1:
            raise ValueError("T3 must be >= 1")
        if self.T4 is not None and self.T4 < 1:
            raise ValueError("T4 must be >= 1")
        if self.sampling not in ("perm", "iid"):
            raise ValueError(f"unknown sampling mode: {self.sampling}")
        if self.repartition not in ("dynamic", "static"):
            raise ValueError(f"unknown repartition mode: {self.repartition}")
        if self.tolerance <= 0.0:
            raise ValueError("tolerance must be > 0")
        if self.max_epochs < 0:
            raise ValueError("max_epochs must be >= 0")
        if self.metrics_every < 1 or self.plan_batch < 1:
            raise ValueError("metrics_every and plan_batch must be >= 1")

    def resolved_bucket_size(self):
        if self.bucket_size is not None:
            return self.bucket_size
        return default_bucket_size(self.cache_line_bytes)

    @property
    def n_rounds(self):
        return self.T1 if self.T1 is not None else self.max_epochs


@dataclass
class EpochMetrics:
    epoch: int
    objective: float
    suboptimality: float | None
    seconds: float
    updates: int
    rel_change: float
    gap: float | None = None


@dataclass
class TrainResult:
    alpha: np.ndarray
    metrics: list
    converged: bool
    total_updates: int
    diverged: bool = False
    reason: str | None = None
    alpha_snapshots: list = field(default_factory=list)


def reduce_replicas(base, replicas):
    """base + sum_r (replica_r - base), ascending r (solvers.py:112-125).

    Host helper kept for API parity; the solver reduces device replicas with
    syscd_reduce_partials in the same ascending order."""
    base = np.asarray(base, dtype=np.float64)
    if not replicas:
        raise ValueError("need at least one replica")
    for r in replicas:
        if np.shape(r) != base.shape:
            raise ValueError("replica length mismatch")
    if len(replicas) == 1:
        return np.array(replicas[0], dtype=np.float64)
    acc = np.zeros_like(base)
    for r in replicas:
        acc += np.asarray(r, dtype=np.float64) - base
    return base + acc


# ---------------------------------------------------------------------------
# GPU engine
# ---------------------------------------------------------------------------
class _Engine:
    """Buffers and launches for one problem shard and one configuration."""

    def __init__(self, problem, cfg, dist):
        torch = _torch()
        self.torch = torch
        self.cfg = cfg
        self.dist = dist
        n = problem.n_coordinates
        B = cfg.resolved_bucket_size()
        sp = shard_plan(n, B, cfg.K, cfg.P, cfg.seed, dist.world, dist.rank)
        self.shard = sp
        self.K_local = sp.K_local
        self.node0 = sp.node0
        buckets = sp.buckets
        ptr = sp.node_ptr
        store_col = sp.bucket_store_col
        if sp.store_cols is None:
            if problem._device is None:
                problem._device = DeviceProblem(problem, dist=dist)
            self.dp = problem._device
        elif problem.data.matrix.global_cols is not None:
            # shard-local problem: it holds exactly this rank's columns
            if problem._device is None or not np.array_equal(problem._device.store_cols,
                                                             sp.store_cols):
                problem._device = DeviceProblem(problem, store_cols=sp.store_cols, dist=dist)
            self.dp = problem._device
        else:
            # full problem on every rank: gather this rank's columns
            self.dp = DeviceProblem(problem, store_cols=sp.store_cols, dist=dist)
        dp = self.dp
        self.single = cfg.K == 1 and cfg.P == 1
        # K=P=1 primal logistic: exact Newton updates on the live v
        # (solvers.py:403-410); every other objective's exact update is the
        # surrogate step with a = gamma and runs in the epoch kernels
        self.exact_logistic = self.single and dp.kind == LOGISTIC
        self.a = dp.gamma * cfg.P * cfg.K
        self.n_parts_local = self.K_local * cfg.P
        # planning
        self._ptr_host = ptr
        self._buckets_dev = torch.from_numpy(np.asarray(buckets, dtype=np.int32)).cuda()
        self._store_col_dev = torch.from_numpy(store_col).cuda()
        self.desc = PlanDesc()
        self.desc.seed = int(cfg.seed)
        self.desc.n_global = int(n)
        self.desc.bucket_size = int(B)
        self.desc.n_nodes_local = int(self.K_local)
        self.desc.node0 = int(self.node0)
        self.desc.P = int(cfg.P)
        self.desc.T3 = -1 if cfg.T3 is None else int(cfg.T3)
        self.desc.T4 = -1 if cfg.T4 is None else int(cfg.T4)
        self.desc.sampling = 0 if cfg.sampling == "perm" else 1
        self.desc.repartition = 0 if cfg.repartition == "dynamic" else 1
        self._ptr_c = (ctypes.c_int32 * (self.K_local + 1))(*ptr.tolist())
        self.desc.node_bucket_ptr = self._ptr_c
        self.desc.node_buckets = self._buckets_dev.data_ptr()
        self.desc.bucket_store_col = self._store_col_dev.data_ptr()
        L = lib()
        self.stride = int(L.syscd_plan_max_updates(ctypes.byref(self.desc)))
        if self.stride < 0:
            call("syscd_plan_max_updates")
        self.R = max(1, min(cfg.plan_batch, cfg.n_rounds * cfg.T2 if cfg.n_rounds else 1))
        # per-round update counts, written by the planner (round_updates[rid]);
        # sized for every round plus the batch planned ahead of the last one
        self.upd_dev = torch.zeros(max(1, cfg.n_rounds * cfg.T2) + 2 * self.R + 1,
                                   dtype=torch.int64, device="cuda")
        self.desc.round_updates = self.upd_dev.data_ptr()
        ws = int(L.syscd_plan_workspace_bytes(ctypes.byref(self.desc), self.R))
        # double-buffered round tables: batch b+1 is planned on a side stream
        # while batch b's epochs run (the permutations are data-independent)
        self.bufs = [_PlanBuf(torch, self.R, self.stride, self.n_parts_local, ws)
                     for _ in range(2)]
        self.cur = 0
        self.side = torch.cuda.Stream()
        # workers
        d = dp.d
        if dp.storage == "dense":
            counts = {self.n_parts_local, cfg.P}
            self.n_workers = max(self._dense_workers(d, c)[0] for c in counts)
            self.cluster = self._dense_workers(d, self.n_parts_local)[1]
            self.part_ld = (d + 31) // 32 * 32
            self.partials = torch.empty(self.n_workers * self.part_ld, dtype=torch.float32,
                                        device="cuda")
            wsb = max(int(lib().syscd_dense_epoch_workspace_bytes(d, c)) for c in counts)
            self.epoch_ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
        else:
            nw = ctypes.c_int32(0)
            call("syscd_sparse_epoch_workers", d, self.n_parts_local, ctypes.byref(nw))
            self.n_workers = nw.value
            self.cluster = 1
            # tagged replica words (tag << 32 | fp32), zero-filled once
            self.dv_work = torch.zeros(self.n_workers * d, dtype=torch.int64, device="cuda")
            self.replica_tag = 1
            self.part_ld = d
            self.partials = torch.empty(d, dtype=torch.float32, device="cuda")
        self.alpha = torch.zeros(dp.n_store, dtype=torch.float32, device="cuda")
        self.v = torch.zeros(d, dtype=torch.float64, device="cuda")
        # u is read by 16-byte bulk copies up to round_up(d, 4): pad it
        self._u_buf = torch.zeros((d + 3) // 4 * 4, dtype=torch.float32, device="cuda")
        self.u = self._u_buf[:d]
        self.dv = torch.empty(d, dtype=torch.float32, device="cuda")
        self.status = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.kernel_events = None  # (start, stop) CUDA events around the epoch kernel
        self.plans_issued = 0      # syscd_plan calls (3 kernel launches each)
        self.launches = 0          # our kernel launches issued (bench accounting)
        dp.grad_into(self.v, self.u)
        # the per-round hot path reuses one argument struct and raw pointers
        self._lib = lib()
        self._workers_for = {}
        self._p_partials = _ptr(self.partials)
        self._p_dv = _ptr(self.dv)
        self._p_v = _ptr(self.v)
        self._p_u = _ptr(self.u)
        self._p_y = _ptr(dp.y)
        if dp.storage == "dense":
            e = DenseEpochArgs()
            e.kind = dp.kind
            e.d = dp.d
            e.lda = dp.lda
            e.A = dp.At.data_ptr()
            e.sq = dp.sq.data_ptr()
            e.alpha = self.alpha.data_ptr()
            e.a = self.a
            e.lam = dp.lam
            e.n_coords = dp.n_coords
            e.iid = 1 if cfg.sampling == "iid" else 0
            e.n_store = dp.n_store
            e.partials = self.partials.data_ptr()
            e.part_ld = self.part_ld
            e.status = self.status.data_ptr()
            e.workspace = self.epoch_ws.data_ptr()
            e.workspace_bytes = self.epoch_ws.numel()
            self._dargs = e
            self._dargs_ref = ctypes.byref(e)

    @staticmethod
    def _dense_workers(d, n_parts):
        nw = ctypes.c_int32(0)
        cl = ctypes.c_int32(0)
        call("syscd_dense_epoch_workers", d, n_parts, ctypes.byref(nw), ctypes.byref(cl))
        return nw.value, cl.value

    # -- one device round (rid) over node range [k0, k1) with lin_vec u -------
    def _plan(self, buf, rid0, stream):
        if rid0 + self.R > self.upd_dev.numel():
            # more rounds than configured (rare): grow the count table once
            self.torch.cuda.synchronize()
            grown = self.torch.zeros(2 * (rid0 + self.R), dtype=self.torch.int64, device="cuda")
            grown[:self.upd_dev.numel()].copy_(self.upd_dev)
            self.torch.cuda.synchronize()
            self.upd_dev = grown
            self.desc.round_updates = grown.data_ptr()
        call("syscd_plan", ctypes.byref(self.desc), int(rid0), self.R, _ptr(buf.seq), self.stride,
             _ptr(buf.wp), _ptr(buf.ws), buf.ws.numel(), ctypes.c_void_p(stream.cuda_stream))
        buf.lo, buf.hi = rid0, rid0 + self.R
        buf.ready.record(stream)
        self.plans_issued += 1

    def _ensure_plan(self, rid):
        """Buffer and row holding round rid's tables (rounds are consumed in
        increasing order; the next batch is prefetched on the side stream)."""
        torch = self.torch
        cur = self.bufs[self.cur]
        if cur.lo is not None and cur.lo <= rid < cur.hi:
            return cur, rid - cur.lo
        main = torch.cuda.current_stream()
        nxt = self.bufs[1 - self.cur]
        if nxt.lo is not None and nxt.lo <= rid < nxt.hi:
            main.wait_event(nxt.ready)
        else:
            # re-plan into nxt: its last consumer (free) AND its last writer
            # (ready: recorded after every plan, also the side-stream
            # prefetch queued after free was recorded) must be done
            main.wait_event(nxt.free)
            main.wait_event(nxt.ready)
            self._plan(nxt, rid, main)
        cur.free.record(main)
        self.cur = 1 - self.cur
        # prefetch the following batch into the buffer just released
        self.side.wait_event(cur.free)
        self._plan(cur, nxt.hi, self.side)
        return nxt, rid - nxt.lo

    def round_ptrs(self, rid):
        """Raw device pointers of round rid's seq and work_prefix rows."""
        buf, r = self._ensure_plan(rid)
        return (buf.seq_ptr + 4 * r * self.stride,
                buf.wp_ptr + 8 * r * (self.n_parts_local + 1))

    def round_tables(self, rid):
        buf, r = self._ensure_plan(rid)
        seq = buf.seq[r * self.stride:]
        wp = buf.wp[r * (self.n_parts_local + 1):(r + 1) * (self.n_parts_local + 1)]
        return seq, wp

    def epoch(self, rid, u, node_lo=0, node_hi=None):
        """Run the partitions of local nodes [node_lo, node_hi) of round rid with
        lin_vec u; leaves their summed replicas in self.dv."""
        cfg, dp = self.cfg, self.dp
        node_hi = self.K_local if node_hi is None else node_hi
        seq_ptr, wp_ptr = self.round_ptrs(rid)
        p0 = node_lo * cfg.P
        nparts = (node_hi - node_lo) * cfg.P
        stream = _stream()
        if dp.storage == "dense":
            e = self._dargs
            e.u = u.data_ptr()
            e.seq = seq_ptr
            e.work_prefix = wp_ptr + 8 * p0
            e.n_parts = nparts
            if self.kernel_events is not None:
                self.kernel_events[0].record()
            check(self._lib.syscd_dense_epoch(self._dargs_ref, stream), "syscd_dense_epoch")
            if self.kernel_events is not None:
                self.kernel_events[1].record()
            nw = self._workers_for.get(nparts)
            if nw is None:
                nw = self._workers_for[nparts] = self._dense_workers(dp.d, nparts)[0]
            check(self._lib.syscd_reduce_partials(self._p_partials, self.part_ld, nw, dp.d,
                                                  self._p_dv, stream), "syscd_reduce_partials")
        else:
            cp, ri, va = dp.csc
            e = SparseEpochArgs()
            e.kind = dp.kind
            e.d = dp.d
            e.col_ptr = cp.data_ptr()
            e.row_idx = ri.data_ptr()
            e.vals = va.data_ptr()
            e.sq = dp.sq.data_ptr()
            e.alpha = self.alpha.data_ptr()
            e.u = u.data_ptr()
            e.seq = seq_ptr
            e.work_prefix = wp_ptr + 8 * p0
            e.n_parts = nparts
            e.a = self.a
            e.lam = dp.lam
            e.n_coords = dp.n_coords
            e.iid = 1 if cfg.sampling == "iid" else 0
            e.dv_work = self.dv_work.data_ptr()
            if self.replica_tag + nparts >= 1 << 32:  # tag space wrapped: re-zero
                self.dv_work.zero_()
                self.replica_tag = 1
            e.replica_tag = self.replica_tag
            self.replica_tag += nparts
            e.n_workers = self.n_workers
            e.delta_v = self.dv.data_ptr()
            e.status = self.status.data_ptr()
            if self.kernel_events is not None:
                self.kernel_events[0].record()
            call("syscd_sparse_epoch", ctypes.byref(e), _stream())
            if self.kernel_events is not None:
                self.kernel_events[1].record()

    def exact_round(self, rid):
        """K=P=1 primal logistic round: exact updates on the live v."""
        dp = self.dp
        seq, wp = self.round_tables(rid)
        e = ExactArgs()
        e.d = dp.d
        if dp.storage == "dense":
            e.lda = dp.lda
            e.A = dp.At.data_ptr()
        else:
            cp, ri, va = dp.csc
            e.col_ptr, e.row_idx, e.vals = cp.data_ptr(), ri.data_ptr(), va.data_ptr()
        e.sq = dp.sq.data_ptr()
        e.alpha = self.alpha.data_ptr()
        e.v = self.v.data_ptr()
        e.y = dp.y.data_ptr()
        e.lam = dp.lam
        e.seq = seq.data_ptr()
        e.work_prefix = wp.data_ptr()
        e.status = self.status.data_ptr()
        call("syscd_exact_logistic_round", ctypes.byref(e), _stream())

    def global_round(self, t1):
        """One outer round (solvers.py:401-424)."""
        cfg, dp = self.cfg, self.dp
        torch = self.torch
        if self.exact_logistic:
            for t2 in range(cfg.T2):
                self.exact_round(t1 * cfg.T2 + t2)
            return
        if cfg.T2 == 1:
            self.epoch(t1, self.u)
            if self.dist.world > 1:
                self.dist.allreduce_(self.dv)
            check(self._lib.syscd_apply_dv(dp.kind, dp.d, self._p_dv, self._p_v, self._p_y,
                                           dp.lam, dp.n_coords, self._p_u, _stream()),
                  "syscd_apply_dv")
            return
        # T2 > 1: node-local rounds with the drift term (solvers.py:373-398).
        # Nodes are independent within a global round, so the node loop is the
        # inner one: round ids are consumed in increasing order (the plan
        # tables are prefetched in that order) with one v_node per local node.
        drift = cfg.K * dp.gamma
        delta_sum = torch.empty(dp.d, dtype=torch.float64, device="cuda")
        u_k = torch.zeros_like(self._u_buf)[:dp.d]
        v_nodes = [self.v.clone() for _ in range(self.K_local)]
        for t2 in range(cfg.T2):
            rid = t1 * cfg.T2 + t2
            for k in range(self.K_local):
                v_node = v_nodes[k]
                if t2 == 0:
                    u_k.copy_(self.u)
                else:
                    dp.grad_into(self.v, u_k, v_node=v_node, drift=drift)
                self.epoch(rid, u_k, k, k + 1)
                call("syscd_apply_dv", dp.kind, dp.d, _ptr(self.dv), _ptr(v_node), None, dp.lam,
                     dp.n_coords, None, _stream())
        for k, v_node in enumerate(v_nodes):  # ascending node order (solvers.py:423)
            call("syscd_node_delta", dp.d, _ptr(v_node), self._p_v, _ptr(delta_sum), int(k == 0),
                 _stream())
        self.dist.allreduce_(delta_sum)
        call("syscd_vec_add", dp.d, self._p_v, _ptr(delta_sum), _stream())
        dp.grad_into(self.v, self.u)

    def updates_last_round(self, rid):
        return int(self.upd_dev[rid].item())

    def check_status(self):
        st = int(self.status.item())
        if st & 2:
            self.status.zero_()
            raise NonFiniteUpdateError("non-finite coordinate update")

    def census_ok(self, rid):
        seq, wp = self.round_tables(rid)
        self.torch.cuda.synchronize()
        tot = int(wp[self.n_parts_local].item())
        s = seq[:tot]
        return int(torch_unique_count(s)) == tot

    def alpha_global(self):
        """alpha in global coordinate order, fp64 host array: an all-gather
        of the per-rank shards (each rank sends only its n_store values)."""
        dp = self.dp
        if self.dist.world == 1:
            return self.alpha.double().cpu().numpy()
        torch = self.torch
        if getattr(self, "_rank_cols", None) is None:
            from .sharding import all_store_cols
            cfg = self.cfg
            self._rank_cols = all_store_cols(dp.n_global, cfg.resolved_bucket_size(), cfg.K, cfg.P,
                                             cfg.seed, self.dist.world)
        m = max(c.size for c in self._rank_cols)
        buf = torch.zeros(m, dtype=torch.float32, device="cuda")
        buf[:dp.n_store] = self.alpha
        parts = self.dist.allgather(buf)
        full = np.empty(dp.n_global)
        for cols, part in zip(self._rank_cols, parts):
            full[cols] = part[:cols.size].double().cpu().numpy()
        return full


class _PlanBuf:
    def __init__(self, torch, R, stride, n_parts, ws_bytes):
        self.seq = torch.empty(R * max(1, stride), dtype=torch.int32, device="cuda")
        self.wp = torch.empty(R * (n_parts + 1), dtype=torch.int64, device="cuda")
        self.seq_ptr = self.seq.data_ptr()
        self.wp_ptr = self.wp.data_ptr()
        self.ws = torch.empty(max(ws_bytes, 256), dtype=torch.uint8, device="cuda")
        self.lo = self.hi = None
        self.ready = torch.cuda.Event()
        self.free = torch.cuda.Event()
        self.free.record()


def torch_unique_count(t):
    import torch
    return torch.unique(t).numel()


def run_syscd(problem, cfg, f_star=None, dist=None):
    """Hierarchical bucketized SySCD on the GPU (solvers.py:337-453)."""
    if cfg.algorithm != "syscd":
        raise ValueError("config.algorithm must be 'syscd'")
    return _run(problem, cfg, f_star, dist)


def run_sequential_scd(problem, cfg, f_star=None, dist=None):
    """Sequential SCD (solvers.py:181-211): one node, one thread, exact
    updates over the shuffled buckets, i.e. run_syscd's K=P=1 round
    (solvers.py:403-410).  Like the reference it ignores cfg.K / P / T2."""
    if cfg.algorithm != "sequential":
        raise ValueError("config.algorithm must be 'sequential'")
    import dataclasses
    one = dataclasses.replace(cfg, algorithm="syscd", K=1, P=1, T2=1)
    return _run(problem, one, f_star, dist)


def run_wild_parallel_scd(problem, cfg, f_star=None):
    """Asynchronous parallel SCD (solvers.py:214-286) on one GPU.

    Every epoch draws the permutation of all n coordinates with key
    (COORD_PERM, epoch, 0) (:250), splits it like np.array_split into P
    chunks and runs P workers that update the shared alpha and v without
    synchronisation (syscd_wild_epoch; primal logistic runs the chunks back
    to back through the exact Newton kernel).  Metrics, divergence handling
    (a non-finite step or F > 1e6 F(0) ends the run with a diverged row) and
    the stopping rule follow :236-282.
    """
    from .partitioning import COORD_PERM, RngStream, permute_within_bucket
    if cfg.algorithm != "wild":
        raise ValueError("config.algorithm must be 'wild'")
    if cfg.K != 1:
        raise ValueError("wild solver uses a flat thread pool (K must be 1)")
    torch = _torch()
    if problem._device is None:
        problem._device = DeviceProblem(problem, dist=Dist.single())
    dp = problem._device
    n, d = dp.n_global, dp.d
    f32 = torch.float32
    alpha = torch.zeros(dp.n_store, dtype=f32, device="cuda")
    v = torch.zeros(d, dtype=torch.float64, device="cuda")
    u_buf = torch.zeros((d + 3) // 4 * 4, dtype=f32, device="cuda")
    dv_buf = torch.zeros_like(u_buf)
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    perm_host = torch.empty(max(n, 1), dtype=torch.int32, pin_memory=True)
    perm_dev = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    wp = torch.tensor([0, n], dtype=torch.int64, device="cuda")
    dp.grad_into(v, u_buf[:d])
    logistic = dp.kind == LOGISTIC

    def evaluate():
        if cfg.compute_gap:
            gap, obj = dp.gap(alpha)
            return obj, gap
        return dp.objective(alpha), None

    init_obj, gap0 = evaluate()
    metrics = [EpochMetrics(0, init_obj, init_obj - f_star if f_star is not None else None,
                            0.0, 0, np.inf, gap0)]
    snaps = []
    prev = alpha.clone()
    converged = diverged = False
    total = 0
    for epoch in range(cfg.n_rounds):
        t0 = time.perf_counter()
        perm = permute_within_bucket((0, n), RngStream(cfg.seed, (COORD_PERM, epoch, 0)))
        perm_host.numpy()[:n] = perm
        perm_dev.copy_(perm_host, non_blocking=True)
        if logistic:
            e = ExactArgs()
            e.d = dp.d
            if dp.storage == "dense":
                e.lda, e.A = dp.lda, dp.At.data_ptr()
            else:
                cp, ri, va = dp.csc
                e.col_ptr, e.row_idx, e.vals = cp.data_ptr(), ri.data_ptr(), va.data_ptr()
            e.sq, e.alpha, e.v, e.y = (dp.sq.data_ptr(), alpha.data_ptr(), v.data_ptr(),
                                        dp.y.data_ptr())
            e.lam = dp.lam
            e.seq, e.work_prefix, e.status = perm_dev.data_ptr(), wp.data_ptr(), status.data_ptr()
            call("syscd_exact_logistic_round", ctypes.byref(e), _stream())
        else:
            w = WildEpochArgs()
            w.kind, w.d = dp.kind, dp.d
            if dp.storage == "dense":
                w.lda, w.A = dp.lda, dp.At.data_ptr()
            else:
                cp, ri, va = dp.csc
                w.col_ptr, w.row_idx, w.vals = cp.data_ptr(), ri.data_ptr(), va.data_ptr()
            w.sq, w.alpha, w.u, w.dv = (dp.sq.data_ptr(), alpha.data_ptr(), u_buf.data_ptr(),
                                        dv_buf.data_ptr())
            w.perm, w.n, w.P = perm_dev.data_ptr(), n, int(cfg.P)
            w.gamma, w.lam, w.n_coords = dp.gamma, dp.lam, dp.n_coords
            w.status = status.data_ptr()
            call("syscd_wild_epoch", ctypes.byref(w), _stream())
            call("syscd_apply_dv", dp.kind, dp.d, _ptr(dv_buf), _ptr(v), _ptr(dp.y), dp.lam,
                 dp.n_coords, _ptr(u_buf), _stream())
            dv_buf.zero_()
        failed = bool(int(status.item()) & 2)  # synchronises
        elapsed = time.perf_counter() - t0
        upd = n
        total += upd
        finite = bool(torch.isfinite(alpha).all())
        obj, gap = evaluate() if finite else (np.inf, None)
        if failed or not np.isfinite(obj) or obj > DIVERGENCE_FACTOR * max(init_obj, 1e-300):
            metrics.append(EpochMetrics(epoch + 1, obj, None, elapsed, upd, np.inf))
            diverged = True
            break
        rel = _rel_change(alpha, prev)
        prev.copy_(alpha)
        sub = obj - f_star if f_star is not None else None
        metrics.append(EpochMetrics(epoch + 1, obj, sub, elapsed, upd, rel, gap))
        if cfg.record_alpha:
            snaps.append(alpha.double().cpu().numpy())
        if cfg.T1 is None and rel < cfg.tolerance:
            converged = True
            break
    return TrainResult(alpha.double().cpu().numpy(), metrics, converged, total,
                       diverged=diverged, reason="diverged" if diverged else None,
                       alpha_snapshots=snaps)


def run_solver(problem, cfg, f_star=None):
    if cfg.algorithm == "sequential":
        return run_sequential_scd(problem, cfg, f_star=f_star)
    if cfg.algorithm == "wild":
        return run_wild_parallel_scd(problem, cfg, f_star=f_star)
    return run_syscd(problem, cfg, f_star=f_star)


def _rel_change(alpha, prev):
    return float((alpha - prev).abs().max() / max(1.0, float(alpha.abs().max())))


def _run(problem, cfg, f_star, dist):
    torch = _torch()
    dist = dist or Dist()
    eng = _Engine(problem, cfg, dist)
    dp = eng.dp

    def metrics_row(epoch, secs, upd, rel):
        if cfg.compute_gap:
            gap, obj = dp.gap(eng.alpha)
        else:
            obj, gap = dp.objective(eng.alpha), None
        sub = obj - f_star if f_star is not None else None
        return EpochMetrics(epoch, obj, sub, secs, upd, rel, gap)

    metrics = [metrics_row(0, 0.0, 0, np.inf)]
    snaps = []
    prev = eng.alpha.clone()
    converged = diverged = False
    total = 0
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    # With a fixed round count, rounds without a metrics row are queued back
    # to back: no host synchronisation, the update counts stay on the device
    # and prev tracks the previous round's alpha with a device copy.  A
    # non-finite step or alpha is then detected at the next metrics row.
    lazy = cfg.T1 is not None and not cfg.verify and not cfg.record_alpha
    pending = 0  # rounds whose update counts have not been read yet
    for t1 in range(cfg.n_rounds):
        last = t1 == cfg.n_rounds - 1
        row_due = (t1 + 1) % cfg.metrics_every == 0 or last
        start.record()
        eng.global_round(t1)
        stop.record()
        if lazy and not row_due:
            prev.copy_(eng.alpha)
            pending += 1
            continue
        stop.synchronize()
        elapsed = start.elapsed_time(stop) / 1e3
        eng.check_status()
        upd = 0
        for t2 in range(cfg.T2):
            upd += eng.updates_last_round(t1 * cfg.T2 + t2)
        if pending:
            lo = (t1 - pending) * cfg.T2
            total_prev = int(eng.upd_dev[lo:t1 * cfg.T2].sum().item())
        else:
            total_prev = 0
        pending = 0
        cnt = torch.tensor([upd, total_prev], dtype=torch.int64, device="cuda")
        dist.allreduce_(cnt)
        upd, total_prev = int(cnt[0].item()), int(cnt[1].item())
        total += upd + total_prev
        if cfg.verify:
            for t2 in range(cfg.T2):
                if cfg.sampling == "perm" and not eng.census_ok(t1 * cfg.T2 + t2):
                    raise AssertionError("write census: coordinate updated twice in one round")
            vv = dp.matvec(eng.alpha)
            scale = max(1.0, float(vv.abs().max()))
            # fp32 replicas: relative consistency 1e-4 instead of the fp64 1e-8
            if float((vv - eng.v).abs().max()) > 1e-4 * scale:
                raise AssertionError("replica consistency: v != A @ alpha after reduction")
        finite = torch.tensor([float(torch.isfinite(eng.alpha).all())], device="cuda")
        if float(dist.allreduce_(finite, op="sum")) < dist.world:
            metrics.append(EpochMetrics(t1 + 1, np.inf, None, elapsed, upd, np.inf))
            diverged = True
            break
        d_rel = (eng.alpha - prev).abs().max().double().reshape(1)
        m_abs = eng.alpha.abs().max().double().reshape(1)
        dist.allreduce_(d_rel, op="max")
        dist.allreduce_(m_abs, op="max")
        rel = float(d_rel) / max(1.0, float(m_abs))
        prev.copy_(eng.alpha)
        stop_now = cfg.T1 is None and rel < cfg.tolerance
        if row_due or stop_now:
            metrics.append(metrics_row(t1 + 1, elapsed, upd, rel))
        if cfg.record_alpha:
            snaps.append(eng.alpha_global())
        if stop_now:
            converged = True
            break
    return TrainResult(eng.alpha_global(), metrics, converged, total, diverged=diverged,
                       reason="diverged" if diverged else None, alpha_snapshots=snaps)
