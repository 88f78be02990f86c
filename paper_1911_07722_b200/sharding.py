"""Static sharding of buckets over GPUs (the NUMA-node level of SySCD).

The reference deals shuffled buckets to K node groups once per run
(static_node_partition, partitioning.py:89-96, key (0,)) and every node
re-partitions its own buckets over its P threads each round
(partitioning.py:99-109).  On a multi-GPU run the node groups are spread over
the ranks: rank r owns nodes [r*K/W, (r+1)*K/W), gathers exactly those
buckets' columns into its own store (in node order), and the only exchange per
round is the all-reduce of dv (solvers.py:423).

shard_plan() is pure host logic (no device), so it is covered by the
world-size-2 gloo tests on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .partitioning import NODE_PARTITION, RngStream, build_buckets, static_node_partition


@dataclass
class ShardPlan:
    K: int
    K_local: int
    node0: int
    buckets: np.ndarray          # global bucket ids of the local nodes, node order
    node_ptr: np.ndarray         # [K_local+1] offsets into buckets
    bucket_store_col: np.ndarray  # store column of each listed bucket's first coordinate
    store_cols: np.ndarray | None  # global column of every store column (None: identity)
    n_store: int


def shard_plan(n, B, K, P, seed, world=1, rank=0):
    layout = build_buckets(n, B)
    if K * P > layout.n_buckets:
        raise ValueError(f"K*P={K * P} exceeds the bucket count {layout.n_buckets}")
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank / world size")
    if K % world != 0:
        raise ValueError(f"K={K} node groups cannot be split over {world} GPUs")
    k_local = K // world
    node0 = rank * k_local
    part = static_node_partition(layout, K, RngStream(seed, (NODE_PARTITION,)))
    nodes = part.assignment[node0:node0 + k_local]
    for nb in nodes:
        if P > len(nb):
            raise ValueError("more threads than buckets on this node")
    buckets = np.array([b for nb in nodes for b in nb], dtype=np.int64)
    ptr = np.zeros(k_local + 1, dtype=np.int32)
    np.cumsum([len(nb) for nb in nodes], out=ptr[1:])
    if world == 1:
        return ShardPlan(K, k_local, node0, buckets, ptr, buckets * B, None, n)
    store_col, store_cols = _bucket_columns(buckets, B, n)
    return ShardPlan(K, k_local, node0, buckets, ptr, store_col, store_cols, int(store_cols.size))


def _bucket_columns(buckets, B, n):
    """(store column of each bucket's first coordinate, global column of every
    store column) for buckets laid out back to back in the given order."""
    lo = buckets * B
    lens = np.minimum(lo + B, n) - lo
    store_col = np.zeros(buckets.size, dtype=np.int64)
    np.cumsum(lens[:-1], out=store_col[1:])
    grid = lo[:, None] + np.arange(B, dtype=np.int64)[None, :]
    store_cols = grid[grid < np.minimum(lo + B, n)[:, None]]
    return store_col, store_cols


def all_store_cols(n, B, K, P, seed, world):
    """Every rank's store columns (rank order): what an all-gather of the
    per-rank alpha shards is scattered by."""
    return [shard_plan(n, B, K, P, seed, world, r).store_cols for r in range(world)]
