"""Multi-GPU host logic on CPU with gloo, world size 2: every rank's shard
covers its nodes' buckets exactly once, the union over ranks is the whole
problem, and the per-round exchange (all-reduce of dv) reproduces the
reference's global reduction v + sum_k (v_k - v) (solvers.py:423)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_07722_b200.sharding import shard_plan
        n, B, K, P, seed = 203, 8, 4, 2, 11
        sp = shard_plan(n, B, K, P, seed, world, rank)
        # per-rank node replicas of a fake round: node k contributes dv_k = (k+1) * e_k-ish
        d = 17
        g = np.random.default_rng(5)
        dv_nodes = g.standard_normal((K, d))
        local = dv_nodes[sp.node0:sp.node0 + sp.K_local].sum(axis=0)
        t = torch.from_numpy(local.copy())
        tdist.all_reduce(t)
        q.put((rank, sp.store_cols.tolist(), sp.node0, sp.K_local, sp.n_store, t.numpy().tolist(),
               dv_nodes.sum(axis=0).tolist()))
    finally:
        tdist.destroy_process_group()


def test_two_rank_sharding_and_reduction(built_lib):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cols = [c for _, sc, _, _, _, _, _ in out for c in sc]
    assert sorted(cols) == list(range(203))           # every coordinate exactly once
    assert [o[2] for o in out] == [0, 2] and all(o[3] == 2 for o in out)
    assert sum(o[4] for o in out) == 203
    for o in out:                                      # all-reduce == serial node sum
        np.testing.assert_allclose(o[5], o[6], rtol=1e-12)


@pytest.mark.parametrize("n_gpus", [1, 2, 4, 8])
def test_bench_workloads_shard_over_n_gpus(built_lib, n_gpus):
    """bench.py --gpus N: every BASELINE config keeps K*P at its one-GPU value
    (within rounding), uses K = N node groups, and shards into N disjoint
    stores covering every coordinate once."""
    from paper_1911_07722_b200.configs import _dims, default_solver
    from paper_1911_07722_b200.sharding import shard_plan
    for cfg_id in range(5):
        one = default_solver(cfg_id, 1)
        cfg = default_solver(cfg_id, n_gpus)
        assert cfg.K == n_gpus
        assert cfg.K * cfg.P <= one.K * one.P * max(1, n_gpus)
        if cfg_id != 3:  # config 3 is K = GPUs, P = 1 by definition
            assert abs(cfg.K * cfg.P - one.K * one.P) < n_gpus
        d, n = _dims(cfg_id, 0.01 if cfg_id != 1 else 0.001)
        B = cfg.resolved_bucket_size()
        if cfg.K * cfg.P > -(-n // B):
            continue  # the scaled-down stand-in has too few buckets for this split
        cols = []
        for r in range(n_gpus):
            sp = shard_plan(n, B, cfg.K, cfg.P, cfg.seed, n_gpus, r)
            cols.extend(sp.store_cols.tolist() if sp.store_cols is not None else range(n))
        assert sorted(cols) == list(range(n))


SHARD_CASES = [(0, 0.05), (1, 0.0002), (2, 0.01), (3, 0.002), (4, 0.00005)]


def _shard_worker(rank, world, port, q):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from host_gen import HostGen
        from paper_1911_07722_b200.configs import _dims, shard_arrays
        from paper_1911_07722_b200.device import Dist
        from paper_1911_07722_b200.sharding import shard_plan
        out = {}
        for cfg_id, scale in SHARD_CASES:
            d, n = _dims(cfg_id, scale)
            sp = shard_plan(n, 4, 2, 1, 0, world, rank)
            arr = shard_arrays(cfg_id, scale, 0, cols=sp.store_cols, dist=Dist(), gen=HostGen(),
                               device="cpu")
            held = arr["csc"][0].numel() - 1 if "csc" in arr else arr["At"].shape[0]
            mat = (arr["csc"][1].reshape(held, -1) if "csc" in arr else arr["At"]).numpy()
            out[cfg_id] = dict(cols=sp.store_cols.tolist(), held=int(held), mat=mat.tolist(),
                               y=arr["y"].tolist() if "y" in arr else None,
                               labels=arr["labels"].tolist() if "labels" in arr else None,
                               lam=arr["lam"])
        q.put((rank, out))
    finally:
        tdist.destroy_process_group()


def test_two_rank_shard_local_generation(built_lib):
    """Each rank generates only its own store columns (O(shard) memory: the
    held matrix has exactly n_store columns); the shards are the columns of
    the one-process matrix, and y / lambda / labels (reduced over the ranks)
    equal the one-process values."""
    from host_gen import HostGen
    from paper_1911_07722_b200.configs import shard_arrays
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for cfg_id, scale in SHARD_CASES:
        full = shard_arrays(cfg_id, scale, 0, gen=HostGen(), device="cpu")
        n = full["n"]
        fm = (full["csc"][1].reshape(n, -1) if "csc" in full else full["At"]).numpy()
        seen = []
        for r in range(world):
            o = out[r][cfg_id]
            assert o["held"] == len(o["cols"]) < n          # a strict shard
            np.testing.assert_array_equal(np.array(o["mat"]), fm[o["cols"]])
            seen += o["cols"]
            if o["y"] is not None:
                np.testing.assert_allclose(o["y"], full["y"].numpy(), rtol=1e-12, atol=1e-12)
            else:
                np.testing.assert_array_equal(o["labels"], full["labels"].numpy()[o["cols"]])
            assert abs(o["lam"] - full["lam"]) <= 1e-12 * full["lam"]
        assert sorted(seen) == list(range(n))
