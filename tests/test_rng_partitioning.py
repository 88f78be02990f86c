"""RNG contract and partitioning mirror against the reference's golden vectors
(tests/golden/rng_kat.json, partition_kat.json from make_golden.py)."""
import numpy as np
import pytest

from paper_1911_07722_b200 import partitioning as P


def test_permutations_bit_exact(built_lib, golden):
    for case in golden("rng_kat.json")["permutations"]:
        got = P.RngStream(case["seed"], tuple(case["key"])).permutation(case["n"])
        assert got.tolist() == case["perm"], case["key"]


def test_integers_bit_exact(built_lib, golden):
    for case in golden("rng_kat.json")["integers"]:
        got = P.RngStream(case["seed"], tuple(case["key"])).integers(case["lo"], case["hi"], 12)
        assert got.tolist() == case["draws"]


def test_large_permutation_matches_numpy(built_lib):
    for n, key in [(131077, (1, 0, 4)), (62500, (1, 0, 29))]:
        ref = np.random.default_rng(np.random.SeedSequence(3, spawn_key=key)).permutation(n)
        assert np.array_equal(P.RngStream(3, key).permutation(n), ref)


def test_static_and_dynamic_partitions(built_lib, golden):
    g = golden("partition_kat.json")
    for c in g["static"]:
        part = P.static_node_partition(P.build_buckets(c["n"], c["B"]), c["K"],
                                       P.RngStream(c["seed"], (0,)))
        assert [list(a) for a in part.assignment] == c["assignment"]
    for c in g["dynamic"]:
        asg = P.dynamic_repartition(tuple(c["buckets"]), c["P"],
                                    P.RngStream(c["seed"], (1, c["k"], c["rid"])))
        assert [list(a) for a in asg.assignment] == c["assignment"]
    for c in g["within"]:
        perm = P.permute_within_bucket((c["lo"], c["hi"]),
                                       P.RngStream(c["seed"], (2, c["rid"], c["b"])))
        assert perm.tolist() == c["coords"]


def test_layout_and_errors(built_lib):
    lay = P.build_buckets(100, 8)
    assert lay.n_buckets == 13 and lay.range_of(12) == (96, 100)
    assert P.default_bucket_size() == 8 and P.default_bucket_size(128) == 16
    assert P.default_bucket_size(4) == 1
    with pytest.raises(ValueError):
        P.build_buckets(0, 8)
    with pytest.raises(ValueError):
        P.static_node_partition(P.build_buckets(16, 8), 3, P.RngStream(0, (0,)))
    with pytest.raises(ValueError):
        P.dynamic_repartition((1, 2), 3, P.RngStream(0, (1,)))
    with pytest.raises(ValueError):
        P.dynamic_repartition((), 1, P.RngStream(0, (1,)))
    with pytest.raises(ValueError):
        P.permute_within_bucket((4, 4), P.RngStream(1, (2,)))


def test_balance_sizes(built_lib):
    part = P.static_node_partition(P.build_buckets(80, 8), 4, P.RngStream(3, (0,)))
    assert sorted(len(a) for a in part.assignment) == [2, 2, 3, 3]
    asg = P.dynamic_repartition(tuple(range(20, 31)), 4, P.RngStream(0, (1, 0, 5)))
    assert sorted(len(a) for a in asg.assignment) == [2, 3, 3, 3]
