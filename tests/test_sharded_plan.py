"""Sharded store host logic (CPU): the ownership map of DDStore
(ddstore.py:95-165, container.py:253-268) and the fetch plan of the
collective exchange -- owner-grouped requests, per-owner counts, and the
permutation that puts the owners' answers back in request order."""

import numpy as np
import pytest

from paper_2406_12909_b200.errors import ConfigError, ValidationError
from paper_2406_12909_b200.store import OwnershipMap, partition_for_readers, plan_fetch


@pytest.mark.parametrize("n,r", [(0, 3), (1, 4), (10, 3), (12, 4), (7, 7), (5, 8)])
def test_partition_contiguous_balanced(n, r):
    rs = partition_for_readers(n, r)
    assert len(rs) == r and rs[0][0] == 0 and rs[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
    sizes = [hi - lo for lo, hi in rs]
    assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)


def test_ownership_replica_subgroups():
    o = OwnershipMap(10, 4, replication_factor=2)
    assert o.group_size == 2 and o.local_ranges == [(0, 5), (5, 10)]
    assert list(o.owners(range(10), 0)) == [0] * 5 + [1] * 5
    assert list(o.owners(range(10), 3)) == [2] * 5 + [3] * 5  # caller's own sub-group
    assert o.range_of(3) == (5, 10) and o.owner_of(7, 1) == 1
    with pytest.raises(ConfigError):
        OwnershipMap(10, 4, replication_factor=3)
    with pytest.raises(ValidationError):
        o.owners([10], 0)


def test_ownership_empty_chunks_skip_to_next_owner():
    o = OwnershipMap(6, 4, chunk_sizes=[0, 2, 0, 4])
    assert list(o.owners(range(6), 0)) == [1, 1, 3, 3, 3, 3]
    o = OwnershipMap(2, 4)  # fewer samples than ranks: trailing empty ranges
    assert list(o.owners([0, 1], 2)) == [0, 1]
    with pytest.raises(ConfigError):
        OwnershipMap(6, 2, chunk_sizes=[1, 2])


@pytest.mark.parametrize("world,rf", [(1, 1), (3, 1), (4, 2), (4, 4)])
def test_plan_fetch_round_trip(world, rf):
    """simulate the all_to_all exchange on the host: each owner answers its
    requests in arrival order; the requester's permutation restores the
    request order exactly (duplicates and empty requests included)"""
    rng = np.random.default_rng(world)
    n = 37
    own = OwnershipMap(n, world, rf)
    reqs = [rng.integers(0, n, size=rng.integers(0, 9)) for _ in range(world)]
    reqs[0] = np.array([5, 5, 36, 0], np.int64)
    plans = [plan_fetch(reqs[r], own, r, world) for r in range(world)]
    # owner o receives from every requester r the slice of r's grouped list
    served = {}
    for r, (grouped, counts, _) in enumerate(plans):
        starts = np.concatenate([[0], np.cumsum(counts)])
        for o in range(world):
            part = grouped[starts[o]:starts[o + 1]]
            lo, hi = own.range_of(o)
            assert ((part >= lo) & (part < hi)).all()  # only owned indices
            if part.size:
                assert own.subgroup_of(o) == own.subgroup_of(r)
            served[(o, r)] = part * 1000 + o  # "payload" tagged with its owner
    for r, (grouped, counts, arrival_to_batch) in enumerate(plans):
        arrival = np.concatenate([served[(o, r)] for o in range(world)]) if world else []
        got = np.asarray(arrival)[arrival_to_batch] // 1000
        np.testing.assert_array_equal(got, reqs[r])
        assert counts.sum() == len(reqs[r])
