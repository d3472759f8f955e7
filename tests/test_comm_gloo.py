"""Multi-process collectives on CPU (gloo, world size 2): the TorchComm that
carries the DP gradient allreduce, in deterministic (rank-ordered) and
default modes, plus the control collectives the train loop uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_12909_b200.comm import TorchComm
    from paper_2406_12909_b200.errors import ValidationError
    try:
        rng = np.random.default_rng(100 + rank)
        vec = rng.normal(size=257) * 10.0 ** rng.integers(-8, 8, size=257)
        det = TorchComm(deterministic=True)
        out_det = det.allreduce_sum(vec)
        fast = TorchComm(deterministic=False)
        t = torch.as_tensor(vec.astype(np.float32))
        fast.allreduce_sum_(t)
        bc = fast.broadcast_obj("budget" if rank == 0 else None)
        gathered = fast.gather_obj(rank * 10)
        mismatch = False
        try:
            det.allreduce_sum(np.zeros(3 + rank))
        except ValidationError:
            mismatch = True
        det.barrier()
        q.put((rank, out_det, t.numpy(), bc, gathered, mismatch))
    finally:
        dist.destroy_process_group()


def test_two_rank_allreduce_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    vecs = []
    for r in range(world):
        rng = np.random.default_rng(100 + r)
        vecs.append(rng.normal(size=257) * 10.0 ** rng.integers(-8, 8, size=257))
    want = vecs[0].copy()
    want += vecs[1]  # ascending rank order (comm.py:143-147)
    for r in range(world):
        np.testing.assert_array_equal(res[r][1], want)          # bitwise ordered sum
        np.testing.assert_array_equal(res[r][2], res[0][2])     # identical bytes on every rank
        assert res[r][3] == "budget"
        assert res[r][5]                                       # count mismatch detected
    assert res[0][4] == [0, 10]
    assert res[1][4] is None


# ---------------------------------------------------------------- buckets
def test_bucket_plan_partitions_payload_in_production_order():
    """plan_buckets (train.py): contiguous buckets of whole gradient groups
    that exactly tile [grad | loss | 1], launched in the backward's order"""
    from paper_2406_12909_b200 import model as M
    from paper_2406_12909_b200.train import plan_buckets

    for L, H, kind, bb in ((6, 512, "pna-agg", 4 << 20), (3, 64, "pna-agg", 4 << 20),
                           (4, 64, "mean-agg", 20_000), (2, 32, "max-agg", 1)):
        cfg = M.ModelConfig(mpnn_kind=kind, mpnn_layers=L, mpnn_width=H, fc_width=H)
        lay = M.param_layout(cfg)
        bs = plan_buckets(lay, cfg, bb)
        spans = sorted((b.lo, b.hi) for b in bs)
        assert spans[0][0] == 0 and spans[-1][1] == lay.Pp + 2
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert sorted(b.order for b in bs) == list(range(len(bs)))
        groups = [g for b in sorted(bs, key=lambda b: b.order) for g in b.groups]
        assert sorted(groups) == sorted(["loss", "head", "force", "embedding"]
                                        + [f"layer{l}" for l in range(L)])
        # the embedding (the backward's last gradient) is in the last bucket
        assert "embedding" in max(bs, key=lambda b: b.order).groups
    cfg = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=6, mpnn_width=512, fc_width=512)
    assert len(plan_buckets(M.param_layout(cfg), cfg, 4 << 20)) == 6


def _bucket_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_12909_b200 import model as M
    from paper_2406_12909_b200.comm import TorchComm
    from paper_2406_12909_b200.train import plan_buckets
    try:
        cfg = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=3, mpnn_width=64, fc_width=64)
        lay = M.param_layout(cfg)
        rng = np.random.default_rng(7 + rank)
        vec = torch.as_tensor(rng.normal(size=lay.Pp + 2).astype(np.float32))
        comm = TorchComm()
        whole = vec.clone()
        comm.allreduce_sum_(whole)
        sliced = vec.clone()
        for b in sorted(plan_buckets(lay, cfg, 40_000), key=lambda b: b.order):
            comm.allreduce_sum_(sliced[b.lo:b.hi])
        q.put((rank, whole.numpy(), sliced.numpy()))
    finally:
        dist.destroy_process_group()


def test_bucketed_allreduce_equals_whole_vector_gloo():
    """the bucket sequence reduces to exactly the bytes of one whole-vector
    allreduce (elementwise sums do not depend on the slicing)"""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=120)
        res[r[0]] = r
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for r in range(world):
        np.testing.assert_array_equal(res[r][1], res[r][2])
        np.testing.assert_array_equal(res[r][2], res[0][2])
