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
