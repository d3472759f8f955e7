"""Data-parallel training over NCCL on 2 GPUs (skipped with fewer): the
trainer's in-graph allreduce of [grad | loss | 1] and the world-size division
inside Adam (train.py:257-262, comm.py:55-77).

* identical batch on both ranks -> parameters bitwise equal to a 1-GPU step
  (x + x = 2x and / 2 are exact);
* different halves of one batch (equal graph and atom counts) -> the same
  update as a 1-GPU step on the union, within the 3xTF32 bar;
* ranks stay bitwise identical to each other (NCCL returns identical bytes);
* the deterministic (rank-ordered all-gather) mode agrees bitwise with the
  default mode for world size 2 (a + b == b + a).
"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _structures(seed, B=8, n=12):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0, 6.0, size=(B * n, 3))
    z = rng.choice(np.array([1, 6, 8]), size=B * n).astype(np.int32)
    e = rng.normal(size=B) * 3.0
    f = rng.normal(size=(B * n, 3))
    return pos, z, e, f


def _step(comm, pos, z, e, f, B, n, steps=2, optimizer="adam", bucket_bytes=4 << 20,
          idle=False, lr=1e-3):
    from oracle import gfm_oracle as O
    from paper_2406_12909_b200 import model as M, train as T

    cfg = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=2, mpnn_width=32, fc_layers=2,
                        fc_width=16)
    flat = O.init_flat(O.config("pna-agg", layers=2, hidden=32, fc_layers=2, fc_width=16), 5)
    tr = T.DataParallelTrainer(cfg, T.TrainConfig(optimizer=optimizer, learning_rate=lr),
                               comm=comm, initial=flat, bucket_bytes=bucket_bytes)
    if idle:  # a rank without a batch (train.py:257-259: zero contribution)
        for _ in range(steps):
            tr.compute(None)
            tr.reduce_and_update()
        return tr.flat_master(), tr.bucketed
    run = T.StructureStepRunner(tr, np.arange(B + 1) * n, 3.0, 8, use_graph=True)
    dev = tr.device
    for _ in range(steps):
        run.step(torch.as_tensor(pos, device=dev), torch.as_tensor(z, device=dev),
                 torch.as_tensor(e, dtype=torch.float32, device=dev),
                 torch.as_tensor(f, dtype=torch.float32, device=dev))
    return tr.flat_master(), tr.bucketed


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    import torch.distributed as dist

    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2406_12909_b200.comm import TorchComm

        comm = TorchComm(deterministic=(mode == "deterministic"))
        pos, z, e, f = _structures(1)
        B, n = 8, 12
        bb = 8 << 10 if mode.endswith("bucketed") else 4 << 20  # several buckets
        if mode.startswith("halves"):  # rank r trains on graphs [4r, 4r + 4)
            h = B // world
            sl = slice(rank * h * n, (rank + 1) * h * n)
            out = _step(comm, pos[sl], z[sl], e[rank * h:(rank + 1) * h], f[sl], h, n,
                        optimizer="sgd", bucket_bytes=bb)
        elif mode.startswith("idle"):  # rank 1 has no batch
            out = _step(comm, pos, z, e, f, B, n, optimizer="sgd", bucket_bytes=bb,
                        idle=rank == 1)
        else:
            out = _step(comm, pos, z, e, f, B, n, bucket_bytes=bb)
        torch.cuda.synchronize()
        comm.barrier()
        q.put((rank, out))
        q.close()
        q.join_thread()  # flush the result before the hard exit below
    finally:
        dist.barrier()
        os._exit(0)  # NCCL communicators captured in CUDA graphs: skip teardown


def _run(mode):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, (out, bucketed) = q.get(timeout=180)
        res[r] = out
        res[f"bucketed{r}"] = bucketed
    for p in procs:
        p.join(timeout=60)
    return res


need2 = pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")


@need2
def test_dp_identical_batches_bitwise_equal_single_gpu():
    from paper_2406_12909_b200.comm import LocalComm

    res = _run("same")
    np.testing.assert_array_equal(res[0], res[1])
    pos, z, e, f = _structures(1)
    single, _ = _step(LocalComm(), pos, z, e, f, 8, 12)
    np.testing.assert_array_equal(res[0], single)


@need2
def test_dp_halves_match_single_gpu_union():
    from paper_2406_12909_b200.comm import LocalComm

    res = _run("halves")
    np.testing.assert_array_equal(res[0], res[1])
    pos, z, e, f = _structures(1)
    single, _ = _step(LocalComm(), pos, z, e, f, 8, 12, optimizer="sgd")
    # SGD: the update is linear in the gradient, so the DP mean of the two
    # half-batch gradients must equal the union gradient (equal graph and
    # atom counts per half) to the 3xTF32 bar, floored at 1% of the max
    from oracle import gfm_oracle as O
    flat = O.init_flat(O.config("pna-agg", layers=2, hidden=32, fc_layers=2, fc_width=16), 5)
    du, ds = res[0] - flat, single - flat
    denom = np.maximum(np.abs(ds), 1e-2 * np.abs(ds).max())
    assert (np.abs(du - ds) / denom).max() <= 5e-4


@need2
def test_dp_deterministic_mode_matches_default():
    a = _run("deterministic")
    b = _run("same")
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[0], a[1])


@need2
def test_dp_bucketed_allreduce_matches_single_allreduce():
    """gradients bucketed (8 KB buckets -> several) and allreduced on a comm
    stream while the backward runs == one allreduce after the backward,
    bitwise (elementwise sums do not depend on the slicing)"""
    a = _run("halves_bucketed")
    b = _run("halves")
    assert a["bucketed0"] and a["bucketed1"] and not b["bucketed0"]
    np.testing.assert_array_equal(a[0], a[1])
    np.testing.assert_array_equal(a[0], b[0])


@need2
def test_dp_idle_rank_runs_the_same_bucket_sequence():
    """rank 1 without a batch contributes zeros through the same bucket
    sequence (train.py:257-259); SGD update = half of rank 0's gradient"""
    from paper_2406_12909_b200.comm import LocalComm

    res = _run("idle_bucketed")
    assert res["bucketed0"] and res["bucketed1"]
    np.testing.assert_array_equal(res[0], res[1])
    pos, z, e, f = _structures(1)
    single, _ = _step(LocalComm(), pos, z, e, f, 8, 12, optimizer="sgd", lr=0.5e-3)
    np.testing.assert_array_equal(res[0], single)
