"""Thread ranks driving GPUs from one process (the reference's thread mode,
cli.py:297-311): the device allreduce (peer copies + float64 sum in rank
order) gives every rank identical bytes == the ordered sum; data-parallel
SGD over two thread ranks on halves of a batch == one rank on the union
(3xTF32 bar) with both ranks' parameters bitwise equal.  Two ranks share
cuda:0 on a 1-GPU box, else use cuda:0 and cuda:1 (NVLink peer copies)."""

import threading

import numpy as np
import pytest
import torch

from oracle import gfm_oracle as O

from paper_2406_12909_b200 import model as M, train as T
from paper_2406_12909_b200.comm import LocalComm, create_thread_comms

pytestmark = pytest.mark.gpu


def _devices():
    return [0, 1] if torch.cuda.device_count() >= 2 else [0, 0]


def _threads(fn, size=2):
    comms = create_thread_comms(size, timeout=120)
    devs = _devices()
    out, err = [None] * size, []

    def work(r):
        try:
            torch.cuda.set_device(devs[r])
            out[r] = fn(comms[r], torch.device("cuda", devs[r]))
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            err.append(e)
            comms[r]._hub.barrier.abort()

    ts = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    if err:
        raise err[0]
    return out


def test_device_allreduce_ordered_and_identical():
    rng = np.random.default_rng(0)
    vals = [rng.standard_normal(100_003).astype(np.float32) for _ in range(2)]

    def fn(c, dev):
        t = torch.as_tensor(vals[c.rank], device=dev)
        c.allreduce_sum_(t)
        return t.cpu().numpy()

    a, b = _threads(fn)
    want = (vals[0].astype(np.float64) + vals[1].astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(a, want)
    np.testing.assert_array_equal(a, b)


def _structures(seed, B=8, n=12):
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0, 6.0, size=(B * n, 3))
    z = rng.choice(np.array([1, 6, 8]), size=B * n).astype(np.int32)
    return pos, z, rng.normal(size=B) * 3.0, rng.normal(size=(B * n, 3))


def _train(comm, dev, pos, z, e, f, B, n):
    cfg = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=2, mpnn_width=32, fc_layers=2,
                        fc_width=16)
    flat = O.init_flat(O.config("pna-agg", layers=2, hidden=32, fc_layers=2, fc_width=16), 5)
    tr = T.DataParallelTrainer(cfg, T.TrainConfig(optimizer="sgd", learning_rate=1e-3),
                               comm=comm, initial=flat, device=dev)
    run = T.StructureStepRunner(tr, np.arange(B + 1) * n, 3.0, 8, use_graph=True)
    for _ in range(2):
        run.step(torch.as_tensor(pos, device=dev), torch.as_tensor(z, device=dev),
                 torch.as_tensor(e, dtype=torch.float32, device=dev),
                 torch.as_tensor(f, dtype=torch.float32, device=dev))
    return tr.flat_master(), flat


def test_thread_ranks_halves_match_union():
    pos, z, e, f = _structures(1)
    B, n, h = 8, 12, 4

    def fn(c, dev):
        sl = slice(c.rank * h * n, (c.rank + 1) * h * n)
        return _train(c, dev, pos[sl], z[sl], e[c.rank * h:(c.rank + 1) * h], f[sl], h, n)

    (p0, flat), (p1, _) = _threads(fn)
    np.testing.assert_array_equal(p0, p1)
    single, _ = _train(LocalComm(), torch.device("cuda", 0), pos, z, e, f, B, n)
    du, ds = p0 - flat, single - flat
    denom = np.maximum(np.abs(ds), 1e-2 * np.abs(ds).max())
    assert (np.abs(du - ds) / denom).max() <= 5e-4


class _Store:
    def __init__(self, groups):
        self._g = groups
        self.ownership = {k: type("O", (), {"n_samples": len(v)})() for k, v in groups.items()}

    def fetch_batch(self, group, idx):
        return [self._g[group][int(i)] for i in idx]


def _groups():
    from paper_2406_12909_b200.records import GraphRecord
    dicts = O.synthetic(14, n_atoms_range=(4, 12), seed=8)
    recs = [GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"]) for d in dicts]
    return {"trainset": recs[:11], "valset": recs[11:]}


def _train_cfg():
    return (M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=2, mpnn_width=16, fc_width=16,
                          batch_size=3), T.TrainConfig(max_epochs=2, patience=5))


def _nccl_worker(rank, world, port, q):
    import os
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        from paper_2406_12909_b200.comm import TorchComm
        mc, cfg = _train_cfg()
        res = T.train(mc, _Store(_groups()), comm=TorchComm(deterministic=True), config=cfg)
        q.put((rank, res.params.flatten(), [m.train_loss for m in res.metrics]))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e), None))
    q.close()
    q.join_thread()
    os._exit(0)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_thread_ranks_train_equals_nccl_processes():
    """train() with two thread ranks (create_thread_comms) == train() with two
    NCCL processes in deterministic mode, bitwise: both sum the [grad | loss
    | 1] payload in ascending rank order in float64"""
    import socket

    import torch.multiprocessing as mp
    mc, cfg = _train_cfg()

    def fn(c, dev):
        res = T.train(mc, _Store(_groups()), comm=c, config=cfg)
        return res.params.flatten(), [m.train_loss for m in res.metrics]

    thr = _threads(fn)
    np.testing.assert_array_equal(thr[0][0], thr[1][0])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (a, b)) for r, a, b in (q.get(timeout=300) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
    assert not isinstance(out[0][0], str), out[0][0]
    np.testing.assert_array_equal(out[0][0], thr[0][0])
    assert out[0][1] == thr[0][1]
