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
