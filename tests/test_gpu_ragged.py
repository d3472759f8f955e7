"""Ragged batches through the captured step (StructureStepRunner with a
capacity layout) against the float64 oracle.

The reference batches structures of any size (model.py:234-285,
generate_synthetic's n_atoms_range, preprocess.py:107-153).  Here each step
has its own graph count (up to the capacity; a short batch as the last batch
of an epoch) and atom counts; the captured graph's node capacity is chosen
per batch and the true counts are read from the device.  Bars as
``test_gpu_parity.py``: float64 1e-10, float32 (3xTF32) 5e-4.
"""

import numpy as np
import pytest
import torch

from oracle import gfm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2406_12909_b200 import model as M, train as T  # noqa: E402
from paper_2406_12909_b200.errors import ValidationError  # noqa: E402
from paper_2406_12909_b200.store import DeviceStructureStore  # noqa: E402
from test_gpu_parity import assert_close_scaled, cfg_of  # noqa: E402

F64, F32 = torch.float64, torch.float32
RC, CAP, BOX = 3.0, 8, 6.0


def _batches():
    # three batches: 12 graphs (short), 16 graphs (full), 5 graphs; sizes 1..30
    out = []
    for seed, count in ((1, 12), (2, 16), (3, 5)):
        recs = O.synthetic(count, n_atoms_range=(1, 30), box_length=BOX, rc=RC, seed=seed,
                           max_nbr=CAP)
        rng = np.random.default_rng(seed)
        for r in recs:  # labels far from predictions (kink-free)
            r["energy"] = float(rng.choice([-1, 1]) * (50 + 10 * rng.uniform()) * len(r["z"]))
            r["forces"] = rng.choice([-1, 1], r["forces"].shape) * (30 + rng.uniform(size=r["forces"].shape))
        out.append(recs)
    return out


def _host(recs, dtype):
    off = np.concatenate([[0], np.cumsum([len(r["z"]) for r in recs])])
    return (torch.as_tensor(np.concatenate([r["pos"] for r in recs])),
            torch.as_tensor(np.concatenate([r["z"] for r in recs]).astype(np.int32)),
            torch.as_tensor(np.array([r["energy"] for r in recs]), dtype=dtype),
            torch.as_tensor(np.concatenate([r["forces"] for r in recs]), dtype=dtype), off)


@pytest.mark.parametrize("use_graph", [False, True])
@pytest.mark.parametrize("dtype,rel,floor", [(F64, 1e-10, 1e-3), (F32, 5e-4, 1e-2)],
                         ids=["f64", "f32"])
def test_ragged_runner_matches_oracle(dtype, rel, floor, use_graph):
    kind = "pna-agg"
    cfg = cfg_of(kind, 2, 32, 2, 16)
    ocfg = O.config(kind, 2, 32, 2, 16)
    flat = O.init_flat(ocfg, 5)
    tr = T.DataParallelTrainer(cfg, T.TrainConfig(), initial=flat, dtype=dtype)
    run = T.StructureStepRunner(tr, None, RC, CAP, max_graphs=16, max_atoms=30,
                                node_caps=[200, 480], use_graph=use_graph)
    batches = _batches()
    pos, z, e, f, off = _host(batches[0], dtype)
    run.load(pos, z, e, f, off)
    if use_graph:
        run.capture(warmup=2)
    m = np.zeros_like(flat)
    v = np.zeros_like(flat)
    t = 0
    used = set()
    for recs in batches:
        bo = O.pack(recs)
        (tot, _, _), grad_o, _ = O.loss_and_grad(ocfg, flat, bo)
        pos, z, e, f, off = _host(recs, dtype)
        loss32 = run.step(pos, z, e, f, off)  # the host read-back is float32
        loss = float(tr.contrib[tr.P].item())
        used.add(run.cur.N)
        assert abs(loss - tot) <= rel * abs(tot), (loss, tot)
        assert abs(loss32 - tot) <= 1e-6 * abs(tot)
        assert_close_scaled(tr.flat_grad(), grad_o, rel, floor, what=f"grad B={len(recs)}")
        flat, m, v, t = O.adam(flat, tr.flat_grad() if dtype == F32 else grad_o, m, v, t)
        if dtype == F64:
            np.testing.assert_allclose(tr.flat_master(), flat, rtol=0, atol=1e-12)
        else:
            flat = tr.flat_master()
    assert used == {200, 480}  # both captured capacities ran


def test_ragged_store_feed_matches_direct_load():
    """DeviceStructureStore.load_runner into a ragged runner == loading the
    same structures from host buffers (bitwise parameters after 2 steps)"""
    recs = O.synthetic(40, n_atoms_range=(3, 24), box_length=BOX, rc=RC, seed=8, max_nbr=CAP)
    cfg = cfg_of("pna-agg", 2, 32, 2, 16)
    flat = O.init_flat(O.config("pna-agg", 2, 32, 2, 16), 1)
    n = np.array([len(r["z"]) for r in recs])
    off = np.concatenate([[0], np.cumsum(n)])
    store = DeviceStructureStore.from_arrays({"trainset": (
        np.concatenate([r["z"] for r in recs]), np.concatenate([r["pos"] for r in recs]),
        np.array([r["energy"] for r in recs]), np.concatenate([r["forces"] for r in recs]),
        off)})
    picks = [np.array([3, 17, 0, 39, 22, 5]), np.array([11, 12, 30, 1])]
    outs = []
    for mode in ("store", "host"):
        tr = T.DataParallelTrainer(cfg, T.TrainConfig(), initial=flat, dtype=F32)
        run = T.StructureStepRunner(tr, None, RC, CAP, max_graphs=8, max_atoms=24)
        for idx in picks:
            sel = [recs[i] for i in idx]
            if mode == "store":
                store.load_runner("trainset", idx, run)
                run.run()
            else:
                pos, z, e, f, o = _host(sel, F32)
                run.load(pos, z, e, f, o)
                run.run()
        torch.cuda.synchronize()
        outs.append(tr.flat_master())
    np.testing.assert_array_equal(outs[0], outs[1])


def test_runner_edge_capacity_overflow_raises():
    recs = O.synthetic(4, n_atoms_range=(20, 20), box_length=4.0, rc=RC, seed=2)
    cfg = cfg_of("sum-agg", 1, 8, 2, 4)
    tr = T.DataParallelTrainer(cfg, T.TrainConfig(), dtype=F32)
    off = np.arange(5) * 20
    run = T.StructureStepRunner(tr, off, RC, 0, e_cap=50)
    pos, z, e, f, _ = _host(recs, F32)
    run.load(pos, z, e, f)
    with pytest.raises(ValidationError, match="e_cap"):
        run.capture(warmup=1)
