"""HBM-resident sample store: gfm_gather_structures against the host
concatenation make_batch performs (model.py:237-250) -- bit-exact -- and
the runner path against the runner's own host-copy path."""

import numpy as np
import pytest
import torch

from oracle import gfm_oracle as O

from paper_2406_12909_b200 import model as M, train as T  # noqa: E402
from paper_2406_12909_b200.errors import ValidationError  # noqa: E402
from paper_2406_12909_b200.records import GraphRecord  # noqa: E402

pytestmark = pytest.mark.gpu


def _records(count, seed, n_range=(4, 12)):
    dicts = O.synthetic(count, n_atoms_range=n_range, seed=seed)
    return [GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"]) for d in dicts]


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_gather_matches_host_concatenation(dtype):
    from paper_2406_12909_b200.store import DeviceStructureStore
    recs = _records(40, 3)
    store = DeviceStructureStore({"trainset": recs})
    idx = np.array([7, 0, 39, 7, 12, 5, 33])  # repeats allowed, any order
    pos, z, e, f, off = store.gather("trainset", idx, dtype=dtype)
    sel = [recs[i] for i in idx]
    np.testing.assert_array_equal(off, np.concatenate([[0], np.cumsum([r.n_atoms for r in sel])]))
    np.testing.assert_array_equal(pos.cpu().numpy(), np.concatenate([r.positions for r in sel]))
    np.testing.assert_array_equal(z.cpu().numpy(), np.concatenate([r.atomic_numbers for r in sel]))
    np.testing.assert_array_equal(e.cpu().numpy(),
                                  np.array([r.energy for r in sel]).astype(e.cpu().numpy().dtype))
    np.testing.assert_array_equal(
        f.cpu().numpy(), np.concatenate([r.forces for r in sel]).astype(f.cpu().numpy().dtype))
    with pytest.raises(ValidationError):
        store.gather("trainset", [40])
    with pytest.raises(ValidationError):
        store.gather("trainset", [])


def test_runner_fed_from_store_matches_host_feed():
    from paper_2406_12909_b200.store import DeviceStructureStore
    recs = _records(24, 5, n_range=(10, 10))  # fixed size: one runner layout
    store = DeviceStructureStore({"trainset": recs})
    mc = M.ModelConfig(mpnn_kind="sum-agg", mpnn_layers=2, mpnn_width=16, fc_width=16)
    tr = T.DataParallelTrainer(mc, T.TrainConfig())
    idx = np.array([3, 17, 8, 21])
    off = store.host_offsets("trainset", idx)
    run = T.StructureStepRunner(tr, off, rc=2.0, use_graph=False)
    sel = [recs[i] for i in idx]
    host = [torch.from_numpy(np.concatenate([r.positions for r in sel])),
            torch.from_numpy(np.concatenate([r.atomic_numbers for r in sel]).astype(np.int32)),
            torch.tensor([r.energy for r in sel], dtype=torch.float32),
            torch.from_numpy(np.concatenate([r.forces for r in sel]).astype(np.float32))]
    run.load(*host)
    want = {k: v.clone() for k, v in run.slot.items()}
    for v in run.slot.values():
        v.zero_()
    store.load_runner("trainset", idx, run)
    for k in want:
        assert torch.equal(run.slot[k], want[k]), k
    run.run()
    torch.cuda.synchronize()
    assert np.isfinite(tr.contrib[tr.P].item())
    with pytest.raises(ValidationError):
        store.load_runner("trainset", idx[:3], run)


def test_train_accepts_device_store():
    from paper_2406_12909_b200.store import DeviceStructureStore
    recs = _records(10, 8)
    store = DeviceStructureStore({"trainset": recs[:7], "valset": recs[7:]})
    mc = M.ModelConfig(mpnn_kind="mean-agg", mpnn_layers=1, mpnn_width=8, fc_width=8,
                       batch_size=4)
    res = T.train(mc, store, config=T.TrainConfig(max_epochs=1), dtype=torch.float64)
    assert res.epochs_run == 1 and np.isfinite(res.metrics[0].val_mae)


def test_store_from_arrays():
    from paper_2406_12909_b200.store import DeviceStructureStore
    recs = _records(9, 6)
    off = np.concatenate([[0], np.cumsum([r.n_atoms for r in recs])])
    arrays = (np.concatenate([r.atomic_numbers for r in recs]),
              np.concatenate([r.positions for r in recs]), np.array([r.energy for r in recs]),
              np.concatenate([r.forces for r in recs]), off)
    a = DeviceStructureStore.from_arrays({"trainset": arrays})
    b = DeviceStructureStore({"trainset": recs})
    assert a.ownership["trainset"].n_samples == 9
    idx = [8, 1, 4]
    for x, y in zip(a.gather("trainset", idx, torch.float64)[:4],
                    b.gather("trainset", idx, torch.float64)[:4]):
        assert torch.equal(x, y)
    with pytest.raises(ValidationError):
        a.fetch_batch("trainset", idx)


def _gather_runner_batch(store, idx, dtype):
    """run the store-mode gather once (eagerly) and return its Batch"""
    mc = M.ModelConfig(mpnn_kind="sum-agg", mpnn_layers=1, mpnn_width=8, fc_width=8)
    tr = T.DataParallelTrainer(mc, T.TrainConfig(), dtype=dtype)
    run = T.StructureStepRunner(tr, None, store=store, max_graphs=len(idx) + 2, use_graph=False)
    run.set_indices(idx)
    with tr.preserved():
        run._eager()
    torch.cuda.synchronize()
    return run.batch


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_store_gather_batch_matches_make_batch(dtype):
    """gfm_gather_batch (per-structure CSR blocks copied with shifted ids)
    == make_batch's CSR / CSC of the same records, bitwise; capacity tail
    nodes edge-free with gnode -1"""
    from paper_2406_12909_b200.store import DeviceStructureStore
    recs = _records(30, 11, n_range=(2, 14))
    store = DeviceStructureStore({"trainset": recs})
    idx = np.array([4, 29, 0, 4, 17, 9])
    b = _gather_runner_batch(store, idx, dtype)
    ref = M.make_batch([recs[i] for i in idx], dtype=dtype)
    N, E = ref.n_nodes, ref.n_edges
    assert int(b.rowptr[N].item()) == E and int(b.rowptr[-1].item()) == E
    for k in ("rowptr", "csc_ptr"):
        np.testing.assert_array_equal(getattr(b, k).cpu().numpy()[:N + 1],
                                      getattr(ref, k).cpu().numpy(), err_msg=k)
    for k in ("col_src", "edge_dst", "csc_eid", "csc_dst", "edge_w", "edge_dx"):
        np.testing.assert_array_equal(getattr(b, k).cpu().numpy()[:E],
                                      getattr(ref, k).cpu().numpy()[:E], err_msg=k)
    np.testing.assert_array_equal(b.graph_of_node.cpu().numpy()[:N],
                                  ref.graph_of_node.cpu().numpy()[:N])
    assert (b.graph_of_node.cpu().numpy()[N:] == -1).all()
    np.testing.assert_array_equal(b.counts.cpu().numpy(), [len(idx), N])


class _HostStore:
    """the reference DDStore surface only (ownership + fetch_batch): train()
    then packs every batch with make_batch on the host"""

    def __init__(self, groups):
        self._g = groups
        self.ownership = {k: type("O", (), {"n_samples": len(v)})() for k, v in groups.items()}

    def fetch_batch(self, group, indices):
        return [self._g[group][int(i)] for i in indices]


def test_train_device_store_matches_host_packing():
    """train() with a DeviceStructureStore (batches gathered on the device
    inside one captured step, ragged, short last batch) == train() packing
    the same batches on the host, float64, 2 epochs"""
    from paper_2406_12909_b200.store import DeviceStructureStore
    recs = _records(23, 12, n_range=(3, 11))
    groups = {"trainset": recs[:19], "valset": recs[19:]}
    mc = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=2, mpnn_width=16, fc_width=16,
                       batch_size=4)
    cfg = T.TrainConfig(max_epochs=2, patience=5)
    dev = T.train(mc, DeviceStructureStore(groups), config=cfg, dtype=torch.float64)
    host = T.train(mc, _HostStore(groups), config=cfg, dtype=torch.float64)
    assert dev.epochs_run == host.epochs_run == 2
    for a, b in zip(dev.metrics, host.metrics):
        assert abs(a.train_loss - b.train_loss) <= 1e-10 * abs(b.train_loss)
        assert abs(a.val_mae - b.val_mae) <= 1e-10 * abs(b.val_mae)
        assert "step" in a.phase_seconds and "forward" in b.phase_seconds
    np.testing.assert_allclose(dev.params.flatten(), host.params.flatten(), rtol=0, atol=1e-10)
