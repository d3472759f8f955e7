"""Container ingest straight into HBM: record payloads
(records.py:126-183) checked (length, CRC32) and decoded on the device ==
the host codec, bitwise; corruption raises CorruptionError like
decode_record; the sharded store built from a reference-written container
by device decode fetches batches == make_batch of the host-decoded records."""

import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import gfm_oracle as O

from paper_2406_12909_b200 import container as C, model as M
from paper_2406_12909_b200.errors import CorruptionError
from paper_2406_12909_b200.records import GraphRecord, decode_record, encode_record
from paper_2406_12909_b200.store import decode_payloads

pytestmark = pytest.mark.gpu
PATH = os.path.join(GOLDEN, "container_tiny")


def _blob(payloads):
    lens = np.array([len(p) for p in payloads], np.int64)
    offs = np.concatenate([[0], np.cumsum(lens)])[:-1].astype(np.int64)
    return np.frombuffer(b"".join(payloads), np.uint8).copy(), offs, lens


def _check(d, recs):
    n = np.array([r.n_atoms for r in recs])
    m = np.array([r.edge_count for r in recs])
    np.testing.assert_array_equal(d["n"], n)
    np.testing.assert_array_equal(d["m"], m)
    cat = lambda xs, dt: np.concatenate([np.asarray(x, dt) for x in xs]) if xs else None
    np.testing.assert_array_equal(d["z"].cpu().numpy(), cat([r.atomic_numbers for r in recs], np.int32))
    np.testing.assert_array_equal(d["pos"].cpu().numpy(), cat([r.positions for r in recs], np.float64))
    np.testing.assert_array_equal(d["forces"].cpu().numpy(), cat([r.forces for r in recs], np.float64))
    np.testing.assert_array_equal(d["energy"].cpu().numpy(), [r.energy for r in recs])
    np.testing.assert_array_equal(d["edges"].cpu().numpy(),
                                  cat([r.edge_index.reshape(-1, 2) for r in recs], np.int32).reshape(-1, 2))
    deg = max((int(np.bincount(r.edge_index[:, 1].astype(np.int64)).max())
               for r in recs if r.edge_count), default=0)
    assert d["max_deg"] == deg


def test_decode_reference_container_payloads():
    man = C.read_manifest(PATH)
    for g in ("trainset", "valset", "testset"):
        n = man.group(g).record_count
        blob, offs, lens = C.read_range_raw(man, g, (0, n), PATH)
        _check(decode_payloads(blob, offs, lens), C.read_group(man, g, PATH))


def test_decode_many_varied_records():
    dicts = O.synthetic(300, n_atoms_range=(1, 40), seed=5)
    recs = [GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"],
                        source_tag="x" * (k % 7) + "é" * (k % 3)) for k, d in enumerate(dicts)]
    payloads = [encode_record(r) for r in recs]
    _check(decode_payloads(*_blob(payloads)), [decode_record(p) for p in payloads])


def test_corruption_detected_on_device():
    dicts = O.synthetic(5, seed=2)
    payloads = [encode_record(GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"]))
                for d in dicts]
    bad = bytearray(payloads[3])
    bad[40] ^= 1
    with pytest.raises(CorruptionError, match="checksum"):
        decode_payloads(*_blob(payloads[:3] + [bytes(bad)] + payloads[4:]))
    with pytest.raises(CorruptionError, match="length"):
        decode_payloads(*_blob(payloads[:2] + [payloads[2][:-5]]))
    with pytest.raises(CorruptionError, match="truncated"):
        decode_payloads(*_blob([bytes(8)]))


def test_sharded_store_from_container_device_decode():
    from paper_2406_12909_b200.comm import LocalComm
    from paper_2406_12909_b200.store import ShardedDeviceStore
    man = C.read_manifest(PATH)
    recs = C.read_group(man, "trainset", PATH)
    dev_st = ShardedDeviceStore.from_container(PATH, LocalComm())
    host_st = ShardedDeviceStore.from_container(PATH, LocalComm(), device_decode=False)
    idx = [4, 0, 2, 4]
    a = dev_st.fetch_device_batch("trainset", idx, dtype=torch.float64)
    b = host_st.fetch_device_batch("trainset", idx, dtype=torch.float64)
    ref = M.make_batch([recs[i] for i in idx], dtype=torch.float64)
    for k in ("z", "pos", "energy_true", "forces_true", "rowptr", "col_src", "csc_ptr"):
        np.testing.assert_array_equal(getattr(a, k).cpu().numpy(), getattr(ref, k).cpu().numpy())
        np.testing.assert_array_equal(getattr(a, k).cpu().numpy(), getattr(b, k).cpu().numpy())
    E = ref.n_edges
    for k in ("edge_w", "edge_dx", "csc_eid", "csc_dst"):
        np.testing.assert_array_equal(getattr(a, k).cpu().numpy()[:E],
                                      getattr(ref, k).cpu().numpy()[:E])


def test_device_store_device_decode_and_device_batches():
    """DeviceStructureStore.from_container(device_decode=True): groups built
    from device-decoded payloads (no host records); fetch_device_batch ==
    make_batch of the host-decoded records, bitwise; train() + evaluate()
    run on it"""
    from paper_2406_12909_b200 import train as T
    from paper_2406_12909_b200.store import DeviceStructureStore
    man = C.read_manifest(PATH)
    recs = C.read_group(man, "trainset", PATH)
    st = DeviceStructureStore.from_container(PATH, device_decode=True)
    assert st.group("trainset").records is None
    idx = [3, 0, 4, 3]
    a = st.fetch_device_batch("trainset", idx, dtype=torch.float64)
    ref = M.make_batch([recs[i] for i in idx], dtype=torch.float64)
    N, E = ref.n_nodes, ref.n_edges
    for k in ("z", "pos", "energy_true", "forces_true", "graph_of_node"):
        np.testing.assert_array_equal(getattr(a, k).cpu().numpy()[:N] if k != "energy_true"
                                      else getattr(a, k).cpu().numpy(),
                                      getattr(ref, k).cpu().numpy()[:N] if k != "energy_true"
                                      else getattr(ref, k).cpu().numpy(), err_msg=k)
    for k in ("rowptr", "csc_ptr"):
        np.testing.assert_array_equal(getattr(a, k).cpu().numpy()[:N + 1],
                                      getattr(ref, k).cpu().numpy(), err_msg=k)
    for k in ("col_src", "edge_dst", "csc_eid", "csc_dst", "edge_w", "edge_dx"):
        np.testing.assert_array_equal(getattr(a, k).cpu().numpy()[:E],
                                      getattr(ref, k).cpu().numpy()[:E], err_msg=k)
    mc = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=2, mpnn_width=16, fc_width=16,
                       batch_size=2)
    res = T.train(mc, st, config=T.TrainConfig(max_epochs=1), dtype=torch.float64)
    assert res.epochs_run == 1 and np.isfinite(res.metrics[0].val_mae)
