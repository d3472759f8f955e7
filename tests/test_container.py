"""Container + record codec (container.py, records.py:126-183) against a
reference-written fixture (golden/container_tiny, made by
oracle/make_container_golden.py with gfmkit's write_container), and the
device store ingested from it (GPU)."""

import os
import shutil

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import gfm_oracle as O

from paper_2406_12909_b200 import container as C  # noqa: E402
from paper_2406_12909_b200.errors import CorruptionError, FormatError  # noqa: E402
from paper_2406_12909_b200.records import decode_record, encode_record  # noqa: E402

PATH = os.path.join(GOLDEN, "container_tiny")
SPLIT = {"trainset": (0, 5), "valset": (5, 7), "testset": (7, 8)}


def test_reads_reference_container():
    man = C.read_manifest(PATH)
    assert (man.version, man.subfile_count, man.total_records) == (1, 2, 8)
    want = O.synthetic(8, seed=21)
    for g, (lo, hi) in SPLIT.items():
        recs = C.read_group(man, g, PATH)
        assert len(recs) == hi - lo
        for k, r in enumerate(recs):
            d = want[lo + k]
            assert r.source_tag == f"s{lo + k}"
            np.testing.assert_array_equal(r.atomic_numbers, d["z"])
            np.testing.assert_array_equal(r.positions, d["pos"])
            np.testing.assert_array_equal(r.edge_index, d["edges"])
            np.testing.assert_array_equal(r.forces, d["forces"])
            assert r.energy == d["energy"]


def test_encode_is_byte_identical_to_reference_payloads():
    man = C.read_manifest(PATH)
    for g in SPLIT:
        ent = man.group(g).entries
        for k, r in enumerate(C.read_group(man, g, PATH)):
            with open(os.path.join(PATH, f"data.{int(ent['subfile'][k])}"), "rb") as fh:
                fh.seek(int(ent["offset"][k]))
                raw = fh.read(int(ent["length"][k]))
            assert encode_record(r) == raw
            assert encode_record(decode_record(raw)) == raw


def test_corruption_detected(tmp_path):
    bad = tmp_path / "c"
    shutil.copytree(PATH, bad)
    blob = bytearray((bad / "data.0").read_bytes())
    blob[40] ^= 1
    (bad / "data.0").write_bytes(bytes(blob))
    man = C.read_manifest(str(bad))
    with pytest.raises(CorruptionError):
        C.read_group(man, "trainset", str(bad))
    m = bytearray((bad / "manifest.gfm").read_bytes())
    m[30] ^= 1
    (bad / "manifest.gfm").write_bytes(bytes(m))
    with pytest.raises(CorruptionError):
        C.read_manifest(str(bad))
    (bad / "manifest.gfm").write_bytes(b"XXXX" + bytes(m[4:]))
    with pytest.raises(FormatError):
        C.read_manifest(str(bad))


@pytest.mark.gpu
def test_device_store_from_container():
    from paper_2406_12909_b200.store import DeviceStructureStore
    store = DeviceStructureStore.from_container(PATH)
    assert {k: v.n_samples for k, v in store.ownership.items()} == {
        g: hi - lo for g, (lo, hi) in SPLIT.items()}
    want = O.synthetic(8, seed=21)
    pos, z, e, f, off = store.gather("trainset", [4, 0], dtype=torch.float64)
    np.testing.assert_array_equal(pos.cpu().numpy(), np.concatenate([want[4]["pos"],
                                                                      want[0]["pos"]]))
    np.testing.assert_array_equal(e.cpu().numpy(), [want[4]["energy"], want[0]["energy"]])


def test_read_range_raw_is_the_payload_bytes():
    """the device ingest's input: per-record (offset, length) into one blob
    holding exactly each record's payload bytes, in index order"""
    man = C.read_manifest(PATH)
    for g, (lo, hi) in SPLIT.items():
        n = hi - lo
        blob, offs, lens = C.read_range_raw(man, g, (0, n), PATH)
        ent = man.group(g).entries
        assert offs.shape == lens.shape == (n,) and int(lens.sum()) == blob.shape[0]
        for k in range(n):
            with open(os.path.join(PATH, f"data.{int(ent['subfile'][k])}"), "rb") as fh:
                fh.seek(int(ent["offset"][k]))
                raw = fh.read(int(ent["length"][k]))
            assert bytes(blob[offs[k]:offs[k] + lens[k]]) == raw
        sub = C.read_range_raw(man, g, (1, n), PATH)
        assert bytes(sub[0]) == bytes(blob[offs[1]:]) if n > 1 else sub[0].size == 0
    with pytest.raises(Exception):
        C.read_range_raw(man, "trainset", (0, 99), PATH)
