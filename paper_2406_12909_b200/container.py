"""Read gfmkit container directories (container.py:48-330 of the reference):
``manifest.gfm`` (GFMC magic, per-group entry tables, CRC32) plus
``data.<k>`` sub-files of encoded records.  The reader feeds the
HBM-resident store (``store.DeviceStructureStore.from_container``): records
are decoded once on the host and ingested into device arrays, after which
no step touches the files.  Writing containers stays with gfmkit.
"""

from __future__ import annotations

import os
import struct
import zlib
from dataclasses import dataclass, field

import numpy as np

from .errors import CorruptionError, FormatError, UnsupportedVersionError, ValidationError
from .records import GraphRecord, decode_record

MANIFEST_MAGIC = b"GFMC"                        # container.py:48
MANIFEST_VERSION = 1                            # container.py:49
MANIFEST_NAME = "manifest.gfm"                  # container.py:50
GROUP_NAMES = ("trainset", "valset", "testset")  # container.py:51
ENTRY_DTYPE = np.dtype([("subfile", "<u4"), ("offset", "<u8"), ("length", "<u8"),
                        ("n_atoms", "<u4"), ("edge_count", "<u4")])  # container.py:53-61


@dataclass
class GroupIndex:
    entries: np.ndarray

    @property
    def record_count(self) -> int:
        return int(self.entries.shape[0])


@dataclass
class ContainerManifest:
    version: int
    subfile_count: int
    total_records: int
    groups: dict = field(default_factory=dict)

    def group(self, name: str) -> GroupIndex:
        if name not in self.groups:
            raise ValidationError(f"unknown group {name!r}; expected one of {sorted(self.groups)}")
        return self.groups[name]


def read_manifest(path: str) -> ContainerManifest:
    """container.py:205-250, same checks and error classes."""
    mpath = os.path.join(path, MANIFEST_NAME)
    if not os.path.exists(mpath):
        raise FormatError(f"no {MANIFEST_NAME} in {path!r}")
    with open(mpath, "rb") as fh:
        blob = fh.read()
    if len(blob) < 4 or blob[:4] != MANIFEST_MAGIC:
        raise FormatError(f"bad manifest magic {blob[:4]!r}, expected {MANIFEST_MAGIC!r}")
    if len(blob) < 24:
        raise CorruptionError("manifest truncated before header")
    version, subfiles, total = struct.unpack_from("<IIQ", blob, 4)
    if version != MANIFEST_VERSION:
        raise UnsupportedVersionError(
            f"manifest version {version} not supported (expected {MANIFEST_VERSION})")
    if zlib.crc32(memoryview(blob)[:-4]) != struct.unpack_from("<I", blob, len(blob) - 4)[0]:
        raise CorruptionError("manifest checksum mismatch")
    (count,) = struct.unpack_from("<I", blob, 20)
    off, groups = 24, {}
    for _ in range(count):
        (nlen,) = struct.unpack_from("<I", blob, off)
        name = blob[off + 4:off + 4 + nlen].decode("utf-8")
        off += 4 + nlen
        (nrec,) = struct.unpack_from("<Q", blob, off)
        off += 8
        nbytes = nrec * ENTRY_DTYPE.itemsize
        if off + nbytes > len(blob) - 4:
            raise CorruptionError(f"manifest truncated inside group {name!r} table")
        groups[name] = GroupIndex(np.frombuffer(blob, ENTRY_DTYPE, nrec, off).copy())
        off += nbytes
    if set(groups) != set(GROUP_NAMES):
        raise FormatError(f"manifest groups {set(groups)} != {set(GROUP_NAMES)}")
    if sum(g.record_count for g in groups.values()) != total:
        raise CorruptionError("manifest group counts do not sum to total_records")
    return ContainerManifest(version, subfiles, total, groups)


def read_range(manifest: ContainerManifest, group: str, index_range, path: str):
    """container.py:271-315: decoded records of [lo, hi), in order.  Reads
    each sub-file once, sequentially, instead of one seek per record."""
    lo, hi = index_range
    g = manifest.group(group)
    if not (0 <= lo <= hi <= g.record_count):
        raise ValidationError(f"range [{lo}, {hi}) out of bounds for group {group!r} "
                              f"with {g.record_count} records")
    ent = g.entries[lo:hi]
    out = [None] * (hi - lo)
    for sub in np.unique(ent["subfile"]):
        mine = np.nonzero(ent["subfile"] == sub)[0]
        with open(os.path.join(path, f"data.{int(sub)}"), "rb") as fh:
            data = fh.read()
        for k in mine:
            o, n = int(ent["offset"][k]), int(ent["length"][k])
            if o + n > len(data):
                raise CorruptionError(f"sub-file data.{int(sub)} truncated at offset {o}")
            out[k] = decode_record(memoryview(data)[o:o + n])
    return out


def read_range_raw(manifest: ContainerManifest, group: str, index_range, path: str,
                   pinned: bool = False):
    """The undecoded payloads of [lo, hi) as one byte blob + per-record
    (offset, length) in it (each sub-file read once) -- for decoding on the
    device (store.decode_payloads).  ``pinned``: the blob lives in page-locked
    host memory (a torch tensor's numpy view), so its upload runs at full
    link speed."""
    lo, hi = index_range
    g = manifest.group(group)
    if not (0 <= lo <= hi <= g.record_count):
        raise ValidationError(f"range [{lo}, {hi}) out of bounds for group {group!r} "
                              f"with {g.record_count} records")
    ent = g.entries[lo:hi]
    lengths = ent["length"].astype(np.int64)
    offsets = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int64)
    if pinned:
        import torch
        blob = torch.empty(max(int(offsets[-1]), 1), dtype=torch.uint8,
                           pin_memory=True).numpy()[:int(offsets[-1])]
    else:
        blob = np.empty(int(offsets[-1]), np.uint8)
    for sub in np.unique(ent["subfile"]):
        mine = np.nonzero(ent["subfile"] == sub)[0]
        with open(os.path.join(path, f"data.{int(sub)}"), "rb") as fh:
            data = np.frombuffer(fh.read(), np.uint8)
        for k in mine:
            o, n = int(ent["offset"][k]), int(ent["length"][k])
            if o + n > data.shape[0]:
                raise CorruptionError(f"sub-file data.{int(sub)} truncated at offset {o}")
            blob[offsets[k]:offsets[k] + n] = data[o:o + n]
    return blob, offsets[:-1].copy(), lengths


def read_group(manifest: ContainerManifest, group: str, path: str) -> list[GraphRecord]:
    """container.py:318-319."""
    return read_range(manifest, group, (0, manifest.group(group).record_count), path)
