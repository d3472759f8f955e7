"""HBM-resident sample store.

Replaces, for the training hot path, DDStore's fetch (ddstore.py:316-490),
``decode_record`` (records.py:154-183) and make_batch's host concatenation
(model.py:237-250): every structure of a group is ingested once into
device arrays (z int32, pos float64, energy/forces float64, CSR-style
offsets), and a batch is assembled by ``gfm_gather_structures`` -- only the
B sample indices cross PCIe per step.  A C3-scale dataset (100-atom
structures, ~10 KB each with labels) holds ~10^7 structures in 180 GB.

``ownership`` / ``fetch_batch`` keep DDStore's surface, so ``train()`` and
``evaluate()`` accept this store unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_handle
from .errors import ValidationError
from .records import MAX_Z


@dataclass
class _Ownership:
    n_samples: int


class _Group:
    def __init__(self, records, device, arrays=None, decoded=None):
        if decoded is not None:
            self._from_decoded(decoded, device)
            return
        if arrays is None:
            if not records:
                raise ValidationError("a store group needs at least one structure")
            cat = np.concatenate
            n = np.array([r.atomic_numbers.shape[0] for r in records], np.int64)
            off = np.concatenate([[0], np.cumsum(n)])
            arrays = (cat([r.atomic_numbers for r in records]), cat([r.positions for r in records]),
                      np.array([r.energy for r in records]), cat([r.forces for r in records]), off)
        z, pos, energy, forces, off = arrays
        self.records = None if records is None else list(records)
        self.host_off = np.asarray(off, np.int64).astype(np.int32)
        self.n_samples = self.host_off.shape[0] - 1
        N = int(self.host_off[-1])
        zz = np.asarray(z).reshape(-1)
        if zz.size != N or (N and (zz.min() < 1 or zz.max() > MAX_Z)):
            raise ValidationError(f"store ingest: {zz.size} atomic numbers for {N} atoms, "
                                  f"each must lie in [1, {MAX_Z}]")
        self.max_atoms = int(np.diff(self.host_off).max()) if self.n_samples else 0
        self.host_m = None
        self.z = torch.as_tensor(np.asarray(z).reshape(N).astype(np.int32), device=device)
        self.pos = torch.as_tensor(np.asarray(pos, np.float64).reshape(N, 3), device=device)
        self.energy = torch.as_tensor(np.asarray(energy, np.float64).reshape(self.n_samples),
                                      device=device)
        self.forces = torch.as_tensor(np.asarray(forces, np.float64).reshape(N, 3), device=device)
        self.off = torch.as_tensor(self.host_off, device=device)
        self.csr = None
        if self.records is not None:
            self._pack_edges(device)

    def _from_decoded(self, d, device):
        """a group decoded on the device (decode_payloads): the same fields
        as the record path, its CSR built from the device arrays -- no host
        records, no host copies of the structures"""
        from .model import batch_from_device
        self.records = None
        n, m = d["n"], d["m"]
        if n.shape[0] == 0:
            raise ValidationError("a store group needs at least one structure")
        self.host_off = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
        self.n_samples = n.shape[0]
        self.max_atoms = int(n.max())
        self.host_m = m.astype(np.int64)
        self.max_edges = int(m.max())
        self.max_deg = int(d["max_deg"])
        self.periodic = False
        self.z, self.pos, self.energy, self.forces = d["z"], d["pos"], d["energy"], d["forces"]
        self.off = torch.as_tensor(self.host_off, device=device)
        S, E = self.n_samples, int(m.sum())
        # record-local edge ids + each structure's node base, one block gather
        edges = torch.empty(max(E, 1), 2, dtype=torch.int32, device=device)
        if E:
            idx = torch.arange(S, dtype=torch.int32, device=device)
            call("gfm_gather_blocks", ptr(idx), S, ptr(d["eoff"]), ptr(d["eoff"]), 2,
                 ptr(d["edges"]), ptr(edges), ptr(self.off), stream_handle())
        e_off = torch.as_tensor(np.concatenate([[0], np.cumsum(m)]).astype(np.int32),
                                device=device)
        b = batch_from_device(self.z, self.pos, self.energy, self.forces,
                              edges[:E, 0].contiguous(), edges[:E, 1].contiguous(), e_off,
                              self.off, self.host_off.astype(np.int64), torch.float64, None,
                              self.max_deg)
        self.csr = dict(rowptr=b.rowptr, col_src=b.col_src, edge_w=b.edge_w, edge_dx=b.edge_dx,
                        csc_ptr=b.csc_ptr, csc_eid=b.csc_eid, csc_dst=b.csc_dst)

    def _pack_edges(self, device):
        """the records' own edges (make_batch semantics, model.py:234-285)
        as one float64 CSR / CSC over the whole group, built once on the
        device; a batch is then a gather of per-structure blocks"""
        from .model import make_batch

        b = make_batch(self.records, device=device, dtype=torch.float64)
        m = np.array([int(np.asarray(r.edge_index).reshape(-1, 2).shape[0]) for r in self.records],
                     np.int64)
        self.host_m = m
        self.max_edges = int(m.max()) if m.size else 0
        self.max_deg = int(b.max_deg)
        self.csr = dict(rowptr=b.rowptr, col_src=b.col_src, edge_w=b.edge_w, edge_dx=b.edge_dx,
                        csc_ptr=b.csc_ptr, csc_eid=b.csc_eid, csc_dst=b.csc_dst)
        self.periodic = bool(b.periodic)


class DeviceStructureStore:
    """``{group: [GraphRecord]}`` ingested into HBM once."""

    def __init__(self, groups: dict, device=None, _arrays: dict | None = None,
                 _decoded: dict | None = None):
        _lib.load(require_device=True)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._groups = {k: _Group(v, self.device) for k, v in groups.items()}
        for k, a in (_arrays or {}).items():
            self._groups[k] = _Group(None, self.device, a)
        for k, d in (_decoded or {}).items():
            self._groups[k] = _Group(None, self.device, decoded=d)
        self.ownership = {k: _Ownership(g.n_samples) for k, g in self._groups.items()}
        self._idx = {}
        self._copy_stream = None

    @classmethod
    def from_arrays(cls, groups: dict, device=None) -> "DeviceStructureStore":
        """``{group: (z (N,), pos (N,3), energy (S,), forces (N,3), offsets
        (S+1,))}`` -- already-concatenated structures (no host records, so
        ``fetch_batch`` is unavailable; use ``gather``/``load_runner``)."""
        return cls({}, device, _arrays=groups)

    @classmethod
    def from_container(cls, path: str, groups=None, device=None,
                       device_decode: bool = False) -> "DeviceStructureStore":
        """Ingest a gfmkit container directory (container.py) into HBM.
        ``device_decode``: payloads checked and decoded on the GPU
        (decode_payloads); the store then keeps no host records
        (``fetch_batch`` is unavailable, ``fetch_device_batch`` serves the
        batches) -- otherwise records are decoded on the host and kept."""
        from .container import GROUP_NAMES, read_group, read_manifest, read_range_raw
        man = read_manifest(path)
        names = [g for g in (groups or GROUP_NAMES) if man.group(g).record_count]
        if device_decode:
            dec = {}
            for g in names:
                blob, offs, lens = read_range_raw(man, g, (0, man.group(g).record_count), path,
                                                  pinned=True)
                dec[g] = decode_payloads(blob, offs, lens, device)
            return cls({}, device, _decoded=dec)
        return cls({g: read_group(man, g, path) for g in names}, device)

    def fetch_device_batch(self, group, indices, dtype=torch.float32):
        """Structures ``indices`` as a model.Batch assembled on the device from
        the group's per-structure CSR blocks (gfm_gather_batch: bitwise the
        CSR / CSC make_batch builds from the same records)."""
        g = self._groups[group]
        if g.csr is None:
            raise ValidationError(f"group {group!r} holds no record edges")
        idx = self._check(g, indices)
        dev = self.device
        host_off, e_off = self.batch_layout(group, idx)
        B, N, E = idx.shape[0], int(host_off[-1]), int(e_off[-1])
        n_per = np.diff(host_off)
        meta = np.concatenate([[B, N], host_off, n_per, e_off]).astype(np.int32)
        meta_d = torch.as_tensor(meta, device=dev)
        idx_d = torch.as_tensor(idx.astype(np.int32), device=dev)
        slot = dict(z=torch.empty(max(N, 1), dtype=torch.int32, device=dev),
                    pos=torch.empty(max(N, 1), 3, dtype=torch.float64, device=dev),
                    e=torch.empty(B, dtype=dtype, device=dev),
                    f=torch.empty(max(N, 1), 3, dtype=dtype, device=dev))
        return gather_batch(g, idx_d, meta_d, B, N, E, dtype, {}, slot, meta_d[2:3 + B],
                            meta_d[3 + B:3 + 2 * B], meta_d[0:2], host_off.astype(np.int64))

    # ---- DDStore surface (ddstore.py:316-490) ----------------------------
    def fetch_batch(self, group, indices):
        recs = self._groups[group].records
        if recs is None:
            raise ValidationError(f"group {group!r} was ingested from arrays; it has no records")
        return [recs[int(i)] for i in indices]

    def close(self):
        self._groups.clear()

    # ---- device batch assembly -------------------------------------------
    def host_offsets(self, group, indices) -> np.ndarray:
        """node offsets of the batch ``indices`` would assemble"""
        g = self._groups[group]
        idx = self._check(g, indices)
        n = g.host_off[idx + 1] - g.host_off[idx]
        return np.concatenate([[0], np.cumsum(n)]).astype(np.int32)

    def _check(self, g, indices):
        idx = np.asarray(indices, np.int64).reshape(-1)
        if idx.size == 0:
            raise ValidationError("cannot build a batch from zero records")
        if idx.min() < 0 or idx.max() >= g.n_samples:
            raise ValidationError(f"sample index out of range [0, {g.n_samples})")
        return idx

    def _launch(self, g, idx, dst_off, z, pos, e, f, dtype):
        # indices go host -> device on a copy stream (so the copy overlaps the
        # step still running on the compute stream) through a ring of pinned /
        # device buffers; a slot is reused only after its last H2D copy (host
        # side) and its last gather (device side) have completed
        B = idx.shape[0]
        main = torch.cuda.current_stream(self.device)
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(device=self.device)
        cs = self._copy_stream
        ring = self._idx.get(B)
        if ring is None:
            ring = self._idx[B] = dict(k=0, slots=[
                [torch.empty(B, dtype=torch.int32).pin_memory(),
                 torch.empty(B, dtype=torch.int32, device=self.device), None, None]
                for _ in range(4)])
        slot = ring["slots"][ring["k"]]
        ring["k"] = (ring["k"] + 1) % len(ring["slots"])
        host, dev, copied, used = slot
        if copied is not None:
            copied.synchronize()
        host.numpy()[:] = idx
        if used is not None:
            cs.wait_event(used)
        with torch.cuda.stream(cs):
            dev.copy_(host, non_blocking=True)
        slot[2] = torch.cuda.Event()
        slot[2].record(cs)
        main.wait_event(slot[2])
        call("gfm_gather_structures", ptr(dev), int(B), ptr(g.off), ptr(dst_off),
             ptr(g.z), ptr(g.pos), ptr(g.energy), ptr(g.forces), ptr(z), ptr(pos), ptr(e), ptr(f),
             _lib.dtype_code(dtype), stream_handle())
        slot[3] = torch.cuda.Event()
        slot[3].record(main)

    def group(self, name) -> "_Group":
        return self._groups[name]

    def batch_layout(self, group, indices):
        """host layout words of a stored-edge batch: (node offsets, edge
        offsets) of structures ``indices``"""
        g = self._groups[group]
        idx = self._check(g, indices)
        n = g.host_off[idx + 1] - g.host_off[idx]
        m = g.host_m[idx]
        return (np.concatenate([[0], np.cumsum(n)]).astype(np.int64),
                np.concatenate([[0], np.cumsum(m)]).astype(np.int64))

    def gather(self, group, indices, dtype=torch.float32):
        """Assemble structures ``indices`` on the device: returns
        (pos f64 (N,3), z i32 (N,), energy (B,), forces (N,3), host_offsets)."""
        g = self._groups[group]
        idx = self._check(g, indices)
        host_off = self.host_offsets(group, idx)
        N, B = int(host_off[-1]), idx.shape[0]
        dev = self.device
        pos = torch.empty(N, 3, dtype=torch.float64, device=dev)
        z = torch.empty(N, dtype=torch.int32, device=dev)
        e = torch.empty(B, dtype=dtype, device=dev)
        f = torch.empty(N, 3, dtype=dtype, device=dev)
        self._launch(g, idx, torch.as_tensor(host_off, device=dev), z, pos, e, f, dtype)
        return pos, z, e, f, host_off

    def load_runner(self, group, indices, runner) -> None:
        """Write structures ``indices`` straight into a StructureStepRunner's
        input slots (a fixed-layout runner needs matching structure sizes; a
        ragged runner takes any batch within its capacity); follow with
        ``runner.run()``."""
        g = self._groups[group]
        idx = self._check(g, indices)
        runner.set_layout(self.host_offsets(group, idx))
        s = runner.slot
        self._launch(g, idx, runner.off, s["z"], s["pos"], s["e"], s["f"], runner.tr.dtype)


def gather_batch(g: "_Group", idx_dev, meta_dev, n_cap_graphs: int, n_nodes: int, e_cap: int,
                 dtype, out: dict, slot: dict, off_view, npg_view, counts_view, host_off_cap):
    """Assemble a training Batch of stored-edge structures on the device
    (gfm_gather_batch) into the buffers of ``out`` / ``slot``; every size is
    read from ``meta_dev``, so the call is CUDA-graph capturable."""
    from .model import Batch

    dev = g.z.device
    Ec = max(int(e_cap), 1)

    def buf(name, shape, dt):
        t = out.get(name)
        if t is None or t.dtype != dt or tuple(t.shape) != tuple(shape):
            t = torch.empty(shape, dtype=dt, device=dev)
            out[name] = t
        return t

    N = int(n_nodes)
    gnode = buf("gnode", (max(N, 1),), torch.int32)
    rowptr = buf("rowptr", (N + 1,), torch.int32)
    csc_ptr = buf("csc_ptr", (N + 1,), torch.int32)
    col_src = buf("col_src", (Ec,), torch.int32)
    edge_dst = buf("edge_dst", (Ec,), torch.int32)
    csc_eid = buf("csc_eid", (Ec,), torch.int32)
    csc_dst = buf("csc_dst", (Ec,), torch.int32)
    edge_w = buf("edge_w", (Ec,), dtype)
    edge_dx = buf("edge_dx", (Ec, 3), dtype)
    c = g.csr
    call("gfm_gather_batch", ptr(idx_dev), ptr(meta_dev), int(n_cap_graphs), N, ptr(g.off),
         ptr(g.z), ptr(g.pos), ptr(g.energy), ptr(g.forces), ptr(c["rowptr"]), ptr(c["col_src"]),
         ptr(c["edge_w"]), ptr(c["edge_dx"]), ptr(c["csc_ptr"]), ptr(c["csc_eid"]),
         ptr(c["csc_dst"]), ptr(slot["z"]), ptr(slot["pos"]), ptr(slot["e"]), ptr(slot["f"]),
         ptr(gnode), ptr(rowptr), ptr(col_src), ptr(edge_dst), ptr(edge_w), ptr(edge_dx),
         ptr(csc_ptr), ptr(csc_eid), ptr(csc_dst), _lib.dtype_code(dtype), stream_handle())
    b = Batch(dtype=dtype, device=dev, z=slot["z"][:N], pos=slot["pos"][:N],
              node_offsets=off_view, n_per_graph=npg_view, graph_of_node=gnode,
              energy_true=slot["e"], forces_true=slot["f"][:N], rowptr=rowptr, col_src=col_src,
              edge_dst=edge_dst, edge_w=edge_w, edge_dx=edge_dx, csc_ptr=csc_ptr,
              csc_eid=csc_eid, csc_dst=csc_dst, order=None, n_nodes=N, e_cap=Ec, _n_edges=None,
              host_offsets=host_off_cap, host_n_per=np.diff(host_off_cap), max_deg=g.max_deg,
              counts=counts_view, periodic=g.periodic)
    return b


# --------------------------------------------------------------------------
# Sharded store: DDStore over NVLink
# --------------------------------------------------------------------------


def decode_payloads(blob, offsets, lengths, device=None) -> dict:
    """Record payloads (records.py:126-183) decoded ON THE DEVICE: the blob
    goes to HBM once, one thread per record checks header, length and CRC32
    (gfm_record_scan; CorruptionError like decode_record), one warp per
    record scatters z / positions / edges / energy / forces into
    concatenated arrays (gfm_record_decode).  Returns the store's group
    arrays: n, m (host int64), z, pos, forces, energy, edges (device), noff /
    eoff / soff (device int64 offsets) and max_deg (host)."""
    from .errors import CorruptionError
    _lib.load(require_device=True)
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    S = int(len(offsets))
    # a page-locked blob (container.read_range_raw(pinned=True)) uploads at
    # link speed; torch.from_numpy keeps the pinned storage's flag
    host = torch.from_numpy(np.ascontiguousarray(blob, np.uint8))
    blob_d = host.to(dev, non_blocking=host.is_pinned())
    off_d = torch.as_tensor(np.asarray(offsets, np.int64), device=dev)
    len_d = torch.as_tensor(np.asarray(lengths, np.int64), device=dev)
    nm = torch.empty(3, max(S, 1), dtype=torch.int32, device=dev)
    s = stream_handle()
    call("gfm_record_scan", ptr(blob_d), ptr(off_d), ptr(len_d), S, ptr(nm[0]), ptr(nm[1]),
         ptr(nm[2]), s)
    n_h, m_h, st = (x[:S].astype(np.int64) for x in nm.cpu().numpy())
    bad = np.nonzero(st)[0]
    if bad.size:
        k = int(bad[0])
        msg = {1: f"record payload truncated ({int(lengths[k])} bytes)",
               2: f"record payload length {int(lengths[k])} != expected",
               3: "record payload checksum mismatch"}[int(st[k])]
        raise CorruptionError(f"record {k}: {msg}")
    noff, eoff = (np.concatenate([[0], np.cumsum(x)]).astype(np.int64) for x in (n_h, m_h))
    N, E = int(noff[-1]), int(eoff[-1])
    t = lambda a: torch.as_tensor(a, device=dev)
    z = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
    pos = torch.empty(max(N, 1), 3, dtype=torch.float64, device=dev)
    forces = torch.empty(max(N, 1), 3, dtype=torch.float64, device=dev)
    energy = torch.empty(max(S, 1), dtype=torch.float64, device=dev)
    edges = torch.empty(max(E, 1), 2, dtype=torch.int32, device=dev)
    deg = torch.zeros(max(N, 1), dtype=torch.int32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    noff_d, eoff_d = t(noff), t(eoff)
    call("gfm_record_decode", ptr(blob_d), ptr(off_d), S, ptr(noff_d), ptr(eoff_d), ptr(z),
         ptr(pos), ptr(forces), ptr(energy), ptr(edges), ptr(deg), ptr(flag), s)
    if int(flag.item()):
        raise ValidationError("edge endpoint out of range")
    if N and (int(z[:N].min()) < 1 or int(z[:N].max()) > MAX_Z):
        raise ValidationError(f"atomic numbers must lie in [1, {MAX_Z}]")
    return dict(n=n_h, m=m_h, noff=noff_d, eoff=eoff_d,
                soff=t(np.arange(S + 1, dtype=np.int64)), z=z[:N], pos=pos[:N],
                forces=forces[:N], energy=energy[:S], edges=edges[:E],
                max_deg=int(deg.max()) if N else 0, shift=None)


def partition_for_readers(record_count: int, reader_count: int):
    """container.py:253-268: contiguous, disjoint, sizes differ by at most
    one, the larger ranges on the lower ids."""
    if reader_count < 1:
        raise ValidationError(f"reader_count must be >= 1, got {reader_count}")
    base, extra = divmod(int(record_count), int(reader_count))
    out, start = [], 0
    for r in range(reader_count):
        size = base + (1 if r < extra else 0)
        out.append((start, start + size))
        start += size
    return out


class OwnershipMap:
    """Who holds which contiguous slice (ddstore.py:95-165): ranks form
    ``replication_factor`` sub-groups of P / R consecutive ranks; each
    sub-group holds the whole group, split by partition_for_readers or by
    explicit ``chunk_sizes`` (empty chunks allowed)."""

    def __init__(self, n_samples: int, n_ranks: int, replication_factor: int = 1,
                 chunk_sizes=None):
        from .errors import ConfigError
        if n_ranks < 1 or replication_factor < 1 or n_ranks % replication_factor:
            raise ConfigError(f"replication_factor {replication_factor} must divide "
                              f"n_ranks {n_ranks} (>= 1)")
        self.n_samples = int(n_samples)
        self.n_ranks = int(n_ranks)
        self.replication_factor = int(replication_factor)
        self.group_size = n_ranks // replication_factor
        if chunk_sizes is None:
            self.local_ranges = partition_for_readers(n_samples, self.group_size)
        else:
            cs = [int(c) for c in chunk_sizes]
            if len(cs) != self.group_size or min(cs, default=0) < 0 or sum(cs) != n_samples:
                raise ConfigError(f"chunk_sizes must be {self.group_size} nonnegative sizes "
                                  f"summing to {n_samples}")
            edges = np.concatenate([[0], np.cumsum(cs)]).astype(int)
            self.local_ranges = [(int(edges[i]), int(edges[i + 1])) for i in range(len(cs))]
        # upper bounds of the non-empty chunks -> their local ids
        self._hi = np.array([hi for lo, hi in self.local_ranges if hi > lo], np.int64)
        self._id = np.array([k for k, (lo, hi) in enumerate(self.local_ranges) if hi > lo],
                            np.int64)

    def subgroup_of(self, rank: int) -> int:
        return rank // self.group_size

    def local_rank(self, rank: int) -> int:
        return rank % self.group_size

    def range_of(self, rank: int):
        return self.local_ranges[self.local_rank(rank)]

    def chunk_sizes(self):
        return [hi - lo for lo, hi in self.local_ranges]

    def owners(self, indices, caller_rank: int) -> np.ndarray:
        """owning rank of every index, within the caller's replica sub-group"""
        idx = np.asarray(indices, np.int64).reshape(-1)
        if idx.size and (idx.min() < 0 or idx.max() >= self.n_samples):
            raise ValidationError(f"index out of range [0, {self.n_samples})")
        local = self._id[np.searchsorted(self._hi, idx, side="right")]
        return self.subgroup_of(caller_rank) * self.group_size + local

    def owner_of(self, global_index: int, caller_rank: int) -> int:
        return int(self.owners([global_index], caller_rank)[0])


def plan_fetch(indices, ownership: OwnershipMap, rank: int, world: int):
    """host plan of one collective fetch: per-owner request lists (in the
    caller's order within each owner), the send counts, and the permutation
    from owner-grouped arrival order back to ``indices`` order"""
    idx = np.asarray(indices, np.int64).reshape(-1)
    own = ownership.owners(idx, rank) if idx.size else np.zeros(0, np.int64)
    order = np.argsort(own, kind="stable")          # owner-grouped, stable
    counts = np.bincount(own, minlength=world).astype(np.int64)
    arrival_to_batch = np.empty_like(order)
    arrival_to_batch[order] = np.arange(order.shape[0])  # batch position -> arrival slot
    return idx[order], counts, arrival_to_batch


class ShardedDeviceStore:
    """DDStore's one-sided remote fetch (ddstore.py:316-490; the paper's MPI
    RMA store) rebuilt over NVLink: every rank keeps only
    its OwnershipMap shard of each group in HBM -- structures and their
    records' own edges -- and a batch is assembled by ONE collective
    exchange: the owners pack the requested structures on the device
    (gfm_gather_blocks), the packed arrays travel with all_to_all_single over
    NCCL, and the requester unpacks them into batch order and builds the
    CSR/CSC (gfm_csr_build).  With a plan (every rank's indices, as the
    global epoch schedule gives them) each rank derives its sends and
    receives from a global size table; without one, request counts and
    indices are exchanged first.

    ``fetch_device_batch`` is collective: every rank of ``comm`` calls it
    once per step (an idle rank with no indices).  Groups come as record
    lists, (shard records, total) or (decode_payloads arrays, total) --
    ``from_container`` decodes the rank's payloads on the device."""

    collective = True

    def __init__(self, groups: dict, comm, replication_factor: int = 1, device=None,
                 chunk_sizes=None):
        """``groups``: {name: full record list} (each rank keeps its shard),
        {name: (records of this rank's shard, total count)} or {name:
        (decode_payloads dict of this rank's shard, total count)}."""
        _lib.load(require_device=True)
        self.comm = comm
        self.rank, self.world = comm.rank, comm.size
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.ownership = {}
        self._g = {}
        self._max_deg = {}
        for name, v in groups.items():
            decoded = None
            if isinstance(v, tuple) and isinstance(v[0], dict):  # (decoded arrays, total)
                decoded, total = v
                recs = None
            elif isinstance(v, tuple):
                recs, total = v
            else:
                recs, total = v, len(v)
            own = OwnershipMap(total, self.world, replication_factor,
                               (chunk_sizes or {}).get(name))
            if decoded is not None:
                lo, hi = own.range_of(self.rank)
                if decoded["n"].shape[0] != hi - lo:
                    raise ValidationError(f"group {name!r}: shard of rank {self.rank} needs "
                                          f"{hi - lo} records, got {decoded['n'].shape[0]}")
                self.ownership[name] = own
                self._g[name] = decoded
                self._max_deg[name] = self._global_max(decoded["max_deg"])
                self._g[name]["sizes"] = self._size_table(own, decoded)
                continue
            lo, hi = own.range_of(self.rank)
            if not isinstance(v, tuple):
                recs = recs[lo:hi]
            if len(recs) != hi - lo:
                raise ValidationError(f"group {name!r}: shard of rank {self.rank} needs "
                                      f"{hi - lo} records, got {len(recs)}")
            self.ownership[name] = own
            periodic = self._global_max(int(any(getattr(r, "edge_shift", None) is not None
                                                 for r in recs)))
            self._g[name] = self._ingest(recs, bool(periodic))
            self._max_deg[name] = self._global_max(self._g[name]["max_deg"])
            self._g[name]["sizes"] = self._size_table(own, self._g[name])

    @classmethod
    def from_container(cls, path: str, comm, groups=None, replication_factor: int = 1,
                       device=None, device_decode: bool = True) -> "ShardedDeviceStore":
        """read only this rank's shard of each group: its payload bytes go to
        HBM undecoded and are checked and decoded there (decode_payloads);
        ``device_decode=False`` decodes on the host (container.read_range)"""
        from .container import GROUP_NAMES, read_manifest, read_range, read_range_raw
        man = read_manifest(path)
        out = {}
        for g in (groups or GROUP_NAMES):
            n = man.group(g).record_count
            if not n:
                continue
            lo, hi = OwnershipMap(n, comm.size, replication_factor).range_of(comm.rank)
            if device_decode:
                blob, offs, lens = read_range_raw(man, g, (lo, hi), path, pinned=True)
                out[g] = (decode_payloads(blob, offs, lens, device), n)
            else:
                out[g] = (read_range(man, g, (lo, hi), path), n)
        return cls(out, comm, replication_factor, device)

    def _global_max(self, x: int) -> int:
        if self.world == 1:
            return int(x)
        vals = self.comm.gather_obj(int(x))
        return int(self.comm.broadcast_obj(max(vals) if self.rank == 0 else None))

    def _size_table(self, own, g):
        """(atoms, edges) of every structure of the group on every rank (one
        host exchange at ingest): with it and a global schedule a fetch needs
        no size or count exchange"""
        if self.world == 1:
            return np.stack([g["n"], g["m"]], 1)
        shards = self.comm.gather_obj(np.stack([g["n"], g["m"]], 1))
        table = None
        if self.rank == 0:
            table = np.zeros((own.n_samples, 2), np.int64)
            for r in range(own.group_size):  # sub-group 0 covers the group
                lo, hi = own.local_ranges[r]
                table[lo:hi] = shards[r]
        return self.comm.broadcast_obj(table)

    def _ingest(self, recs, periodic: bool):
        dev = self.device
        n = np.array([int(np.asarray(r.atomic_numbers).shape[0]) for r in recs], np.int64)
        m = np.array([int(np.asarray(r.edge_index).reshape(-1, 2).shape[0]) for r in recs],
                     np.int64)
        cat = lambda xs, dt, shape: (np.concatenate([np.asarray(x, dt).reshape(shape)
                                                     for x in xs]) if len(xs) else
                                     np.zeros((0,) + shape[1:], dt))
        z = cat([r.atomic_numbers for r in recs], np.int32, (-1,))
        if z.size and (z.min() < 1 or z.max() > MAX_Z):
            raise ValidationError(f"atomic numbers must lie in [1, {MAX_Z}]")
        edges = cat([r.edge_index for r in recs], np.int32, (-1, 2))
        deg = 0
        for r in recs:
            e = np.asarray(r.edge_index, np.int64).reshape(-1, 2)
            if e.size:
                deg = max(deg, int(np.bincount(e[:, 1]).max()))
        t = lambda a: torch.as_tensor(np.ascontiguousarray(a), device=dev)
        return dict(n=n, m=m, noff=t(np.concatenate([[0], np.cumsum(n)])),
                    eoff=t(np.concatenate([[0], np.cumsum(m)])),
                    soff=t(np.arange(len(recs) + 1, dtype=np.int64)),
                    z=t(z), pos=t(cat([r.positions for r in recs], np.float64, (-1, 3))),
                    forces=t(cat([r.forces for r in recs], np.float64, (-1, 3))),
                    energy=t(np.array([float(r.energy) for r in recs], np.float64)),
                    edges=t(edges), max_deg=deg,
                    shift=t(cat([np.zeros((m[k], 3)) if getattr(r, "edge_shift", None) is None
                                 else r.edge_shift for k, r in enumerate(recs)], np.float64,
                                (-1, 3))) if periodic else None)

    # ---- one collective fetch ---------------------------------------------
    def _a2a(self, send, send_splits, recv_splits, row_shape, dtype):
        import torch.distributed as dist
        out = torch.empty((int(sum(recv_splits)),) + row_shape, dtype=dtype, device=self.device)
        if self.world == 1:
            out.copy_(send)
            return out
        dist.all_to_all_single(out, send.contiguous(), [int(x) for x in recv_splits],
                               [int(x) for x in send_splits], group=self.comm.group)
        return out

    def _upload(self, arrays: dict) -> dict:
        """host int32 / int64 arrays -> device views, through ONE pinned
        staging buffer per dtype and an asynchronous copy (no host sync: the
        caching host allocator keeps the staging block alive until its copy
        has run)"""
        out = {}
        for dt, tdt in ((np.int64, torch.int64), (np.int32, torch.int32)):
            items = [(k, np.ascontiguousarray(v, dt).reshape(-1)) for k, v in arrays.items()
                     if np.dtype(v.dtype) == np.dtype(dt)]
            if not items:
                continue
            total = sum(v.shape[0] for _, v in items)
            host = torch.empty(max(total, 1), dtype=tdt, pin_memory=True)
            hv = host.numpy()
            pos = 0
            spans = []
            for k, v in items:
                hv[pos:pos + v.shape[0]] = v
                spans.append((k, pos, v.shape[0]))
                pos += v.shape[0]
            dev = host.to(self.device, non_blocking=True)
            for k, p0, n in spans:
                out[k] = dev[p0:p0 + n]
        return out

    def _gather(self, idx_dev, n_out, src_off_dev, dst_off_dev, rows, src, width, add=None):
        """blocks idx of `src` -> a contiguous buffer in idx order"""
        out = torch.empty((int(rows),) + tuple(src.shape[1:]), dtype=src.dtype, device=self.device)
        if n_out and out.numel():
            call("gfm_gather_blocks", ptr(idx_dev), n_out, ptr(src_off_dev), ptr(dst_off_dev),
                 int(width), ptr(src), ptr(out), ptr(add), stream_handle())
        return out

    def fetch_device_batch(self, group: str, indices, dtype=torch.float32, plan=None):
        """Collective.  Returns a model.Batch of structures ``indices`` (in
        that order) or None when this rank requested nothing.

        ``plan``: every rank's indices for this call (``plan[rank] ==
        indices``), as a global schedule (epoch_schedule) provides them --
        then each rank derives what it serves and receives on the host and
        the exchange is only the payload: no count / index round trips and
        no host synchronisation, so the fetch queues behind the previous
        step's GPU work.  Without it the requests are exchanged first."""
        import torch.distributed as dist

        from .model import batch_from_device
        own = self.ownership[group]
        g = self._g[group]
        table = g["sizes"]
        dev = self.device
        W = self.world
        req, send_counts, arrival_to_batch = plan_fetch(indices, own, self.rank, W)
        lo, _ = own.range_of(self.rank)
        if plan is not None:
            if len(plan) != W or not np.array_equal(
                    np.asarray(plan[self.rank], np.int64).reshape(-1),
                    np.asarray(indices, np.int64).reshape(-1)):
                raise ValidationError("plan must hold every rank's indices, this rank's == indices")
            serve_parts, recv_counts = [], np.zeros(W, np.int64)
            for p in range(W):
                rq, cnt, _ = plan_fetch(plan[p], own, p, W)
                st = int(cnt[:self.rank].sum())
                serve_parts.append(rq[st:st + int(cnt[self.rank])])
                recv_counts[p] = cnt[self.rank]
            serve = np.concatenate(serve_parts) - lo
        else:
            # request counts and indices (all_to_all; two host syncs)
            sc = torch.as_tensor(send_counts, device=dev)
            rc = torch.empty_like(sc)
            if W > 1:
                dist.all_to_all_single(rc, sc, group=self.comm.group)
            else:
                rc.copy_(sc)
            recv_counts = rc.cpu().numpy()
            want = self._a2a(torch.as_tensor(req, device=dev), send_counts, recv_counts, (),
                             torch.int64)
            serve = want.cpu().numpy() - lo                  # local positions I serve
        # every row count from the global size table (host)
        sizes = table[serve + lo] if serve.size else np.zeros((0, 2), np.int64)
        got = table[req] if req.size else np.zeros((0, 2), np.int64)
        peer_of_serve = np.repeat(np.arange(W), recv_counts)
        peer_of_req = np.repeat(np.arange(W), send_counts)
        per_peer = lambda peers, col: np.bincount(peers, weights=col, minlength=W).astype(
            np.int64) if peers.size else np.zeros(W, np.int64)
        s_atoms, s_edges = per_peer(peer_of_serve, sizes[:, 0]), per_peer(peer_of_serve, sizes[:, 1])
        r_atoms, r_edges = per_peer(peer_of_req, got[:, 0]), per_peer(peer_of_req, got[:, 1])
        B = int(arrival_to_batch.shape[0])
        cum = lambda x: np.concatenate([[0], np.cumsum(x)]).astype(np.int64)
        n_arr, m_arr = got[:, 0], got[:, 1]
        src_slot = arrival_to_batch  # batch position b comes from arrival slot src_slot[b]
        n_b, m_b = n_arr[src_slot], m_arr[src_slot]
        host_off = cum(n_b)
        # every small index / offset array of this fetch in one pinned upload
        up = self._upload(dict(
            serve=serve.astype(np.int32), p_noff=cum(sizes[:, 0]), p_eoff=cum(sizes[:, 1]),
            p_soff=np.arange(serve.shape[0] + 1, dtype=np.int64),
            slot=src_slot.astype(np.int32), a_noff=cum(n_arr), a_eoff=cum(m_arr),
            a_soff=np.arange(B + 1, dtype=np.int64), host_off=host_off, e_off64=cum(m_b),
            node_base=host_off[:-1].astype(np.int32), e_off=cum(m_b).astype(np.int32),
            off32=host_off.astype(np.int32)))
        ns = int(serve.shape[0])
        sv = up.get("serve")
        packed = dict(
            z=self._gather(sv, ns, g["noff"], up["p_noff"], sizes[:, 0].sum(), g["z"], 1),
            pos=self._gather(sv, ns, g["noff"], up["p_noff"], sizes[:, 0].sum(), g["pos"], 6),
            forces=self._gather(sv, ns, g["noff"], up["p_noff"], sizes[:, 0].sum(), g["forces"], 6),
            energy=self._gather(sv, ns, g["soff"], up["p_soff"], ns, g["energy"], 2),
            edges=self._gather(sv, ns, g["eoff"], up["p_eoff"], sizes[:, 1].sum(), g["edges"], 2),
            shift=None if g["shift"] is None else
            self._gather(sv, ns, g["eoff"], up["p_eoff"], sizes[:, 1].sum(), g["shift"], 6))
        recv = dict(
            z=self._a2a(packed["z"], s_atoms, r_atoms, (), torch.int32),
            pos=self._a2a(packed["pos"], s_atoms, r_atoms, (3,), torch.float64),
            forces=self._a2a(packed["forces"], s_atoms, r_atoms, (3,), torch.float64),
            energy=self._a2a(packed["energy"], recv_counts, send_counts, (), torch.float64),
            edges=self._a2a(packed["edges"], s_edges, r_edges, (2,), torch.int32),
            shift=None if g["shift"] is None else
            self._a2a(packed["shift"], s_edges, r_edges, (3,), torch.float64))
        if B == 0:
            return None
        sl, N, E = up["slot"], int(host_off[-1]), int(m_b.sum())
        z = self._gather(sl, B, up["a_noff"], up["host_off"], N, recv["z"], 1)
        pos = self._gather(sl, B, up["a_noff"], up["host_off"], N, recv["pos"], 6)
        forces = self._gather(sl, B, up["a_noff"], up["host_off"], N, recv["forces"], 6)
        energy = self._gather(sl, B, up["a_soff"], up["a_soff"], B, recv["energy"], 2)
        # record-local endpoints + the structure's node base in the batch
        edges = self._gather(sl, B, up["a_eoff"], up["e_off64"], E, recv["edges"], 2,
                             add=up["node_base"])
        shift = None if g["shift"] is None else \
            self._gather(sl, B, up["a_eoff"], up["e_off64"], E, recv["shift"], 6)
        return batch_from_device(z, pos, energy.to(dtype), forces.to(dtype),
                                 edges[:, 0].contiguous(), edges[:, 1].contiguous(),
                                 up["e_off"], up["off32"], host_off, dtype, shift,
                                 self._max_deg[group])

    def fetch_batch(self, group, indices):
        raise ValidationError("a sharded store fetches collectively: use fetch_device_batch")

    def close(self):
        self._g.clear()
