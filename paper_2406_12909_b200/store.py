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
    def __init__(self, records, device, arrays=None):
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

    def __init__(self, groups: dict, device=None, _arrays: dict | None = None):
        _lib.load(require_device=True)
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self._groups = {k: _Group(v, self.device) for k, v in groups.items()}
        for k, a in (_arrays or {}).items():
            self._groups[k] = _Group(None, self.device, a)
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
    def from_container(cls, path: str, groups=None, device=None) -> "DeviceStructureStore":
        """Ingest a gfmkit container directory (container.py) into HBM."""
        from .container import GROUP_NAMES, read_group, read_manifest
        man = read_manifest(path)
        return cls({g: read_group(man, g, path) for g in (groups or GROUP_NAMES)
                    if man.group(g).record_count}, device)

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
