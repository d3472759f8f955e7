"""Neighbour lists on the GPU and the synthetic structure generator.

Reference: build_cutoff_edges (preprocess.py:90-104), ToyPotential
(preprocess.py:41-87) and generate_synthetic (preprocess.py:107-153).  The
cutoff search runs in the sm_100a radius kernel (bit-exact float64
predicate); the generator draws structures with the reference's exact rng
call sequence, so equal seeds give equal positions, species and edges.
Labels use a vectorised restatement of the toy potential (same formula;
float64 summation order may differ from the reference in the last bits).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query, stream_handle
from .errors import ValidationError
from .records import MAX_Z, GraphRecord


def default_coefficients() -> np.ndarray:
    return -0.1 * np.arange(1, MAX_Z + 1, dtype=np.float64)


def radius_graph(pos_list, rc: float, max_nbr: int = 0, cells=None, device=None):
    """Batched cutoff search for several structures on the device.

    Returns (rowptr, col_src, edge_dst, shifts_dx, node_offsets) as device
    tensors in dst-sorted CSR order, float64 displacements."""
    _lib.load(require_device=True)
    dev = torch.device(device) if device is not None else torch.device(
        "cuda", torch.cuda.current_device())
    counts = np.array([np.asarray(p).reshape(-1, 3).shape[0] for p in pos_list], np.int64)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    N, B = int(offsets[-1]), len(pos_list)
    pos = torch.from_numpy(np.concatenate([np.asarray(p, np.float64).reshape(-1, 3)
                                           for p in pos_list]) if N else np.zeros((0, 3))).to(dev)
    off = torch.from_numpy(offsets).to(dev)
    s = stream_handle()
    gnode = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
    call("gfm_graph_of_node", ptr(off), B, ptr(gnode), s)
    cells_t = None
    if cells is not None:
        cells_t = torch.as_tensor(np.asarray(cells, np.float64).reshape(B, 3), device=dev)
        if rc >= 0.5 * float(cells_t.min()):
            raise ValidationError("minimum image needs rc < min(cell)/2")
    deg = torch.empty(max(N, 1), dtype=torch.int32, device=dev)
    call("gfm_radius_count", ptr(pos), ptr(off), ptr(gnode), N, ptr(cells_t), float(rc),
         int(max_nbr or 0), ptr(deg), s)
    rowptr = torch.empty(N + 1, dtype=torch.int32, device=dev)
    ws = torch.empty(query("gfm_scan_workspace_bytes", N), dtype=torch.uint8, device=dev)
    call("gfm_exclusive_scan", ptr(deg), N, ptr(rowptr), ptr(ws), s)
    E = int(rowptr[N].item())
    Ec = max(E, 1)
    col_src = torch.empty(Ec, dtype=torch.int32, device=dev)
    edge_dst = torch.empty(Ec, dtype=torch.int32, device=dev)
    w = torch.empty(Ec, dtype=torch.float64, device=dev)
    dx = torch.empty(Ec, 3, dtype=torch.float64, device=dev)
    call("gfm_radius_fill", ptr(pos), ptr(off), ptr(gnode), N, ptr(cells_t), float(rc),
         int(max_nbr or 0), ptr(rowptr), ptr(col_src), ptr(edge_dst), ptr(w), ptr(dx), _lib.F64, s)
    return rowptr, col_src[:E], edge_dst[:E], dx[:E], off, pos


def build_cutoff_edges(positions, cutoff_radius: float, max_nbr: int = 0, cell=None):
    """All ordered pairs (i, j), i != j, |x_i - x_j| <= rc, row-major (src
    ascending, then dst) as uint32 (m, 2) -- preprocess.py:90-104, on the
    GPU.  ``max_nbr`` / ``cell`` are the cap / minimum-image extensions."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1, 3)
    if pos.shape[0] < 2:
        return np.zeros((0, 2), dtype=np.uint32)
    rowptr, col_src, edge_dst, _, _, _ = radius_graph(
        [pos], cutoff_radius, max_nbr, None if cell is None else [cell])
    key = col_src.to(torch.int64) * pos.shape[0] + edge_dst.to(torch.int64)
    order = torch.argsort(key)  # CSR (dst, src) -> reference row-major (src, dst)
    out = torch.stack([col_src[order], edge_dst[order]], 1)
    return out.cpu().numpy().astype(np.uint32)


def toy_labels(z, pos, edges, coefficients=None, d0: float = 1.0):
    """ToyPotential energy / forces (preprocess.py:41-87), vectorised."""
    coeff = default_coefficients() if coefficients is None else np.asarray(coefficients)
    z = np.asarray(z, np.int64)
    e = np.asarray(edges, np.int64).reshape(-1, 2)
    e = e[e[:, 0] < e[:, 1]]
    delta = pos[e[:, 0]] - pos[e[:, 1]]
    d = np.sqrt((delta ** 2).sum(axis=1))
    energy = float(coeff[z - 1].sum() + ((d - d0) ** 2).sum())
    ok = d >= 1e-12
    g = np.zeros_like(delta)
    g[ok] = (2.0 * (d[ok] - d0) / d[ok])[:, None] * delta[ok]
    f = np.zeros_like(pos)
    np.add.at(f, e[:, 0], -g)
    np.add.at(f, e[:, 1], g)
    return energy, f


def generate_synthetic(count, n_atoms_range=(4, 12), element_distribution=None,
                       box_length: float = 6.0, cutoff_radius: float = 2.0, seed: int = 0,
                       max_nbr: int = 0, periodic: bool = False, device=None):
    """Seeded random structures (preprocess.py:107-153): identical rng call
    sequence; edges from the GPU radius kernel (optionally capped /
    periodic, labels always from the uncapped non-periodic toy potential)."""
    if cutoff_radius <= 0:
        raise ValidationError(f"cutoff_radius must be > 0, got {cutoff_radius}")
    lo, hi = n_atoms_range
    if lo < 1 or hi < lo:
        raise ValidationError(f"invalid n_atoms_range {n_atoms_range}")
    element_distribution = element_distribution or {1: 1.0, 6: 1.0, 8: 1.0}
    zs = np.array(sorted(element_distribution), dtype=np.int64)
    if zs.min() < 1 or zs.max() > MAX_Z:
        raise ValidationError("element numbers must lie in [1, 118]")
    w = np.array([element_distribution[int(z)] for z in zs], dtype=np.float64)
    if w.sum() <= 0:
        raise ValidationError("element_distribution has zero total weight")
    probs = w / w.sum()
    rng = np.random.default_rng(seed)
    zl, pl = [], []
    for _ in range(count):
        n = int(rng.integers(lo, hi + 1))
        zl.append(zs[rng.choice(zs.size, size=n, p=probs)].astype(np.uint8))
        pl.append(rng.uniform(0.0, box_length, size=(n, 3)))
    if count == 0:
        return []

    def edges_of(mx, cells):
        rowptr, col_src, edge_dst, dx, off, _ = radius_graph(pl, cutoff_radius, mx, cells, device)
        off = off.cpu().numpy()
        r = rowptr.cpu().numpy()
        cs, ed, dd = col_src.cpu().numpy(), edge_dst.cpu().numpy(), dx.cpu().numpy()
        out = []
        for g in range(count):
            a, b = r[off[g]], r[off[g + 1]]
            src, dst = cs[a:b] - off[g], ed[a:b] - off[g]
            order = np.lexsort((dst, src))
            pair = np.stack([src[order], dst[order]], 1).astype(np.uint32)
            shift = dd[a:b][order] - (pl[g][src[order]] - pl[g][dst[order]])
            out.append((pair, shift))
        return out

    full = edges_of(0, None)
    cells = [(box_length,) * 3] * count if periodic else None
    used = full if (not max_nbr and not periodic) else edges_of(max_nbr, cells)
    records = []
    for g in range(count):
        energy, forces = toy_labels(zl[g], pl[g], full[g][0])
        rec = GraphRecord(zl[g], pl[g], used[g][0], energy, forces)
        if periodic:
            rec.edge_shift = used[g][1]
        records.append(rec)
    return records
