"""Drop-in for ``gfmkit.model`` backed by sm_100a kernels.

Same names, argument meaning and error behaviour as the reference
(``/root/reference/pkg/src/gfmkit/model.py``); the arithmetic runs in the
C-ABI library (``include/gfm_b200.h``) on device tensors.  Differences a
caller sees:

* arrays are ``torch.Tensor`` on the CUDA device (float32 by default, float64
  for exact-parity work) instead of numpy float64; ``ModelParams.flatten()``
  still returns a host float64 numpy vector in the reference's flat order;
* two extra aggregation kinds, ``std-agg`` and ``pna-agg`` (concat of
  sum / mean / max / std, U is H x 4H), which the reference lacks.

There is no CPU fallback: without the built library or a GPU every compute
call raises ``ExtensionMissingError``.
"""

from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query, stream_handle
from .errors import ValidationError
from .records import MAX_Z, GraphRecord

MPNN_KINDS = ("mean-agg", "sum-agg", "max-agg", "std-agg", "pna-agg")
KIND_PARTS = {
    "mean-agg": _lib.PART_MEAN,
    "sum-agg": _lib.PART_SUM,
    "max-agg": _lib.PART_MAX,
    "std-agg": _lib.PART_STD,
    "pna-agg": _lib.PART_SUM | _lib.PART_MEAN | _lib.PART_MAX | _lib.PART_STD,
}


def _n_parts(kind: str) -> int:
    return bin(KIND_PARTS[kind]).count("1")


@dataclass
class ModelConfig:
    """Architecture + loss hyperparameters (model.py:42-86)."""

    mpnn_kind: str = "mean-agg"
    mpnn_layers: int = 3
    mpnn_width: int = 50
    fc_layers: int = 2
    fc_width: int = 50
    batch_size: int = 32
    learning_rate: float = 1e-3
    alpha_energy: float = 1.0
    alpha_forces: float = 100.0

    def __post_init__(self):
        if self.mpnn_kind not in MPNN_KINDS:
            raise ValidationError(f"mpnn_kind {self.mpnn_kind!r} not in {MPNN_KINDS}")
        for name in ("mpnn_layers", "mpnn_width", "fc_width", "batch_size"):
            if int(getattr(self, name)) < 1:
                raise ValidationError(f"{name} must be >= 1")
        if self.fc_layers < 2:
            raise ValidationError("fc_layers must be >= 2 (input and output layers)")
        if self.alpha_energy <= 0 or self.alpha_forces <= 0:
            raise ValidationError("loss weights must be positive")
        if self.learning_rate <= 0:
            raise ValidationError("learning_rate must be positive")

    @property
    def n_parts(self) -> int:
        return _n_parts(self.mpnn_kind)

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "mpnn_kind", "mpnn_layers", "mpnn_width", "fc_layers", "fc_width",
            "batch_size", "learning_rate", "alpha_energy", "alpha_forces")}

    @classmethod
    def from_dict(cls, doc: dict) -> "ModelConfig":
        return cls(**doc)


def _is_egnn(config) -> bool:
    return getattr(config, "model_type", "mpnn") == "egnn"


def param_shapes(config: ModelConfig):
    """(name, shape) in the canonical flat order (ModelParams.arrays,
    model.py:120-132); U is (H, k*H) for k aggregation parts.  An
    EGNNConfig has its own order (egnn.egnn_param_shapes)."""
    if _is_egnn(config):
        from .egnn import egnn_param_shapes
        return egnn_param_shapes(config)
    h, g, k = config.mpnn_width, config.fc_width, config.n_parts
    out = [("embedding", (MAX_Z, h))]
    for l in range(config.mpnn_layers):
        out += [(f"layer_{l}.w", (h, h)), (f"layer_{l}.u", (h, k * h)), (f"layer_{l}.b", (h,))]
    ws = [(g, h)] + [(g, g)] * (config.fc_layers - 2) + [(1, g)]
    bs = [(g,)] * (config.fc_layers - 1) + [(1,)]
    for f in range(config.fc_layers):
        out += [(f"head_{f}.w", ws[f]), (f"head_{f}.b", bs[f])]
    out += [("force.v", (h, h)), ("force.c", (h,)), ("force.u", (h,))]
    return out


def count_params(config: ModelConfig) -> int:
    """Closed form (model.py:89-97) with U widened to k*H:
    118H + L(H^2 + kH^2 + H) + [HG + G + (F-2)(G^2 + G) + G + 1] + H^2 + 2H."""
    if _is_egnn(config):
        from .egnn import egnn_count_params
        return egnn_count_params(config)
    h, l, k = config.mpnn_width, config.mpnn_layers, config.n_parts
    f, g = config.fc_layers, config.fc_width
    head = h * g + g + max(0, f - 2) * (g * g + g) + (g + 1)
    return MAX_Z * h + l * (h * h + k * h * h + h) + head + (h * h + 2 * h)


def _device(device=None) -> torch.device:
    if device is None:
        _lib.load(require_device=True)
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


class ParamLayout:
    """Device layout of the flat parameter vector: the reference's order
    (model.py:120-132) with every array starting on a 16-byte boundary (so
    each weight view is a TMA-loadable tensor).  ``P`` = reference length,
    ``Pp`` = padded device length; padding entries stay exactly 0 (zero
    gradient, zero Adam update)."""

    def __init__(self, config: ModelConfig):
        self.entries = []
        off = 0
        for name, shape in param_shapes(config):
            size = int(np.prod(shape))
            self.entries.append((name, tuple(shape), off, size))
            off += (size + 3) & ~3
        self.Pp = off
        self.P = count_params(config)
        self.index_np = np.concatenate([np.arange(o, o + n) for _, _, o, n in self.entries])
        self._index = {}

    def index(self, device) -> torch.Tensor:
        key = str(device)
        if key not in self._index:
            self._index[key] = torch.as_tensor(self.index_np, device=device)
        return self._index[key]

    def compact(self, padded: torch.Tensor) -> torch.Tensor:
        """padded device vector -> reference-order flat vector"""
        return padded[self.index(padded.device)]

    def pad(self, flat, device, dtype) -> torch.Tensor:
        """reference-order flat vector (numpy or tensor) -> padded device vector"""
        t = flat.detach() if isinstance(flat, torch.Tensor) else torch.from_numpy(
            np.ascontiguousarray(flat, dtype=np.float64))
        if t.dim() != 1 or t.shape[0] != self.P:
            raise ValidationError(f"flat vector has {tuple(t.shape)}, model needs ({self.P},)")
        out = torch.zeros(self.Pp, dtype=dtype, device=device)
        out[self.index(device)] = t.to(device=device, dtype=dtype)
        return out


_LAYOUTS: dict = {}


def param_layout(config: ModelConfig) -> ParamLayout:
    key = tuple(sorted(config.to_dict().items()))
    if key not in _LAYOUTS:
        _LAYOUTS[key] = ParamLayout(config)
    return _LAYOUTS[key]


class ModelParams:
    """All weights as one padded device tensor with named views.

    The element order is the reference's (embedding; per layer W, U, b; per
    head layer A, c; force V, c, u); ``flatten``/``from_flat`` convert to and
    from the reference's float64 flat vector bit-exactly (float64 storage)."""

    def __init__(self, config: ModelConfig, flat: torch.Tensor):
        lay = param_layout(config)
        if flat.dim() != 1 or flat.shape[0] != lay.Pp:
            raise ValidationError(
                f"device parameter vector has {tuple(flat.shape)}, layout needs ({lay.Pp},)")
        self.config = config
        self.layout = lay
        self.flat = flat
        self._views = {name: flat[off:off + size].view(shape)
                       for name, shape, off, size in lay.entries}

    # reference attribute names ------------------------------------------
    @property
    def embedding(self):
        return self._views["embedding"]

    @property
    def layer_w(self):
        return [self._views[f"layer_{l}.w"] for l in range(self.config.mpnn_layers)]

    @property
    def layer_u(self):
        return [self._views[f"layer_{l}.u"] for l in range(self.config.mpnn_layers)]

    @property
    def layer_b(self):
        return [self._views[f"layer_{l}.b"] for l in range(self.config.mpnn_layers)]

    @property
    def head_w(self):
        return [self._views[f"head_{f}.w"] for f in range(self.config.fc_layers)]

    @property
    def head_b(self):
        return [self._views[f"head_{f}.b"] for f in range(self.config.fc_layers)]

    @property
    def force_v(self):
        return self._views["force.v"]

    @property
    def force_c(self):
        return self._views["force.c"]

    @property
    def force_u(self):
        return self._views["force.u"]

    def view(self, name):
        return self._views[name]

    def arrays(self):
        for name, _ in param_shapes(self.config):
            yield name, self._views[name]

    @property
    def n_params(self) -> int:
        return self.layout.P

    @property
    def dtype(self):
        return self.flat.dtype

    def flatten(self) -> np.ndarray:
        return self.layout.compact(self.flat.detach()).to("cpu", torch.float64).numpy().copy()

    @classmethod
    def zeros(cls, config: ModelConfig, device=None, dtype=torch.float32) -> "ModelParams":
        lay = param_layout(config)
        return cls(config, torch.zeros(lay.Pp, dtype=dtype, device=_device(device)))

    @classmethod
    def from_flat(cls, config: ModelConfig, flat, device=None, dtype=None) -> "ModelParams":
        lay = param_layout(config)
        if isinstance(flat, torch.Tensor):
            dev = _device(device) if device or not flat.is_cuda else flat.device
            dtype = dtype or (flat.dtype if flat.is_floating_point() else torch.float32)
        else:
            dev = _device(device)
            dtype = dtype or torch.float32
        return cls(config, lay.pad(flat, dev, dtype))


def init_params_flat(config: ModelConfig, seed: int = 0) -> np.ndarray:
    """init_params (model.py:178-187) on the host, float64: uniform(+-1/sqrt(H))
    drawn from default_rng(seed) in flat order, biases (.b/.c) zero."""
    if _is_egnn(config):
        from .egnn import egnn_init_flat
        return egnn_init_flat(config, seed)
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(config.mpnn_width)
    parts = []
    for name, shape in param_shapes(config):
        if name.endswith(".b") or name.endswith(".c"):
            parts.append(np.zeros(int(np.prod(shape))))
        else:
            parts.append(rng.uniform(-bound, bound, size=shape).ravel())
    return np.concatenate(parts)


def init_params(config: ModelConfig, seed: int = 0, device=None, dtype=torch.float32) -> ModelParams:
    return ModelParams.from_flat(config, init_params_flat(config, seed), device=device, dtype=dtype)


# --------------------------------------------------------------------------
# Batch packing
# --------------------------------------------------------------------------


class Batch:
    """A packed batch on the device (model.py:195-231).

    Node ids are global; edges live in dst-sorted CSR order (rowptr, col_src,
    edge_dst, edge_w, edge_dx) with the src-sorted CSC view (csc_ptr,
    csc_eid, csc_dst) for deterministic backward gathers.  ``order`` maps a
    CSR position to the record edge index (the reference's stable argsort).
    Labels are mutable and read at loss time, as in the reference."""

    counts = None  # device [B, N] of a ragged batch in capacity buffers (else None)
    periodic = False  # edges carry periodic image shifts

    def __init__(self, **kw):
        self.dtype = kw.pop("dtype")
        self._e_true = None
        self._f_true = None
        energy = kw.pop("energy_true")
        forces = kw.pop("forces_true")
        for k, v in kw.items():
            setattr(self, k, v)
        self.energy_true = energy
        self.forces_true = forces

    @property
    def energy_true(self):
        return self._e_true

    @energy_true.setter
    def energy_true(self, value):
        self._e_true = _to_dev(value, self.device, self.dtype).reshape(-1)

    @property
    def forces_true(self):
        return self._f_true

    @forces_true.setter
    def forces_true(self, value):
        self._f_true = _to_dev(value, self.device, self.dtype).reshape(-1, 3).contiguous()

    @property
    def n_graphs(self) -> int:
        return int(self.host_offsets.shape[0] - 1)

    @property
    def n_edges(self) -> int:
        if self._n_edges is None:
            self._n_edges = int(self.rowptr[self.n_nodes].item())
        return self._n_edges

    @property
    def deg(self):
        return self.rowptr[1:] - self.rowptr[:-1]

    @property
    def node_offsets_host(self):
        return self.host_offsets


def _to_dev(value, device, dtype):
    if isinstance(value, torch.Tensor):
        return value.detach().to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.asarray(value, dtype=np.float64), dtype=dtype, device=device)


def _i32(a, device):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device, non_blocking=True)


def make_batch(records, device=None, dtype=torch.float32) -> Batch:
    """make_batch (model.py:234-285): host concatenation, then the CSR/CSC,
    edge weights and displacements are built on the device."""
    if not records:
        raise ValidationError("cannot build a batch from zero records")
    dev = _device(device)
    code = _lib.dtype_code(dtype)
    n_per = np.array([int(np.asarray(r.atomic_numbers).shape[0]) for r in records], np.int64)
    offsets = np.concatenate([[0], np.cumsum(n_per)])
    z = np.concatenate([np.asarray(r.atomic_numbers, np.int64) for r in records])
    pos = np.concatenate([np.asarray(r.positions, np.float64).reshape(-1, 3) for r in records])
    forces = np.concatenate([np.asarray(r.forces, np.float64).reshape(-1, 3) for r in records])
    energy = np.array([float(r.energy) for r in records], np.float64)
    e_per = np.array([int(np.asarray(r.edge_index).reshape(-1, 2).shape[0]) for r in records])
    e_off = np.concatenate([[0], np.cumsum(e_per)])
    if e_off[-1]:
        src = np.concatenate([np.asarray(r.edge_index, np.int64).reshape(-1, 2)[:, 0] + offsets[g]
                              for g, r in enumerate(records)])
        dst = np.concatenate([np.asarray(r.edge_index, np.int64).reshape(-1, 2)[:, 1] + offsets[g]
                              for g, r in enumerate(records)])
    else:
        src = dst = np.zeros(0, np.int64)
    shifts = [getattr(r, "edge_shift", None) for r in records]
    shift = None
    if any(s is not None for s in shifts):
        shift = np.concatenate([np.zeros((e_per[g], 3)) if s is None else np.asarray(s, np.float64)
                                for g, s in enumerate(shifts)])
    N, E, B = int(offsets[-1]), int(e_off[-1]), len(records)
    if E and (src.max() >= N or dst.max() >= N or min(src.min(), dst.min()) < 0):
        raise ValidationError("edge endpoint out of range")
    t_pos = torch.from_numpy(pos).to(dev, non_blocking=True)
    t_src, t_dst = _i32(src, dev), _i32(dst, dev)
    t_eoff, t_off = _i32(e_off, dev), _i32(offsets, dev)
    t_shift = torch.from_numpy(shift).to(dev) if shift is not None else None
    return batch_from_device(_i32(z, dev), t_pos, energy, forces, t_src, t_dst, t_eoff, t_off,
                             offsets, dtype, t_shift,
                             int(np.bincount(dst, minlength=1).max()) if E else 0)


def batch_from_device(z, pos, energy, forces, src, dst, edge_offsets, node_offsets,
                      host_offsets, dtype=torch.float32, shift=None, max_deg=None) -> Batch:
    """make_batch's device half (model.py:234-285): structures already
    concatenated on the device -- z i32 [N], pos f64 [N,3], energy [B],
    forces [N,3], record edges as global src / dst i32 [E] with per-graph edge
    offsets (device, B+1) -- into the dst-sorted CSR + src-sorted CSC batch.
    ``max_deg`` bounds any row (enables the uint8 argmax; None = unknown)."""
    dev = pos.device
    code = _lib.dtype_code(dtype)
    offsets = np.asarray(host_offsets, np.int64)
    n_per = np.diff(offsets)
    N, B = int(offsets[-1]), int(offsets.shape[0] - 1)
    E = int(src.shape[0])
    f = dict(device=dev)
    t_pos, t_src, t_dst, t_eoff, t_off, t_shift = pos, src, dst, edge_offsets, node_offsets, shift
    Ec = max(E, 1)
    rowptr = torch.empty(N + 1, dtype=torch.int32, **f)
    csc_ptr = torch.empty(N + 1, dtype=torch.int32, **f)
    col_src = torch.empty(Ec, dtype=torch.int32, **f)
    edge_dst = torch.empty(Ec, dtype=torch.int32, **f)
    order = torch.empty(Ec, dtype=torch.int32, **f)
    csc_eid = torch.empty(Ec, dtype=torch.int32, **f)
    csc_dst = torch.empty(Ec, dtype=torch.int32, **f)
    edge_w = torch.empty(Ec, dtype=dtype, **f)
    edge_dx = torch.empty(Ec, 3, dtype=dtype, **f)
    ws = torch.empty(query("gfm_csr_workspace_bytes", N, E, B), dtype=torch.uint8, **f)
    s = stream_handle()
    call("gfm_csr_build", ptr(t_src), ptr(t_dst), ptr(t_eoff), B, ptr(t_pos), ptr(t_shift), N, E,
         ptr(rowptr), ptr(col_src), ptr(edge_dst), ptr(edge_w), ptr(edge_dx), ptr(order),
         ptr(csc_ptr), ptr(csc_eid), ptr(csc_dst), code, ptr(ws), s)
    gnode = torch.empty(max(N, 1), dtype=torch.int32, **f)
    call("gfm_graph_of_node", ptr(t_off), B, ptr(gnode), s)
    b = Batch(dtype=dtype, device=dev, z=z, pos=t_pos, node_offsets=t_off,
              n_per_graph=_i32(n_per, dev), graph_of_node=gnode, energy_true=energy,
              forces_true=forces, rowptr=rowptr, col_src=col_src, edge_dst=edge_dst,
              edge_w=edge_w, edge_dx=edge_dx, csc_ptr=csc_ptr, csc_eid=csc_eid,
              csc_dst=csc_dst, order=order, n_nodes=N, e_cap=E, _n_edges=E,
              host_offsets=offsets, host_n_per=n_per, max_deg=max_deg,
              periodic=shift is not None)
    b._keep = (t_src, t_dst, t_eoff, t_shift, ws)
    return b


def radius_batch(pos: torch.Tensor, z: torch.Tensor, node_offsets: torch.Tensor,
                 host_offsets: np.ndarray, rc: float, max_nbr: int = 0, cells=None,
                 energy_true=None, forces_true=None, dtype=torch.float32, e_cap=None,
                 out: dict | None = None, fused: bool | None = None,
                 max_atoms: int | None = None) -> Batch:
    """Batch assembly from device-resident raw structures: the radius graph
    (build_cutoff_edges, preprocess.py:90-104, plus cap / minimum-image
    extensions) is built on the GPU directly as the dst-sorted CSR.

    ``e_cap`` bounds the edge buffers (default: exact count, one host sync);
    pass ``n_nodes * max_nbr`` to stay sync-free (CUDA-graph capture).
    ``fused`` (default: when ``e_cap`` is given and the graphs are small
    enough) builds everything in one per-graph kernel (gfm_radius_batch).

    Capacity mode (ragged batches, fused path only): ``node_offsets`` is a
    device array whose contents change per step, ``host_offsets`` only fixes
    the graph capacity B (its length) and ``max_atoms`` bounds any graph's
    size; ``pos`` may hold more rows than ``node_offsets[B]`` (the tail is
    edge-free and graph-less).  ``out["n_per_graph"]`` / ``out["counts"]``
    (device [B, N]) preset by the caller are used as the batch's per-graph
    sizes and true counts."""
    dev = pos.device
    code = _lib.dtype_code(dtype)
    N = int(pos.shape[0])
    B = int(host_offsets.shape[0] - 1)
    s = stream_handle()
    o = out if out is not None else {}

    def buf(name, shape, dt):
        t = o.get(name)
        if t is None or t.dtype != dt or tuple(t.shape) != tuple(shape):
            t = torch.empty(shape, dtype=dt, device=dev)
            o[name] = t
        return t

    gnode = buf("gnode", (max(N, 1),), torch.int32)
    n_per = np.diff(host_offsets)
    if max_atoms is None:
        max_atoms = int(n_per.max()) if n_per.size else 0
    can_fuse = e_cap is not None and B > 0 and max_atoms <= _FUSED_MAX_ATOMS and (
        bool(max_nbr) or max_atoms <= _FUSED_UNCAPPED_ATOMS)
    if fused and not can_fuse:
        raise ValidationError("fused batch assembly needs e_cap and graphs of <= 256 atoms")
    if o.get("counts") is not None and not (can_fuse and fused is not False):
        raise ValidationError("ragged (capacity) batches need the fused assembly: e_cap given, "
                              "graphs of <= 256 atoms")
    if can_fuse and fused is not False:
        # one fused kernel: neighbour search + CSR + CSC + graph_of_node
        Ec = max(int(e_cap), 1)
        rowptr = buf("rowptr", (N + 1,), torch.int32)
        col_src = buf("col_src", (Ec,), torch.int32)
        edge_dst = buf("edge_dst", (Ec,), torch.int32)
        edge_w = buf("edge_w", (Ec,), dtype)
        edge_dx = buf("edge_dx", (Ec, 3), dtype)
        csc_ptr = buf("csc_ptr", (N + 1,), torch.int32)
        csc_eid = buf("csc_eid", (Ec,), torch.int32)
        csc_dst = buf("csc_dst", (Ec,), torch.int32)
        ws = buf("rb_ws", (query("gfm_radius_batch_workspace_bytes", B),), torch.uint8)
        call("gfm_radius_batch", ptr(pos), ptr(node_offsets), B, N, max_atoms, ptr(cells),
             float(rc), int(max_nbr or 0), ptr(gnode), ptr(rowptr), ptr(col_src), ptr(edge_dst),
             ptr(edge_w), ptr(edge_dx), ptr(csc_ptr), ptr(csc_eid), ptr(csc_dst), Ec, ptr(ws),
             code, s)
        return _radius_batch_result(o, dev, dtype, z, pos, node_offsets, gnode, host_offsets,
                                    energy_true, forces_true, rowptr, col_src, edge_dst, edge_w,
                                    edge_dx, csc_ptr, csc_eid, csc_dst, e_cap, None,
                                    _deg_bound(max_atoms, max_nbr), cells is not None)
    call("gfm_graph_of_node", ptr(node_offsets), B, ptr(gnode), s)
    deg = buf("deg", (max(N, 1),), torch.int32)
    cells_t = None if cells is None else cells
    call("gfm_radius_count", ptr(pos), ptr(node_offsets), ptr(gnode), N, ptr(cells_t), float(rc),
         int(max_nbr or 0), ptr(deg), s)
    rowptr = buf("rowptr", (N + 1,), torch.int32)
    sws = buf("scan_ws", (query("gfm_scan_workspace_bytes", N),), torch.uint8)
    call("gfm_exclusive_scan", ptr(deg), N, ptr(rowptr), ptr(sws), s)
    if e_cap is None:
        e_cap = int(rowptr[N].item())
        n_edges = e_cap
    else:
        n_edges = None
    Ec = max(int(e_cap), 1)
    col_src = buf("col_src", (Ec,), torch.int32)
    edge_dst = buf("edge_dst", (Ec,), torch.int32)
    edge_w = buf("edge_w", (Ec,), dtype)
    edge_dx = buf("edge_dx", (Ec, 3), dtype)
    call("gfm_radius_fill", ptr(pos), ptr(node_offsets), ptr(gnode), N, ptr(cells_t), float(rc),
         int(max_nbr or 0), ptr(rowptr), ptr(col_src), ptr(edge_dst), ptr(edge_w), ptr(edge_dx),
         code, s)
    csc_ptr = buf("csc_ptr", (N + 1,), torch.int32)
    csc_eid = buf("csc_eid", (Ec,), torch.int32)
    csc_dst = buf("csc_dst", (Ec,), torch.int32)
    ws = buf("csr_ws", (query("gfm_csr_workspace_bytes", N, Ec, B),), torch.uint8)
    call("gfm_csc_from_csr", ptr(rowptr), ptr(col_src), ptr(edge_dst), ptr(node_offsets), B, N,
         int(e_cap), ptr(csc_ptr), ptr(csc_eid), ptr(csc_dst), ptr(ws), s)
    return _radius_batch_result(o, dev, dtype, z, pos, node_offsets, gnode, host_offsets,
                                energy_true, forces_true, rowptr, col_src, edge_dst, edge_w,
                                edge_dx, csc_ptr, csc_eid, csc_dst, e_cap, n_edges,
                                _deg_bound(max_atoms, max_nbr), cells is not None)


def radius_batch_overflowed(out: dict, n_graphs: int) -> bool:
    """True when the last fused radius_batch into ``out`` found more edges
    than its e_cap (the batch was emitted edge-free; reads one int, syncs)"""
    ws = out.get("rb_ws")
    if ws is None:
        return False
    k = query("gfm_radius_batch_overflow_index", int(n_graphs))
    return bool(ws[4 * k:4 * k + 4].view(torch.int32).item())


# fused batch assembly limits (gfm_radius_batch: <= 256 atoms per graph; the
# uncapped neighbour lists must fit in shared memory)
_FUSED_MAX_ATOMS = 256
_FUSED_UNCAPPED_ATOMS = 96


def _deg_bound(max_atoms: int, max_nbr: int) -> int:
    """upper bound of any CSR row length of a radius batch"""
    full = max(max_atoms - 1, 0)
    return min(int(max_nbr), full) if max_nbr else full


def _radius_batch_result(o, dev, dtype, z, pos, node_offsets, gnode, host_offsets, energy_true,
                         forces_true, rowptr, col_src, edge_dst, edge_w, edge_dx, csc_ptr,
                         csc_eid, csc_dst, e_cap, n_edges, max_deg, periodic=False):
    B = int(host_offsets.shape[0] - 1)
    N = int(pos.shape[0])
    n_per = np.diff(host_offsets)
    npg = o.get("n_per_graph")
    if npg is None:
        npg = _i32(n_per, dev)
        o["n_per_graph"] = npg
    if energy_true is None:
        energy_true = torch.zeros(B, dtype=dtype, device=dev)
    if forces_true is None:
        forces_true = torch.zeros(N, 3, dtype=dtype, device=dev)
    return Batch(dtype=dtype, device=dev, z=z, pos=pos, node_offsets=node_offsets,
                 n_per_graph=npg, graph_of_node=gnode, energy_true=energy_true,
                 forces_true=forces_true, rowptr=rowptr, col_src=col_src, edge_dst=edge_dst,
                 edge_w=edge_w, edge_dx=edge_dx, csc_ptr=csc_ptr, csc_eid=csc_eid,
                 csc_dst=csc_dst, order=None, n_nodes=N, e_cap=int(e_cap), _n_edges=n_edges,
                 host_offsets=np.asarray(host_offsets), host_n_per=n_per, max_deg=max_deg,
                 counts=o.get("counts"), periodic=periodic)


# --------------------------------------------------------------------------
# Forward
# --------------------------------------------------------------------------


class _Scratch:
    """Reusable device buffers keyed by name (stable addresses let a whole
    step be captured into a CUDA graph)."""

    def __init__(self, device):
        self.device = device
        self.bufs = {}
        self.ones_ready = {}  # wgrad workspace -> (address, rows) its ones operand was written for

    def get(self, name, shape, dtype, zero: bool = False):
        shape = tuple(int(x) for x in shape)
        t = self.bufs.get(name)
        if t is None or t.dtype != dtype or tuple(t.shape) != shape:
            t = (torch.zeros if zero else torch.empty)(shape, dtype=dtype, device=self.device)
            self.bufs[name] = t
        return t

    def bytes(self, name, n, zero: bool = False):
        """``zero``: zero-filled when (re)allocated (workspaces whose
        counters the kernels keep at zero between calls)"""
        return self.get(name, (max(int(n), 1),), torch.uint8, zero)

    def side_stream(self):
        """second stream for work with no consumer until a later join (one
        per device and thread, shared by every scratch: API calls without a
        scratch object do not create a stream per call)"""
        if _ONE_STREAM:  # GFM_ONE_STREAM=1: everything on the caller's stream (A/B runs)
            return torch.cuda.current_stream(self.device)
        if getattr(self, "_side", None) is None:
            key = (str(self.device), threading.get_ident())
            st = _SIDE_STREAMS.get(key)
            if st is None:
                st = _SIDE_STREAMS[key] = torch.cuda.Stream(device=self.device)
            self._side = st
        return self._side


_SIDE_STREAMS: dict = {}
_ONE_STREAM = os.environ.get("GFM_ONE_STREAM") == "1"


def _scratch_for(owner, device):
    return owner if owner is not None else _Scratch(device)


# GFM_W_CSC=0: the backward gathers read w[eid] (A/B runs)
_W_CSC = os.environ.get("GFM_W_CSC", "1") != "0"


def _argmax_flag(batch) -> int:
    """uint8 argmax storage when every CSR row is known to hold <= 256 edges;
    local gathers when the batch is made of small graphs"""
    md = getattr(batch, "max_deg", None)
    f = _lib.FLAG_ARGMAX_U8 if md is not None and md <= 256 else 0
    n_per = getattr(batch, "host_n_per", None)
    if n_per is not None and len(n_per) and int(np.max(n_per)) <= _LOCAL_GRAPH_ATOMS:
        f |= _lib.FLAG_GATHER_LOCAL
    return f


# graphs up to this size count as local for the backward gathers (a graph's
# rows: <= 4096 x H floats, L2-resident while its edges are gathered)
_LOCAL_GRAPH_ATOMS = 4096


def forward_batch(params: ModelParams, batch: Batch, cache: dict | None = None,
                  scratch: _Scratch | None = None, flags: int = 0):
    """forward_batch (model.py:344-400): returns (e_pred (B,), f_pred (N, 3))
    as device tensors; fills ``cache`` with what the backward needs.  For an
    EGNNConfig, f_pred = -dE/dx0 (egnn.forces)."""
    cfg = params.config
    if _is_egnn(cfg):
        from . import egnn
        _, e_pred, f_pred = egnn.forces(params, batch, scratch)
        if scratch is None:
            return e_pred[:batch.n_graphs].clone(), f_pred[:batch.n_nodes].clone()
        return e_pred, f_pred
    dt = params.dtype
    if batch.dtype != dt:
        raise ValidationError(f"batch dtype {batch.dtype} != params dtype {dt}")
    code = _lib.dtype_code(dt)
    sc = _scratch_for(scratch, batch.device)
    s = stream_handle()
    N, H, B = batch.n_nodes, cfg.mpnn_width, batch.n_graphs
    parts, K = KIND_PARTS[cfg.mpnn_kind], cfg.n_parts
    G = cfg.fc_width
    h = sc.get("h0", (N, H), dt)
    call("gfm_embed", ptr(batch.z), N, ptr(params.embedding), H, ptr(h), code, s)
    layers = []
    am_flag = _argmax_flag(batch)
    for l in range(cfg.mpnn_layers):
        agg = sc.get(f"agg{l}", (N, K * H), dt)
        argmax = sc.get(f"argmax{l}", (N, H), torch.uint8 if am_flag & _lib.FLAG_ARGMAX_U8 else torch.int32) \
            if parts & _lib.PART_MAX else None
        smean = sc.get(f"smean{l}", (N, H), dt) if parts & _lib.PART_STD else None
        call("gfm_agg_fwd", ptr(h), N, H, ptr(batch.rowptr), ptr(batch.col_src),
             ptr(batch.edge_w), parts, ptr(agg), ptr(argmax), ptr(smean), code, flags | am_flag,
             s)
        h_out = sc.get(f"h{l + 1}", (N, H), dt)
        call("gfm_linear_fwd", ptr(h), H, H, ptr(agg), K * H, K * H,
             ptr(params.view(f"layer_{l}.w")), H, ptr(params.view(f"layer_{l}.u")), K * H,
             ptr(params.view(f"layer_{l}.b")), N, None, H, 1, ptr(h_out), H, code, s)
        layers.append(dict(h_in=h, agg=agg, argmax=argmax, smean=smean, h_out=h_out))
        h = h_out
    # the two heads only share h: the energy head runs on a side stream (a
    # parallel CUDA-graph branch) while the force head runs here
    main = torch.cuda.current_stream(batch.device)
    side = sc.side_stream()
    fork = torch.cuda.Event()
    fork.record(main)
    side.wait_event(fork)
    ss = side.cuda_stream
    ys = [h]
    y = h
    for f in range(cfg.fc_layers - 1):
        kin = y.shape[1]
        y2 = sc.get(f"y{f + 1}", (N, G), dt)
        call("gfm_linear_fwd", ptr(y), kin, kin, None, 0, 0, ptr(params.view(f"head_{f}.w")), kin,
             None, 0, ptr(params.view(f"head_{f}.b")), N, None, G, 1, ptr(y2), G, code, ss)
        ys.append(y2)
        y = y2
    node_e = sc.get("node_e", (max(N, 1),), dt)
    e_pred = sc.get("e_pred", (B,), dt)
    F = cfg.fc_layers
    call("gfm_energy_readout", ptr(y), N, G, ptr(params.view(f"head_{F - 1}.w")),
         ptr(params.view(f"head_{F - 1}.b")), ptr(batch.node_offsets), B, ptr(node_e),
         ptr(e_pred), code, ss)
    f_pred = sc.get("f_pred", (N, 3), dt)
    P = sc.get("force_P", (N, H), dt)  # h V^T, reused by the backward
    call("gfm_force_fwd", ptr(h), H, N, ptr(batch.rowptr), ptr(batch.col_src), ptr(batch.edge_dx),
         ptr(params.force_v), ptr(params.force_c), ptr(params.force_u), ptr(P), ptr(f_pred), code,
         flags, s)
    join = torch.cuda.Event()
    join.record(side)
    main.wait_event(join)
    if cache is not None:
        cache.update(layers=layers, h_final=h, head_inputs=ys, force_P=P)
    if scratch is None:
        return e_pred.clone(), f_pred.clone()
    return e_pred, f_pred


def predict(params: ModelParams, records):
    """Per-graph energies and per-graph force arrays (model.py:403-411)."""
    batch = make_batch(records, device=params.flat.device, dtype=params.dtype)
    e_pred, f_packed = forward_batch(params, batch)
    off = batch.host_offsets
    return e_pred, [f_packed[off[g]:off[g + 1]] for g in range(batch.n_graphs)]


def forward(params: ModelParams, records):
    """One record, a list of records, or a prepacked Batch (model.py:414-421)."""
    if isinstance(records, Batch):
        return forward_batch(params, records)
    if isinstance(records, GraphRecord) or hasattr(records, "atomic_numbers"):
        e_pred, forces = predict(params, [records])
        return float(e_pred[0]), forces[0]
    return predict(params, records)


# --------------------------------------------------------------------------
# Loss
# --------------------------------------------------------------------------


class LossBreakdown:
    """L1 MTL loss terms (model.py:429-434).  Values live on the device and
    are read (one sync) on first access."""

    def __init__(self, values: torch.Tensor, residuals_fn):
        self.values = values
        self._res_fn = residuals_fn
        self._host = None
        self._res = None

    def _h(self):
        if self._host is None:
            self._host = self.values.detach().to("cpu", torch.float64).numpy()
        return self._host

    @property
    def total(self) -> float:
        return float(self._h()[0])

    @property
    def energy_term(self) -> float:
        return float(self._h()[1])

    @property
    def force_term(self) -> float:
        return float(self._h()[2])

    @property
    def per_graph_residuals(self):
        if self._res is None:
            self._res = self._res_fn()
        return self._res


def _loss_kernel(e_pred, f_pred, e_true, f_true, n_per, alpha_e, alpha_f, scratch=None,
                 contrib=None, counts=None):
    dt = e_pred.dtype
    code = _lib.dtype_code(dt)
    sc = _scratch_for(scratch, e_pred.device)
    B, N = int(e_pred.shape[0]), int(f_pred.shape[0])
    vals = sc.get("loss", (3,), dt)
    de = sc.get("de", (max(B, 1),), dt)
    df = sc.get("df", (max(N, 1), 3), dt)
    ws = sc.bufs.get("loss_ws")
    if ws is None:  # zero once; the kernel re-arms its ticket after every call
        ws = torch.zeros(query("gfm_loss_workspace_bytes"), dtype=torch.uint8, device=e_pred.device)
        sc.bufs["loss_ws"] = ws
    call("gfm_loss_seeds", ptr(e_pred), ptr(e_true), ptr(n_per), B, ptr(f_pred), ptr(f_true), N,
         ptr(counts), float(alpha_e), float(alpha_f), ptr(vals), ptr(de), ptr(df), ptr(contrib),
         ptr(ws), code, stream_handle())
    return vals, de, df


def mtl_loss(e_pred, f_pred, e_true, f_true, n_per_graph, alpha_energy: float = 1.0,
             alpha_forces: float = 100.0) -> LossBreakdown:
    """L1 multitask loss (model.py:437-462) on the device."""
    dev = e_pred.device if isinstance(e_pred, torch.Tensor) else _device()
    dt = e_pred.dtype if isinstance(e_pred, torch.Tensor) and e_pred.is_floating_point() \
        else torch.float64
    ep = _to_dev(e_pred, dev, dt).reshape(-1)
    et = _to_dev(e_true, dev, dt).reshape(-1)
    npg = torch.as_tensor(np.asarray(n_per_graph.cpu() if isinstance(n_per_graph, torch.Tensor)
                                     else n_per_graph).reshape(-1).astype(np.int32), device=dev)
    fp = _to_dev(f_pred, dev, dt)
    ft = _to_dev(f_true, dev, dt)
    if ep.shape != et.shape or ep.shape[0] != npg.shape[0]:
        raise ValidationError(
            f"energy shapes differ: {tuple(ep.shape)} vs {tuple(et.shape)} vs {tuple(npg.shape)}")
    if fp.shape != ft.shape:
        raise ValidationError(f"force shapes differ: {tuple(fp.shape)} vs {tuple(ft.shape)}")
    vals, _, _ = _loss_kernel(ep, fp.reshape(-1, 3).contiguous(), et, ft.reshape(-1, 3).contiguous(),
                              npg, alpha_energy, alpha_forces)
    return LossBreakdown(vals.clone(), lambda: (ep - et) / npg.to(dt))


def batch_loss(params: ModelParams, batch: Batch) -> LossBreakdown:
    e_pred, f_pred = forward_batch(params, batch)
    c = params.config
    return mtl_loss(e_pred, f_pred, batch.energy_true, batch.forces_true, batch.n_per_graph,
                    c.alpha_energy, c.alpha_forces)


# --------------------------------------------------------------------------
# Backward
# --------------------------------------------------------------------------


def loss_and_grad(params: ModelParams, batch: Batch, precomputed=None,
                  scratch: _Scratch | None = None, grad_out: torch.Tensor | None = None,
                  contrib: torch.Tensor | None = None, flags: int = 0, grad_ready=None):
    """Loss plus exact analytic gradient as a flat vector (model.py:483-565).

    ``grad_out`` (length P, params dtype) receives the gradient in place;
    ``contrib`` (float32) receives [loss.total, 1.0] for the DP allreduce.
    ``grad_ready(group, stream)``, when given, is called as soon as a group of
    gradient entries is final on ``stream`` -- "loss", "head", "force",
    "layer{L-1}" ... "layer0", "embedding", in that order of production -- so
    the trainer can allreduce finished buckets while the backward runs."""
    cfg = params.config
    if _is_egnn(cfg):
        from . import egnn
        return egnn.loss_and_grad(params, batch, scratch=scratch, grad_out=grad_out,
                                  contrib=contrib)
    dt = params.dtype
    code = _lib.dtype_code(dt)
    sc = _scratch_for(scratch, batch.device)
    if precomputed is None:
        cache: dict = {}
        e_pred, f_pred = forward_batch(params, batch, cache, scratch=sc, flags=flags)
    else:
        cache, e_pred, f_pred = precomputed
    s = stream_handle()
    N, H, B, G = batch.n_nodes, cfg.mpnn_width, batch.n_graphs, cfg.fc_width
    parts, K = KIND_PARTS[cfg.mpnn_kind], cfg.n_parts
    F = cfg.fc_layers
    vals, de, df = _loss_kernel(e_pred, f_pred, batch.energy_true, batch.forces_true,
                                batch.n_per_graph, cfg.alpha_energy, cfg.alpha_forces,
                                scratch=sc, contrib=contrib, counts=batch.counts)
    main_s = torch.cuda.current_stream(batch.device)
    if grad_ready is not None:
        grad_ready("loss", main_s)
    grad = grad_out if grad_out is not None else torch.zeros(params.layout.Pp, dtype=dt,
                                                             device=batch.device)
    gp = ModelParams(cfg, grad)

    # weight gradients: split-K partials on a side stream (nothing downstream
    # consumes them until the end), so each tensor-core GEMM overlaps the
    # L2-bound gathers of the main stream; all reductions in one batched
    # launch after the last layer (each call keeps its own workspace and its
    # inputs stay untouched: per-layer dz buffers)
    jobs = []
    main = torch.cuda.current_stream(batch.device)
    side = sc.side_stream()

    def flush_jobs():
        """reduce the weight-gradient partials issued so far (side stream)"""
        if jobs:
            arr = (_lib.ReduceJob * len(jobs))(*jobs)
            call("gfm_splitk_reduce_batch", arr, len(jobs), code, side.cuda_stream)
            jobs.clear()

    def wgrad(dY, ldd, n_out, X1, ld1, K1, X2, ld2, K2, g1, g2, gb, tag, inputs_on_side=False):
        nb = query("gfm_linear_bwd_weight_workspace_bytes", N, n_out, K1, K2, 1, code)
        key = f"wgrad_ws_{tag}"
        ws = sc.bytes(key, nb)
        # the workspace's ones operand survives between calls: fill it once
        bias = 2 if sc.ones_ready.get(key) == (ws.data_ptr(), N) else 1
        job = _lib.ReduceJob()
        if not inputs_on_side:  # inputs produced on the main stream
            ready = torch.cuda.Event()
            ready.record(main)
            side.wait_event(ready)
        call("gfm_linear_bwd_weight_partials", ptr(dY), ldd, N, None, n_out, ptr(X1), ld1, K1,
             ptr(X2), ld2, K2, bias, ptr(g1), ptr(g2), ptr(gb), ptr(ws), ctypes.byref(job),
             code, side.cuda_stream)
        jobs.append(job)
        sc.ones_ready[key] = (ws.data_ptr(), N)

    # energy head (model.py:520-533) on the side stream, concurrent with the
    # force head's edge passes on this one; they meet at dh_energy
    fork = torch.cuda.Event()
    fork.record(main)
    side.wait_event(fork)
    ss = side.cuda_stream
    ys = cache["head_inputs"]
    # ds as an [N][4] column (cols 1..3 zero) so its rows are 16B aligned and
    # the weight-gradient GEMM below can stream it with TMA
    ds = sc.get("ds", (max(N, 1), 4), dt)
    dz = sc.get("dz_head", (N, G), dt)
    call("gfm_energy_seed", ptr(de), ptr(batch.graph_of_node), N, G,
         ptr(params.view(f"head_{F - 1}.w")), ptr(ys[F - 1]), ptr(ds), 4, ptr(dz), code, ss)
    wgrad(ds, 4, 1, ys[F - 1], G, G, None, 0, 0, gp.view(f"head_{F - 1}.w"), None,
          gp.view(f"head_{F - 1}.b"), f"head{F - 1}", inputs_on_side=True)
    dh_e = sc.get("dh_energy", (N, H), dt)
    for f in range(F - 2, -1, -1):
        kin = ys[f].shape[1]
        wgrad(dz, G, G, ys[f], kin, kin, None, 0, 0, gp.view(f"head_{f}.w"), None,
              gp.view(f"head_{f}.b"), f"head{f}", inputs_on_side=True)
        if f > 0:
            dz2 = sc.get(f"dz_head{f}", (N, kin), dt)
            call("gfm_linear_bwd_data", ptr(dz), G, N, None, G, ptr(params.view(f"head_{f}.w")),
                 kin, kin, None, 0, 0, ptr(dz2), kin, None, 0, ptr(ys[f]), kin, code, ss)
            dz = dz2
        else:
            call("gfm_linear_bwd_data", ptr(dz), G, N, None, G, ptr(params.view(f"head_{f}.w")),
                 kin, kin, None, 0, 0, ptr(dh_e), H, None, 0, None, 0, code, ss)
    if grad_ready is not None:  # bucketed allreduce: reduce the head's partials now
        flush_jobs()
        grad_ready("head", side)
    head_done = torch.cuda.Event()
    head_done.record(side)

    # force head (model.py:535-547) -> dz of the last message-passing layer
    dzl = sc.get("dz_layer", (N, H), dt)
    ws = sc.bytes("force_bwd_ws", query("gfm_force_bwd_workspace_bytes", H, N, code))
    call("gfm_force_bwd_edges", ptr(cache["h_final"]), ptr(cache["force_P"]), H, N,
         ptr(batch.rowptr), ptr(batch.col_src), ptr(batch.edge_dx), ptr(batch.csc_ptr),
         ptr(batch.csc_eid), ptr(batch.csc_dst), ptr(params.force_v), ptr(params.force_c),
         ptr(params.force_u), ptr(df), None, None, None, ptr(ws), code, flags, s)
    # grad_V = S^T h, grad_c, grad_u: off the critical path on the side stream
    edges_done = torch.cuda.Event()
    edges_done.record(main)
    side.wait_event(edges_done)
    call("gfm_force_bwd_grads", ptr(cache["h_final"]), H, N, ptr(gp.force_v), ptr(gp.force_c),
         ptr(gp.force_u), ptr(ws), code, ss)
    if grad_ready is not None:
        grad_ready("force", side)
    main.wait_event(head_done)
    call("gfm_force_bwd_finish", ptr(cache["h_final"]), H, N, ptr(params.force_v), ptr(dh_e),
         ptr(dzl), ptr(ws), code, s)

    # message-passing layers (model.py:549-562)
    dz = dzl
    agg_ws = sc.bytes("agg_bwd_ws", query("gfm_agg_bwd_workspace_bytes", N, H, parts, code))
    # PNA on the float32 tensor-core engine: backward-data GEMM + agg prep
    # fused into its epilogue for wide layers (H >= 256: with the CTA-pair
    # GEMM the C3 step is 1% faster; at C2 (H 64) the separate float4 prep
    # pass is 1.5% faster).  GFM_FUSED_PREP=1 / 0 forces it on / off.
    fp_env = os.environ.get("GFM_FUSED_PREP")
    fused_prep = ((fp_env == "1" or (fp_env is None and H >= 256)) and dt == torch.float32
                  and parts == 15 and H % 4 == 0 and N > 0
                  and query("gfm_get_gemm_mode") != 0 and not flags & _lib.FLAG_SCALAR)
    up_ws = sc.bytes("up_ws", query("gfm_layer_bwd_data_agg_workspace_bytes", H)) \
        if fused_prep else None
    # edge weights in CSC order once per step: the gathers then read w[q]
    # with their CSC slot instead of a dependent random w[eid]
    w_agg, w_flag = batch.edge_w, 0
    if _W_CSC and batch.edge_w.shape[0] > 0:
        w_agg = sc.get("w_csc", tuple(batch.edge_w.shape), dt)
        call("gfm_permute", ptr(batch.csc_eid), int(batch.edge_w.shape[0]),
             ptr(batch.rowptr) + 4 * N, ptr(batch.edge_w), ptr(w_agg), code, s)
        w_flag = _lib.FLAG_W_CSC
    for l in range(cfg.mpnn_layers - 1, -1, -1):
        lay = cache["layers"][l]
        wgrad(dz, H, H, lay["h_in"], H, H, lay["agg"], K * H, K * H, gp.view(f"layer_{l}.w"),
              gp.view(f"layer_{l}.u"), gp.view(f"layer_{l}.b"), f"layer{l}")
        if grad_ready is not None:
            flush_jobs()
            grad_ready(f"layer{l}", side)
        dh_in = sc.get("dh_in", (N, H), dt)
        out = sc.get(f"dz_l{l}", (N, H), dt)
        if fused_prep:
            # dh_in = dz W and the gather's inputs (G | coef in agg_ws, dmax)
            # straight from the GEMM epilogue: no [N][4H] dagg, no prep pass
            dmax = sc.get("dmax", (N, H), dt)
            call("gfm_layer_bwd_data_agg", ptr(dz), N, H, ptr(params.view(f"layer_{l}.w")),
                 ptr(params.view(f"layer_{l}.u")), ptr(lay["agg"]), ptr(lay["smean"]),
                 ptr(batch.rowptr), ptr(dh_in), agg_ws.data_ptr(),
                 agg_ws.data_ptr() + 4 * N * H, ptr(dmax), ptr(up_ws), s)
            call("gfm_agg_bwd", ptr(dmax), ptr(lay["agg"]), ptr(lay["smean"]), ptr(lay["argmax"]),
                 ptr(lay["h_in"]), ptr(batch.rowptr), ptr(batch.csc_ptr), ptr(batch.csc_eid),
                 ptr(batch.csc_dst), ptr(w_agg), N, H, parts, ptr(dh_in),
                 ptr(lay["h_in"]) if l > 0 else None, ptr(out), ptr(agg_ws), code,
                 flags | _argmax_flag(batch) | _lib.FLAG_AGG_PREPPED | w_flag, s)
        else:
            dagg = sc.get("dagg", (N, K * H), dt)
            call("gfm_linear_bwd_data", ptr(dz), H, N, None, H, ptr(params.view(f"layer_{l}.w")),
                 H, H, ptr(params.view(f"layer_{l}.u")), K * H, K * H, ptr(dh_in), H, ptr(dagg),
                 K * H, None, 0, code, s)
            call("gfm_agg_bwd", ptr(dagg), ptr(lay["agg"]), ptr(lay["smean"]), ptr(lay["argmax"]),
                 ptr(lay["h_in"]), ptr(batch.rowptr), ptr(batch.csc_ptr), ptr(batch.csc_eid),
                 ptr(batch.csc_dst), ptr(w_agg), N, H, parts, ptr(dh_in),
                 ptr(lay["h_in"]) if l > 0 else None, ptr(out), ptr(agg_ws), code,
                 flags | _argmax_flag(batch) | w_flag, s)
        dz = out
    # the batched reduction follows the weight-gradient GEMMs on the side
    # stream while the embedding gradient runs here; join before returning
    flush_jobs()
    ews = sc.bytes("emb_ws", query("gfm_embedding_grad_workspace_bytes", N, H, code))
    call("gfm_embedding_grad", ptr(batch.z), N, ptr(dz), H, ptr(gp.embedding), ptr(ews), code, s)
    if grad_ready is not None:
        grad_ready("embedding", main_s)
    done = torch.cuda.Event()
    done.record(side)
    main.wait_event(done)

    e_true, n_per = batch.energy_true, batch.n_per_graph
    lb = LossBreakdown(vals if scratch is not None else vals.clone(),
                       lambda: (e_pred - e_true) / n_per.to(e_pred.dtype))
    # API callers get the reference-order flat gradient; grad_out callers
    # (the trainer) keep the padded device layout
    return lb, (grad if grad_out is not None else params.layout.compact(grad))


def backward(params: ModelParams, batch_or_records):
    """Exact gradient of the multitask loss w.r.t. the flat parameters."""
    batch = batch_or_records if isinstance(batch_or_records, Batch) else make_batch(
        batch_or_records, device=params.flat.device, dtype=params.dtype)
    _, grad = loss_and_grad(params, batch)
    return grad
