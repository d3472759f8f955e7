"""Data-parallel MTL training step and loop (drop-in for ``gfmkit.train``).

Reference: train.py:59-338.  One process per GPU; each step a rank runs
forward + backward on its own batch into a float32 ``[grad | loss | 1]``
vector, the vector is summed across ranks by the ``Comm`` (NCCL over
NVLink), a device-side non-finite guard is raised if any entry is bad, and
the Adam / SGD kernel divides by the world size and updates float64 master
weights plus the float32 working copy -- identical bytes on every rank, so
parameters stay bitwise equal across ranks (train.py:1-10).

The guard is sticky on the device: once set, every later update is skipped,
which is exactly the reference's "update discarded, training aborted"
(train.py:264-274) without a host round trip per step.
"""

from __future__ import annotations

import contextlib
import json
import os
import logging
import struct
import time
import zlib
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_handle
from .comm import Comm, LocalComm
from .errors import ConfigError, CorruptionError, FormatError, UnsupportedVersionError, ValidationError
from .model import (ModelConfig, ModelParams, _Scratch, count_params, forward_batch, param_layout,
                    init_params_flat, loss_and_grad, make_batch)
from .records import MAX_Z
from .schedule import epoch_schedule
from .telemetry import DeviceClock, PhaseClock

log = logging.getLogger(__name__)

OPTIMIZERS = ("adam", "sgd")
BC_TABLE_LEN = 1 << 20  # steps with host-exact Adam bias corrections (16 MB)


@dataclass
class TrainConfig:
    """train.py:59-82."""

    max_epochs: int = 30
    patience: int = 10
    base_seed: int = 0
    optimizer: str = "adam"
    learning_rate: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    wall_clock_budget_s: float | None = None
    checkpoint_path: str | None = None

    def __post_init__(self):
        if self.optimizer not in OPTIMIZERS:
            raise ConfigError(f"optimizer must be one of {OPTIMIZERS}, got {self.optimizer!r}")
        if self.max_epochs < 0:
            raise ConfigError(f"max_epochs must be >= 0, got {self.max_epochs}")
        if self.patience < 1:
            raise ConfigError(f"patience must be >= 1, got {self.patience}")
        if self.learning_rate <= 0:
            raise ConfigError(f"learning_rate must be > 0, got {self.learning_rate}")


class OptimizerState:
    """Adam moments (float64, on the device) and step counter (train.py:85-93)."""

    def __init__(self, m, v, t: int = 0):
        self.m = m
        self.v = v
        self.t = t

    @classmethod
    def zeros(cls, n: int, device=None) -> "OptimizerState":
        dev = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        return cls(torch.zeros(n, dtype=torch.float64, device=dev),
                   torch.zeros(n, dtype=torch.float64, device=dev), 0)


def _dev_f64(x, device):
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=device, dtype=torch.float64).contiguous()
    return torch.as_tensor(np.asarray(x, dtype=np.float64), device=device)


def apply_update(flat, grad, cfg: TrainConfig, state: OptimizerState):
    """One optimiser step (train.py:96-108) on the device; returns a NEW
    float64 vector (numpy in -> numpy out) and mutates ``state``.  Bit-identical
    to the reference for identical float64 inputs."""
    _lib.load(require_device=True)
    dev = state.m.device if isinstance(state.m, torch.Tensor) else torch.device("cuda")
    if not isinstance(state.m, torch.Tensor):
        state.m = _dev_f64(state.m, dev)
        state.v = _dev_f64(state.v, dev)
    as_numpy = not isinstance(flat, torch.Tensor)
    master = _dev_f64(flat, dev).clone()
    g = grad.detach() if isinstance(grad, torch.Tensor) else torch.as_tensor(
        np.asarray(grad, np.float64))
    g = g.to(dev).contiguous()
    if g.dtype not in (torch.float32, torch.float64):
        g = g.to(torch.float64)
    n = master.shape[0]
    if g.shape[0] != n:
        raise ValidationError(f"grad has {g.shape[0]} entries, params {n}")
    state.t += 1
    s = stream_handle()
    code = _lib.dtype_code(g.dtype)
    if cfg.optimizer == "sgd":
        call("gfm_sgd_step", ptr(g), code, n, 1.0, ptr(master), float(cfg.learning_rate), None,
             None, s)
    else:
        bc = torch.tensor([1.0 - cfg.beta1 ** state.t, 1.0 - cfg.beta2 ** state.t],
                          dtype=torch.float64, device=dev)
        call("gfm_adam_step", ptr(g), code, n, 1.0, ptr(master), ptr(state.m), ptr(state.v),
             ptr(bc), float(cfg.learning_rate), float(cfg.beta1), float(cfg.beta2),
             float(cfg.eps), None, None, s)
    return master.cpu().numpy() if as_numpy else master


class EarlyStopper:
    """Stop when the metric has not decreased for ``patience`` epochs (train.py:111-126)."""

    def __init__(self, patience: int):
        self.patience = patience
        self.best = np.inf
        self.since_improvement = 0

    def update(self, value: float) -> bool:
        if value < self.best:
            self.best = value
            self.since_improvement = 0
        else:
            self.since_improvement += 1
        return self.since_improvement >= self.patience


@dataclass
class EpochMetrics:
    epoch: int
    train_loss: float
    val_mae: float
    val_energy_mae: float
    val_force_mae: float
    epoch_time_s: float
    phase_seconds: dict = field(default_factory=dict)
    device_phase_seconds: dict = field(default_factory=dict)  # DeviceClock (CUDA events)

    def to_dict(self) -> dict:
        return dict(epoch=self.epoch, train_loss=self.train_loss, val_mae=self.val_mae,
                    val_energy_mae=self.val_energy_mae, val_force_mae=self.val_force_mae,
                    epoch_time_s=self.epoch_time_s, phase_seconds=dict(self.phase_seconds),
                    device_phase_seconds=dict(self.device_phase_seconds))


@dataclass
class TrainResult:
    params: ModelParams
    metrics: list
    stop_reason: str
    nan_event: bool
    epochs_run: int


class DataParallelTrainer:
    """The hot path: device-resident parameters, optimiser state and
    scratch; ``step(batch)`` = forward + backward + allreduce + guard + update
    with no host synchronisation.  Float32 compute by default (float64 for
    exact-parity runs)."""

    def __init__(self, model_config: ModelConfig, train_config: TrainConfig | None = None,
                 comm: Comm | None = None, device=None, initial=None,
                 dtype=torch.float32, flags: int = 0, bucket_bytes: int = 64 << 20):
        _lib.load(require_device=True)
        self.cfg = model_config
        self.tcfg = train_config or TrainConfig()
        self.comm = comm or LocalComm()
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        self.dtype = dtype
        self.flags = flags
        # device buffers use the padded parameter layout (16-byte aligned
        # arrays); P is the padded length, the allreduce payload is
        # [grad (P) | loss | 1]
        self.layout = param_layout(model_config)
        P = self.layout.Pp
        self.P = P
        if initial is None:
            flat = init_params_flat(model_config, self.tcfg.base_seed)
        elif isinstance(initial, ModelParams):
            flat = initial.flatten()
        else:
            flat = np.asarray(initial, np.float64)
        self.master = self.layout.pad(flat, self.device, torch.float64)
        self.m = torch.zeros_like(self.master)
        self.v = torch.zeros_like(self.master)
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.bc = torch.zeros(2, dtype=torch.float64, device=self.device)
        # host-computed bias corrections 1 - beta ** t (train.py:104-105, the
        # reference's libm pow), looked up by the device step counter; filled
        # ahead of the host's step count in chunks (fixed address: captured
        # steps keep reading the same table)
        self.bc_table = torch.zeros(2 * BC_TABLE_LEN, dtype=torch.float64, device=self.device)
        self._bc_filled = 0
        self._ensure_bc(1024)
        self.flag = torch.zeros(2, dtype=torch.int32, device=self.device)  # [non-finite, ticket]
        self.contrib = torch.zeros(P + 2, dtype=dtype, device=self.device)
        if dtype == torch.float32:
            self.work = torch.empty(P, dtype=torch.float32, device=self.device)
            call("gfm_cast_f64_to_f32", ptr(self.master), P, ptr(self.work), stream_handle())
        else:
            self.work = self.master
        self.params = ModelParams(model_config, self.work)
        self.scratch = _Scratch(self.device)
        self.steps = 0
        # bucketed, backward-overlapped gradient allreduce (N > 1, MPNN): each
        # bucket is summed on a comm stream as soon as its gradients are final.
        # Default 64 MB buckets, i.e. one allreduce for every benched config:
        # at C3 on 4 B200 (34 MB payload) 4 MB buckets measured 22.2 ms/step,
        # 16 MB 21.8, one allreduce 21.45 (profiles/r02_bucket_ab.txt) -- NCCL
        # kernels overlapping the persistent (one CTA per SM) GEMMs cost the
        # GEMMs more than the overlap hides
        if os.environ.get("GFM_BUCKET_MB"):  # A/B knob: bucket size in MB (0 = one bucket)
            mb = float(os.environ["GFM_BUCKET_MB"])
            bucket_bytes = int(mb * (1 << 20)) if mb > 0 else 1 << 62
        self.buckets = plan_buckets(self.layout, model_config, bucket_bytes,
                                    self.contrib.element_size())
        self.bucketed = (self.comm.size > 1 and len(self.buckets) > 1
                         and getattr(model_config, "model_type", "mpnn") == "mpnn"
                         and hasattr(self.comm, "allreduce_sum_"))
        self._comm_stream = torch.cuda.Stream(device=self.device) if self.bucketed else None
        self._reduced = False

    def _ensure_bc(self, steps_ahead: int):
        """make the bias-correction table cover step counts < steps_ahead"""
        want = min(int(steps_ahead), BC_TABLE_LEN)
        if want <= self._bc_filled or self.tcfg.optimizer != "adam":
            return
        hi = min(BC_TABLE_LEN, max(want, 2 * self._bc_filled, 1024))
        b1, b2 = self.tcfg.beta1, self.tcfg.beta2
        vals = [x for t in range(self._bc_filled, hi)
                for x in ((1.0 - b1 ** t, 1.0 - b2 ** t) if t else (0.0, 0.0))]
        self.bc_table[2 * self._bc_filled:2 * hi].copy_(
            torch.tensor(vals, dtype=torch.float64))
        self._bc_filled = hi

    def compute(self, batch, scratch=None, precomputed=None):
        """forward + backward into ``contrib`` (or zeros when no batch).
        ``scratch``: activation buffers to use (default: the trainer's own;
        a runner keeps one per captured shape); ``precomputed``: a forward
        already run into that scratch (cache, e_pred, f_pred)."""
        P = self.P
        self._reduced = False
        if batch is None:
            self.contrib.zero_()
            return
        sc = scratch if scratch is not None else self.scratch
        if self.dtype == torch.float32:
            hook = self._bucket_hook() if self.bucketed else None
            loss_and_grad(self.params, batch, precomputed=precomputed, scratch=sc,
                          grad_out=self.contrib[:P], contrib=self.contrib[P:], flags=self.flags,
                          grad_ready=hook)
            if hook is not None:
                self._join_buckets()
        else:
            lb, _ = loss_and_grad(self.params, batch, precomputed=precomputed, scratch=sc,
                                  grad_out=self.contrib[:P], flags=self.flags)
            self.contrib[P:P + 1].copy_(lb.values[:1])
            self.contrib[P + 1].fill_(1.0)

    def _bucket_hook(self):
        """grad_ready callback: launch each bucket's allreduce on the comm
        stream once all its groups are final (same order on every rank)"""
        waiting = [set(b.groups) for b in self.buckets]
        events = [[] for _ in self.buckets]
        cs = self._comm_stream

        def ready(group, stream):
            ev = torch.cuda.Event()
            ev.record(stream)
            for k, b in enumerate(self.buckets):
                if group in waiting[k]:
                    waiting[k].discard(group)
                    events[k].append(ev)
                    if not waiting[k]:
                        for e in events[k]:
                            cs.wait_event(e)
                        with torch.cuda.stream(cs):
                            self.comm.allreduce_sum_(self.contrib[b.lo:b.hi])
        self._reduced = True
        return ready

    def _join_buckets(self):
        torch.cuda.current_stream(self.device).wait_stream(self._comm_stream)

    def reduce_and_update(self):
        P = self.P
        s = stream_handle()
        if self.bucketed and not self._reduced:
            # an idle rank (or a caller that bypassed compute) runs the same
            # bucket sequence so the collectives line up across ranks
            cs = self._comm_stream
            cs.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(cs):
                for b in sorted(self.buckets, key=lambda b: b.order):
                    self.comm.allreduce_sum_(self.contrib[b.lo:b.hi])
            self._join_buckets()
        elif not self.bucketed:
            _allreduce(self.comm, self.contrib)
        self._reduced = False
        code = _lib.dtype_code(self.dtype)
        adam = self.tcfg.optimizer == "adam"
        capturing = torch.cuda.is_current_stream_capturing()
        if not capturing:  # a captured replay's caller advances the count
            self._ensure_bc(self.steps + 2)
        # train.py:262-274 guard, fused with the device's applied-step counter
        # (and Adam's bias corrections)
        call("gfm_nonfinite_advance", ptr(self.contrib), P + 1, code, ptr(self.flag),
             ptr(self.t_dev), float(self.tcfg.beta1), float(self.tcfg.beta2),
             ptr(self.bc) if adam else None, ptr(self.bc_table), self._bc_filled, s)
        out32 = self.work if self.dtype == torch.float32 else None
        world = float(self.comm.size)
        if adam:
            call("gfm_adam_step", ptr(self.contrib), code, P, world, ptr(self.master), ptr(self.m),
                 ptr(self.v), ptr(self.bc), float(self.tcfg.learning_rate),
                 float(self.tcfg.beta1), float(self.tcfg.beta2), float(self.tcfg.eps),
                 ptr(self.flag), ptr(out32), s)
        else:
            call("gfm_sgd_step", ptr(self.contrib), code, P, world, ptr(self.master),
                 float(self.tcfg.learning_rate), ptr(self.flag), ptr(out32), s)
        if not capturing:
            self.steps += 1

    def step(self, batch, scratch=None):
        self.compute(batch, scratch)
        self.reduce_and_update()
        return self.contrib[self.P:self.P + 2]

    def state_tensors(self):
        """every device tensor a step mutates (for snapshot / restore)"""
        ts = [self.master, self.m, self.v, self.t_dev, self.bc, self.flag, self.contrib]
        if self.work is not self.master:
            ts.append(self.work)
        return ts

    @contextlib.contextmanager
    def preserved(self):
        """run steps (e.g. capture warm-ups) without changing the training
        state: parameters, moments, counters and flags are restored after"""
        saved = [t.clone() for t in self.state_tensors()]
        steps = self.steps
        try:
            yield self
        finally:
            for t, c in zip(self.state_tensors(), saved):
                t.copy_(c)
            self.steps = steps

    @property
    def nan_event(self) -> bool:
        return bool(self.flag[0].item())

    def current_params(self) -> ModelParams:
        return ModelParams(self.cfg, self.master.clone())

    def optimizer_state(self) -> "OptimizerState":
        """Adam moments in the reference's flat order plus the applied-step
        count ``t`` (train.py:100: every applied update, SGD included; a
        discarded non-finite step does not count)."""
        lay = self.layout
        t = int(self.t_dev.item())  # applied updates only (device counter)
        return OptimizerState(lay.compact(self.m).cpu().numpy(), lay.compact(self.v).cpu().numpy(),
                              t)

    def flat_master(self) -> np.ndarray:
        """float64 master parameters in the reference's flat order"""
        return self.layout.compact(self.master).cpu().numpy()

    def flat_grad(self) -> np.ndarray:
        """last step's (summed) gradient in the reference's flat order"""
        return self.layout.compact(self.contrib[:self.P]).to(torch.float64).cpu().numpy()


@dataclass
class Bucket:
    """a contiguous slice [lo, hi) of the [grad | loss | 1] payload and the
    gradient groups whose completion it waits for; ``order`` = its launch
    position (buckets complete in the backward's production order)"""
    lo: int
    hi: int
    groups: tuple
    order: int


def plan_buckets(layout, config, bucket_bytes: int, elem_bytes: int = 4):
    """Gradient buckets in reverse layer order: the payload
    [embedding | layer_0 .. layer_{L-1} | head | force | loss, 1] is cut, from
    the end, into contiguous buckets of >= bucket_bytes made of whole groups,
    so each bucket's allreduce can start when the backward has finished its
    groups ("loss"/"head"/"force" first, "embedding" last)."""
    ent = {name: (off, size) for name, _, off, size in layout.entries}
    if getattr(config, "model_type", "mpnn") != "mpnn":
        return [Bucket(0, layout.Pp + 2, ("all",), 0)]
    L = config.mpnn_layers
    names = [n for n, _, _, _ in layout.entries]
    groups = [("embedding", ["embedding"])]
    groups += [(f"layer{l}", [n for n in names if n.startswith(f"layer_{l}.")]) for l in range(L)]
    groups += [("head", [n for n in names if n.startswith("head_")]),
               ("force", [n for n in names if n.startswith("force.")])]
    starts = [ent[g[1][0]][0] for g in groups] + [layout.Pp]
    spans = [(g[0], starts[k], starts[k + 1]) for k, g in enumerate(groups)]
    spans.append(("loss", layout.Pp, layout.Pp + 2))
    # production order of the groups in loss_and_grad
    produced = ["loss", "head", "force"] + [f"layer{l}" for l in range(L - 1, -1, -1)] +         ["embedding"]
    buckets, cur = [], []
    for name, lo, hi in reversed(spans):  # from the end of the payload
        cur.append((name, lo, hi))
        if sum(h - l for _, l, h in cur) * elem_bytes >= bucket_bytes:
            buckets.append(cur)
            cur = []
    if cur:
        if buckets and sum(h - l for _, l, h in cur) * elem_bytes < bucket_bytes // 4:
            buckets[-1].extend(cur)  # a small remainder joins the last bucket
        else:
            buckets.append(cur)
    out = []
    for grp in buckets:
        gs = tuple(n for n, _, _ in grp)
        done = max(produced.index(n) for n in gs)
        out.append(Bucket(min(l for _, l, _ in grp), max(h for _, _, h in grp), gs, done))
    order = sorted(range(len(out)), key=lambda k: out[k].order)
    for pos, k in enumerate(order):
        out[k].order = pos
    return out


@contextlib.contextmanager
def _dphase(dclk, name):
    if dclk is None:
        yield
    else:
        with dclk.phase(name):
            yield


def _allreduce(comm, contrib: torch.Tensor):
    """In-place sum of the step payload across ranks.  Comm objects of this
    package reduce the device tensor directly (NCCL); any other object with
    the reference's Comm contract (comm.py:55-77, e.g. gfmkit's StarComm)
    goes through the host: float64 allreduce_sum of the payload, copied back."""
    fn = getattr(comm, "allreduce_sum_", None)
    if fn is not None:
        fn(contrib)
        return
    if getattr(comm, "size", 1) == 1:
        return
    out = comm.allreduce_sum(contrib.detach().to("cpu", torch.float64).numpy())
    contrib.copy_(torch.as_tensor(np.asarray(out), dtype=contrib.dtype))


class _Shape:
    """One captured step shape of a runner: node capacity N, edge capacity,
    its own activation scratch and batch buffers (so graphs captured for
    different shapes never share a reallocated buffer) and its CUDA graphs."""

    def __init__(self, n_nodes: int, e_cap: int, device):
        self.N = int(n_nodes)
        self.e_cap = int(e_cap)
        self.bufs: dict = {}
        self.scratch = _Scratch(device)
        self.graph = None
        self.stage_graphs = None
        self.batch = None


class StructureStepRunner:
    """Training step on raw structures: device batch assembly (radius graph
    -> CSR/CSC) + forward + backward + allreduce + update, captured into a
    CUDA graph and replayed.

    Fixed layout: ``host_offsets`` gives the per-graph atom counts of every
    batch.  Ragged layout (``host_offsets=None``, ``max_graphs``,
    ``max_atoms``): each batch has its own sizes (up to ``max_graphs``
    structures of up to ``max_atoms`` atoms, as generate_synthetic's
    ``n_atoms_range`` produces, preprocess.py:107-153; model.py:234-285
    batches any sizes).  The step is captured once per node capacity in
    ``node_caps`` (default: one, ``max_graphs * max_atoms``); a batch runs in
    the smallest capacity holding it, its true graph / node counts read from
    the device ([B, N] ``counts``), the tail nodes edge-free and seedless.

    ``load(...)`` copies a batch's raw inputs (host pinned or device tensors)
    into stable device slots; ``run()`` executes one step; ``step(...)`` =
    load + run + loss read-back (the end-to-end public call)."""

    def __init__(self, trainer: DataParallelTrainer, host_offsets=None, rc: float = 5.0,
                 max_nbr: int = 0, cells=None, use_graph: bool = True, e_cap: int | None = None,
                 *, max_graphs: int | None = None, max_atoms: int | None = None,
                 node_caps=None, store=None, group: str = "trainset"):
        self.tr = trainer
        dev = trainer.device
        self.rc = float(rc)
        self.max_nbr = int(max_nbr or 0)
        # store mode: batches are gathered from a DeviceStructureStore's
        # per-structure CSR blocks (the records' own edges) inside the graph
        self.store = store
        self.group = group
        if store is not None:
            g = store.group(group)
            if g.csr is None:
                raise ValidationError(f"store group {group!r} holds no edges (ingest records)")
            host_offsets = None
            max_atoms = max_atoms or g.max_atoms
            if e_cap is None:
                e_cap = int(max_graphs) * max(g.max_edges, 1)
        self.ragged = host_offsets is None
        if self.ragged:
            if not max_graphs or not max_atoms:
                raise ValidationError("a ragged runner needs max_graphs and max_atoms")
            self.B = int(max_graphs)
            self.max_atoms = int(max_atoms)
            caps = sorted({int(c) for c in (node_caps or [self.B * self.max_atoms])})
            if caps[-1] > self.B * self.max_atoms or caps[0] < 1:
                raise ValidationError("node capacities must lie in [1, max_graphs * max_atoms]")
            # the graph-capacity layout handed to radius_batch: B graphs
            self.host_off = np.zeros(self.B + 1, np.int32)
        else:
            self.host_off = np.asarray(host_offsets, np.int32)
            self.B = int(self.host_off.shape[0] - 1)
            n = np.diff(self.host_off)
            self.max_atoms = int(n.max()) if n.size else 0
            caps = [int(self.host_off[-1])]
        self.N = caps[-1]
        # per-step layout words: [counts (2) | node offsets (B+1) | n_per (B) |
        # edge offsets (B+1), store mode]
        self.meta = torch.zeros(3 * self.B + 4, dtype=torch.int32, device=dev)
        self.counts = self.meta[0:2] if self.ragged else None
        self.off = self.meta[2:self.B + 3]
        self.npg = self.meta[self.B + 3:2 * self.B + 3]
        self.idx = torch.zeros(self.B, dtype=torch.int32, device=dev)
        if not self.ragged:
            self._write_meta(self.host_off, sync=True)
        self._meta_ring = [[torch.empty(self.meta.shape[0] + self.B, dtype=torch.int32)
                            .pin_memory(), None] for _ in range(3)]
        self._meta_k = 0
        self.cells = None if cells is None else torch.as_tensor(
            np.asarray(cells, np.float64).reshape(self.B, 3), device=dev)

        def edge_cap(n_nodes):
            if e_cap is not None:
                return int(e_cap)
            if self.max_nbr:
                return n_nodes * self.max_nbr
            if self.ragged:
                return (n_nodes // max(self.max_atoms, 1) + 1) * self.max_atoms * \
                    max(self.max_atoms - 1, 0)
            n = np.diff(self.host_off).astype(np.int64)
            return int((n * (n - 1)).sum())

        self.shapes = [_Shape(c, edge_cap(c), dev) for c in caps]
        self.e_cap = self.shapes[-1].e_cap
        dt = trainer.dtype
        self.slot = dict(pos=torch.zeros(self.N, 3, dtype=torch.float64, device=dev),
                         z=torch.ones(self.N, dtype=torch.int32, device=dev),
                         e=torch.zeros(self.B, dtype=dt, device=dev),
                         f=torch.zeros(self.N, 3, dtype=dt, device=dev))
        self.cur = self.shapes[-1]
        # thread-rank comms rendezvous on the host: no graph capture
        self.use_graph = use_graph and getattr(trainer.comm, "capturable", True)
        self.loss_host = torch.empty(2, dtype=torch.float32).pin_memory()
        # pipelined stepping: two pinned loss slots, each with its copy event
        self._loss_slots = [torch.empty(2, dtype=torch.float32).pin_memory() for _ in range(2)]
        self._loss_events = [None, None]
        self._slot = 0
        self._stage = None

    # ---- compatibility views ---------------------------------------------
    @property
    def graph(self):
        return self.cur.graph

    @graph.setter
    def graph(self, g):
        self.cur.graph = g

    @property
    def batch(self):
        return self.cur.batch

    @property
    def bufs(self):
        return self.cur.bufs

    # ---- layout --------------------------------------------------------------
    def _write_meta(self, offsets, sync=False, eoffsets=None, idx=None):
        off = np.asarray(offsets, np.int64)
        B_true = off.shape[0] - 1
        host = np.zeros(self.meta.shape[0] + self.B, np.int32)  # meta | idx
        host[0], host[1] = B_true, off[-1]
        host[2:2 + B_true + 1] = off
        host[2 + B_true + 1:self.B + 3] = off[-1]  # empty capacity graphs
        host[self.B + 3:self.B + 3 + B_true] = np.diff(off)
        if eoffsets is not None:
            eo = np.asarray(eoffsets, np.int64)
            e0 = 2 * self.B + 3
            host[e0:e0 + B_true + 1] = eo
            host[e0 + B_true + 1:e0 + self.B + 1] = eo[-1]
        nm = self.meta.shape[0]
        if idx is not None:
            host[nm:nm + B_true] = idx
        if sync:
            self.meta.copy_(torch.from_numpy(host[:nm]))
            return
        buf = self._meta_ring[self._meta_k]
        self._meta_k = (self._meta_k + 1) % len(self._meta_ring)
        if buf[1] is not None:
            buf[1].synchronize()  # that staging buffer's last copy is done
        buf[0].numpy()[:] = host
        self.meta.copy_(buf[0][:nm], non_blocking=True)
        if idx is not None:
            self.idx.copy_(buf[0][nm:], non_blocking=True)
        buf[1] = torch.cuda.Event()
        buf[1].record()

    def set_indices(self, indices) -> _Shape:
        """Store mode: the next batch = store structures ``indices`` (host
        ints).  Their layout words and the indices go to the device (one
        small copy); the captured step gathers the structures itself."""
        if self.store is None:
            raise ValidationError("set_indices needs a runner built with store=")
        idx = np.asarray(indices, np.int64).reshape(-1)
        off, eoff = self.store.batch_layout(self.group, idx)
        return self.set_layout(off, eoffsets=eoff, idx=idx)

    def set_layout(self, offsets, eoffsets=None, idx=None) -> _Shape:
        """Ragged: the next batch's node offsets (host, B_true + 1 entries)
        -> device layout words; selects the smallest capacity holding it."""
        off = np.asarray(offsets, np.int64).reshape(-1)
        if not self.ragged:
            if not np.array_equal(off, self.host_off):
                raise ValidationError("batch structure sizes do not match the runner's layout")
            return self.cur
        n = np.diff(off)
        if off.shape[0] - 1 > self.B or off.shape[0] < 2:
            raise ValidationError(f"a batch holds 1..{self.B} structures, got {off.shape[0] - 1}")
        if n.size and (n.max() > self.max_atoms or n.min() < 0):
            raise ValidationError(f"structures hold 0..{self.max_atoms} atoms")
        N = int(off[-1])
        for sh in self.shapes:
            if N <= sh.N:
                self.cur = sh
                break
        else:
            raise ValidationError(f"batch of {N} atoms exceeds the runner's capacity {self.N}")
        if eoffsets is not None and int(np.asarray(eoffsets)[-1]) > self.cur.e_cap:
            raise ValidationError(f"batch of {int(np.asarray(eoffsets)[-1])} edges exceeds "
                                  f"e_cap={self.cur.e_cap}")
        self._write_meta(off, eoffsets=eoffsets, idx=idx)
        return self.cur

    def load(self, pos, z, energy, forces, offsets=None):
        """copy one batch's inputs into the device slots (ragged: with its
        node ``offsets``; tensors may be pinned host or device memory)"""
        if self.ragged:
            if offsets is None:
                raise ValidationError("a ragged runner needs each batch's node offsets")
            self.set_layout(offsets)
        N = int(pos.reshape(-1, 3).shape[0])
        Bt = int(energy.reshape(-1).shape[0])
        if not isinstance(z, torch.Tensor) or not z.is_cuda:
            zz = np.asarray(z.numpy() if isinstance(z, torch.Tensor) else z)
            if zz.size and (zz.min() < 1 or zz.max() > MAX_Z):
                raise ValidationError(f"atomic numbers must lie in [1, {MAX_Z}]")
        for key, v, n in (("pos", pos, N), ("z", z, N), ("e", energy, Bt), ("f", forces, N)):
            dst = self.slot[key][:n]
            dst.copy_(torch.as_tensor(v).reshape(dst.shape), non_blocking=True)

    # ---- the step ------------------------------------------------------------
    def _eager(self, sh: _Shape | None = None, slot=None):
        from .model import radius_batch

        sh = sh or self.cur
        sl = slot or self.slot
        if self.store is not None:
            from .store import gather_batch
            sh.batch = gather_batch(self.store.group(self.group), self.idx, self.meta, self.B,
                                    sh.N, sh.e_cap, self.tr.dtype, sh.bufs, sl, self.off,
                                    self.npg, self.counts, self.host_off)
            self.tr.step(sh.batch, scratch=sh.scratch)
            return
        sh.bufs["n_per_graph"] = self.npg
        sh.bufs["counts"] = self.counts
        sh.batch = radius_batch(sl["pos"][:sh.N], sl["z"][:sh.N], self.off, self.host_off,
                                self.rc, self.max_nbr, self.cells, sl["e"], sl["f"][:sh.N],
                                self.tr.dtype, e_cap=sh.e_cap, out=sh.bufs,
                                max_atoms=self.max_atoms)
        self.tr.step(sh.batch, scratch=sh.scratch)

    def capture(self, warmup: int = 2):
        """Warm up eagerly (allocates every buffer) and record one step per
        capacity.  The training state is restored afterwards: capturing adds
        no training step."""
        with self.tr.preserved():
            for sh in self.shapes:
                for _ in range(warmup):
                    self._eager(sh)
                torch.cuda.synchronize()
                self._check_overflow(sh)
            if self.use_graph:
                for sh in self.shapes:
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g):
                        self._eager(sh)
                    sh.graph = g
            torch.cuda.synchronize()
        return self

    def _check_overflow(self, sh):
        from .model import radius_batch_overflowed

        if self.store is None and radius_batch_overflowed(sh.bufs, self.B):
            raise ValidationError(f"a batch had more than e_cap={sh.e_cap} edges; raise e_cap")

    def run(self):
        self.tr.steps += 1
        self.tr._ensure_bc(self.tr.steps + 2)
        if self.cur.graph is not None:
            self.cur.graph.replay()
        else:
            self._eager()
            self.tr.steps -= 1  # tr.step counted it

    def step(self, pos, z, energy, forces, offsets=None) -> float:
        """End to end: inputs (host or device) -> step -> mean loss on host."""
        self.load(pos, z, energy, forces, offsets)
        self.run()
        P = self.tr.P
        self.loss_host.copy_(self.tr.contrib[P:P + 2].float(), non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self._check_overflow(self.cur)
        tot, cnt = float(self.loss_host[0]), float(self.loss_host[1])
        return tot / cnt if cnt else float("nan")

    def _build_stages(self):
        """Two device staging copies of the input slots (+ the copy stream)."""
        dev = self.tr.device
        self._stage = [{k: torch.empty_like(v) for k, v in self.slot.items()} for _ in range(2)]
        for st in self._stage:
            st["z"].fill_(1)
        self._copy_stream = torch.cuda.Stream(device=dev)
        self._stage_free = [None, None]
        self._stage_i = 0

    def _capture_stages(self, sh):
        """One captured step per staging copy, each reading its staging
        buffers directly (no stage -> slot copy; the stage stays busy until
        the step's ``_stage_free`` event).  Capture records without executing,
        so building these never adds a training step."""
        torch.cuda.synchronize()
        graphs = []
        for k in range(2):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._eager(sh, self._stage[k])
            graphs.append(g)
        sh.stage_graphs = graphs

    def step_pipelined(self, pos, z, energy, forces, offsets=None):
        """As ``step``, but pipelined: the host->device copy of this step's
        inputs runs on a copy stream into one of two staging buffers while the
        previous step computes, and the host reads this step's loss one call
        later (asynchronous loss logging).  The caller must not modify a
        (pinned) input buffer until two calls later.  Returns the previous
        step's mean loss (None on the first call); call ``drain()`` after the
        last step for its loss."""
        if self._stage is None:
            self._build_stages()
        main = torch.cuda.current_stream(self.tr.device)
        if self.ragged:
            if offsets is None:
                raise ValidationError("a ragged runner needs each batch's node offsets")
            self.set_layout(offsets)
        sh = self.cur
        k = self._stage_i
        cs = self._copy_stream
        if self._stage_free[k] is not None:
            cs.wait_event(self._stage_free[k])  # the step that last read stage k is done
        ins = (("pos", pos), ("z", z), ("e", energy), ("f", forces))
        if any(isinstance(v, torch.Tensor) and v.is_cuda for _, v in ins):
            cs.wait_stream(main)  # device inputs produced on the compute stream
        N = int(pos.reshape(-1, 3).shape[0])
        Bt = int(energy.reshape(-1).shape[0])
        with torch.cuda.stream(cs):
            for key, v in ins:
                n = Bt if key == "e" else N
                dst = self._stage[k][key][:n]
                dst.copy_(torch.as_tensor(v).reshape(dst.shape), non_blocking=True)
                if isinstance(v, torch.Tensor) and v.is_cuda:
                    v.record_stream(cs)
        copied = torch.cuda.Event()
        copied.record(cs)
        main.wait_event(copied)
        if self.use_graph and sh.stage_graphs is None and sh.batch is not None:
            self._capture_stages(sh)  # buffers exist (an earlier eager step allocated them)
        self.tr.steps += 1
        self.tr._ensure_bc(self.tr.steps + 2)
        if sh.stage_graphs is not None:
            sh.stage_graphs[k].replay()
        else:
            self._eager(sh, self._stage[k])
            self.tr.steps -= 1
        free = torch.cuda.Event()
        free.record(main)
        self._stage_free[k] = free
        self._stage_i = k ^ 1
        P = self.tr.P
        k = self._slot
        self._loss_slots[k].copy_(self.tr.contrib[P:P + 2].float(), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self._loss_events[k] = ev
        self._slot = k ^ 1
        return self._read_slot(k ^ 1)

    def drain(self):
        """Loss of the last ``step_pipelined`` call (waits for it)."""
        return self._read_slot(self._slot ^ 1)

    def _read_slot(self, k):
        ev = self._loss_events[k]
        if ev is None:
            return None
        ev.synchronize()
        self._loss_events[k] = None
        tot, cnt = float(self._loss_slots[k][0]), float(self._loss_slots[k][1])
        return tot / cnt if cnt else float("nan")


# --------------------------------------------------------------------------
# GFMP checkpoints (train.py:341-423): the reference's byte format, so a
# model trained here loads in the reference's ensemble/HPO/uq tooling and
# vice versa.  Layout (little-endian):
#   b"GFMP" | u32 version | u64 len(cfg) | cfg json (sort_keys) |
#   u64 n | u64 t | i64 epoch | i64 base_seed | f64 flat[n] | f64 m[n] |
#   f64 v[n] | u32 crc32(everything before it)
# --------------------------------------------------------------------------

CHECKPOINT_MAGIC = b"GFMP"        # train.py:55
CHECKPOINT_VERSION = 1            # train.py:56
_CKPT_HEAD = struct.Struct("<IQ")
_CKPT_COUNTS = struct.Struct("<QQq")


@dataclass
class Checkpoint:
    """train.py:349-355."""
    model_config: ModelConfig
    flat: np.ndarray
    opt_state: OptimizerState
    epoch: int
    base_seed: int


def _host_f64(x) -> np.ndarray:
    if isinstance(x, torch.Tensor):
        x = x.detach().to("cpu", torch.float64).numpy()
    return np.ascontiguousarray(x, dtype="<f8")


def save_checkpoint(path: str, model_config: ModelConfig, flat, opt_state: OptimizerState,
                    epoch: int, base_seed: int) -> None:
    """train.py:358-381.  ``flat``/``m``/``v`` may be numpy or device tensors
    in the reference's flat order; the file is byte-identical to the
    reference's for the same values."""
    flat = _host_f64(flat)
    m, v = _host_f64(opt_state.m), _host_f64(opt_state.v)
    n = flat.shape[0]
    if flat.ndim != 1 or m.shape != (n,) or v.shape != (n,):
        raise ValidationError(f"checkpoint vectors disagree: flat {flat.shape}, m {m.shape}, "
                              f"v {v.shape}")
    cfg = json.dumps(model_config.to_dict(), sort_keys=True).encode()
    body = b"".join((CHECKPOINT_MAGIC, _CKPT_HEAD.pack(CHECKPOINT_VERSION, len(cfg)), cfg,
                     _CKPT_COUNTS.pack(n, int(opt_state.t), int(epoch)),
                     struct.pack("<q", int(base_seed)), flat.tobytes(), m.tobytes(),
                     v.tobytes()))
    with open(path, "wb") as fh:
        fh.write(body + struct.pack("<I", zlib.crc32(body)))


def load_checkpoint(path: str) -> Checkpoint:
    """train.py:384-423, same checks and error classes: bad magic ->
    FormatError; wrong version -> UnsupportedVersionError; bad crc or
    length -> CorruptionError.  Returns host (numpy) vectors."""
    with open(path, "rb") as fh:
        blob = fh.read()
    magic = len(CHECKPOINT_MAGIC)
    if len(blob) < 4 or blob[:magic] != CHECKPOINT_MAGIC:
        raise FormatError(f"{path!r} is not a checkpoint (bad magic)")
    if len(blob) < 8:
        raise CorruptionError(f"checkpoint {path!r} truncated")
    body = memoryview(blob)[:-4]
    if zlib.crc32(body) != struct.unpack("<I", blob[-4:])[0]:
        raise CorruptionError(f"checkpoint {path!r} failed its checksum")
    version, cfg_len = _CKPT_HEAD.unpack_from(body, magic)
    if version != CHECKPOINT_VERSION:
        raise UnsupportedVersionError(
            f"checkpoint version {version} not supported (want {CHECKPOINT_VERSION})")
    off = magic + _CKPT_HEAD.size
    doc = json.loads(bytes(body[off:off + cfg_len]))
    if doc.get("model_type") == "egnn":
        from .egnn import EGNNConfig
        model_config = EGNNConfig.from_dict(doc)
    else:
        model_config = ModelConfig.from_dict(doc)
    off += cfg_len
    n, t, epoch = _CKPT_COUNTS.unpack_from(body, off)
    off += _CKPT_COUNTS.size
    (base_seed,) = struct.unpack_from("<q", body, off)
    off += 8
    if len(body) != off + 24 * n:
        raise CorruptionError(f"checkpoint {path!r} truncated: {len(body)} bytes, "
                              f"expected {off + 24 * n}")
    vecs = np.frombuffer(body, dtype="<f8", count=3 * n, offset=off).reshape(3, n).copy()
    return Checkpoint(model_config=model_config, flat=vecs[0].copy(),
                      opt_state=OptimizerState(vecs[1].copy(), vecs[2].copy(), t),
                      epoch=epoch, base_seed=base_seed)


def _fetch_batch(store, group: str, indices, device, dtype, plan=None):
    """one batch from any store: a collective store (store.ShardedDeviceStore)
    is called on every rank, with or without indices (``plan``: every rank's
    indices of this call, from the global schedule); None = nothing here"""
    if getattr(store, "collective", False):
        return store.fetch_device_batch(group, indices, dtype=dtype, plan=plan)
    if not len(indices):
        return None
    from .store import DeviceStructureStore
    if isinstance(store, DeviceStructureStore) and store.group(group).csr is not None:
        # assembled on the device from the stored CSR blocks (== make_batch)
        return store.fetch_device_batch(group, indices, dtype=dtype)
    return make_batch(store.fetch_batch(group, indices), device=device, dtype=dtype)


def evaluate(params: ModelParams, store, comm: Comm, group: str = "valset",
             batch_size: int = 64) -> tuple[float, float]:
    """Per-atom energy MAE and force-component MAE over a group
    (train.py:160-189): rank r scores ``r::P``; sums are allreduced."""
    ownership = store.ownership.get(group)
    if ownership is None:
        raise ValidationError(f"group {group!r} not loaded on rank {comm.rank}")
    n = ownership.n_samples
    dev = params.flat.device
    acc = torch.zeros(4, dtype=torch.float64, device=dev)
    mine = np.arange(comm.rank, n, comm.size)
    collective = getattr(store, "collective", False)
    # a collective (sharded) store needs every rank in every fetch: all ranks
    # run rank 0's batch count, shorter ones with empty requests
    n_rows = -(-n // comm.size) if collective else mine.shape[0]
    for lo in range(0, n_rows, batch_size):
        plan = [np.arange(r, n, comm.size)[lo:lo + batch_size] for r in range(comm.size)] \
            if collective else None
        batch = _fetch_batch(store, group, mine[lo:lo + batch_size], dev, params.dtype, plan)
        if batch is None:
            continue
        e_pred, f_pred = forward_batch(params, batch)
        # numpy's pairwise sums of this batch added to the running float64
        # totals in the reference's order (train.py:180-183)
        call("gfm_eval_errors", ptr(e_pred), ptr(batch.energy_true), ptr(batch.n_per_graph),
             batch.n_graphs, ptr(f_pred), ptr(batch.forces_true), batch.n_nodes, ptr(acc),
             _lib.dtype_code(e_pred.dtype), stream_handle())
    totals = comm.allreduce_sum(acc.cpu().numpy())
    energy_mae = totals[0] / totals[1] if totals[1] else 0.0
    force_mae = totals[2] / totals[3] if totals[3] else 0.0
    return float(energy_mae), float(force_mae)


def train(model_config: ModelConfig, store, comm: Comm | None = None,
          config: TrainConfig | None = None, clock: PhaseClock | None = None,
          initial: ModelParams | None = None, schedule_fn=None, device=None,
          dtype=torch.float32, nan_check_every: int = 16,
          device_clock: "DeviceClock | None" = None) -> TrainResult:
    """The data-parallel training loop on this rank (train.py:192-338).

    With a ``store.DeviceStructureStore`` holding records, every batch is
    assembled on the device from the store's per-structure CSR blocks inside
    one captured step (StructureStepRunner store mode): per step only the
    batch's indices and layout words cross PCIe.  Otherwise batches are
    packed from fetched records (``make_batch``).  The sticky non-finite
    guard (train.py:264-274) freezes parameters on the device at once; the
    host reads it every ``nan_check_every`` steps and at each epoch end.
    ``device_clock`` (telemetry.DeviceClock) records CUDA-event device time
    per phase beside ``clock``'s host wall time."""
    from .store import DeviceStructureStore

    comm = comm or LocalComm()
    config = config or TrainConfig()
    clock = clock or PhaseClock()
    trainer = DataParallelTrainer(model_config, config, comm, device=device, initial=initial,
                                  dtype=dtype)
    ownership = store.ownership.get("trainset")
    if ownership is None:
        raise ValidationError(f"trainset not loaded on rank {comm.rank}")
    runner = None
    if isinstance(store, DeviceStructureStore) and store.group("trainset").csr is not None:
        runner = StructureStepRunner(trainer, None, store=store, group="trainset",
                                     max_graphs=model_config.batch_size)
    captured = False
    dclk = device_clock
    n_train = ownership.n_samples
    start = time.monotonic()
    stopper = EarlyStopper(config.patience)
    metrics = []
    stop_reason = "max_epochs"
    nan_event = False
    P = trainer.P
    epoch = 0
    for epoch in range(1, config.max_epochs + 1):
        t0 = time.perf_counter()
        before = clock.totals()
        dbefore = dclk.totals() if dclk is not None else {}
        if schedule_fn is not None:
            per_rank = schedule_fn(epoch)
            mine = per_rank[comm.rank]
            steps = max(len(b) for b in per_rank)
        else:
            sched = epoch_schedule(n_train, comm.size, model_config.batch_size, config.base_seed,
                                   epoch)
            per_rank = [sched.for_rank(r) for r in range(comm.size)]
            mine = per_rank[comm.rank]
            steps = sched.max_batches()
        acc = torch.zeros(2, dtype=torch.float64, device=trainer.device)
        for step in range(steps):
            has = step < len(mine) and len(mine[step])
            if has and runner is not None:
                # device assembly + forward + backward + allreduce + update:
                # one captured graph (device time under "step")
                with clock.phase("dataload"):
                    runner.set_indices(mine[step])
                if not captured:
                    runner.capture(warmup=1)
                    captured = True
                with clock.phase("step"), _dphase(dclk, "step"):
                    runner.run()
            else:
                with clock.phase("dataload"), _dphase(dclk, "dataload"):
                    # the global schedule: a collective store plans its
                    # exchange without request round trips
                    plan = [b[step] if step < len(b) else [] for b in per_rank]
                    batch = _fetch_batch(store, "trainset", mine[step] if has else [],
                                         trainer.device, dtype, plan)
                if batch is not None:
                    with clock.phase("forward"), _dphase(dclk, "forward"):
                        cache: dict = {}
                        e_pred, f_pred = forward_batch(trainer.params, batch, cache,
                                                       scratch=trainer.scratch)
                    with clock.phase("backward"), _dphase(dclk, "backward"):
                        trainer.compute(batch, precomputed=(cache, e_pred, f_pred))
                    with clock.phase("sync"), _dphase(dclk, "sync"):
                        trainer.reduce_and_update()
                else:  # no batch for this rank: zero contribution (train.py:257-259)
                    with clock.phase("sync"), _dphase(dclk, "sync"):
                        trainer.compute(None)
                        trainer.reduce_and_update()
            acc += trainer.contrib[P:P + 2].to(torch.float64)
            if (step + 1) % max(1, nan_check_every) == 0 or step == steps - 1:
                if trainer.nan_event:  # train.py:264-274 (the device skipped the update)
                    log.warning("rank %d: non-finite loss at epoch %d (by step %d); update "
                                "discarded, training aborted", comm.rank, epoch, step)
                    nan_event = True
                    stop_reason = "nan"
                    break
        if nan_event:
            break
        params = ModelParams(model_config, trainer.work)
        ve, vf = evaluate(params, store, comm)
        after = clock.totals()
        dafter = dclk.totals() if dclk is not None else {}
        loss_sum, loss_count = acc.cpu().numpy()
        metrics.append(EpochMetrics(
            epoch=epoch, train_loss=loss_sum / loss_count if loss_count else float("nan"),
            val_mae=ve + vf, val_energy_mae=ve, val_force_mae=vf,
            epoch_time_s=time.perf_counter() - t0,
            phase_seconds={k: after[k] - before.get(k, 0.0) for k in after},
            device_phase_seconds={k: dafter[k] - dbefore.get(k, 0.0) for k in dafter}))
        if stopper.update(ve + vf):
            stop_reason = "early_stop"
            break
        over = (config.wall_clock_budget_s is not None
                and time.monotonic() - start >= config.wall_clock_budget_s)
        if comm.broadcast_obj("budget" if over else None) is not None:
            stop_reason = "budget"
            break
    if config.checkpoint_path and comm.rank == 0:  # train.py:323-331
        save_checkpoint(config.checkpoint_path, model_config, trainer.flat_master(),
                        trainer.optimizer_state(), epoch=epoch, base_seed=config.base_seed)
    return TrainResult(params=trainer.current_params(), metrics=metrics,
                       stop_reason=stop_reason, nan_event=nan_event,
                       epochs_run=len(metrics) + (1 if nan_event else 0))
