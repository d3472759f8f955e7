"""EGNN-style variant with coordinate updates and autograd forces (C4).

BASELINE.json configs[3]; the reference has no EGNN and no autograd forces
(``/root/reference/SPEC.md:8, 352``), so the model is the restatement in
``oracle/egnn_oracle.py`` (pinned there by finite differences and torch
double backward), built on the reference's conventions: embedding, tanh
node update, sum-pooled MLP energy head and the L1 MTL loss
(``/root/reference/pkg/src/gfmkit/model.py:344-400, 437-462``).

Forces are F = -dE/dx0 through every layer's distances and coordinate
updates.  Training needs dL/dtheta of a loss holding F (second
derivatives); it runs as reverse-over-forward on the device:

1. primal forward (node GEMMs on the tensor cores, ``gfm_egnn_edge_fwd``);
2. reverse pass for dE/dx0 -> F (``gfm_egnn_edge_bwd``, backward-data GEMMs);
3. L1 loss and seeds (``gfm_loss_seeds``: de = dL/dE, v = dL/dF);
4. tangent forward from xdot0 = v (tangent rows of the stacked buffers);
5. one reverse pass over primal + tangent rows with seeds (de, -1): every
   GEMM runs once on the stacked [primal; tangent] 2N rows, the edge and
   tanh kernels mix the two.

The API mirrors ``model``: ``EGNNConfig`` + the shared ``ModelParams`` /
``init_params`` / ``forward_batch`` / ``loss_and_grad`` (which dispatch on
the config type), so ``DataParallelTrainer`` and ``StructureStepRunner``
train it unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, query, stream_handle
from .errors import ValidationError
from .records import MAX_Z

COORD_INIT_SCALE = 0.1  # oracle/egnn_oracle.py: ux drawn like every weight, then scaled


@dataclass
class EGNNConfig:
    """Architecture + loss hyperparameters of the EGNN variant."""

    egnn_layers: int = 3
    egnn_width: int = 64
    fc_layers: int = 2
    fc_width: int = 64
    batch_size: int = 256
    learning_rate: float = 1e-3
    alpha_energy: float = 1.0
    alpha_forces: float = 100.0

    model_type = "egnn"

    def __post_init__(self):
        for name in ("egnn_layers", "egnn_width", "fc_width", "batch_size"):
            if int(getattr(self, name)) < 1:
                raise ValidationError(f"{name} must be >= 1")
        if self.egnn_width % 32 or self.egnn_width > 512 or \
                (self.egnn_width // 32) & (self.egnn_width // 32 - 1):
            raise ValidationError("egnn_width must be 32, 64, 128, 256 or 512")
        if self.fc_layers < 2:
            raise ValidationError("fc_layers must be >= 2 (input and output layers)")
        if self.alpha_energy <= 0 or self.alpha_forces <= 0:
            raise ValidationError("loss weights must be positive")

    # ModelConfig-compatible views used by the shared layout / trainer code
    @property
    def mpnn_width(self) -> int:
        return self.egnn_width

    @property
    def mpnn_layers(self) -> int:
        return self.egnn_layers

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "egnn_layers", "egnn_width", "fc_layers", "fc_width", "batch_size",
            "learning_rate", "alpha_energy", "alpha_forces")} | {"model_type": "egnn"}

    @classmethod
    def from_dict(cls, doc: dict) -> "EGNNConfig":
        d = dict(doc)
        d.pop("model_type", None)
        return cls(**d)


def egnn_param_shapes(config: EGNNConfig):
    """flat order of oracle/egnn_oracle.py:param_shapes: embedding; per layer
    w, wa, wb (adjacent: the backward's dh = [dz | dA | dB] [w; wa; wb] is
    one GEMM), u, wd, c, ux, b; the MPNN's energy head."""
    H, G = config.egnn_width, config.fc_width
    out = [("embedding", (MAX_Z, H))]
    for l in range(config.egnn_layers):
        out += [(f"egnn_{l}.w", (H, H)), (f"egnn_{l}.wa", (H, H)), (f"egnn_{l}.wb", (H, H)),
                (f"egnn_{l}.u", (H, H)), (f"egnn_{l}.wd", (H,)), (f"egnn_{l}.c", (H,)),
                (f"egnn_{l}.ux", (H,)), (f"egnn_{l}.b", (H,))]
    ws = [(G, H)] + [(G, G)] * (config.fc_layers - 2) + [(1, G)]
    bs = [(G,)] * (config.fc_layers - 1) + [(1,)]
    for f in range(config.fc_layers):
        out += [(f"head_{f}.w", ws[f]), (f"head_{f}.b", bs[f])]
    return out


def egnn_count_params(config: EGNNConfig) -> int:
    return sum(int(np.prod(s)) for _, s in egnn_param_shapes(config))


def egnn_init_flat(config: EGNNConfig, seed: int = 0) -> np.ndarray:
    """init_params convention (model.py:178-187) + ux scaled by 0.1
    (oracle/egnn_oracle.py:init_flat)."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(config.egnn_width)
    parts = []
    for name, shape in egnn_param_shapes(config):
        if name.endswith(".b") or name.endswith(".c"):
            parts.append(np.zeros(int(np.prod(shape))))
        else:
            v = rng.uniform(-bound, bound, size=shape).ravel()
            parts.append(v * COORD_INIT_SCALE if name.endswith(".ux") else v)
    return np.concatenate(parts)


# --------------------------------------------------------------------------
# device passes
# --------------------------------------------------------------------------


class _Bufs:
    """stacked activation buffers of one batch shape (primal rows 0..N-1,
    tangent rows N..2N-1)"""

    def __init__(self, sc, cfg, N, E, B, dt):
        H, G, L, F = cfg.egnn_width, cfg.fc_width, cfg.egnn_layers, cfg.fc_layers
        g = sc.get
        self.hs = [g(f"eg_h{l}", (2 * N, H), dt) for l in range(L + 1)]
        if not getattr(sc, "_eg_h0_zeroed", None) == self.hs[0].data_ptr():
            self.hs[0][N:].zero_()  # h0 has no tangent (the embedding ignores x)
            sc._eg_h0_zeroed = self.hs[0].data_ptr()
        self.xs = [g(f"eg_x{l}", (max(N, 1), 3), dt) for l in range(L)]
        self.xds = [g(f"eg_xd{l}", (max(N, 1), 3), dt) for l in range(L)]
        self.AB = [g(f"eg_ab{l}", (2 * N, 2 * H), dt) for l in range(L)]
        self.agg = [g(f"eg_agg{l}", (2 * N, H), dt) for l in range(L)]
        self.zt = [g(f"eg_zt{l}", (max(N, 1), H), dt) for l in range(L)]
        widths = [H] + [G] * (F - 1)
        self.ys = [self.hs[L]] + [g(f"eg_y{f}", (2 * N, G), dt) for f in range(1, F)]
        self.yzt = [None] + [g(f"eg_yzt{f}", (max(N, 1), G), dt) for f in range(1, F)]
        self.widths = widths
        self.node_e = g("eg_ne", (max(N, 1),), dt)
        self.node_ed = g("eg_ned", (max(N, 1),), dt)
        self.e_pred = g("eg_e", (max(B, 1),), dt)
        self.e_dot = g("eg_ed", (max(B, 1),), dt)
        self.f_pred = g("eg_f", (max(N, 1), 3), dt)
        self.xb = [g(f"eg_xb{k}", (max(N, 1), 3), dt) for k in range(2)]
        self.xdb = [g(f"eg_xdb{k}", (max(N, 1), 3), dt) for k in range(2)]
        self.gbuf = g("eg_gbuf", (2 * N, 3 * H), dt)      # [dz | dA | dB]
        self.aggb = g("eg_aggb", (2 * N, H), dt)
        self.hb = [g(f"eg_hb{k}", (2 * N, H), dt) for k in range(2)]     # dL/dh (layers)
        self.yb = [g(f"eg_yb{k}", (2 * N, G), dt) for k in range(2)]     # dL/dy (head)
        self.zb = g("eg_zb", (2 * N, G), dt)
        self.ds = g("eg_ds", (2 * N, 4), dt)
        self.preb = g("eg_preb", (max(E, 1), H), dt)
        self.predb = g("eg_predb", (max(E, 1), H), dt)
        self.rb = g("eg_rb", (max(E, 1), 3), dt)
        self.rdb = g("eg_rdb", (max(E, 1), 3), dt)
        self.part = g("eg_part", (max(N, 1), 2 * H), dt)
        ones = sc.bufs.get("eg_ones")
        if ones is None or ones.shape[0] < max(B, 1) or ones.dtype != dt:
            ones = torch.ones(max(B, 1), dtype=dt, device=sc.device)
            sc.bufs["eg_ones"] = ones
        self.ones = ones


def _check_batch(batch):
    if getattr(batch, "periodic", False):
        raise ValidationError("the EGNN variant takes non-periodic batches (molecules)")


class _Pass:
    """launch helpers bound to one (params, batch, scratch)"""

    def __init__(self, params, batch, sc):
        self.p = params
        self.b = batch
        self.sc = sc
        self.cfg = params.config
        self.dt = params.dtype
        self.code = _lib.dtype_code(self.dt)
        self.s = stream_handle()
        self.N = batch.n_nodes
        self.E = batch.e_cap
        self.B = batch.n_graphs
        self.buf = _Bufs(sc, self.cfg, self.N, self.E, self.B, self.dt)

    def v(self, name):
        return self.p.view(name)

    def row(self, t, r0):
        """pointer to row r0 of a 2D tensor"""
        return t.data_ptr() + r0 * t.stride(0) * t.element_size()

    def col(self, t, c0, r0=0):
        return t.data_ptr() + (r0 * t.stride(0) + c0) * t.element_size()

    def fwd(self, X1, ld1, K1, W1, M, n_out, Y, ldy, X2=None, ld2=0, K2=0, W2=None, bias=None,
            act=0):
        call("gfm_linear_fwd", X1, ld1, K1, X2, ld2, K2, W1, K1, W2, K2, bias, M, None, n_out,
             act, Y, ldy, self.code, self.s)

    def bwd_data(self, dY, ldd, M, n_out, W1, K1, out1, ldo1):
        call("gfm_linear_bwd_data", dY, ldd, M, None, n_out, W1, K1, K1, None, 0, 0, out1, ldo1,
             None, 0, None, 0, self.code, self.s)

    def wgrad(self, dY, ldd, M, n_out, X1, ld1, K1, g1, X2=None, ld2=0, K2=0, g2=None, tag=""):
        nb = query("gfm_linear_bwd_weight_workspace_bytes", M, n_out, K1, K2, 0, self.code)
        ws = self.sc.bytes(f"eg_wg_{tag}", nb)
        call("gfm_linear_bwd_weight", dY, ldd, M, None, n_out, X1, ld1, K1, X2, ld2, K2, 0,
             ptr(g1), ptr(g2), None, ptr(ws), self.code, self.s)

    def colsum(self, X, rows, cols, ld, out):
        ws = self.sc.bytes(f"eg_cs_{cols}", query("gfm_colsum_workspace_bytes", rows, cols),
                           zero=True)
        call("gfm_colsum", X, rows, cols, ld, ptr(out), 0, ptr(ws), self.code, self.s)

    # ---- passes -------------------------------------------------------------
    def forward(self, tangent: bool):
        """primal (tangent=False) or tangent rows of the forward pass"""
        cfg, b, bf, N = self.cfg, self.b, self.buf, self.N
        H, L, F, G = cfg.egnn_width, cfg.egnn_layers, cfg.fc_layers, cfg.fc_width
        r0 = N if tangent else 0
        if not tangent:
            call("gfm_embed", ptr(b.z), N, ptr(self.v("embedding")), H, ptr(bf.hs[0]), self.code,
                 self.s)
            if self.dt == torch.float32:
                call("gfm_cast_f64_to_f32", ptr(b.pos), 3 * N, ptr(bf.xs[0]), self.s)
            else:
                call("gfm_scale", ptr(b.pos), 3 * N, 1.0, ptr(bf.xs[0]), self.code, self.s)
        for l in range(L):
            v = lambda n: self.v(f"egnn_{l}.{n}")
            coord = 1 if l < L - 1 else 0
            # A | B = h [wa; wb]^T  ([wa; wb] are adjacent rows in the layout)
            self.fwd(self.row(bf.hs[l], r0), H, H, ptr(v("wa")), N, 2 * H,
                     self.row(bf.AB[l], r0), 2 * H)
            if not tangent:
                call("gfm_egnn_edge_fwd", ptr(bf.AB[l]), 2 * H, None, ptr(bf.xs[l]), None, N, H,
                     ptr(b.rowptr), ptr(b.col_src), ptr(v("wd")), ptr(v("c")), ptr(v("ux")),
                     coord, ptr(bf.agg[l]), H, None, ptr(bf.xs[l + 1]) if coord else None, None,
                     self.code, self.s)
                self.fwd(ptr(bf.hs[l]), H, H, ptr(v("w")), N, H, ptr(bf.hs[l + 1]), H,
                         X2=ptr(bf.agg[l]), ld2=H, K2=H, W2=ptr(v("u")), bias=ptr(v("b")),
                         act=1)
            else:
                call("gfm_egnn_edge_fwd", ptr(bf.AB[l]), 2 * H, self.row(bf.AB[l], N),
                     ptr(bf.xs[l]), ptr(bf.xds[l]), N, H, ptr(b.rowptr), ptr(b.col_src),
                     ptr(v("wd")), ptr(v("c")), ptr(v("ux")), coord, None, H,
                     self.row(bf.agg[l], N), None, ptr(bf.xds[l + 1]) if coord else None,
                     self.code, self.s)
                self.fwd(self.row(bf.hs[l], N), H, H, ptr(v("w")), N, H, ptr(bf.zt[l]), H,
                         X2=self.row(bf.agg[l], N), ld2=H, K2=H, W2=ptr(v("u")))
                call("gfm_egnn_tanh_fwd", None, ptr(bf.zt[l]), H, None, N, H, ptr(bf.hs[l + 1]),
                     self.row(bf.hs[l + 1], N), H, self.code, self.s)
        for f in range(F - 1):
            kin = bf.widths[f]
            if not tangent:
                self.fwd(ptr(bf.ys[f]), kin, kin, ptr(self.v(f"head_{f}.w")), N, G,
                         ptr(bf.ys[f + 1]), G, bias=ptr(self.v(f"head_{f}.b")), act=1)
            else:
                self.fwd(self.row(bf.ys[f], N), kin, kin, ptr(self.v(f"head_{f}.w")), N, G,
                         ptr(bf.yzt[f + 1]), G)
                call("gfm_egnn_tanh_fwd", None, ptr(bf.yzt[f + 1]), G, None, N, G,
                     ptr(bf.ys[f + 1]), self.row(bf.ys[f + 1], N), G, self.code, self.s)
        if not tangent:
            call("gfm_egnn_energy", ptr(bf.ys[F - 1]), None, bf.widths[F - 1], N,
                 bf.widths[F - 1], ptr(self.v(f"head_{F - 1}.w")),
                 ptr(self.v(f"head_{F - 1}.b")), ptr(b.node_offsets), self.B, ptr(bf.node_e),
                 None, ptr(bf.e_pred), None, self.code, self.s)

    def reverse(self, de, dual: bool, grad=None):
        """Reverse pass.  dual=False: seeds dE_g = de (ones) over the primal
        rows, result dL/dx0 in the returned (N, 3) buffer.  dual=True: seeds
        (de, -1) over primal + tangent rows, parameter gradients into
        ``grad`` (a ModelParams view of the flat gradient)."""
        cfg, b, bf, N = self.cfg, self.b, self.buf, self.N
        H, L, F, G = cfg.egnn_width, cfg.egnn_layers, cfg.fc_layers, cfg.fc_width
        rows = 2 * N if dual else N
        # head seeds + energy-head backward (model.py:520-533, dual)
        yb, yb_next = bf.yb
        call("gfm_egnn_head_seed", ptr(de), ptr(b.graph_of_node), N, rows, -1.0 if dual else 0.0,
             ptr(self.v(f"head_{F - 1}.w")), G, ptr(bf.ds), ptr(yb), G, self.code, self.s)
        if dual:
            self.wgrad(ptr(bf.ds), 4, rows, 1, ptr(bf.ys[F - 1]), G, G, grad.view(f"head_{F - 1}.w"),
                       tag="hl")
            self.colsum(ptr(bf.ds), N, 1, 4, grad.view(f"head_{F - 1}.b"))
        hb, hb_next = bf.hb
        for f in range(F - 2, -1, -1):
            kin = bf.widths[f]
            zt = bf.yzt[f + 1]
            call("gfm_egnn_tanh_bwd", ptr(bf.ys[f + 1]), G, ptr(zt) if dual else None, G,
                 ptr(yb), self.row(yb, N) if dual else None, G, N, G, ptr(bf.zb),
                 self.row(bf.zb, N) if dual else None, G, self.code, self.s)
            if dual:
                self.wgrad(ptr(bf.zb), G, rows, G, ptr(bf.ys[f]), kin, kin,
                           grad.view(f"head_{f}.w"), tag=f"h{f}")
                self.colsum(ptr(bf.zb), N, G, G, grad.view(f"head_{f}.b"))
            out = hb if f == 0 else yb_next  # f == 0: dL/dh of the last layer (width H)
            self.bwd_data(ptr(bf.zb), G, rows, G, ptr(self.v(f"head_{f}.w")), kin, ptr(out), kin)
            yb, yb_next = yb_next, yb
        # message-passing layers, last to first
        xb, xb_new = bf.xb
        xdb, xdb_new = bf.xdb
        ld3 = 3 * H
        for l in range(L - 1, -1, -1):
            v = lambda n: self.v(f"egnn_{l}.{n}")
            coord = 1 if l < L - 1 else 0
            # node update adjoints: [dz] -> gbuf[:, 0:H]
            call("gfm_egnn_tanh_bwd", ptr(bf.hs[l + 1]), H, ptr(bf.zt[l]) if dual else None, H,
                 ptr(hb), self.row(hb, N) if dual else None, H, N, H, ptr(bf.gbuf),
                 self.row(bf.gbuf, N) if dual else None, ld3, self.code, self.s)
            self.bwd_data(ptr(bf.gbuf), ld3, rows, H, ptr(v("u")), H, ptr(bf.aggb), H)
            call("gfm_egnn_edge_bwd", ptr(bf.AB[l]), 2 * H, self.row(bf.AB[l], N) if dual else None,
                 ptr(bf.xs[l]), ptr(bf.xds[l]) if dual else None, N, H, ptr(b.rowptr),
                 ptr(b.col_src), ptr(b.csc_ptr), ptr(b.csc_eid), ptr(v("wd")), ptr(v("c")),
                 ptr(v("ux")), coord, ptr(bf.aggb), H, self.row(bf.aggb, N) if dual else None,
                 ptr(xb) if coord else None, ptr(xdb) if (coord and dual) else None,
                 self.col(bf.gbuf, H), ld3, self.col(bf.gbuf, H, N) if dual else None,
                 ptr(bf.preb), ptr(bf.predb) if dual else None, ptr(bf.rb),
                 ptr(bf.rdb) if dual else None, ptr(xb_new), ptr(xdb_new) if dual else None,
                 ptr(bf.part), self.code, self.s)
            if dual:
                g = lambda n: grad.view(f"egnn_{l}.{n}")
                self.wgrad(ptr(bf.gbuf), ld3, rows, H, ptr(bf.hs[l]), H, H, g("w"),
                           X2=ptr(bf.agg[l]), ld2=H, K2=H, g2=g("u"), tag=f"n{l}")
                # [d wa; d wb] (2H x H, adjacent in the layout) = [dA | dB]^T h
                self.wgrad(self.col(bf.gbuf, H), ld3, rows, 2 * H, ptr(bf.hs[l]), H, H, g("wa"),
                           tag=f"e{l}")
                self.colsum(ptr(bf.gbuf), N, H, ld3, g("b"))
                self.colsum(self.col(bf.gbuf, H), N, H, ld3, g("c"))
                self.colsum(ptr(bf.part), N, H, 2 * H, g("wd"))
                self.colsum(self.col(bf.part, H), N, H, 2 * H, g("ux"))
            # dh = [dz | dA | dB] [w; wa; wb]
            self.bwd_data(ptr(bf.gbuf), ld3, rows, 3 * H, ptr(v("w")), H, ptr(hb_next), H)
            hb, hb_next = hb_next, hb
            xb, xb_new = xb_new, xb
            xdb, xdb_new = xdb_new, xdb
        if dual:
            ews = self.sc.bytes("eg_emb_ws", query("gfm_embedding_grad_workspace_bytes", N, H,
                                                   self.code))
            call("gfm_embedding_grad", ptr(b.z), N, ptr(hb), H, ptr(grad.embedding), ptr(ews),
                 self.code, self.s)
        return xb


def forces(params, batch, scratch=None):
    """(e_pred (B,), f_pred (N, 3)): energies and F = -dE/dx0 (autograd
    forces through every distance and coordinate update)."""
    from .model import _scratch_for

    _check_batch(batch)
    sc = _scratch_for(scratch, batch.device)
    ps = _Pass(params, batch, sc)
    ps.forward(False)
    xb = ps.reverse(ps.buf.ones, dual=False)
    call("gfm_scale", ptr(xb), 3 * ps.N, -1.0, ptr(ps.buf.f_pred), ps.code, ps.s)
    return ps, ps.buf.e_pred, ps.buf.f_pred


def loss_and_grad(params, batch, scratch=None, grad_out=None, contrib=None):
    """L1 MTL loss on (E, F = -dE/dx0) and its exact gradient (reverse over
    the primal + tangent forward).  Same return as model.loss_and_grad."""
    from .model import LossBreakdown, ModelParams, _loss_kernel

    cfg = params.config
    ps, e_pred, f_pred = forces(params, batch, scratch)
    vals, de, df = _loss_kernel(e_pred[:ps.B], f_pred[:ps.N], batch.energy_true,
                                batch.forces_true, batch.n_per_graph, cfg.alpha_energy,
                                cfg.alpha_forces, scratch=ps.sc, contrib=contrib,
                                counts=batch.counts)
    grad = grad_out if grad_out is not None else torch.zeros(params.layout.Pp, dtype=ps.dt,
                                                             device=batch.device)
    gp = ModelParams(cfg, grad)
    # tangent forward from xdot0 = dL/dF, then the dual reverse pass
    call("gfm_scale", ptr(df), 3 * ps.N, 1.0, ptr(ps.buf.xds[0]), ps.code, ps.s)
    ps.forward(True)
    ps.reverse(de, dual=True, grad=gp)
    lb = LossBreakdown(vals if scratch is not None else vals.clone(),
                       lambda: (e_pred - batch.energy_true) / batch.n_per_graph.to(e_pred.dtype))
    return lb, (grad if grad_out is not None else params.layout.compact(grad))
