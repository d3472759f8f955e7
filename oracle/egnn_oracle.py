"""float64 numpy restatement of the EGNN-style variant (C4) -- TEST ORACLE.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  The reference has no
EGNN and no autograd forces (``/root/reference/SPEC.md:8, 352``; its force
head is an edge-pair MLP, not -grad E).  BASELINE.json configs[3] asks for
"EGNN-style equivariant message-passing with coordinate updates and autograd
forces"; this module restates it with the reference's conventions
(embedding, tanh node update, sum-pooled energy head, L1 MTL loss:
``/root/reference/pkg/src/gfmkit/model.py:344-400, 437-462``) and the E(n)
equivariant layer of Satorras et al. (2021) as HydraGNN's EGCL uses it:

    r_e   = x_src - x_dst (+ shift)            d2_e = r_e . r_e
    m_e   = tanh(A_dst + B_src + wd * d2_e + c)   A = h Wa^T, B = h Wb^T
    s_e   = m_e . ux                            (coordinate weight, scalar)
    agg_i = sum_{e -> i} m_e
    x'_i  = x_i - (1 / max(deg_i, 1)) sum_{e -> i} r_e s_e   (layers 0..L-2)
    h'_i  = tanh(h_i W^T + agg_i U^T + b)

energy E_g = sum-pooled head(h_L) (model.py:365-373); forces F = -dE/dx0
(autograd forces: the graph is fixed, positions are differentiated through
every layer's distances and coordinate updates).

Training needs dL/dtheta of a loss that contains F = -dE/dx0, i.e. second
derivatives.  With seeds de = dL/dE and v = dL/dF (the L1 seeds of
model.py:510-516):  dL/dtheta = d/dtheta [ sum_g de_g E_g - v . dE/dx0 ],
and v . dE/dx0 = Edot is the directional derivative of E along v -- one
forward-mode (tangent) pass from xdot0 = v.  So the gradient is ONE reverse
pass over the primal + tangent forward with seeds (E: de, Edot: -1):
reverse-over-forward, which is what the GPU kernels implement.  Every linear
op acts on primal and tangent rows alike (stacked [p; pdot] GEMMs); only the
elementwise ops (tanh, distances, coordinate products) mix them.

Pinned by (tests/test_egnn_oracle.py): F against central finite differences
of E in x0; dL/dtheta against central differences of the loss; both against
torch autograd double backward in float64; E(3) invariance of E and
equivariance of F.
"""

from __future__ import annotations

import numpy as np

MAX_Z = 118
COORD_INIT_SCALE = 0.1  # ux drawn like every weight, then scaled (small coordinate steps)


def config(layers=3, hidden=64, fc_layers=2, fc_width=64, alpha_energy=1.0,
           alpha_forces=100.0):
    if fc_layers < 2:
        raise ValueError("fc_layers must be >= 2")
    return dict(L=int(layers), H=int(hidden), F=int(fc_layers), G=int(fc_width),
                aE=float(alpha_energy), aF=float(alpha_forces))


def param_shapes(cfg):
    """flat order: embedding; per layer w (node update, on h), wa, wb (edge
    MLP on h_dst / h_src), u (node update, on agg), wd, c (edge MLP distance
    weight and bias), ux (coordinate weight), b (node update bias); energy
    head as the MPNN.  [w; wa; wb] are adjacent so the backward's
    dh = [dz | dA | dB] [w; wa; wb] is one GEMM."""
    H, G = cfg["H"], cfg["G"]
    out = [("embedding", (MAX_Z, H))]
    for l in range(cfg["L"]):
        out += [(f"egnn_{l}.w", (H, H)), (f"egnn_{l}.wa", (H, H)), (f"egnn_{l}.wb", (H, H)),
                (f"egnn_{l}.u", (H, H)), (f"egnn_{l}.wd", (H,)), (f"egnn_{l}.c", (H,)),
                (f"egnn_{l}.ux", (H,)), (f"egnn_{l}.b", (H,))]
    ws = [(G, H)] + [(G, G)] * (cfg["F"] - 2) + [(1, G)]
    bs = [(G,)] * (cfg["F"] - 1) + [(1,)]
    for f in range(cfg["F"]):
        out += [(f"head_{f}.w", ws[f]), (f"head_{f}.b", bs[f])]
    return out


def n_params(cfg):
    return sum(int(np.prod(s)) for _, s in param_shapes(cfg))


def unflatten(cfg, flat):
    flat = np.asarray(flat, dtype=np.float64)
    views, off = {}, 0
    for name, shape in param_shapes(cfg):
        size = int(np.prod(shape))
        views[name] = flat[off:off + size].reshape(shape)
        off += size
    return views


def init_flat(cfg, seed=0):
    """init_params convention (model.py:178-187): uniform(+-1/sqrt(H)) in
    flat order from default_rng(seed), names ending .b / .c stay zero;
    the coordinate weights ux are then scaled by COORD_INIT_SCALE."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(cfg["H"])
    flat = np.zeros(n_params(cfg))
    views = unflatten(cfg, flat)
    for name, shape in param_shapes(cfg):
        if name.endswith(".b") or name.endswith(".c"):
            continue
        views[name][...] = rng.uniform(-bound, bound, size=shape)
        if name.endswith(".ux"):
            views[name][...] *= COORD_INIT_SCALE
    return flat


def _sum_to(idx, vals, n):
    out = np.zeros((n,) + vals.shape[1:])
    np.add.at(out, idx, vals)
    return out


def forward(cfg, flat, b, x0=None, tangent=None, cache=None):
    """Primal (and, with ``tangent`` = xdot0 (N, 3), tangent) forward.
    ``b`` = oracle.gfm_oracle.pack(records) (uses src, dst, z, offsets,
    deg and the per-edge shift folded into dx - pos[src] + pos[dst]).
    Returns e_pred (B,) [, edot (B,)]."""
    P = unflatten(cfg, flat)
    src, dst = b["src"], b["dst"]
    N, L = b["z"].shape[0], cfg["L"]
    x = np.array(b["pos"] if x0 is None else x0, dtype=np.float64)
    shift = b["dx"] - (b["pos"][src] - b["pos"][dst])  # constant image offsets
    cinv = 1.0 / np.maximum(b["deg"], 1).astype(np.float64)
    h = P["embedding"][b["z"] - 1]
    dual = tangent is not None
    xd = np.array(tangent, dtype=np.float64) if dual else None
    hd = np.zeros_like(h) if dual else None
    layers = []
    for l in range(L):
        p = lambda n: P[f"egnn_{l}.{n}"]
        A, B = h @ p("wa").T, h @ p("wb").T
        r = x[src] - x[dst] + shift
        d2 = (r * r).sum(axis=1)
        m = np.tanh(A[dst] + B[src] + d2[:, None] * p("wd") + p("c"))
        s = m @ p("ux")
        agg = _sum_to(dst, m, N)
        lay = dict(h=h, x=x, A=A, B=B, r=r, d2=d2, m=m, s=s, agg=agg)
        if dual:
            Ad, Bd = hd @ p("wa").T, hd @ p("wb").T
            rd = xd[src] - xd[dst]
            d2d = 2.0 * (r * rd).sum(axis=1)
            pred = Ad[dst] + Bd[src] + d2d[:, None] * p("wd")
            md = (1.0 - m * m) * pred
            sd = md @ p("ux")
            aggd = _sum_to(dst, md, N)
            lay.update(hd=hd, xd=xd, rd=rd, d2d=d2d, pred=pred, md=md, sd=sd, aggd=aggd)
        if l < L - 1:
            x_new = x - cinv[:, None] * _sum_to(dst, r * s[:, None], N)
            if dual:
                xd = xd - cinv[:, None] * _sum_to(dst, rd * s[:, None] + r * sd[:, None], N)
        else:
            x_new = x
        z = h @ p("w").T + agg @ p("u").T + p("b")
        h_new = np.tanh(z)
        lay["h_out"] = h_new
        if dual:
            zd = hd @ p("w").T + aggd @ p("u").T
            hd = (1.0 - h_new * h_new) * zd
            lay.update(zd=zd, hd_out=hd)
        layers.append(lay)
        h, x = h_new, x_new
    ys, yds = [h], [hd]
    y, yd = h, hd
    F = cfg["F"]
    for f in range(F - 1):
        y = np.tanh(y @ P[f"head_{f}.w"].T + P[f"head_{f}.b"])
        ys.append(y)
        if dual:
            yd = (1.0 - y * y) * (yd @ P[f"head_{f}.w"].T)
            yds.append(yd)
    node_e = (y @ P[f"head_{F - 1}.w"].T)[:, 0] + P[f"head_{F - 1}.b"][0]
    e_pred = np.add.reduceat(node_e, b["offsets"][:-1]) if N else np.zeros(0)
    if cache is not None:
        cache.update(layers=layers, ys=ys, yds=yds, cinv=cinv)
    if dual:
        ed = (yd @ P[f"head_{F - 1}.w"].T)[:, 0]
        return e_pred, np.add.reduceat(ed, b["offsets"][:-1])
    return e_pred


def energy_total(cfg, flat, b, x0=None):
    return float(forward(cfg, flat, b, x0).sum())


def forces(cfg, flat, b, cache=None):
    """F = -dE_total/dx0 by one reverse pass (seed dE_g = 1)."""
    c = {} if cache is None else cache
    e_pred = forward(cfg, flat, b, cache=c)
    grads = _reverse(cfg, flat, b, c, np.ones(e_pred.shape[0]), None, want_params=False)
    return e_pred, -grads["x0"]


def _reverse(cfg, flat, b, c, de, edot_seed, want_params=True):
    """Reverse pass over the cached forward.  Primal seeds dL/dE_g = de;
    with ``edot_seed`` (a scalar, the seed of sum_g Edot_g) the cache must
    hold the tangent forward and the pass runs over primal + tangent."""
    P = unflatten(cfg, flat)
    G_ = unflatten(cfg, np.zeros_like(flat)) if want_params else None
    src, dst = b["src"], b["dst"]
    N, L, F = b["z"].shape[0], cfg["L"], cfg["F"]
    dual = edot_seed is not None
    gnode = np.repeat(np.arange(len(b["offsets"]) - 1), np.diff(b["offsets"]))
    ys, yds = c["ys"], c["yds"]
    # head (model.py:520-533), dual: node_e = y a + c, ndot = ydot a
    ne_bar = de[gnode]
    a = P[f"head_{F - 1}.w"]
    if want_params:
        G_[f"head_{F - 1}.w"][...] += ne_bar @ ys[-1]
        G_[f"head_{F - 1}.b"][...] += ne_bar.sum()
    yb = ne_bar[:, None] * a
    if dual:
        G_[f"head_{F - 1}.w"][...] += edot_seed * yds[-1].sum(axis=0)
        ydb = edot_seed * np.ones((N, 1)) * a
    for f in range(F - 2, -1, -1):
        y = ys[f + 1]
        if dual:
            zd = yds[f] @ P[f"head_{f}.w"].T
            zb = (1.0 - y * y) * (yb - 2.0 * y * zd * ydb)
            zdb = (1.0 - y * y) * ydb
        else:
            zb = (1.0 - y * y) * yb
        if want_params:
            G_[f"head_{f}.w"][...] += zb.T @ ys[f] + (zdb.T @ yds[f] if dual else 0.0)
            G_[f"head_{f}.b"][...] += zb.sum(axis=0)
        yb = zb @ P[f"head_{f}.w"]
        if dual:
            ydb = zdb @ P[f"head_{f}.w"]
    hb, xb = yb, np.zeros((N, 3))
    hdb = ydb if dual else None
    xdb = np.zeros((N, 3)) if dual else None
    cinv = c["cinv"]
    for l in range(L - 1, -1, -1):
        lay = c["layers"][l]
        p = lambda n: P[f"egnn_{l}.{n}"]
        gp = (lambda n: G_[f"egnn_{l}.{n}"]) if want_params else None
        hn = lay["h_out"]
        # node update: h' = tanh(z), hdot' = (1 - h'^2) zdot
        if dual:
            zb = (1.0 - hn * hn) * (hb - 2.0 * hn * lay["zd"] * hdb)
            zdb = (1.0 - hn * hn) * hdb
        else:
            zb = (1.0 - hn * hn) * hb
        if want_params:
            gp("w")[...] += zb.T @ lay["h"] + (zdb.T @ lay["hd"] if dual else 0.0)
            gp("u")[...] += zb.T @ lay["agg"] + (zdb.T @ lay["aggd"] if dual else 0.0)
            gp("b")[...] += zb.sum(axis=0)
        hb_in = zb @ p("w")
        aggb = zb @ p("u")
        if dual:
            hdb_in = zdb @ p("w")
            aggdb = zdb @ p("u")
        r, m, s = lay["r"], lay["m"], lay["s"]
        ci = cinv[dst][:, None]
        # coordinate update (layers 0..L-2): x' = x - ci sum r s,
        # xdot' = xdot - ci sum (rdot s + r sdot)
        rb = np.zeros_like(r)
        sb = np.zeros(r.shape[0])
        if dual:
            rdb = np.zeros_like(r)
            sdb = np.zeros(r.shape[0])
        if l < L - 1:
            xbd = xb[dst]
            rb += -ci * s[:, None] * xbd
            sb += -(ci[:, 0]) * (r * xbd).sum(axis=1)
            if dual:
                xdbd = xdb[dst]
                rd, sd = lay["rd"], lay["sd"]
                rdb += -ci * s[:, None] * xdbd
                sb += -(ci[:, 0]) * (rd * xdbd).sum(axis=1)
                rb += -ci * sd[:, None] * xdbd
                sdb += -(ci[:, 0]) * (r * xdbd).sum(axis=1)
        xb_in = xb.copy()
        xdb_in = xdb.copy() if dual else None
        # s = m . ux ; sdot = mdot . ux
        mb = aggb[dst] + sb[:, None] * p("ux")
        if want_params:
            gp("ux")[...] += sb @ m
        if dual:
            md = lay["md"]
            mdb = aggdb[dst] + sdb[:, None] * p("ux")
            if want_params:
                gp("ux")[...] += sdb @ md
            # mdot = (1 - m^2) predot
            predb = (1.0 - m * m) * mdb
            mb = mb - 2.0 * m * lay["pred"] * mdb
        preb = (1.0 - m * m) * mb
        # pre = A_dst + B_src + wd d2 + c ; predot = Ad_dst + Bd_src + wd d2dot
        d2b = preb @ p("wd")
        if want_params:
            gp("wd")[...] += lay["d2"] @ preb
            gp("c")[...] += preb.sum(axis=0)
        Ab = _sum_to(dst, preb, N)
        Bb = _sum_to(src, preb, N)
        rb += 2.0 * r * d2b[:, None]
        if dual:
            d2db = predb @ p("wd")
            if want_params:
                gp("wd")[...] += lay["d2d"] @ predb
            Adb = _sum_to(dst, predb, N)
            Bdb = _sum_to(src, predb, N)
            # d2dot = 2 r . rdot
            rb += 2.0 * lay["rd"] * d2db[:, None]
            rdb += 2.0 * r * d2db[:, None]
        # r = x_src - x_dst (+ shift), rdot = xdot_src - xdot_dst
        xb_in += _sum_to(src, rb, N) - _sum_to(dst, rb, N)
        if dual:
            xdb_in += _sum_to(src, rdb, N) - _sum_to(dst, rdb, N)
        # A = h wa^T, B = h wb^T (and the tangent rows)
        if want_params:
            gp("wa")[...] += Ab.T @ lay["h"] + (Adb.T @ lay["hd"] if dual else 0.0)
            gp("wb")[...] += Bb.T @ lay["h"] + (Bdb.T @ lay["hd"] if dual else 0.0)
        hb_in += Ab @ p("wa") + Bb @ p("wb")
        if dual:
            hdb_in += Adb @ p("wa") + Bdb @ p("wb")
        hb, xb = hb_in, xb_in
        if dual:
            hdb, xdb = hdb_in, xdb_in
    out = dict(x0=xb)
    if dual:
        out["xd0"] = xdb
    if want_params:
        np.add.at(G_["embedding"], b["z"] - 1, hb)  # model.py:564
        out["grad"] = np.concatenate([G_[n].ravel() for n, _ in param_shapes(cfg)])
    return out


def mtl_loss(e_pred, f_pred, e_true, f_true, n_per, aE, aF):
    """model.py:437-462"""
    r = (e_pred - e_true) / n_per
    et = float(np.abs(r).mean())
    ft = float(np.abs(f_pred - f_true).mean()) if f_true.size else 0.0
    return aE * et + aF * ft, et, ft, r


def loss_and_grad(cfg, flat, b):
    """(total, energy, force), flat gradient, (e_pred, f_pred)."""
    c = {}
    e_pred, f_pred = forces(cfg, flat, b, c)
    total, et, ft, r = mtl_loss(e_pred, f_pred, b["e_true"], b["f_true"], b["n_per"],
                                cfg["aE"], cfg["aF"])
    B, N = b["n_per"].shape[0], b["z"].shape[0]
    de = cfg["aE"] * np.sign(r) / (b["n_per"] * B)                      # model.py:511
    v = cfg["aF"] * np.sign(f_pred - b["f_true"]) / (3.0 * N)           # model.py:516
    # dL/dtheta = d/dtheta [sum de E - v . dE/dx0]: tangent forward from v,
    # one reverse pass over primal + tangent with seeds (de, -1)
    cd = {}
    forward(cfg, flat, b, tangent=v, cache=cd)
    g = _reverse(cfg, flat, b, cd, de, -1.0, want_params=True)
    return (total, et, ft), g["grad"], (e_pred, f_pred)


def batch_loss(cfg, flat, b):
    e_pred, f_pred = forces(cfg, flat, b)
    return mtl_loss(e_pred, f_pred, b["e_true"], b["f_true"], b["n_per"], cfg["aE"],
                    cfg["aF"])[0]
