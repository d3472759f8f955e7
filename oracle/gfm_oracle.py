"""float64 numpy restatement of the gfmkit training hot path (TEST ORACLE).

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  Every function cites
the reference code it restates (paths relative to
``/root/reference/pkg/src/gfmkit/``).  The arithmetic lives in numpy (the
reference pins ``numpy>=1.24``, ``pkg/pyproject.toml:11``; this image has
numpy 2.3.5), so the restatement uses the same numpy primitives where the
reference's floating-point order matters (``add.reduceat`` segment sums,
``add.at`` scatters, ``maximum.reduceat``).

Pinned (checked bit-for-bit or to 1e-12 against vectors produced by the
reference itself, ``tests/golden/``): mean/sum/max MPNN forward, L1 MTL loss,
hand-written backward, Adam/SGD, epoch schedule, ordered allreduce, and
uncapped non-periodic cutoff edges + synthetic generator.

Not pinnable to reference outputs (the reference has no implementation;
restated from its conventions): ``std-agg``, ``pna-agg`` (= concat[sum,
mean, max, std], U is H x 4H), the per-destination neighbour cap, and
minimum-image periodic edges.  Their gradients are pinned by central finite
differences with the reference's own harness (``tests/test_oracle_fd.py``,
a port of test_gradients.py:27-108: 20 kink-free batches, step 1e-4,
rel 1e-5, floor 1e-4), ``std-agg`` against ``numpy.std`` and ``pna-agg`` as
the exact concatenation of the golden-pinned sum/mean/max blocks.

Data model: a *record* is a dict with keys ``z`` (u8 n), ``pos`` (f64 n x 3),
``edges`` (u32 m x 2, columns [src, dst]), ``energy`` (f64), ``forces``
(f64 n x 3) and optionally ``shift`` (f64 m x 3, periodic image offset added
to ``pos[src] - pos[dst]``).
"""

from __future__ import annotations

import math

import numpy as np

MAX_Z = 118  # records.py:33
KINDS = ("mean-agg", "sum-agg", "max-agg", "std-agg", "pna-agg")
PARTS = {  # model.py:39 (first three); std/pna are restated extensions
    "mean-agg": ("mean",),
    "sum-agg": ("sum",),
    "max-agg": ("max",),
    "std-agg": ("std",),
    "pna-agg": ("sum", "mean", "max", "std"),
}
STD_CLAMP = 1e-5  # PyG StdAggregation convention: clamp(var, 1e-5), sqrt, <= sqrt(1e-5) -> 0


# ---------------------------------------------------------------------------
# Configuration and flat parameter layout            (model.py:42-187)
# ---------------------------------------------------------------------------


def config(kind="mean-agg", layers=3, hidden=50, fc_layers=2, fc_width=50,
           alpha_energy=1.0, alpha_forces=100.0):
    """Plain-dict model configuration (ModelConfig, model.py:42-69)."""
    if kind not in KINDS:
        raise ValueError(kind)
    if fc_layers < 2:
        raise ValueError("fc_layers must be >= 2")
    return dict(kind=kind, L=int(layers), H=int(hidden), F=int(fc_layers),
                G=int(fc_width), aE=float(alpha_energy), aF=float(alpha_forces))


def param_shapes(cfg):
    """(name, shape) in the canonical flat order (ModelParams.arrays,
    model.py:120-132); U widens to (H, kH) for multi-aggregator kinds."""
    H, G, k = cfg["H"], cfg["G"], len(PARTS[cfg["kind"]])
    out = [("embedding", (MAX_Z, H))]
    for l in range(cfg["L"]):
        out += [(f"layer_{l}.w", (H, H)), (f"layer_{l}.u", (H, k * H)),
                (f"layer_{l}.b", (H,))]
    ws = [(G, H)] + [(G, G)] * (cfg["F"] - 2) + [(1, G)]
    bs = [(G,)] * (cfg["F"] - 1) + [(1,)]
    for f in range(cfg["F"]):
        out += [(f"head_{f}.w", ws[f]), (f"head_{f}.b", bs[f])]
    out += [("force.v", (H, H)), ("force.c", (H,)), ("force.u", (H,))]
    return out


def n_params(cfg):
    """count_params (model.py:89-97), generalised to U of width kH."""
    return sum(int(np.prod(s)) for _, s in param_shapes(cfg))


def unflatten(cfg, flat):
    """name -> view into ``flat`` (ModelParams.from_flat, model.py:164-175)."""
    flat = np.asarray(flat, dtype=np.float64)
    if flat.shape != (n_params(cfg),):
        raise ValueError(f"flat has {flat.shape}, model needs ({n_params(cfg)},)")
    views, off = {}, 0
    for name, shape in param_shapes(cfg):
        size = int(np.prod(shape))
        views[name] = flat[off:off + size].reshape(shape)
        off += size
    return views


def init_flat(cfg, seed=0):
    """init_params (model.py:178-187): uniform(+-1/sqrt(H)) drawn in flat
    order from default_rng(seed), skipping names ending in .b / .c."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(cfg["H"])
    flat = np.zeros(n_params(cfg))
    views = unflatten(cfg, flat)
    for name, shape in param_shapes(cfg):
        if name.endswith(".b") or name.endswith(".c"):
            continue
        views[name][...] = rng.uniform(-bound, bound, size=shape)
    return flat


# ---------------------------------------------------------------------------
# Neighbour lists and synthetic data                  (preprocess.py:41-153)
# ---------------------------------------------------------------------------


def _pair_geometry(pos, cell):
    """delta[i, j] = pos[i] - pos[j] (+ minimum-image shift when ``cell``)."""
    delta = pos[:, None, :] - pos[None, :, :]
    shift = None
    if cell is not None:
        L = np.asarray(cell, dtype=np.float64).reshape(3)
        shift = -L * np.rint(delta / L)
        delta = delta + shift
    dist = np.sqrt((delta ** 2).sum(axis=2))  # ((dx^2 + dy^2) + dz^2), no FMA
    return dist, shift


def cutoff_edges(pos, rc, max_nbr=None, cell=None):
    """build_cutoff_edges (preprocess.py:90-104): every ordered pair i != j
    with |x_i - x_j| <= rc, emitted row-major as [src=i, dst=j].

    Extensions (UNPINNED): ``max_nbr`` keeps, per destination j, the
    ``max_nbr`` nearest sources by (float64 distance, then source index);
    ``cell`` (orthorhombic box lengths) applies the minimum-image convention
    (requires rc < min(cell)/2).  Returns (edges u32 m x 2, shift f64 m x 3).
    """
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
    n = pos.shape[0]
    if cell is not None and rc >= 0.5 * float(np.min(cell)):
        raise ValueError("minimum image needs rc < min(cell)/2")
    if n < 2:
        return np.zeros((0, 2), np.uint32), np.zeros((0, 3))
    dist, shift = _pair_geometry(pos, cell)
    mask = dist <= rc
    np.fill_diagonal(mask, False)
    if max_nbr is not None:
        for j in range(n):
            cand = np.nonzero(mask[:, j])[0]
            if cand.size > max_nbr:
                keep = cand[np.lexsort((cand, dist[cand, j]))[:max_nbr]]
                mask[:, j] = False
                mask[keep, j] = True
    edges = np.argwhere(mask)
    if shift is None:
        sh = np.zeros((edges.shape[0], 3))
    else:
        sh = shift[edges[:, 0], edges[:, 1]]
    return edges.astype(np.uint32), sh


def toy_energy_forces(z, pos, edges, d0=1.0):
    """ToyPotential.energy/forces (preprocess.py:41-87): C*_Z = -0.1 Z plus a
    harmonic term over src < dst pairs; forces are the exact -grad."""
    z = np.asarray(z, dtype=np.int64)
    e = float((-0.1 * np.arange(1, MAX_Z + 1, dtype=np.float64))[z - 1].sum())
    f = np.zeros_like(pos)
    for s, d in np.asarray(edges, dtype=np.int64).reshape(-1, 2):
        if s < d:
            r = float(np.linalg.norm(pos[s] - pos[d]))
            e += (r - d0) ** 2
            if r >= 1e-12:
                g = 2.0 * (r - d0) * (pos[s] - pos[d]) / r
                f[s] -= g
                f[d] += g
    return e, f


def synthetic(count, n_atoms_range=(4, 12), elements=None, box_length=6.0,
              rc=2.0, seed=0, max_nbr=None, periodic=False):
    """generate_synthetic (preprocess.py:107-153): identical rng call
    sequence (integers, choice, uniform per structure) so the same seed
    yields the same structures.  ``max_nbr`` / ``periodic`` are extensions:
    labels always come from the uncapped, non-periodic toy potential."""
    lo, hi = n_atoms_range
    elements = elements or {1: 1.0, 6: 1.0, 8: 1.0}
    zs = np.array(sorted(elements), dtype=np.int64)
    w = np.array([elements[int(z)] for z in zs], dtype=np.float64)
    probs = w / w.sum()
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(count):
        n = int(rng.integers(lo, hi + 1))
        z = zs[rng.choice(zs.size, size=n, p=probs)].astype(np.uint8)
        pos = rng.uniform(0.0, box_length, size=(n, 3))
        full, _ = cutoff_edges(pos, rc)
        energy, forces = toy_energy_forces(z, pos, full)
        cell = (box_length,) * 3 if periodic else None
        if max_nbr is None and cell is None:
            edges, shift = full, np.zeros((full.shape[0], 3))
        else:
            edges, shift = cutoff_edges(pos, rc, max_nbr=max_nbr, cell=cell)
        out.append(dict(z=z, pos=pos, edges=edges, shift=shift,
                        energy=float(energy), forces=forces))
    return out


# ---------------------------------------------------------------------------
# Batch packing                                        (model.py:195-285)
# ---------------------------------------------------------------------------


def pack(records):
    """make_batch (model.py:234-285) with segments expressed as CSR.

    Keys: z, pos, src, dst (original edge order), w, dx, offsets, n_per,
    gnode, e_true, f_true, order (stable dst sort), rowptr (N+1), deg.
    """
    if not records:
        raise ValueError("cannot build a batch from zero records")
    n_per = np.array([r["z"].shape[0] for r in records], dtype=np.int64)
    offsets = np.concatenate([[0], np.cumsum(n_per)])
    z = np.concatenate([np.asarray(r["z"], np.int64) for r in records])
    pos = np.concatenate([np.asarray(r["pos"], np.float64) for r in records])
    src = np.concatenate([np.asarray(r["edges"], np.int64)[:, 0] + offsets[g]
                          for g, r in enumerate(records)])
    dst = np.concatenate([np.asarray(r["edges"], np.int64)[:, 1] + offsets[g]
                          for g, r in enumerate(records)])
    shift = np.concatenate([np.asarray(r.get("shift", np.zeros((len(r["edges"]), 3))),
                                       np.float64).reshape(-1, 3) for r in records])
    dx = pos[src] - pos[dst]
    if np.any(shift):
        dx = dx + shift
    w = 1.0 / (1.0 + np.sqrt((dx ** 2).sum(axis=1)))
    order = np.argsort(dst, kind="stable")
    deg = np.bincount(dst, minlength=z.shape[0]).astype(np.int64)
    rowptr = np.concatenate([[0], np.cumsum(deg)])
    return dict(z=z, pos=pos, src=src, dst=dst, w=w, dx=dx, offsets=offsets,
                n_per=n_per, gnode=np.repeat(np.arange(len(records)), n_per),
                e_true=np.array([r["energy"] for r in records], np.float64),
                f_true=np.concatenate([np.asarray(r["forces"], np.float64)
                                       for r in records]),
                order=order, rowptr=rowptr, deg=deg)


# ---------------------------------------------------------------------------
# Aggregation                                          (model.py:293-341)
# ---------------------------------------------------------------------------


def _segments(b):
    """Non-empty dst segments of the sorted edge list (model.py:260-266)."""
    starts = b["rowptr"][:-1]
    nz = b["deg"] > 0
    return np.nonzero(nz)[0], starts[nz]


def aggregate(b, msg, kind, cache=None):
    """_aggregate (model.py:293-322) for one or several parts.  Output is
    concat over PARTS[kind] of (N, H) blocks.  Sums use numpy's reduceat
    order (m[first] + pairwise(rest)); max keeps the FIRST sorted-edge
    argmax per (segment, column); empty neighbourhoods give 0."""
    N, H = b["z"].shape[0], msg.shape[1]
    parts = PARTS[kind]
    out = np.zeros((N, len(parts) * H))
    if msg.shape[0] == 0:
        if cache is not None:
            cache["argmax"] = np.zeros((0, H), np.int64)
        return out
    seg_dst, seg_start = _segments(b)
    ms = msg[b["order"]]
    deg = b["deg"][seg_dst][:, None].astype(np.float64)
    s1 = np.add.reduceat(ms, seg_start, axis=0)
    for p, part in enumerate(parts):
        blk = out[:, p * H:(p + 1) * H]
        if part == "sum":
            blk[seg_dst] = s1
        elif part == "mean":
            blk[seg_dst] = s1 / deg
        elif part == "max":
            mx = np.maximum.reduceat(ms, seg_start, axis=0)
            blk[seg_dst] = mx
            if cache is not None:
                e = ms.shape[0]
                lens = np.diff(np.concatenate([seg_start, [e]]))
                hit = ms == np.repeat(mx, lens, axis=0)
                pos_ = np.where(hit, np.arange(e)[:, None], e)
                cache["argmax"] = np.minimum.reduceat(pos_, seg_start, axis=0)
                cache["seg_dst"] = seg_dst
        elif part == "std":
            s2 = np.add.reduceat(ms * ms, seg_start, axis=0)
            mean = s1 / deg
            var = s2 / deg - mean * mean
            std = np.where(var > STD_CLAMP, np.sqrt(np.maximum(var, STD_CLAMP)), 0.0)
            blk[seg_dst] = std
            if cache is not None:
                full_mean = np.zeros((N, H))
                full_std = np.zeros((N, H))
                full_mean[seg_dst] = mean
                full_std[seg_dst] = std
                cache["std_mean"], cache["std_val"] = full_mean, full_std
    return out


def aggregate_backward(b, dagg, msg, kind, cache):
    """_aggregate_backward (model.py:325-341): d agg -> d msg (E, H) in the
    ORIGINAL edge order."""
    E = b["src"].shape[0]
    parts = PARTS[kind]
    H = dagg.shape[1] // len(parts)
    dmsg = np.zeros((E, H))
    if E == 0:
        return dmsg
    dst = b["dst"]
    for p, part in enumerate(parts):
        d = dagg[:, p * H:(p + 1) * H]
        if part == "sum":
            dmsg += d[dst]
        elif part == "mean":
            dmsg += d[dst] / b["deg"][dst][:, None]
        elif part == "max":
            am = cache["argmax"]
            routed = np.zeros((E, H))
            cols = np.tile(np.arange(H), am.shape[0])
            np.add.at(routed, (am.ravel(), cols), d[cache["seg_dst"]].ravel())
            back = np.zeros((E, H))
            back[b["order"]] = routed
            dmsg += back
        elif part == "std":
            std = cache["std_val"][dst]
            safe = np.where(std > 0, std, 1.0)
            coef = np.where(std > 0, d[dst] / (b["deg"][dst][:, None] * safe), 0.0)
            dmsg += coef * (msg - cache["std_mean"][dst])
    return dmsg


# ---------------------------------------------------------------------------
# Forward, loss, backward                              (model.py:344-565)
# ---------------------------------------------------------------------------


def forward(cfg, flat, b, cache=None):
    """forward_batch (model.py:344-400): returns (e_pred (B,), f_pred (N,3))."""
    P = unflatten(cfg, flat)
    h = P["embedding"][b["z"] - 1]
    layers = []
    for l in range(cfg["L"]):
        msg = h[b["src"]] * b["w"][:, None]
        ac = {} if cache is not None else None
        agg = aggregate(b, msg, cfg["kind"], ac)
        h_out = np.tanh(h @ P[f"layer_{l}.w"].T + agg @ P[f"layer_{l}.u"].T
                        + P[f"layer_{l}.b"])
        # msg is recomputed by the backward (h_in[src] * w) instead of kept:
        # at GFM scale every cached E x H float64 array is ~1 GB
        layers.append(dict(h_in=h, agg=agg, h_out=h_out, ac=ac))
        del msg
        h = h_out
    ys = [h]
    y = h
    for f in range(cfg["F"] - 1):
        y = np.tanh(y @ P[f"head_{f}.w"].T + P[f"head_{f}.b"])
        ys.append(y)
    node_e = y @ P[f"head_{cfg['F'] - 1}.w"].T + P[f"head_{cfg['F'] - 1}.b"]
    e_pred = np.add.reduceat(node_e[:, 0], b["offsets"][:-1])
    N = h.shape[0]
    f_pred = np.zeros((N, 3))
    pair = h[b["dst"]] + h[b["src"]]
    t = np.tanh(pair @ P["force.v"].T + P["force.c"])
    m = t @ P["force.u"]
    if b["src"].size:
        np.add.at(f_pred, b["dst"], m[:, None] * b["dx"])
    if cache is not None:
        cache.update(layers=layers, h=h, ys=ys, pair=pair, t=t, m=m)
    return e_pred, f_pred


def mtl_loss(e_pred, f_pred, e_true, f_true, n_per, aE=1.0, aF=100.0):
    """mtl_loss (model.py:437-462): returns (total, energy, force, residuals)."""
    r = (np.asarray(e_pred, np.float64) - e_true) / np.asarray(n_per, np.float64)
    et = float(np.abs(r).mean())
    ft = float(np.abs(np.asarray(f_pred) - f_true).mean()) if f_true.size else 0.0
    return aE * et + aF * ft, et, ft, r


def loss_and_grad(cfg, flat, b):
    """loss_and_grad (model.py:483-565): (total, energy, force), flat grad."""
    cache = {}
    e_pred, f_pred = forward(cfg, flat, b, cache)
    total, et, ft, r = mtl_loss(e_pred, f_pred, b["e_true"], b["f_true"],
                                b["n_per"], cfg["aE"], cfg["aF"])
    P = unflatten(cfg, flat)
    grad = np.zeros_like(flat)
    Gd = unflatten(cfg, grad)
    B, N = b["n_per"].shape[0], b["z"].shape[0]
    de = cfg["aE"] * np.sign(r) / (b["n_per"] * B)
    df = cfg["aF"] * np.sign(f_pred - b["f_true"]) / (3.0 * N)

    # energy head (model.py:520-533)
    ys = cache["ys"]
    F = cfg["F"]
    ds = de[b["gnode"]][:, None]
    Gd[f"head_{F - 1}.w"][...] += ds.T @ ys[-1]
    Gd[f"head_{F - 1}.b"][...] += ds.sum(axis=0)
    dy = ds @ P[f"head_{F - 1}.w"]
    for f in range(F - 2, -1, -1):
        dz = dy * (1.0 - ys[f + 1] ** 2)
        Gd[f"head_{f}.w"][...] += dz.T @ ys[f]
        Gd[f"head_{f}.b"][...] += dz.sum(axis=0)
        dy = dz @ P[f"head_{f}.w"]
    dh = dy

    # force head (model.py:535-547)
    if b["src"].size:
        dm = (df[b["dst"]] * b["dx"]).sum(axis=1)
        t = cache["t"]
        Gd["force.u"][...] += t.T @ dm
        dpre = dm[:, None] * P["force.u"][None, :] * (1.0 - t ** 2)
        Gd["force.v"][...] += dpre.T @ cache["pair"]
        Gd["force.c"][...] += dpre.sum(axis=0)
        dpair = dpre @ P["force.v"]
        np.add.at(dh, b["dst"], dpair)
        np.add.at(dh, b["src"], dpair)

    # message-passing layers (model.py:549-562)
    for l in range(cfg["L"] - 1, -1, -1):
        lay = cache["layers"][l]
        dz = dh * (1.0 - lay["h_out"] ** 2)
        Gd[f"layer_{l}.b"][...] += dz.sum(axis=0)
        Gd[f"layer_{l}.w"][...] += dz.T @ lay["h_in"]
        Gd[f"layer_{l}.u"][...] += dz.T @ lay["agg"]
        dh_in = dz @ P[f"layer_{l}.w"]
        dagg = dz @ P[f"layer_{l}.u"]
        msg = lay["h_in"][b["src"]] * b["w"][:, None]
        dmsg = aggregate_backward(b, dagg, msg, cfg["kind"], lay["ac"])
        del msg
        if b["src"].size:
            np.add.at(dh_in, b["src"], dmsg * b["w"][:, None])
        dh = dh_in
    np.add.at(Gd["embedding"], b["z"] - 1, dh)  # model.py:564
    return (total, et, ft), grad, (e_pred, f_pred)


def batch_loss(cfg, flat, b):
    e_pred, f_pred = forward(cfg, flat, b)
    return mtl_loss(e_pred, f_pred, b["e_true"], b["f_true"], b["n_per"],
                    cfg["aE"], cfg["aF"])[0]


# ---------------------------------------------------------------------------
# Optimiser, schedule, collective                      (train.py, ddstore.py, comm.py)
# ---------------------------------------------------------------------------


def adam(flat, grad, m, v, t, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
    """apply_update, adam branch (train.py:96-108); returns (new, m, v, t)."""
    t += 1
    m = b1 * m + (1.0 - b1) * grad
    v = b2 * v + (1.0 - b2) * grad * grad
    m_hat = m / (1.0 - b1 ** t)
    v_hat = v / (1.0 - b2 ** t)
    return flat - lr * m_hat / (np.sqrt(v_hat) + eps), m, v, t


def sgd(flat, grad, lr):
    """apply_update, sgd branch (train.py:102-103)."""
    return flat - lr * grad


def schedule(n_samples, n_ranks, batch_size, seed, epoch):
    """epoch_permutation + epoch_schedule (ddstore.py:515-543): permutation
    index k goes to rank k mod P, each rank's stream chunked by batch_size."""
    perm = np.random.default_rng([int(seed), int(epoch)]).permutation(n_samples)
    return [[perm[r::n_ranks][i:i + batch_size]
             for i in range(0, perm[r::n_ranks].shape[0], batch_size)]
            for r in range(n_ranks)]


def ordered_allreduce_sum(vecs):
    """StarComm._allreduce (comm.py:124-151): sum in ascending rank order."""
    total = np.array(vecs[0], dtype=np.float64, copy=True)
    for v in vecs[1:]:
        total += v
    return total


def train_step_contribution(cfg, flat, b):
    """One rank's allreduce payload (train.py:252-259): [grad | loss | 1]."""
    (total, _, _), grad, _ = loss_and_grad(cfg, flat, b)
    return np.concatenate([grad, [total, 1.0]])


def numpy_pairwise_sum(a):
    """numpy's pairwise_sum for a strided double run (n<8 sequential from
    0.0; n<=128 eight accumulators; else split at n/2 rounded down to a
    multiple of 8).  Used by tests to document the order the fp64 GPU
    aggregation reproduces; reduceat(seg) == seg[0] + pairwise(seg[1:])."""
    n = len(a)
    if n < 8:
        r = 0.0
        for x in a:
            r += x
        return r
    if n <= 128:
        r = [a[j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += a[i + j]
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += a[i]
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return numpy_pairwise_sum(a[:n2]) + numpy_pairwise_sum(a[n2:])


def gflops_per_step(cfg, n_nodes, n_edges):
    """Algorithmic GEMM work of one training step (fwd + bwd), for reports."""
    H, G, k = cfg["H"], cfg["G"], len(PARTS[cfg["kind"]])
    node = 2.0 * n_nodes * (1 + k) * H * H * cfg["L"] * 3
    force = 2.0 * n_edges * H * H * 4
    head = 2.0 * n_nodes * H * G * 3
    return (node + force + head) / 1e9


__all__ = [n for n in dir() if not n.startswith("_")] + ["math"]


# ---------------------------------------------------------------------------
# Ensemble spread                                      (ensemble.py:121-186)
# ---------------------------------------------------------------------------


def population_sigma(stack, axis=0):
    """ensemble.py:121-130: std with ddof=0, exactly 0 where members agree."""
    arr = np.asarray(stack, dtype=np.float64)
    spread = arr.max(axis=axis) - arr.min(axis=axis)
    return np.where(spread == 0.0, 0.0, np.std(arr, axis=axis, ddof=0))


def reduce_force_sigma(sigma_comp, offsets, how="max"):
    """ensemble.py:133-148: per-structure max | mean | rms of the (n, 3)
    component spreads."""
    out = np.zeros(len(offsets) - 1)
    for g in range(out.shape[0]):
        blk = sigma_comp[offsets[g]:offsets[g + 1]]
        out[g] = (blk.max() if how == "max" else blk.mean() if how == "mean"
                  else np.sqrt(np.mean(blk ** 2)))
    return out


def ensemble_predict(members, records, how="max"):
    """ensemble.py:159-186; ``members`` = [(cfg dict, flat)].  Checked
    bit-identical (0.0 max diff, all three reductions) against the
    reference's ensemble_predict on synthetic(6, seed=9), 3 members."""
    b = pack(records)
    outs = [forward(cfg, flat, b) for cfg, flat in members]
    e = np.stack([o[0] for o in outs])
    f = np.stack([o[1] for o in outs])
    return (e.mean(axis=0), population_sigma(e),
            reduce_force_sigma(population_sigma(f), b["offsets"], how))
