"""Pin the EGNN restatement (oracle/egnn_oracle.py; no reference exists).

* forces == -dE/dx0 by central finite differences of the energy;
* dL/dtheta (reverse over the primal + tangent forward) == finite
  differences of the loss, with the reference's FD harness
  (test_gradients.py:27-108: kink-free targets, step 1e-4, rel 1e-5,
  floor 1e-4; fourth-order central differences);
* both == torch.autograd in float64 (F by autograd.grad(create_graph=True),
  dL/dtheta by double backward) to 1e-10 -- an independent implementation;
* E(3): energies invariant and forces equivariant under rotation +
  translation.
"""

import numpy as np
import pytest
import torch

from oracle import egnn_oracle as EG
from oracle import gfm_oracle as O


def _batch(seed, count=3, n=(3, 7), rc=2.5, box=5.0, max_nbr=None):
    recs = O.synthetic(count, n_atoms_range=n, box_length=box, rc=rc, seed=seed,
                       max_nbr=max_nbr)
    return O.pack(recs)


def _kink_free(cfg, flat, b, rng):
    e, f = EG.forces(cfg, flat, b)
    sign = lambda shape: np.where(rng.uniform(size=shape) < 0.5, -1.0, 1.0)
    b["e_true"] = e + (0.5 + rng.uniform(0, 0.5, e.shape)) * sign(e.shape) * b["n_per"]
    b["f_true"] = f + (0.3 + rng.uniform(0, 0.5, f.shape)) * sign(f.shape)
    return b


@pytest.mark.parametrize("seed", range(3))
def test_forces_are_minus_energy_gradient(seed):
    cfg = EG.config(layers=3, hidden=8, fc_layers=2, fc_width=6)
    flat = EG.init_flat(cfg, seed)
    b = _batch(seed)
    _, f = EG.forces(cfg, flat, b)
    h = 1e-5
    x0 = b["pos"].copy()
    fd = np.zeros_like(x0)
    for i in range(x0.shape[0]):
        for k in range(3):
            xp, xm = x0.copy(), x0.copy()
            xp[i, k] += h
            xm[i, k] -= h
            fd[i, k] = -(EG.energy_total(cfg, flat, b, xp) - EG.energy_total(cfg, flat, b, xm)) / (2 * h)
    np.testing.assert_allclose(f, fd, rtol=1e-6, atol=1e-8)


@pytest.mark.parametrize("seed", range(6))
def test_parameter_gradient_matches_finite_differences(seed):
    cfg = EG.config(layers=2 + seed % 2, hidden=3, fc_layers=2, fc_width=2)
    flat = EG.init_flat(cfg, 100 + seed)
    rng = np.random.default_rng(seed)
    b = _kink_free(cfg, flat, _batch(seed, max_nbr=3 if seed % 3 == 0 else None), rng)
    _, analytic, _ = EG.loss_and_grad(cfg, flat, b)
    # fourth-order central differences (step 1e-4): the loss holds F = -dE/dx,
    # so its third derivatives are larger than the MPNN's and the plain
    # central difference's h^2 term reaches ~1e-5 on a few coordinates
    step = 1e-4
    numeric = np.zeros_like(flat)

    def at(k, d):
        q = flat.copy()
        q[k] += d
        return EG.batch_loss(cfg, q, b)

    for k in range(flat.size):
        numeric[k] = (8 * (at(k, step) - at(k, -step)) - (at(k, 2 * step) - at(k, -2 * step))) \
            / (12 * step)
    rel = np.abs(analytic - numeric) / np.maximum(np.maximum(np.abs(analytic), np.abs(numeric)),
                                                  1e-4)
    assert rel.max() < 1e-5, f"worst rel err {rel.max():.3e} at {int(rel.argmax())}"


def _torch_model(cfg, flat, b):
    """the same model in torch float64: F by autograd.grad(create_graph=True)"""
    P = {k: torch.tensor(v, dtype=torch.float64, requires_grad=True)
         for k, v in EG.unflatten(cfg, flat.copy()).items()}
    src, dst = torch.as_tensor(b["src"]), torch.as_tensor(b["dst"])
    N = b["z"].shape[0]
    x0 = torch.tensor(b["pos"], dtype=torch.float64, requires_grad=True)
    shift = torch.as_tensor(b["dx"] - (b["pos"][b["src"]] - b["pos"][b["dst"]]))
    cinv = torch.as_tensor(1.0 / np.maximum(b["deg"], 1))
    h = P["embedding"][torch.as_tensor(b["z"] - 1)]
    x = x0
    for l in range(cfg["L"]):
        p = lambda n: P[f"egnn_{l}.{n}"]
        A, B = h @ p("wa").T, h @ p("wb").T
        r = x[src] - x[dst] + shift
        d2 = (r * r).sum(1)
        m = torch.tanh(A[dst] + B[src] + d2[:, None] * p("wd") + p("c"))
        s = m @ p("ux")
        agg = torch.zeros(N, cfg["H"], dtype=torch.float64).index_add(0, dst, m)
        if l < cfg["L"] - 1:
            x = x - cinv[:, None] * torch.zeros(N, 3, dtype=torch.float64).index_add(
                0, dst, r * s[:, None])
        h = torch.tanh(h @ p("w").T + agg @ p("u").T + p("b"))
    y = h
    F = cfg["F"]
    for f in range(F - 1):
        y = torch.tanh(y @ P[f"head_{f}.w"].T + P[f"head_{f}.b"])
    node_e = (y @ P[f"head_{F - 1}.w"].T)[:, 0] + P[f"head_{F - 1}.b"][0]
    gn = torch.as_tensor(np.repeat(np.arange(len(b["offsets"]) - 1), np.diff(b["offsets"])))
    e = torch.zeros(len(b["offsets"]) - 1, dtype=torch.float64).index_add(0, gn, node_e)
    (gx,) = torch.autograd.grad(e.sum(), x0, create_graph=True)
    f = -gx
    n = torch.as_tensor(b["n_per"], dtype=torch.float64)
    loss = cfg["aE"] * ((e - torch.as_tensor(b["e_true"])) / n).abs().mean() + \
        cfg["aF"] * (f - torch.as_tensor(b["f_true"])).abs().mean()
    keys = [k for k, _ in EG.param_shapes(cfg)]
    # the last layer's coordinate weights feed nothing (no update after it)
    grads = torch.autograd.grad(loss, [P[k] for k in keys], allow_unused=True)
    return (e.detach().numpy(), f.detach().numpy(), float(loss),
            np.concatenate([(torch.zeros_like(P[k]) if g is None else g).detach().numpy().ravel()
                            for k, g in zip(keys, grads)]))


@pytest.mark.parametrize("seed", range(3))
def test_matches_torch_autograd_double_backward(seed):
    cfg = EG.config(layers=3, hidden=16, fc_layers=3, fc_width=12)
    flat = EG.init_flat(cfg, seed)
    rng = np.random.default_rng(seed)
    b = _kink_free(cfg, flat, _batch(seed, count=4, n=(4, 12), max_nbr=6), rng)
    (tot, _, _), grad, (e, f) = EG.loss_and_grad(cfg, flat, b)
    te, tf, tl, tg = _torch_model(cfg, flat, b)
    np.testing.assert_allclose(e, te, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(f, tf, rtol=1e-10, atol=1e-12)
    assert abs(tot - tl) <= 1e-12 * abs(tl)
    np.testing.assert_allclose(grad, tg, rtol=1e-9, atol=1e-12)


def test_e3_invariance_and_equivariance():
    cfg = EG.config(layers=3, hidden=16, fc_layers=2, fc_width=16)
    flat = EG.init_flat(cfg, 3)
    b = _batch(5, count=3, n=(5, 9))
    e, f = EG.forces(cfg, flat, b)
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    t = rng.normal(size=3)
    b2 = dict(b)
    b2["pos"] = b["pos"] @ Q.T + t
    b2["dx"] = b["dx"] @ Q.T
    e2, f2 = EG.forces(cfg, flat, b2)
    np.testing.assert_allclose(e2, e, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(f2, f @ Q.T, rtol=1e-9, atol=1e-12)
