"""Golden vectors for the GFM-scale (C3-shape) whole-model parity test.

TEST INFRASTRUCTURE ONLY.  Runs the float64 oracle (``gfm_oracle``) once at
the C3 model shape -- pna-agg, 6 layers, hidden 512, fc 2 x 512, periodic
100-atom crystals in a 12 A cell, rc 5 A, max 32 neighbours -- on 84
structures (N = 8,400 > 8,192, so the GPU's tensor-core GEMMs run several
128-row tiles per CTA and split their weight-gradient K dimension), and
writes ``tests/golden/c3_shape.npz``:

* the inputs' checksum (the test regenerates them with ``O.synthetic``);
* kink-free targets: every force residual >= 0.3 and every per-atom energy
  residual >= 0.5 from the oracle's own prediction (test_gradients.py:47-60);
* e_pred (B), f_pred (N, 3), the loss triple, and the gradient at a fixed
  subset of coordinates (all of the embedding, biases, force head u / c and
  energy head output; every 7th entry of the 512 x 512 head / force
  matrices; every 97th of the 6 x (W, U) layer matrices) -- the full 8.45M
  float64 gradient would be 68 MB.

About 5 minutes and 16 GB of RAM on 8 cores:
``python oracle/make_c3_golden.py``.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import gfm_oracle as O  # noqa: E402

SPEC = dict(count=84, n_atoms=100, box=12.0, rc=5.0, max_nbr=32, seed=5, kind="pna-agg",
            layers=6, hidden=512, fc_layers=2, fc_width=512, param_seed=0, target_seed=11)


def inputs():
    s = SPEC
    return O.synthetic(s["count"], n_atoms_range=(s["n_atoms"], s["n_atoms"]),
                       box_length=s["box"], rc=s["rc"], seed=s["seed"], max_nbr=s["max_nbr"],
                       periodic=True)


def checksum(recs):
    return np.array([float(np.sum([r["pos"].sum() for r in recs])),
                     float(sum(int(r["edges"].shape[0]) for r in recs)),
                     float(np.sum([(r["edges"].astype(np.float64) * [1.0, 3.0]).sum()
                                   for r in recs]))])


def grad_index(cfg):
    """fixed subset of flat gradient coordinates"""
    idx, off = [], 0
    for name, shape in O.param_shapes(cfg):
        n = int(np.prod(shape))
        if name.startswith("layer_") and not name.endswith(".b"):
            step = 97
        elif n >= 512 * 512:
            step = 7
        else:
            step = 1
        idx.append(off + np.arange(0, n, step))
        off += n
    return np.concatenate(idx).astype(np.int64)


def main():
    s = SPEC
    t0 = time.time()
    recs = inputs()
    cfg = O.config(s["kind"], s["layers"], s["hidden"], s["fc_layers"], s["fc_width"])
    flat = O.init_flat(cfg, s["param_seed"])
    b = O.pack(recs)
    e0, f0 = O.forward(cfg, flat, b)
    rng = np.random.default_rng(s["target_seed"])
    sign = lambda shape: np.where(rng.uniform(size=shape) < 0.5, -1.0, 1.0)
    e_true = e0 + (0.5 + rng.uniform(0.0, 0.5, e0.shape)) * sign(e0.shape) * b["n_per"]
    f_true = f0 + (0.3 + rng.uniform(0.0, 0.5, f0.shape)) * sign(f0.shape)
    b["e_true"], b["f_true"] = e_true, f_true
    (tot, et, ft), grad, (e, f) = O.loss_and_grad(cfg, flat, b)
    idx = grad_index(cfg)
    out = os.path.join(ROOT, "tests", "golden", "c3_shape.npz")
    np.savez_compressed(out, checksum=checksum(recs), e_true=e_true, f_true=f_true, e_pred=e,
                        f_pred=f, loss=np.array([tot, et, ft]), grad_idx=idx, grad_val=grad[idx],
                        n_params=np.array(flat.shape[0]), n_edges=np.array(b["src"].shape[0]),
                        numpy_version=np.array(np.__version__))
    print(f"wrote {out}: N={b['z'].shape[0]} E={b['src'].shape[0]} P={flat.shape[0]} "
          f"coords={idx.shape[0]} loss={tot:.6f} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
