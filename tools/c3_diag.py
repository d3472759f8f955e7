"""Where does float32 error enter at the C3 shape?  Runs the C3-golden batch
through the float64 kernels and the float32 kernels (tc3 / simt GEMM
engines) and prints the relative error of every layer's aggregation parts,
h_out, the head and e_pred / f_pred against float64.

    python tools/c3_diag.py"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import gfm_oracle as O  # noqa: E402
from oracle.make_c3_golden import SPEC, inputs  # noqa: E402
from paper_2406_12909_b200 import _lib, model as M  # noqa: E402

s = SPEC
recs = inputs()
cfg = M.ModelConfig(mpnn_kind=s["kind"], mpnn_layers=s["layers"], mpnn_width=s["hidden"],
                    fc_layers=s["fc_layers"], fc_width=s["fc_width"])
flat = O.init_flat(O.config(s["kind"], s["layers"], s["hidden"], s["fc_layers"], s["fc_width"]),
                   s["param_seed"])
B, n = len(recs), s["n_atoms"]
off = (np.arange(B + 1) * n).astype(np.int32)
dev = torch.device("cuda")
pos = torch.as_tensor(np.concatenate([r["pos"] for r in recs]), device=dev)
z = torch.as_tensor(np.concatenate([r["z"] for r in recs]).astype(np.int32), device=dev)
cells = torch.full((B, 3), s["box"], dtype=torch.float64, device=dev)


def run(dtype, mode):
    _lib.call("gfm_set_gemm_mode", mode)
    b = M.radius_batch(pos, z, torch.as_tensor(off, device=dev), off, s["rc"], s["max_nbr"],
                       cells, dtype=dtype, e_cap=B * n * s["max_nbr"])
    p = M.ModelParams.from_flat(cfg, flat, dtype=dtype)
    cache = {}
    e, f = M.forward_batch(p, b, cache)
    torch.cuda.synchronize()
    out = dict(e=e.double().cpu().numpy(), f=f.double().cpu().numpy())
    for l, lay in enumerate(cache["layers"]):
        out[f"agg{l}"] = lay["agg"].double().cpu().numpy()
        out[f"h{l + 1}"] = lay["h_out"].double().cpu().numpy()
        if lay["smean"] is not None:
            out[f"smean{l}"] = lay["smean"].double().cpu().numpy()
    for k, y in enumerate(cache["head_inputs"]):
        out[f"y{k}"] = y.double().cpu().numpy()
    _lib.call("gfm_set_gemm_mode", 1)
    return out


ref = run(torch.float64, 0)
H = s["hidden"]
for name, dt, mode in (("f32 tc3", torch.float32, 1), ("f32 simt", torch.float32, 0)):
    got = run(dt, mode)
    print(f"== {name}")
    for k in ref:
        a, b_ = got[k], ref[k]
        if k.startswith("agg"):
            for pi, pn in enumerate(("sum", "mean", "max", "std")):
                aa, bb = a[:, pi * H:(pi + 1) * H], b_[:, pi * H:(pi + 1) * H]
                sc = np.abs(bb).max()
                err = np.abs(aa - bb)
                print(f"{k}.{pn}: max abs {err.max():.3e} scale {sc:.3e} "
                      f"rel-to-scale {err.max() / sc:.3e}  zero-flips "
                      f"{int(((aa == 0) != (bb == 0)).sum())}")
        else:
            sc = np.abs(b_).max()
            err = np.abs(a - b_)
            rel = err / np.maximum(np.abs(b_), 1e-2 * sc)
            print(f"{k}: max abs {err.max():.3e} scale {sc:.3e} max rel(floor 1%) {rel.max():.3e}")
