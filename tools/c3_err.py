"""Error survey of the float32 engines at the C3 shape against the oracle
golden (tests/golden/c3_shape.npz): per output / gradient array, the max
elementwise relative error with the denominator floored at 1e-2 and 1e-3 of
the array's max, and the 99.9th percentile.

    python tools/c3_err.py [tc3,mixed,tc1,simt]"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from conftest import golden  # noqa: E402
from oracle.make_c3_golden import SPEC, inputs  # noqa: E402
from paper_2406_12909_b200 import _lib, model as M  # noqa: E402
from test_gpu_c3_fd import _c3_step  # noqa: E402
from test_gpu_parity import cfg_of  # noqa: E402


def stats(got, want):
    sc = max(float(np.abs(want).max()), 1e-30)
    out = []
    for fl in (1e-2, 1e-3):
        err = np.abs(got - want) / np.maximum(np.abs(want), fl * sc)
        out.append(err.max())
    err = np.abs(got - want) / np.maximum(np.abs(want), 1e-2 * sc)
    out.append(np.quantile(err, 0.999))
    return out


g = golden("c3_shape.npz")
recs = inputs()
s = SPEC
cfg = cfg_of(s["kind"], s["layers"], s["hidden"], s["fc_layers"], s["fc_width"])
MODES = {"simt": 0, "tc3": 1, "tc1": 2, "mixed": 3}
names = (sys.argv[1] if len(sys.argv) > 1 else "tc3,mixed,simt").split(",")
summary = {}
for name in names:
    mode = MODES[name]
    _lib.call("gfm_set_gemm_mode", mode)
    worst = [0.0, 0.0]
    loss, grad, e, f = _c3_step(g, recs, torch.float32)
    print(f"== {name}: loss rel {abs(loss - g['loss'][0]) / abs(g['loss'][0]):.3e}")
    for k, got, want in (("e_pred", e, g["e_pred"]), ("f_pred", f, g["f_pred"])):
        a, b, c = stats(got, want)
        print(f"{k:14s} max(fl 1e-2) {a:.3e} max(fl 1e-3) {b:.3e} q999 {c:.3e}")
    idx = g["grad_idx"]
    off = 0
    for pname, shape in M.param_shapes(cfg):
        n = int(np.prod(shape))
        sel = (idx >= off) & (idx < off + n)
        a, b, c = stats(grad[idx[sel]], g["grad_val"][sel])
        print(f"{pname:14s} max(fl 1e-2) {a:.3e} max(fl 1e-3) {b:.3e} q999 {c:.3e}")
        worst = [max(worst[0], a), max(worst[1], c)]
        off += n
    summary[name] = worst
print("# gradients, worst over parameter arrays: max(fl 1e-2) / q999")
for name, (a, c) in summary.items():
    print(f"{name:6s} {a:.3e} {c:.3e}")
_lib.call("gfm_set_gemm_mode", 1)
