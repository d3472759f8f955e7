"""Time the aggregation kernels at a bench config's in-step shape (device
radius graph of bench.py's synthetic batch, uint8 argmax as in the step):
gfm_agg_fwd and gfm_agg_bwd (prep + CSC gather), CUDA events, L2 flushed
before every launch.  Env knobs (GFM_AGG_*) select kernel variants.

    python tools/agg_time.py [c3|c2]
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, packed  # noqa: E402
from paper_2406_12909_b200 import _lib, model as M  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c3"
W = CONFIGS[cfgname]
B, n = W["batch"], W["atoms"][1]
dev = torch.device("cuda")
z, pos, e, f, off = packed(B, W, 0)
cells = torch.full((B, 3), W["box"], dtype=torch.float64, device=dev) if W["periodic"] else None
b = M.radius_batch(torch.as_tensor(pos, device=dev), torch.as_tensor(z, device=dev),
                   torch.as_tensor(off, device=dev), off, W["rc"], W["max_nbr"], cells,
                   dtype=torch.float32, e_cap=B * n * W["max_nbr"])
N, E, H = b.n_nodes, b.n_edges, W["hidden"]
parts, K = 15, 4
flags = M._argmax_flag(b)
P = _lib.ptr
sh = _lib.stream_handle()
h = torch.randn(N, H, device=dev)
agg = torch.empty(N, K * H, device=dev)
am = torch.empty(N, H, dtype=torch.uint8, device=dev)
sm = torch.empty(N, H, device=dev)
dagg = torch.randn(N, K * H, device=dev)
dh = torch.randn(N, H, device=dev)
out = torch.empty(N, H, device=dev)
ws = torch.empty(_lib.query("gfm_agg_bwd_workspace_bytes", N, H, parts, _lib.F32),
                 dtype=torch.uint8, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def fwd():
    _lib.call("gfm_agg_fwd", P(h), N, H, P(b.rowptr), P(b.col_src), P(b.edge_w), parts, P(agg),
              P(am), P(sm), _lib.F32, flags, sh)


# edge weights in CSC order as in the step (GFM_W_CSC=0: w[eid] gathers)
W_CSC = os.environ.get("GFM_W_CSC", "1") != "0"
w_b = b.edge_w
if W_CSC:
    w_b = torch.empty_like(b.edge_w)
    _lib.call("gfm_permute", P(b.csc_eid), E, None, P(b.edge_w), P(w_b), _lib.F32, sh)


def bwd():
    _lib.call("gfm_agg_bwd", P(dagg), P(agg), P(sm), P(am), P(h), P(b.rowptr), P(b.csc_ptr),
              P(b.csc_eid), P(b.csc_dst), P(w_b), N, H, parts, P(dh), P(h), P(out), P(ws),
              _lib.F32, flags | (_lib.FLAG_W_CSC if W_CSC else 0), sh)


def timeit(fn, reps=30):
    for _ in range(3):
        fn()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        fn()
        a1.record()
        torch.cuda.synchronize()
        tot += a0.elapsed_time(a1)
    return tot / reps * 1e3


fwd()
tf, tb = timeit(fwd), timeit(bwd)
ref = out.clone()
knobs = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("GFM_AGG"))
print(f"{cfgname} N={N} E={E} H={H} [{knobs or 'default'}]  fwd {tf:7.1f} us  bwd {tb:7.1f} us",
      flush=True)
np.save(os.path.join(ROOT, "gpurun_out", f"aggout_{cfgname}_{knobs.replace(' ', '_') or 'default'}.npy"),
        out.cpu().numpy()[:2000])
