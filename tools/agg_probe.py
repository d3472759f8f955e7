"""Time gfm_agg_fwd / gfm_agg_bwd / force fwd+bwd on the bench workload's
batch (CUDA events, L2 flushed between reps).
Usage: python tools/agg_probe.py [--config c3]   (GFM_AGG_TILE=1 for A/B)"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import CONFIGS, WORKLOAD, make_structures  # noqa: E402
from paper_2406_12909_b200 import _lib, model as M, train as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--once", action="store_true", help="one fwd + one bwd call (ncu target)")
a = ap.parse_args()
WORKLOAD.update(CONFIGS[a.config])
B, n = WORKLOAD["batch"], WORKLOAD["atoms"]
cfg = M.ModelConfig(mpnn_kind=WORKLOAD["kind"], mpnn_layers=WORKLOAD["layers"],
                    mpnn_width=WORKLOAD["hidden"], fc_layers=2, fc_width=WORKLOAD["fc_width"],
                    batch_size=B)
tr = T.DataParallelTrainer(cfg, T.TrainConfig())
cells = [[WORKLOAD["box"]] * 3] * B if WORKLOAD["periodic"] else None
runner = T.StructureStepRunner(tr, (np.arange(B + 1) * n).astype(np.int32), WORKLOAD["rc"],
                               WORKLOAD["max_nbr"], cells=cells, use_graph=False)
z, pos, e, f = make_structures(B, 0)
dev = tr.device
runner.load(torch.as_tensor(pos.reshape(-1, 3), device=dev),
            torch.as_tensor(z.reshape(-1), device=dev),
            torch.as_tensor(e, dtype=torch.float32, device=dev),
            torch.as_tensor(f.reshape(-1, 3), dtype=torch.float32, device=dev))
runner.run()
torch.cuda.synchronize()
b = runner.batch
N, E, H = b.n_nodes, b.n_edges, cfg.mpnn_width
parts, K = M.KIND_PARTS[cfg.mpnn_kind], cfg.n_parts
sh = _lib.stream_handle()
P = _lib.ptr
h = torch.randn(N, H, device=dev)
agg = torch.empty(N, K * H, device=dev)
am = torch.empty(N, H, dtype=torch.int32, device=dev)
sm = torch.empty(N, H, device=dev)
dagg = torch.randn(N, K * H, device=dev)
dh = torch.randn(N, H, device=dev)
out = torch.empty(N, H, device=dev)
ws = torch.empty(_lib.query("gfm_agg_bwd_workspace_bytes", N, H, parts, _lib.F32),
                 dtype=torch.uint8, device=dev)
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)


def fwd():
    _lib.call("gfm_agg_fwd", P(h), N, H, P(b.rowptr), P(b.col_src), P(b.edge_w), parts, P(agg),
              P(am), P(sm), _lib.F32, 0, sh)


def bwd():
    _lib.call("gfm_agg_bwd", P(dagg), P(agg), P(sm), P(am), P(h), P(b.rowptr), P(b.csc_ptr),
              P(b.csc_eid), P(b.csc_dst), P(b.edge_w), N, H, parts, P(dh), P(h), P(out), P(ws),
              _lib.F32, 0, sh)


def timeit(fn):
    fn()
    tot = 0.0
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / a.reps * 1e3


if a.once:
    fwd()
    bwd()
    torch.cuda.synchronize()
    print("once ok")
    sys.exit(0)
tf, tb = timeit(fwd), timeit(bwd)
fb = E * H * 4 + 8 * E + 4 * (N + 1) + K * N * H * 4 + 8 * N * H
comp_f = N * H * 4 + 8 * E + 4 * (N + 1) + K * N * H * 4 + 8 * N * H
comp_b = 5 * N * H * 4 + 8 * E + 4 * (N + 1) + 2 * N * H * 4 + N * H * 4 * 2
print(f"{a.config} N={N} E={E} H={H} tile={'on' if os.environ.get('GFM_AGG_TILE') == '1' else 'off'}"
      f"  fwd {tf:8.1f} us ({comp_f / tf / 1e3:6.0f} GB/s compulsory, {fb / tf / 1e3:6.0f} GB/s survey)"
      f"  bwd {tb:8.1f} us ({comp_b / tb / 1e3:6.0f} GB/s compulsory)")
