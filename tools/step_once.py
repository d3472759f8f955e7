"""Run the bench workload's training step eagerly a few times (for ncu launch
lists / full captures).  Usage: python tools/step_once.py [--config c3] [--steps 3]"""

import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import CONFIGS, packed  # noqa: E402
from paper_2406_12909_b200 import model as M, train as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--batch", type=int, default=None)
a = ap.parse_args()
W = CONFIGS[a.config]
B, n = a.batch or W["batch"], W["atoms"][1]
if W["kind"] == "egnn":
    from paper_2406_12909_b200.egnn import EGNNConfig
    cfg = EGNNConfig(egnn_layers=W["layers"], egnn_width=W["hidden"], fc_layers=W["fc_layers"],
                     fc_width=W["fc_width"], batch_size=B)
else:
    cfg = M.ModelConfig(mpnn_kind=W["kind"], mpnn_layers=W["layers"], mpnn_width=W["hidden"],
                        fc_layers=2, fc_width=W["fc_width"], batch_size=B)
tr = T.DataParallelTrainer(cfg, T.TrainConfig())
cells = [[W["box"]] * 3] * B if W["periodic"] else None
runner = T.StructureStepRunner(tr, (np.arange(B + 1) * n).astype(np.int32), W["rc"],
                               W["max_nbr"], cells=cells, use_graph=False)
z, pos, e, f, _ = packed(B, W, 0)
dev = tr.device
runner.load(torch.as_tensor(pos, device=dev), torch.as_tensor(z, device=dev),
            torch.as_tensor(e, dtype=torch.float32, device=dev),
            torch.as_tensor(f, dtype=torch.float32, device=dev))
for _ in range(a.steps):
    runner.run()
torch.cuda.synchronize()
print("ok", float(tr.contrib[tr.P]))
