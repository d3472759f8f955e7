"""Generate tests/golden/checkpoint_tiny.gfmp with the REFERENCE's own
``save_checkpoint`` (gfmkit/train.py:358-381).  Test infrastructure only.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python oracle/make_checkpoint_golden.py

The fixture records a tiny model so the GFMP byte format is pinned
without a large file (P = 263): init_params(seed=3), m ~ N(0,1), v ~ U[0,1) from
default_rng(5), t = 7, epoch = 5, base_seed = 11.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                   "checkpoint_tiny.gfmp")

CONFIG = dict(mpnn_kind="max-agg", mpnn_layers=1, mpnn_width=2, fc_layers=2, fc_width=2,
              batch_size=4, learning_rate=2e-3, alpha_energy=1.0, alpha_forces=100.0)


def main() -> None:
    sys.path.insert(0, REF)
    from gfmkit.model import ModelConfig, init_params
    from gfmkit.train import OptimizerState, save_checkpoint

    cfg = ModelConfig(**CONFIG)
    flat = init_params(cfg, seed=3).flatten()
    rng = np.random.default_rng(5)
    state = OptimizerState(m=rng.standard_normal(flat.shape[0]),
                           v=rng.random(flat.shape[0]), t=7)
    save_checkpoint(OUT, cfg, flat, state, epoch=5, base_seed=11)
    print(f"wrote {OUT}: P={flat.shape[0]} numpy {np.__version__}")


if __name__ == "__main__":
    main()
