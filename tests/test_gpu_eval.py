"""evaluate() (train.py:160-189): the per-batch sums on the device
(gfm_eval_errors: numpy's pairwise sums, float64 running totals in the
reference's order) == the reference's numpy loop over the same predictions,
bitwise; ragged sizes and a short last batch."""

import numpy as np
import pytest
import torch

from oracle import gfm_oracle as O

from paper_2406_12909_b200 import model as M, train as T
from paper_2406_12909_b200.comm import LocalComm
from paper_2406_12909_b200.records import GraphRecord

pytestmark = pytest.mark.gpu


class _Store:
    def __init__(self, recs):
        self.recs = recs
        self.ownership = {"valset": type("O", (), {"n_samples": len(recs)})()}

    def fetch_batch(self, group, idx):
        return [self.recs[int(i)] for i in idx]


def test_evaluate_sums_bitwise_vs_numpy_loop():
    dicts = O.synthetic(23, n_atoms_range=(3, 60), seed=4)
    recs = [GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"]) for d in dicts]
    mc = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=2, mpnn_width=16, fc_width=16)
    params = M.ModelParams.from_flat(mc, M.init_params_flat(mc, seed=3), dtype=torch.float64)
    store = _Store(recs)
    got = T.evaluate(params, store, LocalComm(), batch_size=10)
    sum_e = sum_f = n_graphs = n_comp = 0.0
    for lo in range(0, len(recs), 10):
        b = M.make_batch(recs[lo:lo + 10], dtype=torch.float64)
        e, f = M.forward_batch(params, b)
        e, f = e.cpu().numpy(), f.cpu().numpy()
        n_per = np.diff(b.host_offsets)
        sum_e += float(np.abs((e - b.energy_true.cpu().numpy()) / n_per).sum())
        sum_f += float(np.abs(f - b.forces_true.cpu().numpy()).sum())
        n_graphs += b.n_graphs
        n_comp += 3.0 * b.n_nodes
    assert got == (sum_e / n_graphs, sum_f / n_comp)
