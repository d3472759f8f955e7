"""float32 error survey of the EGNN variant at the benched C4 shape against
the float64 oracle (max elementwise relative error, floor 1% of each
array's max).  python tools/c4_err.py"""
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from oracle import egnn_oracle as EG, gfm_oracle as O
from paper_2406_12909_b200 import model as M
from paper_2406_12909_b200.egnn import EGNNConfig
from test_gpu_parity import as_records
recs = O.synthetic(256, n_atoms_range=(32, 32), box_length=8.0, rc=5.0, seed=31, max_nbr=20)
ocfg = EG.config(layers=3, hidden=64, fc_layers=2, fc_width=64)
cfg = EGNNConfig(egnn_layers=3, egnn_width=64, fc_layers=2, fc_width=64, batch_size=256)
flat = EG.init_flat(ocfg, 3)
bo = O.pack(recs)
(tot, _, _), grad_o, (e_o, f_o) = EG.loss_and_grad(ocfg, flat, bo)
def err(got, want, fl=1e-2):
    sc = max(float(np.abs(want).max()), 1e-30)
    return float((np.abs(got - want) / np.maximum(np.abs(want), fl * sc)).max())
params = M.ModelParams.from_flat(cfg, flat, dtype=torch.float32)
b = M.make_batch(as_records(recs), dtype=torch.float32)
e, f = M.forward_batch(params, b)
print("e", err(e.cpu().numpy(), e_o), "f", err(f.cpu().numpy(), f_o))
lb, grad = M.loss_and_grad(params, b)
print("loss", abs(lb.total - tot) / abs(tot))
g = grad.cpu().numpy(); off = 0; worst = 0
for name, shape in M.param_shapes(cfg):
    n = int(np.prod(shape)); x = err(g[off:off+n], grad_o[off:off+n]); worst = max(worst, x); print(name, x); off += n
print("worst grad", worst)
