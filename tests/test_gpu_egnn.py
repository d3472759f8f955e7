"""EGNN variant (C4) on the GPU against its float64 oracle
(oracle/egnn_oracle.py, pinned by FD and torch double backward).

Energies, autograd forces F = -dE/dx0, the L1 MTL loss and the parameter
gradient (reverse over the primal + tangent forward) through the C-ABI
kernels.  Bars: float64 1e-9 relative; float32 (3xTF32 tensor-core GEMMs)
5e-4 on energies / forces / loss and 5e-3 on gradients (elementwise,
denominator floored at 1e-2 of the array's max).
"""

import numpy as np
import pytest
import torch

from oracle import egnn_oracle as EG
from oracle import gfm_oracle as O

pytestmark = pytest.mark.gpu

from paper_2406_12909_b200 import model as M, train as T  # noqa: E402
from paper_2406_12909_b200.egnn import EGNNConfig  # noqa: E402
from test_gpu_parity import as_records, assert_close_scaled  # noqa: E402

F64, F32 = torch.float64, torch.float32


def _case(seed, count=6, n=(6, 20), H=32, L=3, G=32, cap=8):
    recs = O.synthetic(count, n_atoms_range=n, box_length=6.0, rc=3.0, seed=seed, max_nbr=cap)
    ocfg = EG.config(layers=L, hidden=H, fc_layers=2, fc_width=G)
    cfg = EGNNConfig(egnn_layers=L, egnn_width=H, fc_layers=2, fc_width=G)
    flat = EG.init_flat(ocfg, seed)
    bo = O.pack(recs)
    e, f = EG.forces(ocfg, flat, bo)
    rng = np.random.default_rng(seed)
    sign = lambda shape: np.where(rng.uniform(size=shape) < 0.5, -1.0, 1.0)
    bo["e_true"] = e + (0.5 + rng.uniform(0, 0.5, e.shape)) * sign(e.shape) * bo["n_per"]
    bo["f_true"] = f + (0.3 + rng.uniform(0, 0.5, f.shape)) * sign(f.shape)
    return recs, ocfg, cfg, flat, bo


@pytest.mark.parametrize("seed", range(3))
@pytest.mark.parametrize("dtype,rel,grel", [(F64, 1e-9, 1e-9), (F32, 5e-4, 5e-3)],
                         ids=["f64", "f32"])
def test_egnn_vs_oracle(seed, dtype, rel, grel):
    recs, ocfg, cfg, flat, bo = _case(seed, H=32 if seed < 2 else 64)
    (tot, _, _), grad_o, (e_o, f_o) = EG.loss_and_grad(ocfg, flat, bo)
    params = M.ModelParams.from_flat(cfg, flat, dtype=dtype)
    b = M.make_batch(as_records(recs), dtype=dtype)
    b.energy_true, b.forces_true = bo["e_true"], bo["f_true"]
    e, f = M.forward_batch(params, b)
    fl = 1e-3 if dtype == F64 else 1e-2
    assert_close_scaled(e.cpu().numpy(), e_o, rel, fl, what="e_pred")
    assert_close_scaled(f.cpu().numpy(), f_o, rel, fl, what="forces = -dE/dx")
    lb, grad = M.loss_and_grad(params, b)
    assert abs(lb.total - tot) <= rel * abs(tot), (lb.total, tot)
    g = grad.cpu().numpy()
    off = 0
    for name, shape in M.param_shapes(cfg):
        n = int(np.prod(shape))
        assert_close_scaled(g[off:off + n], grad_o[off:off + n], grel, fl, what=f"grad {name}")
        off += n


def test_egnn_trainer_runner_step_matches_oracle_adam():
    """C4-style training step through DataParallelTrainer + the captured
    StructureStepRunner (device radius graph): loss and the Adam update
    against the oracle in float64."""
    B, n, box, rc, cap = 8, 16, 6.0, 3.0, 8
    recs = O.synthetic(B, n_atoms_range=(n, n), box_length=box, rc=rc, seed=4, max_nbr=cap)
    ocfg = EG.config(layers=3, hidden=32, fc_layers=2, fc_width=32)
    cfg = EGNNConfig(egnn_layers=3, egnn_width=32, fc_layers=2, fc_width=32, batch_size=B)
    flat = EG.init_flat(ocfg, 1)
    tr = T.DataParallelTrainer(cfg, T.TrainConfig(), initial=flat, dtype=F64)
    run = T.StructureStepRunner(tr, np.arange(B + 1) * n, rc, cap)
    pos = torch.as_tensor(np.concatenate([r["pos"] for r in recs]))
    z = torch.as_tensor(np.concatenate([r["z"] for r in recs]).astype(np.int32))
    e = torch.as_tensor(np.array([r["energy"] for r in recs]), dtype=F64)
    f = torch.as_tensor(np.concatenate([r["forces"] for r in recs]), dtype=F64)
    run.load(pos, z, e, f)
    run.capture(warmup=2)
    bo = O.pack(recs)
    m = np.zeros_like(flat)
    v = np.zeros_like(flat)
    t = 0
    for _ in range(2):
        (tot, _, _), grad_o, _ = EG.loss_and_grad(ocfg, flat, bo)
        run.load(pos, z, e, f)
        run.run()
        torch.cuda.synchronize()
        assert abs(float(tr.contrib[tr.P].item()) - tot) <= 1e-9 * abs(tot)
        flat, m, v, t = EG_adam(flat, grad_o, m, v, t)
        np.testing.assert_allclose(tr.flat_master(), flat, rtol=0, atol=1e-9)


def EG_adam(flat, grad, m, v, t):
    return O.adam(flat, grad, m, v, t)


@pytest.mark.parametrize("rows,cols", [(1, 1), (255, 33), (1000, 64), (4097, 130)])
def test_colsum_one_launch_deterministic(rows, cols):
    """gfm_colsum (chunk partials + last-block final in one launch): float64
    sums of the columns, bitwise repeatable with the workspace reused (the
    tickets reset), accumulate mode adds to the output"""
    from paper_2406_12909_b200 import _lib
    rng = np.random.default_rng(rows)
    ld = cols + 3
    X = torch.as_tensor(rng.standard_normal((rows, ld)), dtype=torch.float32, device="cuda")
    ws = torch.zeros(_lib.query("gfm_colsum_workspace_bytes", rows, cols), dtype=torch.uint8,
                     device="cuda")
    s = _lib.stream_handle()
    outs = []
    for _ in range(3):
        out = torch.empty(cols, dtype=torch.float32, device="cuda")
        _lib.call("gfm_colsum", _lib.ptr(X), rows, cols, ld, _lib.ptr(out), 0, _lib.ptr(ws),
                  _lib.F32, s)
        outs.append(out.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])
    want = X.double().cpu().numpy()[:, :cols].sum(axis=0)
    np.testing.assert_allclose(outs[0], want, rtol=1e-6, atol=1e-5)
    acc = torch.ones(cols, dtype=torch.float32, device="cuda")
    _lib.call("gfm_colsum", _lib.ptr(X), rows, cols, ld, _lib.ptr(acc), 1, _lib.ptr(ws),
              _lib.F32, s)
    np.testing.assert_allclose(acc.cpu().numpy(), want + 1.0, rtol=1e-6, atol=1e-5)


# float32 at this shape (tools/c4_err.py): e 3.8e-6, forces 9.1e-4 (8,192
# atoms x 20 neighbours: the reverse pass accumulates more 3xTF32 rounding
# than the small cases), loss 3.6e-8, gradients <= 1.03e-3
@pytest.mark.parametrize("dtype,rel,frel,grel", [(F64, 1e-9, 1e-9, 1e-9),
                                                 (F32, 5e-4, 2e-3, 5e-3)], ids=["f64", "f32"])
def test_egnn_c4_shape_vs_oracle(dtype, rel, frel, grel):
    """the benched C4 configuration itself: 256 molecules x 32 atoms, EGNN L3
    H64 fc 2x64, box 8 A, rc 5 A, 20 neighbours -- energies, forces, loss
    and the full parameter gradient against the float64 oracle"""
    recs = O.synthetic(256, n_atoms_range=(32, 32), box_length=8.0, rc=5.0, seed=31, max_nbr=20)
    ocfg = EG.config(layers=3, hidden=64, fc_layers=2, fc_width=64)
    cfg = EGNNConfig(egnn_layers=3, egnn_width=64, fc_layers=2, fc_width=64, batch_size=256)
    flat = EG.init_flat(ocfg, 3)
    bo = O.pack(recs)
    (tot, _, _), grad_o, (e_o, f_o) = EG.loss_and_grad(ocfg, flat, bo)
    params = M.ModelParams.from_flat(cfg, flat, dtype=dtype)
    b = M.make_batch(as_records(recs), dtype=dtype)
    e, f = M.forward_batch(params, b)
    fl = 1e-3 if dtype == F64 else 1e-2
    assert_close_scaled(e.cpu().numpy(), e_o, rel, fl, what="e_pred")
    assert_close_scaled(f.cpu().numpy(), f_o, frel, fl, what="forces = -dE/dx")
    lb, grad = M.loss_and_grad(params, b)
    assert abs(lb.total - tot) <= rel * abs(tot), (lb.total, tot)
    g = grad.cpu().numpy()
    off = 0
    for name, shape in M.param_shapes(cfg):
        n = int(np.prod(shape))
        assert_close_scaled(g[off:off + n], grad_o[off:off + n], grel, fl, what=f"grad {name}")
        off += n
