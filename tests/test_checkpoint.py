"""GFMP checkpoints (train.py:341-423) and the train() loop that writes them
(train.py:192-338).

CPU: the reference-written fixture ``golden/checkpoint_tiny.gfmp`` (made by
oracle/make_checkpoint_golden.py with the reference's own save_checkpoint)
loads, and re-saving it is byte-identical; the error classes match.
GPU: train() over an in-memory store, float64, against the oracle's
schedule + loss_and_grad + Adam loop (1e-9 relative), and the checkpoint it
writes holds the final parameters, moments and step count.
"""

import os
import struct
import zlib

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from oracle import gfm_oracle as O

from paper_2406_12909_b200 import model as M, train as T  # noqa: E402
from paper_2406_12909_b200.errors import (CorruptionError, FormatError,  # noqa: E402
                                          UnsupportedVersionError)
from paper_2406_12909_b200.records import GraphRecord  # noqa: E402
from paper_2406_12909_b200.schedule import RecordStore  # noqa: E402

FIXTURE = os.path.join(GOLDEN, "checkpoint_tiny.gfmp")


def _tiny_cfg():
    return M.ModelConfig(mpnn_kind="max-agg", mpnn_layers=1, mpnn_width=2, fc_layers=2,
                         fc_width=2, batch_size=4, learning_rate=2e-3)


def test_reference_checkpoint_loads_and_resaves_byte_identical(tmp_path):
    ck = T.load_checkpoint(FIXTURE)
    assert ck.model_config == _tiny_cfg()
    assert (ck.epoch, ck.base_seed, ck.opt_state.t) == (5, 11, 7)
    assert ck.flat.shape == (M.count_params(ck.model_config),) == (263,)
    np.testing.assert_array_equal(ck.flat, M.init_params_flat(ck.model_config, seed=3))
    rng = np.random.default_rng(5)
    np.testing.assert_array_equal(ck.opt_state.m, rng.standard_normal(263))
    np.testing.assert_array_equal(ck.opt_state.v, rng.random(263))
    out = tmp_path / "resaved.gfmp"
    T.save_checkpoint(str(out), ck.model_config, ck.flat, ck.opt_state, ck.epoch, ck.base_seed)
    with open(FIXTURE, "rb") as a:
        assert out.read_bytes() == a.read()


def test_checkpoint_accepts_tensors(tmp_path):
    ck = T.load_checkpoint(FIXTURE)
    st = T.OptimizerState(torch.from_numpy(ck.opt_state.m), torch.from_numpy(ck.opt_state.v),
                          ck.opt_state.t)
    out = tmp_path / "t.gfmp"
    T.save_checkpoint(str(out), ck.model_config, torch.from_numpy(ck.flat), st, 5, 11)
    with open(FIXTURE, "rb") as a:
        assert out.read_bytes() == a.read()


def _rewrite(tmp_path, blob, fix_crc=True):
    if fix_crc:
        body = blob[:-4]
        blob = body + struct.pack("<I", zlib.crc32(body))
    p = tmp_path / "bad.gfmp"
    p.write_bytes(blob)
    return str(p)


def test_checkpoint_errors(tmp_path):
    with open(FIXTURE, "rb") as fh:
        blob = fh.read()
    with pytest.raises(FormatError):
        T.load_checkpoint(_rewrite(tmp_path, b"XXXX" + blob[4:]))
    flipped = bytearray(blob)
    flipped[200] ^= 1
    with pytest.raises(CorruptionError):
        T.load_checkpoint(_rewrite(tmp_path, bytes(flipped), fix_crc=False))
    with pytest.raises(UnsupportedVersionError):
        T.load_checkpoint(_rewrite(tmp_path, blob[:4] + struct.pack("<I", 2) + blob[8:]))
    with pytest.raises(CorruptionError):  # drop one float64, crc recomputed
        T.load_checkpoint(_rewrite(tmp_path, blob[:-12] + blob[-4:]))
    with pytest.raises(CorruptionError):
        T.load_checkpoint(_rewrite(tmp_path, b"GFMP", fix_crc=False))


@pytest.mark.gpu
@pytest.mark.parametrize("optimizer", ["adam", "sgd"])
def test_train_loop_matches_oracle_and_checkpoints(tmp_path, optimizer):
    dicts = O.synthetic(11, seed=4)
    recs = [GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"]) for d in dicts]
    store = RecordStore({"trainset": recs[:8], "valset": recs[8:]})
    mc = M.ModelConfig(mpnn_kind="mean-agg", mpnn_layers=2, mpnn_width=8, fc_layers=2,
                       fc_width=8, batch_size=3)
    path = str(tmp_path / "model.gfmp")
    tc = T.TrainConfig(max_epochs=2, patience=10, base_seed=2, optimizer=optimizer,
                       learning_rate=1e-3, checkpoint_path=path)
    res = T.train(mc, store, config=tc, dtype=torch.float64)
    assert res.epochs_run == 2 and not res.nan_event

    ocfg = O.config("mean-agg", 2, 8, 2, 8)
    flat = O.init_flat(ocfg, seed=tc.base_seed)
    m, v, t = np.zeros_like(flat), np.zeros_like(flat), 0
    for epoch in (1, 2):
        losses = []
        for idx in O.schedule(8, 1, mc.batch_size, tc.base_seed, epoch)[0]:
            (loss, _, _), g, _ = O.loss_and_grad(ocfg, flat, O.pack([dicts[i] for i in idx]))
            losses.append(loss)
            if optimizer == "adam":
                flat, m, v, t = O.adam(flat, g, m, v, t, lr=tc.learning_rate)
            else:
                flat, t = O.sgd(flat, g, tc.learning_rate), t + 1
    got = res.params.flatten()
    np.testing.assert_allclose(got, flat, rtol=1e-9, atol=1e-12)
    # epoch metrics: mean step loss (train.py:276-283) and evaluate() on the
    # valset with the epoch's final parameters (train.py:160-189)
    last = res.metrics[-1]
    np.testing.assert_allclose(last.train_loss, np.mean(losses), rtol=1e-10)
    vb = O.pack(dicts[8:])
    e, f = O.forward(ocfg, flat, vb)
    np.testing.assert_allclose(last.val_energy_mae,
                               np.mean(np.abs((e - vb["e_true"]) / vb["n_per"])), rtol=1e-9)
    np.testing.assert_allclose(last.val_force_mae, np.mean(np.abs(f - vb["f_true"])), rtol=1e-9)

    ck = T.load_checkpoint(path)
    assert ck.model_config == mc and ck.epoch == 2 and ck.base_seed == 2
    assert ck.opt_state.t == t == 6
    np.testing.assert_array_equal(ck.flat, got)
    np.testing.assert_allclose(ck.opt_state.m, m, rtol=1e-9, atol=1e-15)
    np.testing.assert_allclose(ck.opt_state.v, v, rtol=1e-9, atol=1e-20)
