"""Ensemble inference (ensemble.py:121-186): the device spread reductions
against the oracle's numpy restatement (CPU tensors), and ensemble_predict
through the sm_100a forward against the oracle (GPU, float64, 1e-10)."""

import numpy as np
import pytest
import torch

from oracle import gfm_oracle as O

from paper_2406_12909_b200 import ensemble as EN, model as M, train as T  # noqa: E402
from paper_2406_12909_b200.errors import ConfigError, ValidationError  # noqa: E402
from paper_2406_12909_b200.records import GraphRecord  # noqa: E402


@pytest.mark.parametrize("how", EN.FORCE_REDUCTIONS)
def test_spread_reductions_match_oracle(how):
    rng = np.random.default_rng(0)
    f = rng.standard_normal((4, 23, 3))
    f[:, 5] = f[0, 5]  # all members agree on node 5: exactly zero spread
    offsets = np.array([0, 4, 4 + 9, 23])
    gnode = torch.from_numpy(np.repeat(np.arange(3), np.diff(offsets)).astype(np.int32))
    sig = EN.population_sigma(torch.from_numpy(f))
    want = O.population_sigma(f)
    np.testing.assert_allclose(sig.numpy(), want, rtol=1e-14, atol=0)
    assert np.all(sig.numpy()[5] == 0.0)
    got = EN.reduce_force_sigma(sig, gnode, 3, how).numpy()
    np.testing.assert_allclose(got, O.reduce_force_sigma(want, offsets, how), rtol=1e-14)


def test_reduction_name_checked():
    with pytest.raises(ConfigError):
        EN.reduce_force_sigma(torch.zeros(2, 3), torch.zeros(2, dtype=torch.int32), 1, "median")
    with pytest.raises(ValidationError):
        EN.ensemble_predict([], [])


@pytest.mark.gpu
@pytest.mark.parametrize("how", EN.FORCE_REDUCTIONS)
def test_ensemble_predict_matches_oracle(how):
    dicts = O.synthetic(6, seed=9)
    recs = [GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"]) for d in dicts]
    mc = M.ModelConfig(mpnn_kind="max-agg", mpnn_layers=2, mpnn_width=16, fc_layers=2,
                       fc_width=16)
    flats = [M.init_params_flat(mc, seed=s) for s in (1, 2, 3)]
    members = [T.Checkpoint(mc, f, T.OptimizerState(None, None, 0), 0, 0) for f in flats]
    got = EN.ensemble_predict(members, recs, how)
    ocfg = O.config("max-agg", 2, 16, 2, 16)
    e_mean, e_sig, f_sig = O.ensemble_predict([(ocfg, f) for f in flats], dicts, how)
    assert got.member_count == 3
    np.testing.assert_allclose(got.energy_mean, e_mean, rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(got.energy_sigma, e_sig, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(got.force_sigma, f_sig, rtol=1e-9, atol=1e-12)
    one = EN.ensemble_predict(members[:1], recs, how)
    assert np.all(one.energy_sigma == 0.0) and np.all(one.force_sigma == 0.0)
