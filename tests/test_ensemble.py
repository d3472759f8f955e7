"""Ensemble inference (ensemble.py:121-186): the device spread reductions
against the oracle's numpy restatement (bitwise, float64), and
ensemble_predict through the sm_100a forward against the oracle (GPU,
float64, 1e-10)."""

import numpy as np
import pytest
import torch

from oracle import gfm_oracle as O

from paper_2406_12909_b200 import ensemble as EN, model as M, train as T  # noqa: E402
from paper_2406_12909_b200.errors import ConfigError, ValidationError  # noqa: E402
from paper_2406_12909_b200.records import GraphRecord  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("how", EN.FORCE_REDUCTIONS)
def test_spread_reductions_match_oracle(how):
    """gfm_member_stats / gfm_force_sigma_reduce == numpy (the oracle's
    restatement of ensemble.py:121-148), bitwise in float64 -- including a
    structure of 300 atoms (900 components: numpy's pairwise recursion)"""
    rng = np.random.default_rng(0)
    f = rng.standard_normal((4, 323, 3))
    f[:, 5] = f[0, 5]  # all members agree on node 5: exactly zero spread
    offsets = np.array([0, 4, 4 + 9, 23, 323])
    sig = EN.population_sigma(torch.from_numpy(f).cuda())
    want = O.population_sigma(f)
    np.testing.assert_array_equal(sig.cpu().numpy(), want)
    assert np.all(sig.cpu().numpy()[5] == 0.0)
    mean, _ = EN.member_stats(torch.from_numpy(f).cuda())
    np.testing.assert_array_equal(mean.cpu().numpy(), f.mean(axis=0))
    off = torch.as_tensor(offsets.astype(np.int32)).cuda()
    got = EN.reduce_force_sigma(sig, off, how).cpu().numpy()
    np.testing.assert_array_equal(got, O.reduce_force_sigma(want, offsets, how))


def test_reduction_name_checked():
    with pytest.raises(ConfigError):
        EN.reduce_force_sigma(torch.zeros(2, 3), torch.zeros(2, dtype=torch.int32), "median")
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
