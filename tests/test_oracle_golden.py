"""Pin the CPU oracle restatement against vectors made by the reference.

The goldens (tests/golden/*.npz) were produced by oracle/make_golden.py from
/root/reference/pkg/src/gfmkit itself.  These tests need neither the
reference nor a GPU.
"""

import numpy as np
import pytest

from conftest import golden, records_from
from oracle import gfm_oracle as O

REF_KINDS = ("mean-agg", "sum-agg", "max-agg")


def test_golden_numpy_version_matches():
    g = golden("misc.npz")
    assert str(g["numpy_version"]) == np.__version__


@pytest.mark.parametrize("kind", REF_KINDS)
def test_c1_forward_loss_grad(kind):
    g = golden("c1_model.npz")
    recs = records_from(g, "rec_")
    cfg = O.config(kind, layers=3, hidden=64, fc_layers=2, fc_width=64)
    flat = O.init_flat(cfg, 0)
    np.testing.assert_array_equal(flat, g["mean-agg_flat"])
    b = O.pack(recs)
    (total, et, ft), grad, (e, f) = O.loss_and_grad(cfg, flat, b)
    np.testing.assert_allclose(e, g[f"{kind}_e_pred"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(f, g[f"{kind}_f_pred"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose([total, et, ft], g[f"{kind}_loss"], rtol=1e-12)
    np.testing.assert_allclose(grad, g[f"{kind}_grad"], rtol=1e-9, atol=1e-13)


def test_c1_layer0_aggregation_bitwise():
    g = golden("c1_model.npz")
    b = O.pack(records_from(g, "rec_"))
    cfg = O.config("mean-agg", layers=3, hidden=64, fc_layers=2, fc_width=64)
    flat = O.init_flat(cfg, 0)
    cache = {}
    O.forward(cfg, flat, b, cache)
    np.testing.assert_array_equal(cache["layers"][0]["agg"], g["mean-agg_layer0_agg"])


def test_c1_adam_first_step():
    g = golden("c1_model.npz")
    flat = g["mean-agg_flat"]
    new, m, v, t = O.adam(flat, g["mean-agg_grad"], 0 * flat, 0 * flat, 0)
    np.testing.assert_array_equal(new - flat, g["mean-agg_adam1"])


@pytest.mark.parametrize("case_id", range(6))
@pytest.mark.parametrize("kind", REF_KINDS)
def test_small_cases(case_id, kind):
    g = golden("small_models.npz")
    recs = records_from(g, f"case{case_id}_rec_")
    p = f"case{case_id}_{kind}_"
    cfg = O.config(kind, layers=2, hidden=8, fc_layers=3, fc_width=6)
    flat = O.init_flat(cfg, case_id + 7)
    np.testing.assert_array_equal(flat, g[p + "flat"])
    b = O.pack(recs)
    b["e_true"], b["f_true"] = g[p + "energy_true"], g[p + "forces_true"]
    (total, et, ft), grad, (e, f) = O.loss_and_grad(cfg, flat, b)
    np.testing.assert_allclose(e, g[p + "e_pred"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(f, g[p + "f_pred"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose([total, et, ft], g[p + "loss"], rtol=1e-12)
    np.testing.assert_allclose(grad, g[p + "grad"], rtol=1e-10, atol=1e-13)


@pytest.mark.parametrize("case_id", range(3))
@pytest.mark.parametrize("kind", REF_KINDS)
def test_aggregate_isolated_bitwise(case_id, kind):
    g = golden("aggregate.npz")
    p = f"agg{case_id}_"
    src, dst, pos = g[p + "src"], g[p + "dst"], g[p + "pos"]
    n = pos.shape[0]
    rec = dict(z=np.ones(n, np.uint8), pos=pos, edges=np.stack([src, dst], 1),
               energy=0.0, forces=np.zeros((n, 3)))
    b = O.pack([rec])
    msg = g[p + "msg"]
    c = {}
    a = O.aggregate(b, msg, kind, c)
    np.testing.assert_array_equal(a, g[p + kind + "_fwd"])
    d = O.aggregate_backward(b, g[p + kind + "_dagg"], msg, kind, c)
    np.testing.assert_array_equal(d, g[p + kind + "_bwd"])


def test_reduceat_order_is_first_plus_pairwise():
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 8, 9, 16, 17, 40, 129, 300):
        m = rng.normal(size=(n, 5))
        got = np.add.reduceat(m, [0], axis=0)[0]
        want = [m[0, c] + O.numpy_pairwise_sum(list(m[1:, c])) for c in range(5)]
        np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("case_id", range(4))
def test_cutoff_edges_exact(case_id):
    g = golden("neighbors.npz")
    p = f"nb{case_id}_"
    edges, _ = O.cutoff_edges(g[p + "pos"], float(g[p + "rc"]))
    np.testing.assert_array_equal(edges, g[p + "edges"])


def test_synthetic_generator_matches_reference():
    g = golden("neighbors.npz")
    want = records_from(g, "synth_")
    got = O.synthetic(6, seed=42)
    assert len(got) == len(want)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a["z"], b["z"])
        np.testing.assert_array_equal(a["pos"], b["pos"])
        np.testing.assert_array_equal(a["edges"], b["edges"])
        assert a["energy"] == b["energy"]
        np.testing.assert_array_equal(a["forces"], b["forces"])


def test_c1_records_regenerate():
    g = golden("c1_model.npz")
    want = records_from(g, "rec_")
    got = O.synthetic(32, n_atoms_range=(32, 32), box_length=8.0, rc=5.0, seed=0)
    for a, b in zip(got, want):
        np.testing.assert_array_equal(a["edges"], b["edges"])
        np.testing.assert_array_equal(a["pos"], b["pos"])


def test_adam_trajectory_bitwise():
    g = golden("misc.npz")
    flat = g["adam_init"]
    m = np.zeros_like(flat)
    v = np.zeros_like(flat)
    t = 0
    for k in range(5):
        flat, m, v, t = O.adam(flat, g["adam_grads"][k], m, v, t)
        np.testing.assert_array_equal(flat, g["adam_traj"][k])


def test_schedule_matches():
    g = golden("misc.npz")
    sched = O.schedule(103, 4, 8, 7, 3)
    np.testing.assert_array_equal(np.concatenate([np.concatenate(b) for b in sched]), g["sched"])


def test_ordered_allreduce_bitwise():
    g = golden("misc.npz")
    np.testing.assert_array_equal(O.ordered_allreduce_sum(list(g["allreduce_in"])), g["allreduce_out"])
