"""Generate golden vectors from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python oracle/make_golden.py

Writes ``tests/golden/*.npz``.  These pin the oracle restatement
(``oracle/gfm_oracle.py``) and give the GPU parity tests fixed answers that
do not need /root/reference at run time.  The numpy version used is stored
in every file (numpy does not promise Generator streams across versions).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "tests", "golden")


def _records_arrays(records):
    """Flatten a list of GraphRecord into concatenated arrays."""
    return dict(
        n_atoms=np.array([r.n_atoms for r in records], np.int64),
        n_edges=np.array([r.edge_count for r in records], np.int64),
        z=np.concatenate([r.atomic_numbers for r in records]).astype(np.uint8),
        pos=np.concatenate([r.positions for r in records]),
        edges=np.concatenate([r.edge_index for r in records]).astype(np.uint32),
        energy=np.array([r.energy for r in records]),
        forces=np.concatenate([r.forces for r in records]),
    )


def _model_case(model, train, cfg, records, seed, kink_free=None):
    params = model.init_params(cfg, seed=seed)
    batch = model.make_batch(records)
    if kink_free is not None:
        batch.energy_true, batch.forces_true = kink_free(model, params, batch)
    cache = {}
    e_pred, f_pred = model.forward_batch(params, batch, cache)
    loss, grad = model.loss_and_grad(params, batch, (cache, e_pred, f_pred))
    flat = params.flatten()
    state = train.OptimizerState.zeros(flat.shape[0])
    tcfg = train.TrainConfig(optimizer="adam", learning_rate=1e-3)
    new = train.apply_update(flat, grad, tcfg, state)
    return dict(
        flat=flat, e_pred=e_pred, f_pred=f_pred,
        loss=np.array([loss.total, loss.energy_term, loss.force_term]),
        grad=grad, adam1=new, energy_true=batch.energy_true,
        forces_true=batch.forces_true,
        layer0_agg=cache["layers"][0]["agg"],
        h_final=cache["h_final"],
    )


def _kink_free(model, params, batch, seed=5):
    rng = np.random.default_rng(seed)
    e_pred, f_pred = model.forward_batch(params, batch)
    sgn = lambda s: np.where(rng.uniform(size=s) < 0.5, -1.0, 1.0)
    e_true = e_pred + (0.5 + rng.uniform(0, 0.5, e_pred.shape)) * sgn(e_pred.shape) * batch.n_per_graph
    f_true = f_pred + (0.3 + rng.uniform(0, 0.5, f_pred.shape)) * sgn(f_pred.shape)
    return e_true, f_true


def main():
    sys.path.insert(0, REF)
    from gfmkit import comm, ddstore, model, preprocess, train
    from gfmkit.records import GraphRecord

    os.makedirs(OUT, exist_ok=True)
    meta = dict(numpy_version=np.array(np.__version__))

    # 1. C1-shaped model cases (32 graphs x 32 atoms, box 8, rc 5, H 64, L 3)
    recs = preprocess.generate_synthetic(32, n_atoms_range=(32, 32), box_length=8.0,
                                         cutoff_radius=5.0, seed=0)
    out = dict(meta, **{f"rec_{k}": v for k, v in _records_arrays(recs).items()})
    for kind in model.MPNN_KINDS:
        cfg = model.ModelConfig(mpnn_kind=kind, mpnn_layers=3, mpnn_width=64,
                                fc_layers=2, fc_width=64, batch_size=32)
        case = _model_case(model, train, cfg, recs, seed=0)
        for k, v in case.items():
            if k in ("flat", "adam1", "h_final", "layer0_agg") and kind != "mean-agg":
                continue
            if k == "adam1":
                v = v - case["flat"]  # store the update, not the params
            out[f"{kind}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "c1_model.npz"), **out)

    # 2. small configs, every kind, several seeds, kink-free targets,
    #    plus random records with duplicate / self-loop / asymmetric edges
    small = dict(meta)
    rng = np.random.default_rng(1234)
    for case_id in range(6):
        if case_id < 4:
            recs = preprocess.generate_synthetic(
                5, n_atoms_range=(2, 9), cutoff_radius=2.5, seed=100 + case_id)
        else:  # conftest.make_random_record-style inputs (pkg/tests/conftest.py:7-23)
            recs = []
            for _ in range(5):
                n = int(rng.integers(1, 12))
                m = int(rng.integers(0, max(1, n * (n - 1)) + 1)) if n > 1 else 0
                e = rng.integers(0, n, size=(m, 2), dtype=np.uint32) if m else np.zeros((0, 2), np.uint32)
                recs.append(GraphRecord(rng.integers(1, 119, size=n, dtype=np.uint8),
                                        rng.normal(size=(n, 3)), e, float(rng.normal()),
                                        rng.normal(size=(n, 3))))
        for k, v in _records_arrays(recs).items():
            small[f"case{case_id}_rec_{k}"] = v
        for kind in model.MPNN_KINDS:
            cfg = model.ModelConfig(mpnn_kind=kind, mpnn_layers=2, mpnn_width=8,
                                    fc_layers=3, fc_width=6, batch_size=5)
            res = _model_case(model, train, cfg, recs, seed=case_id + 7,
                              kink_free=_kink_free)
            for k, v in res.items():
                small[f"case{case_id}_{kind}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "small_models.npz"), **small)

    # 3. aggregation in isolation (random messages, Poisson-ish segments)
    agg = dict(meta)
    for case_id, (n_nodes, n_edges, H) in enumerate([(50, 700, 8), (200, 1500, 32), (40, 0, 4)]):
        r = np.random.default_rng(case_id)
        dst = r.integers(0, n_nodes, n_edges)
        src = r.integers(0, n_nodes, n_edges)
        pos = r.normal(size=(n_nodes, 3))
        rec = GraphRecord(np.ones(n_nodes, np.uint8), pos,
                          np.stack([src, dst], 1).astype(np.uint32), 0.0,
                          np.zeros((n_nodes, 3)))
        batch = model.make_batch([rec])
        msg = r.normal(size=(n_edges, H))
        agg[f"agg{case_id}_src"] = src
        agg[f"agg{case_id}_dst"] = dst
        agg[f"agg{case_id}_pos"] = pos
        agg[f"agg{case_id}_msg"] = msg
        for kind in model.MPNN_KINDS:
            c = {}
            a = model._aggregate(batch, msg, kind, c)
            agg[f"agg{case_id}_{kind}_fwd"] = a
            dagg = r.normal(size=(n_nodes, H))
            agg[f"agg{case_id}_{kind}_dagg"] = dagg
            agg[f"agg{case_id}_{kind}_bwd"] = model._aggregate_backward(batch, dagg, kind, c)
    np.savez_compressed(os.path.join(OUT, "aggregate.npz"), **agg)

    # 4. neighbour lists, synthetic generator, toy potential
    nb = dict(meta)
    for case_id, (n, box, rc) in enumerate([(32, 8.0, 5.0), (100, 12.0, 5.0), (7, 3.0, 1.5), (1, 5.0, 2.0)]):
        r = np.random.default_rng(50 + case_id)
        pos = r.uniform(0, box, size=(n, 3))
        nb[f"nb{case_id}_pos"] = pos
        nb[f"nb{case_id}_rc"] = np.array(rc)
        nb[f"nb{case_id}_edges"] = preprocess.build_cutoff_edges(pos, rc)
    recs = preprocess.generate_synthetic(6, seed=42)
    for k, v in _records_arrays(recs).items():
        nb[f"synth_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "neighbors.npz"), **nb)

    # 5. optimiser, schedule, ordered allreduce
    misc = dict(meta)
    r = np.random.default_rng(9)
    flat = r.normal(size=257)
    misc["adam_init"] = flat.copy()
    st = train.OptimizerState.zeros(257)
    tc = train.TrainConfig(optimizer="adam", learning_rate=1e-3)
    traj, grads = [], []
    for _ in range(5):
        g = r.normal(size=257) * 10.0 ** r.integers(-6, 2, size=257)
        grads.append(g)
        flat = train.apply_update(flat, g, tc, st)
        traj.append(flat.copy())
    misc["adam_grads"] = np.stack(grads)
    misc["adam_traj"] = np.stack(traj)
    sched = ddstore.epoch_schedule(103, 4, 8, 7, 3)
    misc["sched"] = np.concatenate([np.concatenate(b) for b in sched.per_rank])
    misc["sched_lens"] = np.array([[len(x) for x in b] + [0] * (4 - len(b)) for b in sched.per_rank])
    comms = comm.create_thread_comms(3)
    vecs = [r.normal(size=64) * 10.0 ** r.integers(-8, 8, size=64) for _ in range(3)]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(3) as pool:
        res = list(pool.map(lambda k: comms[k].allreduce_sum(vecs[k]), range(3)))
    misc["allreduce_in"] = np.stack(vecs)
    misc["allreduce_out"] = res[0]
    np.savez_compressed(os.path.join(OUT, "misc.npz"), **misc)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
