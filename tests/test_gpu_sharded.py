"""Sharded HBM store (DDStore's remote fetch over NVLink, ddstore.py:316-490):
a batch fetched collectively from the ranks' shards == make_batch of the
same records (model.py:234-285), bitwise; train() over the sharded store ==
train() packing the same batches on the host.  World size 1 always, 2 when
two GPUs are visible (NCCL all_to_all)."""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import gfm_oracle as O

pytestmark = pytest.mark.gpu

FIELDS_N1 = ("rowptr", "csc_ptr")
FIELDS_E = ("col_src", "edge_dst", "csc_eid", "csc_dst", "order", "edge_w", "edge_dx")


def _records(count, seed, n_range=(2, 14), periodic=False):
    from paper_2406_12909_b200.records import GraphRecord
    out = []
    rng = np.random.default_rng(seed + 100)
    for d in O.synthetic(count, n_atoms_range=n_range, seed=seed):
        r = GraphRecord(d["z"], d["pos"], d["edges"], d["energy"], d["forces"])
        if periodic:
            r.edge_shift = rng.integers(-1, 2, size=(r.edge_index.shape[0], 3)) * 4.0
        out.append(r)
    return out


def _compare(b, ref):
    assert b.n_nodes == ref.n_nodes and b.n_edges == ref.n_edges
    np.testing.assert_array_equal(b.host_offsets, ref.host_offsets)
    for k in ("z", "pos", "energy_true", "forces_true", "graph_of_node", "n_per_graph",
              "node_offsets") + FIELDS_N1 + FIELDS_E:
        x, y = getattr(b, k), getattr(ref, k)
        if k in FIELDS_E:
            x, y = x[:ref.n_edges], y[:ref.n_edges]
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy(), err_msg=k)


class _HostStore:
    def __init__(self, groups):
        self._g = groups
        self.ownership = {k: type("O", (), {"n_samples": len(v)})() for k, v in groups.items()}

    def fetch_batch(self, group, indices):
        return [self._g[group][int(i)] for i in indices]


@pytest.mark.parametrize("periodic", [False, True])
@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_sharded_fetch_single_rank_matches_make_batch(dtype, periodic):
    from paper_2406_12909_b200 import model as M
    from paper_2406_12909_b200.comm import LocalComm
    from paper_2406_12909_b200.store import ShardedDeviceStore
    recs = _records(30, 11, periodic=periodic)
    st = ShardedDeviceStore({"trainset": recs}, LocalComm())
    idx = [4, 29, 0, 4, 17, 9]
    _compare(st.fetch_device_batch("trainset", idx, dtype=dtype),
             M.make_batch([recs[i] for i in idx], dtype=dtype))
    assert st.fetch_device_batch("trainset", [], dtype=dtype) is None


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    import torch.distributed as dist

    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    out = {}
    try:
        from paper_2406_12909_b200 import model as M, train as T
        from paper_2406_12909_b200.comm import TorchComm
        from paper_2406_12909_b200.store import ShardedDeviceStore
        comm = TorchComm()
        recs = _records(41, 7)
        st = ShardedDeviceStore({"trainset": recs}, comm)
        lo, hi = st.ownership["trainset"].range_of(rank)
        out["shard"] = (lo, hi)
        # requests crossing both shards, duplicates, one rank idle in step 2
        all_reqs = [[[40, 0, 21, 20, 3, 40], [1, 39]], [[5, 6, 33], []]]
        reqs = all_reqs[rank]
        ok = []
        # exchanged requests, then the planned (global schedule) exchange
        for step, idx in enumerate(reqs + reqs):
            plan = [all_reqs[r][step % 2] for r in range(world)] if step >= 2 else None
            b = st.fetch_device_batch("trainset", idx, dtype=torch.float64, plan=plan)
            if not idx:
                ok.append(b is None)
                continue
            try:
                _compare(b, M.make_batch([recs[i] for i in idx], dtype=torch.float64))
                ok.append(True)
            except AssertionError as e:
                ok.append(str(e)[:400])
        out["fetch"] = ok
        # train() over the sharded store == train() over a host-packing store
        groups = {"trainset": recs[:33], "valset": recs[33:]}
        mc = M.ModelConfig(mpnn_kind="pna-agg", mpnn_layers=2, mpnn_width=16, fc_width=16,
                           batch_size=4)
        cfg = T.TrainConfig(max_epochs=2, patience=5)
        a = T.train(mc, ShardedDeviceStore(groups, comm), comm=comm, config=cfg,
                    dtype=torch.float64)
        b = T.train(mc, _HostStore(groups), comm=comm, config=cfg, dtype=torch.float64)
        out["train"] = (a.params.flatten(), b.params.flatten(),
                        [(m.train_loss, m.val_mae) for m in a.metrics],
                        [(m.train_loss, m.val_mae) for m in b.metrics])
        torch.cuda.synchronize()
        comm.barrier()
    except Exception as e:  # report, do not hang the peer
        out["error"] = repr(e)
    q.put((rank, out))
    q.close()
    q.join_thread()
    os._exit(0)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_sharded_fetch_two_ranks_nccl():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
    for r in (0, 1):
        assert "error" not in res[r], res[r].get("error")
        assert res[r]["fetch"] == [True] * 4, res[r]["fetch"]
    assert res[0]["shard"] == (0, 21) and res[1]["shard"] == (21, 41)
    pa, pb, ma, mb = res[0]["train"]
    np.testing.assert_array_equal(pa, pb)
    np.testing.assert_array_equal(pa, res[1]["train"][0])
    assert ma == mb
