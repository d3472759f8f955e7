"""Benchmark: training graphs/s of the data-parallel energy+force MTL step.

Headline workload (BASELINE.json configs[2], "C3", the north-star GFM-scale
target): HydraGNN-PNA stand-in -- pna-agg (sum|mean|max|std), 6 message-
passing layers, hidden 512, fc 2 x 512 -- on synthetic 100-atom periodic
crystals (12 A cubic cell, radius 5 A, max 32 neighbours), 512 graphs per
GPU per step.  Nested in the same line: ``c2`` (configs[1]: pna L3 H64,
1024 x 32-atom molecules, max 20 neighbours), ``ragged`` (C2 with 20..44
atoms per structure through the capacity-bucketed runner) and ``c4_egnn``
(configs[3]: the EGNN variant with autograd forces, 256 graphs).

A step = device batch assembly (radius graph -> CSR/CSC) from device-
resident raw structures + forward + backward + gradient allreduce (NCCL) +
Adam, captured once in a CUDA graph and replayed.  N > 1: one process per
GPU (torchrun), per-GPU batch fixed (weak scaling).  Synthetic structures
follow the reference's generate_synthetic (preprocess.py:107-153: same rng
call sequence, ToyPotential labels -- per-element constant + harmonic pairs
within the cutoff, forces its exact negative gradient).

    python bench.py [--gpus N --steps K --warmup W] [--config c3|c2]
                    [--impl reference] [--no-nested]

Prints ONE JSON line on rank 0.  ``--impl reference`` times the CPU side
instead: the numpy float64 oracle port of the reference step on the same
config over all host cores (the line's value), beside the reference's own
gfmkit data-parallel path (``scaling.run_strong_scaling(transport=
"process")``, mean-agg -- the reference has no PNA) when baseline/_ref holds
the installed reference.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]: the single-GPU kernel roofline config
    "c2": dict(kind="pna-agg", layers=3, hidden=64, fc_layers=2, fc_width=64, atoms=(32, 32),
               box=8.0, rc=5.0, max_nbr=20, batch=1024, periodic=False, cpu_sample=32,
               desc="C2: pna-agg L3 H64 fc2x64, 32-atom graphs, box 8 A, rc 5 A, max 20 "
                    "neighbours, 1024 graphs/GPU"),
    # BASELINE.json configs[2]: GFM scale, data parallel (the headline)
    "c3": dict(kind="pna-agg", layers=6, hidden=512, fc_layers=2, fc_width=512, atoms=(100, 100),
               box=12.0, rc=5.0, max_nbr=32, batch=512, periodic=True, cpu_sample=2,
               desc="C3: pna-agg L6 H512 fc2x512, 100-atom periodic crystals, 12 A cell, "
                    "rc 5 A, max 32 neighbours, 512 graphs/GPU"),
    # BASELINE.json configs[3]: EGNN variant, coordinate updates, autograd forces
    "c4": dict(kind="egnn", layers=3, hidden=64, fc_layers=2, fc_width=64, atoms=(32, 32),
               box=8.0, rc=5.0, max_nbr=20, batch=256, periodic=False, cpu_sample=8,
               desc="C4: EGNN L3 H64 fc2x64 (coordinate updates, forces = -dE/dx by "
                    "reverse-over-forward), 32-atom molecules, box 8 A, rc 5 A, max 20 "
                    "neighbours, 256 graphs/GPU"),
    # C2 with ragged structures (mean 32 atoms): the capacity-bucketed runner
    "c2r": dict(kind="pna-agg", layers=3, hidden=64, fc_layers=2, fc_width=64, atoms=(20, 44),
                box=8.0, rc=5.0, max_nbr=20, batch=1024, periodic=False, cpu_sample=32,
                desc="C2-ragged: as C2 with 20..44 atoms per structure (mean 32)"),
}
METRIC = "training graphs/sec (energy+forces MTL) at 1/2/4/8 B200; aggregation HBM GB/s"
UNIT = "graphs/s"
DTYPE = "f32 (3xTF32 tensor-core GEMMs, stated bound 5e-4 rel)"
# --gemm: engine code and the dtype label it puts on the line
GEMM_MODES = {
    "tc3": (1, DTYPE),
    "mixed": (3, "f32 (3xTF32 tensor-core GEMMs; weight-gradient GEMMs 1xTF32, bounds in "
                 "DESIGN.md section 4)"),
    "tc1": (2, "f32 storage, 1xTF32 tensor-core GEMMs (~1e-3 rel)"),
    "simt": (0, "f32 (IEEE fp32 FFMA GEMMs)"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--config", default="c3", choices=["c2", "c3"])
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--gemm", default="tc3", choices=list(GEMM_MODES),
                    help="float32 GEMM engine (gfm_set_gemm_mode)")
    ap.add_argument("--no-graph", action="store_true", help="disable CUDA-graph capture")
    ap.add_argument("--no-nested", action="store_true", help="skip the nested c2 / ragged lines")
    ap.add_argument("--cpu-sample-s", type=float, default=12.0)
    ap.add_argument("--ref-ranks", default="1,2,4,8,all",
                    help="rank counts of the reference's own DP timing (--impl reference)")
    return ap.parse_args()


# ---------------------------------------------------------------- synthetic data
def synthetic(count, W, seed):
    """generate_synthetic (preprocess.py:107-153): per structure n =
    integers(lo, hi + 1), species choice over {H, C, O}, positions uniform in
    the box; ToyPotential labels (preprocess.py:41-87: -0.1 Z per atom +
    sum over pairs within rc of (r - 1)^2, forces = -grad), vectorised.
    Returns (z list, pos list, energy array, forces list)."""
    lo, hi = W["atoms"]
    zs = np.array([1, 6, 8])
    rng = np.random.default_rng(seed)
    Z, P, E, F = [], [], np.zeros(count), []
    for g in range(count):
        n = int(rng.integers(lo, hi + 1))
        z = zs[rng.choice(3, size=n, p=np.full(3, 1.0 / 3.0))]
        pos = rng.uniform(0.0, W["box"], size=(n, 3))
        d = pos[:, None, :] - pos[None, :, :]
        r = np.sqrt((d ** 2).sum(axis=2))
        pair = np.triu(r <= W["rc"], 1)
        i, j = np.nonzero(pair)
        rr = r[i, j]
        e = float((-0.1 * z).sum() + ((rr - 1.0) ** 2).sum())
        gvec = (2.0 * (rr - 1.0) / np.maximum(rr, 1e-12))[:, None] * d[i, j]
        f = np.zeros((n, 3))
        np.add.at(f, i, -gvec)
        np.add.at(f, j, gvec)
        Z.append(z.astype(np.int32))
        P.append(pos)
        E[g] = e
        F.append(f)
    return Z, P, E, F


def packed(count, W, seed):
    Z, P, E, F = synthetic(count, W, seed)
    off = np.concatenate([[0], np.cumsum([len(z) for z in Z])]).astype(np.int32)
    return np.concatenate(Z), np.concatenate(P), E, np.concatenate(F), off


# ---------------------------------------------------------------- CPU legs
def _cpu_worker(args):
    seed, n_graphs, budget_s, W = args
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import gfm_oracle as O

    cfg = O.config(W["kind"], W["layers"], W["hidden"], W["fc_layers"], W["fc_width"])
    flat = O.init_flat(cfg, 0)
    m = np.zeros_like(flat)
    v = np.zeros_like(flat)
    Z, P, E, F = synthetic(n_graphs, W, seed)
    recs = []
    for g in range(n_graphs):
        cell = (W["box"],) * 3 if W["periodic"] else None
        edges, shift = O.cutoff_edges(P[g], W["rc"], max_nbr=W["max_nbr"], cell=cell)
        recs.append(dict(z=Z[g], pos=P[g], edges=edges, shift=shift, energy=E[g], forces=F[g]))
    steps, t = 0, 0
    t0 = time.perf_counter()
    while True:
        b = O.pack(recs)
        _, grad, _ = O.loss_and_grad(cfg, flat, b)
        flat, m, v, t = O.adam(flat, grad, m, v, t)
        steps += 1
        if time.perf_counter() - t0 >= budget_s:
            break
    return steps * n_graphs, time.perf_counter() - t0


def host_info():
    """cores used, CPU model and numpy / BLAS versions of this host"""
    info = dict(cores=len(os.sched_getaffinity(0)))
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    info["numpy"] = np.__version__
    try:
        from threadpoolctl import threadpool_info
        blas = [d for d in threadpool_info() if d.get("user_api") == "blas"]
        if blas:
            info["blas"] = f"{blas[0].get('internal_api')} {blas[0].get('version')}"
    except Exception:
        pass
    return info


def cpu_oracle_rate(budget_s, W, procs=None):
    """graphs/s of the numpy oracle step (make_batch + fwd + bwd + Adam, the
    reference's train.py:247-277 minus the fetch) over all host cores: one
    single-threaded process per core, each stepping its own sample."""
    import multiprocessing as mp

    procs = procs or len(os.sched_getaffinity(0))
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, [(1000 + k, W["cpu_sample"], budget_s, W)
                                     for k in range(procs)])
    graphs = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return graphs / wall, procs, (f"{procs} processes x {W['cpu_sample']}-graph samples of "
                                  f"the config (numpy float64 oracle port, "
                                  f"OPENBLAS_NUM_THREADS=1), ~{budget_s:.0f} s each")


def reference_dp(W, rank_counts, budget_s=8.0):
    """The reference's own data-parallel CPU path:
    gfmkit.scaling.run_strong_scaling(transport="process") over a container
    of gfmkit.generate_synthetic structures, OPENBLAS_NUM_THREADS =
    cores / ranks.  mean-agg (the reference has no PNA / cap / PBC: its
    edges are all pairs within rc in the non-periodic box)."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "gfmkit")):
        return dict(unavailable="baseline/_ref has no installed gfmkit")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import tempfile

    from gfmkit.container import write_container
    from gfmkit.model import ModelConfig
    from gfmkit.preprocess import generate_synthetic
    from gfmkit.scaling import run_strong_scaling

    cores = len(os.sched_getaffinity(0))
    counts = sorted({cores if c == "all" else int(c) for c in rank_counts if c})
    counts = [c for c in counts if c <= cores]
    lo, hi = W["atoms"]
    bs = W["cpu_sample"]
    # enough samples for every rank to take a few batches at the largest count
    n_total = max(counts) * bs * 2
    recs = generate_synthetic(n_total, n_atoms_range=(lo, hi), box_length=W["box"],
                              cutoff_radius=W["rc"], seed=0)
    mc = ModelConfig(mpnn_kind="mean-agg", mpnn_layers=W["layers"], mpnn_width=W["hidden"],
                     fc_layers=W["fc_layers"], fc_width=W["fc_width"], batch_size=bs)
    out = []
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "c")
        write_container({"trainset": recs, "valset": recs[:1], "testset": recs[:1]}, 4, path)
        for p in counts:
            os.environ["OPENBLAS_NUM_THREADS"] = str(max(1, cores // p))
            t0 = time.perf_counter()
            rep = run_strong_scaling(path, [p], mc, transport="process", warmup_epochs=1,
                                     scratch_dir=tmp, oversubscribe=False)
            pt = rep.points[0]
            epoch = max(t.epoch_time_s for t in pt.rank_timings)
            out.append(dict(ranks=p, blas_threads=max(1, cores // p), graphs=n_total,
                            epoch_s=epoch, value=n_total / epoch, lif=pt.lif["epoch"],
                            wait_fractions=pt.wait_fractions,
                            wall_s=time.perf_counter() - t0))
    best = max(out, key=lambda r: r["value"])
    return dict(value=best["value"], unit=UNIT, kind="reference", model="mean-agg (no PNA in "
                "the reference)", impl="gfmkit.scaling.run_strong_scaling(transport='process')",
                points=out,
                sample=f"{n_total} generate_synthetic structures ({lo}..{hi} atoms, box "
                       f"{W['box']} A, rc {W['rc']} A, uncapped, non-periodic), batch {bs}, "
                       "1 warm-up + 1 timed epoch per rank count", **host_info())


def run_reference(args, W):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    rate, cores, sample = cpu_oracle_rate(args.cpu_sample_s, W)
    try:
        dp = reference_dp(W, args.ref_ranks.split(","))
    except Exception as exc:  # the reference's harness failing must not lose the line
        dp = dict(unavailable=f"{type(exc).__name__}: {exc}")
    line = dict(metric=METRIC, value=rate, unit=UNIT, n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, higher_is_better=True, scaling="weak", vs_baseline=None,
                dtype="f64", data="synthetic", impl="reference",
                config=dict(workload=W["desc"], global_batch=W["batch"] * args.gpus),
                cpu_baseline=dict(value=rate, unit=UNIT, kind="port", sample=sample,
                                  **host_info()),
                reference_dp=dp,
                e2e=dict(value=rate, unit=UNIT, h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- clocks sampler
class ClockSampler:
    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._th.join(10)

    def summary(self):
        if not self.rows:
            return dict(sm_mhz=None, sm_max_mhz=None, reasons=["nvidia-smi unavailable"])
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        pw = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        return dict(sm_mhz=float(np.median(sm)) if sm else None,
                    sm_max_mhz=max(mx) if mx else None, reasons=reasons, samples=len(self.rows),
                    power_w=float(np.median(pw)) if pw else None)


# ---------------------------------------------------------------- native leg
class Ctx:
    """process-wide state shared by the measurements of one run"""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        from paper_2406_12909_b200 import _lib
        from paper_2406_12909_b200.comm import LocalComm, TorchComm

        self.args = args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
            self.comm = TorchComm()
        else:
            self.comm = LocalComm()
        _lib.load(require_device=True)
        self.peaks = {}
        try:
            self.peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        self.flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=self.dev)

    def barrier(self):
        if self.world > 1:
            self.comm.barrier()

    def max_over_ranks(self, x):
        import torch
        import torch.distributed as dist

        t = torch.tensor([float(x)], dtype=torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather(self, x):
        import torch
        import torch.distributed as dist

        t = torch.tensor([float(x)], dtype=torch.float64, device=self.dev)
        if self.world == 1:
            return [float(x)]
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t)
        return [float(o.item()) for o in out]

    def launch_ms(self, fn, stream, reps=20):
        """mean device time of fn (CUDA events on the launch stream, L2
        flushed before every launch)"""
        import torch

        for _ in range(3):
            fn()
        tot = 0.0
        for _ in range(reps):
            self.flush.zero_()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            fn()
            a1.record(stream)
            torch.cuda.synchronize()
            tot += a0.elapsed_time(a1)
        return tot / reps


def _trainer(ctx, W, B):
    from paper_2406_12909_b200 import model as M
    from paper_2406_12909_b200 import train as T

    cfg = M.ModelConfig(mpnn_kind=W["kind"], mpnn_layers=W["layers"], mpnn_width=W["hidden"],
                        fc_layers=W["fc_layers"], fc_width=W["fc_width"], batch_size=B)
    tr = T.DataParallelTrainer(cfg, T.TrainConfig(optimizer="adam", learning_rate=1e-3),
                               comm=ctx.comm, device=ctx.dev)
    return cfg, tr


def measure_step(ctx, W, full=True):
    """graphs/s of the captured step (inputs resident in HBM), e2e from
    pinned host buffers, e2e from the HBM sample store, and (full) the
    kernel rooflines, neighbour-list timing, launches and LIF."""
    import torch

    from paper_2406_12909_b200 import train as T

    args = ctx.args
    B = args.batch if (args.batch and W is CONFIGS[args.config]) else W["batch"]
    n = W["atoms"][1]
    N = B * n
    cfg, tr = _trainer(ctx, W, B)
    host_off = (np.arange(B + 1) * n).astype(np.int32)
    cells = [[W["box"]] * 3] * B if W["periodic"] else None
    runner = T.StructureStepRunner(tr, host_off, W["rc"], W["max_nbr"], cells=cells,
                                   use_graph=not args.no_graph)
    dev = ctx.dev
    pool = []
    for k in range(8):
        z, pos, energy, forces, _ = packed(B, W, 1000 * ctx.rank + k)
        pool.append(dict(z=torch.as_tensor(z, device=dev), pos=torch.as_tensor(pos, device=dev),
                         e=torch.as_tensor(energy, dtype=torch.float32, device=dev),
                         f=torch.as_tensor(forces, dtype=torch.float32, device=dev)))

    def load_slot(k):
        d = pool[k % len(pool)]
        runner.load(d["pos"], d["z"], d["e"], d["f"])

    s = torch.cuda.current_stream()
    load_slot(0)
    try:
        runner.capture(warmup=max(args.warmup, 3))
    except Exception as exc:  # e.g. a collective that refuses capture: run eagerly
        print(f"[bench] CUDA-graph capture failed ({exc}); eager launches", file=sys.stderr)
        runner.graph = None
        runner.use_graph = False
    for i in range(max(args.warmup, 3)):
        load_slot(i)
        runner.run()
    torch.cuda.synchronize()

    # ---- timed region: K steps, inputs already in HBM (8-batch pool)
    ctx.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(ctx.local) as clk:
        ev0.record(s)
        for i in range(args.steps):
            load_slot(i)
            runner.run()
        ev1.record(s)
        torch.cuda.synchronize()
    ctx.barrier()
    ms = ctx.max_over_ranks(ev0.elapsed_time(ev1))
    out = dict(value=ctx.world * B * args.steps / (ms / 1e3), ms_per_step=ms / args.steps,
               clocks=clk.summary(), per_gpu_batch=B, nodes_per_gpu=N,
               cuda_graph=runner.graph is not None)

    # ---- e2e: the public call (StructureStepRunner.step_pipelined) from pinned
    # host buffers: every step copies its inputs host->device and its loss back
    host = []
    for k in range(4):
        z, pos, energy, forces, _ = packed(B, W, 5000 + 1000 * ctx.rank + k)
        host.append(dict(z=torch.as_tensor(z).pin_memory(), pos=torch.as_tensor(pos).pin_memory(),
                         e=torch.as_tensor(energy, dtype=torch.float32).pin_memory(),
                         f=torch.as_tensor(forces, dtype=torch.float32).pin_memory()))
    h2d = sum(v.numel() * v.element_size() for v in host[0].values())
    d2h = runner.loss_host.numel() * runner.loss_host.element_size()

    def e2e_step(i):
        hb = host[i % len(host)]
        return runner.step_pipelined(hb["pos"], hb["z"], hb["e"], hb["f"])

    for i in range(2):
        e2e_step(i)
    runner.drain()
    ctx.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    losses = [e2e_step(i) for i in range(args.steps)]
    losses.append(runner.drain())
    torch.cuda.synchronize()
    assert all(x is not None and np.isfinite(x) for x in losses[1:]), losses
    e2e_s = ctx.max_over_ranks(time.perf_counter() - t0)
    out["e2e"] = dict(value=ctx.world * B * args.steps / e2e_s, unit=UNIT,
                      h2d_bytes_per_step=h2d, d2h_bytes_per_step=d2h,
                      note="StructureStepRunner.step_pipelined: pinned host inputs copied and "
                           "the loss read back every step (read one step late)")
    if not full:
        out["runner"] = runner
        return out

    # ---- e2e from the HBM-resident sample store: the
    # dataset is ingested once; per step only the B sample indices go
    # host->device and the loss comes back (read one step late)
    from paper_2406_12909_b200.store import DeviceStructureStore
    parts = [packed(B, W, 9000 + 1000 * ctx.rank + k) for k in range(8)]
    S = 8 * B
    store = DeviceStructureStore.from_arrays({"trainset": (
        np.concatenate([p[0] for p in parts]), np.concatenate([p[1] for p in parts]),
        np.concatenate([p[2] for p in parts]), np.concatenate([p[3] for p in parts]),
        np.arange(S + 1) * n)}, device=dev)
    rng = np.random.default_rng(77 + ctx.rank)
    loss_slots = [torch.empty(2, dtype=torch.float32).pin_memory() for _ in range(2)]
    loss_ev = [None, None]
    P = tr.P

    def store_step(i):
        store.load_runner("trainset", rng.choice(S, B, replace=False), runner)
        runner.run()
        k = i % 2
        loss_slots[k].copy_(tr.contrib[P:P + 2].float(), non_blocking=True)
        loss_ev[k] = torch.cuda.Event()
        loss_ev[k].record()
        j = 1 - k
        if loss_ev[j] is None:
            return None
        loss_ev[j].synchronize()
        return float(loss_slots[j][0]) / float(loss_slots[j][1])

    for i in range(3):
        store_step(i)
    ctx.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    slosses = [store_step(i) for i in range(args.steps)]
    loss_ev[(args.steps - 1) % 2].synchronize()
    torch.cuda.synchronize()
    assert all(x is not None and np.isfinite(x) for x in slosses), slosses
    st_s = ctx.max_over_ranks(time.perf_counter() - t0)
    out["e2e_device_store"] = dict(
        value=ctx.world * B * args.steps / st_s, unit=UNIT, h2d_bytes_per_step=4 * B,
        d2h_bytes_per_step=d2h,
        note="dataset resident in HBM (store.DeviceStructureStore); per step: B int32 sample "
             "indices H2D, loss D2H")
    del store

    # ---- sharded store (DDStore's remote fetch over NVLink, N > 1): every
    # rank holds 1/N of a group of these structures with 29 record edges per
    # atom; a batch of B random indices (mostly remote) is fetched by one
    # collective exchange (counts, indices, sizes, packed arrays by NCCL
    # all_to_all) and assembled into the CSR on the requester
    if ctx.world > 1:
        out["sharded_store_fetch"] = measure_sharded_fetch(ctx, W, B, n)

    # ---- load balance (scaling.py:54-72): each rank's compute time (batch
    # assembly + forward + backward, no collective) over its pool
    from paper_2406_12909_b200.telemetry import compute_lif, wait_fraction
    load_slot(0)
    runner._eager()
    torch.cuda.synchronize()
    b = runner.batch

    def compute_only():
        from paper_2406_12909_b200.model import radius_batch
        radius_batch(runner.slot["pos"], runner.slot["z"], runner.off, runner.host_off,
                     runner.rc, runner.max_nbr, runner.cells, runner.slot["e"], runner.slot["f"],
                     tr.dtype, e_cap=runner.e_cap, out=runner.bufs)
        tr.compute(b, scratch=runner.cur.scratch)

    busy = ctx.launch_ms(compute_only, s, reps=10)
    times = ctx.gather(busy)
    out["load_balance"] = dict(compute_ms_per_rank=times, lif=compute_lif(times),
                               wait_fraction=wait_fraction(times),
                               note="scaling.py:54-72 on each rank's device compute time")

    # ---- kernel rooflines (CUDA events on the launch stream, L2 flushed
    # before every launch) on this step's batch, with the step's own flags
    out.update(rooflines(ctx, W, cfg, b, s))

    # ---- neighbour lists, GPU batch assembly per graph
    from paper_2406_12909_b200 import model as M

    def nbr_call():
        M.radius_batch(runner.slot["pos"], runner.slot["z"], runner.off, runner.host_off,
                       runner.rc, runner.max_nbr, runner.cells, runner.slot["e"],
                       runner.slot["f"], tr.dtype, e_cap=runner.e_cap, out=runner.bufs)

    nbr_ms = ctx.launch_ms(nbr_call, s)
    out["neighbour_list"] = dict(gpu_ms_per_batch=nbr_ms, gpu_us_per_graph=nbr_ms * 1e3 / B,
                                 note="radius_batch on the step's input slots, L2 flushed")
    out["edges_per_gpu"] = b.n_edges

    # ---- launches per step (one extra untimed eager step under the profiler):
    # every kernel of this repository (gfm:: and tc:: namespaces)
    try:
        from torch.profiler import ProfilerActivity, profile

        load_slot(1)
        with tr.preserved():
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                runner._eager()
                torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        ours = [nm for nm in names if "gfm::" in nm or "tc::" in nm]
        out["gpu_launches"] = len(ours) * args.steps
        out["launches_per_step"] = len(ours)
    except Exception:
        out["gpu_launches"] = None
    out["runner"] = runner
    return out


def rooflines(ctx, W, cfg, b, s):
    """The aggregation kernels as the step runs them (uint8 argmax) and the
    largest GEMM, against MEASURED_PEAKS.json.  ``frac`` uses SURVEY 8(d)'s
    algorithmic bytes only."""
    import torch

    from paper_2406_12909_b200 import _lib
    from paper_2406_12909_b200 import model as M

    dev = ctx.dev
    N, E = b.n_nodes, b.n_edges
    H, K = cfg.mpnn_width, cfg.n_parts
    parts = M.KIND_PARTS[cfg.mpnn_kind]
    flags = M._argmax_flag(b)
    h_in = torch.randn(N, H, device=dev)
    agg = torch.empty(N, K * H, device=dev)
    am = torch.empty(N, H, dtype=torch.uint8 if flags & _lib.FLAG_ARGMAX_U8 else torch.int32, device=dev)
    sm_ = torch.empty(N, H, device=dev)
    dagg = torch.randn(N, K * H, device=dev)
    dh_b = torch.randn(N, H, device=dev)
    out_b = torch.empty(N, H, device=dev)
    ws_b = torch.empty(_lib.query("gfm_agg_bwd_workspace_bytes", N, H, parts, _lib.F32),
                       dtype=torch.uint8, device=dev)
    sh = _lib.stream_handle()
    P_ = _lib.ptr

    def agg_fwd_call():
        _lib.call("gfm_agg_fwd", P_(h_in), N, H, P_(b.rowptr), P_(b.col_src), P_(b.edge_w),
                  parts, P_(agg), P_(am), P_(sm_), _lib.F32, flags, sh)

    # the step's backward reads the edge weights in CSC order (GFM_FLAG_W_CSC)
    w_csc = torch.empty_like(b.edge_w)
    _lib.call("gfm_permute", P_(b.csc_eid), int(b.edge_w.shape[0]), P_(b.rowptr) + 4 * N,
              P_(b.edge_w), P_(w_csc), _lib.F32, sh)

    def agg_bwd_call():
        _lib.call("gfm_agg_bwd", P_(dagg), P_(agg), P_(sm_), P_(am), P_(h_in), P_(b.rowptr),
                  P_(b.csc_ptr), P_(b.csc_eid), P_(b.csc_dst), P_(w_csc), N, H, parts,
                  P_(dh_b), P_(h_in), P_(out_b), P_(ws_b), _lib.F32, flags | _lib.FLAG_W_CSC, sh)

    agg_fwd_call()
    # at H >= 256 the step computes the prep (G | coef, dmax) in the
    # backward-data GEMM's epilogue and launches the gather alone
    # (GFM_FLAG_AGG_PREPPED): time that launch; below, prep + gather
    prepped = H >= 256 and parts == 15 and os.environ.get("GFM_FUSED_PREP") != "0"
    agg_bwd_call()  # the prep pass fills G | coef in the workspace
    dmax = dagg.view(N, K, H)[:, 2].contiguous()

    def agg_bwd_gather():
        _lib.call("gfm_agg_bwd", P_(dmax), P_(agg), P_(sm_), P_(am), P_(h_in), P_(b.rowptr),
                  P_(b.csc_ptr), P_(b.csc_eid), P_(b.csc_dst), P_(w_csc), N, H, parts,
                  P_(dh_b), P_(h_in), P_(out_b), P_(ws_b), _lib.F32,
                  flags | _lib.FLAG_W_CSC | _lib.FLAG_AGG_PREPPED, sh)

    fwd_ms = ctx.launch_ms(agg_fwd_call, s)
    bwd_ms = ctx.launch_ms(agg_bwd_gather if prepped else agg_bwd_call, s)
    s4 = 4
    # SURVEY 8(d) C5 formulas, fused mode (ii), s = 4 bytes, pna (k = 4, max + std):
    # fwd: E*H*s + 4E (src) + 4E (w) + 4(N+1) + k*N*H*s + 4*N*H argmax
    fwd_bytes = E * H * s4 + 8 * E + 4 * (N + 1) + K * N * H * s4 + 4 * N * H
    # bwd (CSC gather): E*H*s + 8E + 4(N+1) + N*H*s + E*H*4 argmax (max) + E*H*s (std)
    bwd_bytes = E * H * s4 + 8 * E + 4 * (N + 1) + N * H * s4 + E * H * 4 + E * H * s4
    peak = float(ctx.peaks.get("hbm_gbs", 6550.0))
    l2 = {}
    traffic = {}
    try:
        l2 = json.load(open(os.path.join(ROOT, "profiles", "r01_l2_bw.json")))
    except Exception:
        pass
    name = "c3" if H >= 256 else "c2"
    for rnd in ("r02", "r01"):
        try:
            tr_ = json.load(open(os.path.join(ROOT, "profiles", f"{rnd}_agg_traffic_{name}.json")))
            # the captured launch must store argmax the same way (u8 or int32)
            if tr_.get("config") == name and (tr_.get("flags", 0) & 2) == (flags & 2):
                traffic = tr_
                break
        except Exception:
            continue

    def roof(kernel, nbytes, ms_, key, note):
        ach = nbytes / (ms_ / 1e3) / 1e9
        l2p = l2.get("l2_read_gbs")
        t = traffic.get(key)
        if key == "agg_bwd_dram_bytes" and prepped and traffic.get("kernels"):
            # the gather launch alone (the capture lists prep and gather)
            t = sum(k["dram_bytes"] for k in traffic["kernels"]
                    if "k_agg_bwd_vec" in k["name"]) or None
        return dict(kernel=kernel, bound="hbm", achieved=ach, peak=peak, unit="GB/s",
                    frac=ach / peak, traffic=t, launch_ms=ms_, algorithmic_bytes=nbytes,
                    dram_frac=(t / (ms_ / 1e3) / 1e9 / peak) if t else None,
                    traffic_source=traffic.get("source") if t else None,
                    l2_peak=l2p, l2_frac=ach / l2p if l2p else None,
                    peak_source="MEASURED_PEAKS.json hbm_gbs" if ctx.peaks else "fallback",
                    note=note)

    res = dict(
        roofline=roof("gfm_agg_bwd (pna CSC gather, uint8 argmax as in the step"
                      + ("; prep fused into the backward-data GEMM: the gather launch alone)"
                         if prepped else "; prep + gather)"), bwd_bytes,
                      bwd_ms, "agg_bwd_dram_bytes",
                      "frac = SURVEY 8(d) bwd bytes (argmax counted at 4 B/elem as 8(d) "
                      "states; the step stores 1 B) / time / HBM peak.  The per-edge row "
                      "gathers are mostly L2 hits: dram_frac is ncu's DRAM bytes / time"),
        roofline_agg_fwd=roof("gfm_agg_fwd (pna: sum|mean|max|std)", fwd_bytes, fwd_ms,
                              "agg_fwd_dram_bytes", "SURVEY 8(d) fwd bytes"))

    # ---- the largest GEMM: a layer's weight gradient [dW | dU | db] =
    # dz^T [h | agg | 1], M = N rows (split-K), 512 x (H + kH) outputs
    dz = torch.randn(N, H, device=dev)
    g1 = torch.empty(H, H, device=dev)
    g2 = torch.empty(H, K * H, device=dev)
    gb = torch.empty(H, device=dev)
    nb = _lib.query("gfm_linear_bwd_weight_workspace_bytes", N, H, H, K * H, 1, _lib.F32)
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)

    def wgrad_call():
        _lib.call("gfm_linear_bwd_weight", P_(dz), H, N, None, H, P_(h_in), H, H, P_(agg),
                  K * H, K * H, 1, P_(g1), P_(g2), P_(gb), P_(ws), _lib.F32, sh)

    wg_ms = ctx.launch_ms(wgrad_call, s)
    flops = 2.0 * N * H * (H + K * H + 1)
    tf = flops / (wg_ms / 1e3) / 1e12
    pk = float(ctx.peaks.get("bf16_tflops_sustained", 1379.5))
    res["roofline_gemm"] = dict(
        kernel="layer weight gradient (tcgen05 3xTF32 split-K + ordered reduce)", bound="tensor",
        achieved=tf, peak=pk, unit="TFLOP/s", frac=tf / pk, launch_ms=wg_ms,
        algorithmic_flops=flops, issued_tf32_tflops=3.0 * tf, issued_frac_of_tf32=3.0 * tf / (pk / 2),
        tensor_pipe_active="72% (ncu, profiles/r02_ncu_wgrad.txt)",
        note="useful fp32 flops; each product costs 3 TF32 MMAs (hi*hi + hi*lo + lo*hi); peak "
             "= MEASURED_PEAKS bf16 sustained; TF32 MMAs run at half the bf16 rate, so the "
             "issued TF32 rate is compared with peak / 2")
    return res


def measure_sharded_fetch(ctx, W, B, n):
    import torch

    from paper_2406_12909_b200.records import GraphRecord
    from paper_2406_12909_b200.store import ShardedDeviceStore
    S = 8 * B * ctx.world  # group size: 8 batches per rank
    own = None
    rng = np.random.default_rng(123)  # the same group on every rank
    from paper_2406_12909_b200.store import OwnershipMap
    own = OwnershipMap(S, ctx.world)
    lo, hi = own.range_of(ctx.rank)
    recs = []
    deg = 29
    for k in range(S):
        z, pos = rng.integers(1, 9, n), rng.uniform(0, W["box"], (n, 3))
        if lo <= k < hi:
            src = rng.integers(0, n, n * deg)
            dst = np.repeat(np.arange(n), deg)
            recs.append(GraphRecord(z, pos, np.stack([src, dst], 1), float(k), pos * 0.1))
    store = ShardedDeviceStore({"trainset": (recs, S)}, ctx.comm, device=ctx.dev)
    pick = np.random.default_rng(1000)  # the global schedule: every rank knows every batch
    steps = [[pick.choice(S, B, replace=False) for _ in range(ctx.world)] for _ in range(12)]
    res = {}
    for mode in ("exchanged", "planned"):
        for k in range(2):
            store.fetch_device_batch("trainset", steps[k][ctx.rank],
                                     plan=steps[k] if mode == "planned" else None)
        ctx.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(2, 12):
            b = store.fetch_device_batch("trainset", steps[k][ctx.rank],
                                         plan=steps[k] if mode == "planned" else None)
        torch.cuda.synchronize()
        res[mode] = ctx.max_over_ranks(time.perf_counter() - t0) / 10
    dt = res["planned"]
    # bytes a rank receives per batch: (N-1)/N of the structures are remote
    per_struct = n * (4 + 24 + 24) + 8 + n * deg * 8
    moved = B * per_struct * (ctx.world - 1) / ctx.world
    return dict(ms_per_batch=dt * 1e3, ms_per_batch_exchanged=res["exchanged"] * 1e3,
                batch=B, atoms=n, edges_per_atom=deg,
                remote_bytes_per_rank=moved, remote_gbs_per_rank=moved / dt / 1e9,
                nodes=b.n_nodes, edges=b.n_edges,
                note="store.ShardedDeviceStore.fetch_device_batch, wall time, max over ranks: "
                     "planned = the global schedule known to every rank (payload all_to_all "
                     "only, no host sync); exchanged = requests, counts exchanged first")


def measure_egnn(ctx, W):
    """C4: the EGNN variant's full training step (forward, forces by the
    reverse pass, loss, tangent forward, reverse over primal + tangent,
    allreduce, Adam) through the same captured runner."""
    import torch

    from paper_2406_12909_b200 import train as T
    from paper_2406_12909_b200.egnn import EGNNConfig

    args = ctx.args
    B, n = W["batch"], W["atoms"][1]
    cfg = EGNNConfig(egnn_layers=W["layers"], egnn_width=W["hidden"], fc_layers=W["fc_layers"],
                     fc_width=W["fc_width"], batch_size=B)
    tr = T.DataParallelTrainer(cfg, T.TrainConfig(optimizer="adam", learning_rate=1e-3),
                               comm=ctx.comm, device=ctx.dev)
    runner = T.StructureStepRunner(tr, (np.arange(B + 1) * n).astype(np.int32), W["rc"],
                                   W["max_nbr"], use_graph=not args.no_graph)
    dev = ctx.dev
    pool = []
    for k in range(4):
        z, pos, energy, forces, _ = packed(B, W, 7000 + 1000 * ctx.rank + k)
        pool.append((torch.as_tensor(pos, device=dev), torch.as_tensor(z, device=dev),
                     torch.as_tensor(energy, dtype=torch.float32, device=dev),
                     torch.as_tensor(forces, dtype=torch.float32, device=dev)))
    runner.load(*pool[0])
    runner.capture(warmup=3)
    for i in range(3):
        runner.load(*pool[i % 4])
        runner.run()
    ctx.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    for i in range(args.steps):
        runner.load(*pool[i % 4])
        runner.run()
    ev1.record(s)
    torch.cuda.synchronize()
    ms = ctx.max_over_ranks(ev0.elapsed_time(ev1))
    loss = float(tr.contrib[tr.P].item())
    assert np.isfinite(loss)
    return dict(value=ctx.world * B * args.steps / (ms / 1e3), unit=UNIT,
                ms_per_step=ms / args.steps, workload=W["desc"], params=tr.layout.P,
                note="EGNNConfig through DataParallelTrainer + StructureStepRunner (CUDA graph)")


def measure_ragged(ctx, W, fixed_value):
    """C2 with 20..44-atom structures (mean 32) through the ragged runner:
    two captured node capacities (mean + 4 sigma, and the maximum)."""
    import torch

    from paper_2406_12909_b200 import train as T

    args = ctx.args
    B = W["batch"]
    lo, hi = W["atoms"]
    _, tr = _trainer(ctx, W, B)
    sd = np.sqrt(((hi - lo + 1) ** 2 - 1) / 12.0) * np.sqrt(B)
    cap_q = int(np.ceil((B * (lo + hi) / 2 + 4 * sd) / 256.0) * 256)
    runner = T.StructureStepRunner(tr, None, W["rc"], W["max_nbr"], max_graphs=B,
                                   max_atoms=hi, node_caps=[min(cap_q, B * hi), B * hi],
                                   use_graph=not args.no_graph)
    dev = ctx.dev
    pool = []
    for k in range(8):
        z, pos, energy, forces, off = packed(B, W, 3000 + 1000 * ctx.rank + k)
        pool.append((torch.as_tensor(pos, device=dev), torch.as_tensor(z, device=dev),
                     torch.as_tensor(energy, dtype=torch.float32, device=dev),
                     torch.as_tensor(forces, dtype=torch.float32, device=dev), off))
    runner.load(*pool[0])
    runner.capture(warmup=3)
    for i in range(3):
        runner.load(*pool[i % 8])
        runner.run()
    ctx.barrier()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(s)
    for i in range(args.steps):
        runner.load(*pool[i % 8])
        runner.run()
    ev1.record(s)
    torch.cuda.synchronize()
    ms = ctx.max_over_ranks(ev0.elapsed_time(ev1))
    value = ctx.world * B * args.steps / (ms / 1e3)
    mean_atoms = float(np.mean([p[4][-1] for p in pool])) / B
    return dict(value=value, unit=UNIT, ms_per_step=ms / args.steps, workload=W["desc"],
                node_caps=[sh.N for sh in runner.shapes], mean_atoms_per_graph=mean_atoms,
                vs_fixed_c2=value / fixed_value if fixed_value else None,
                note="ragged runner (capacity buckets, device counts); same model and per-GPU "
                     "batch as C2; vs_fixed_c2 = this / the fixed-size C2 value")


def run_native(args):
    import torch

    ctx = Ctx(args)
    from paper_2406_12909_b200 import _lib
    _lib.call("gfm_set_gemm_mode", GEMM_MODES[args.gemm][0])
    W = CONFIGS[args.config]
    main = measure_step(ctx, W, full=True)
    main.pop("runner")
    nested = {}
    if not args.no_nested:
        torch.cuda.empty_cache()
        if args.config != "c2":
            c2 = measure_step(ctx, CONFIGS["c2"], full=False)
            c2.pop("runner")
            nested["c2"] = dict(value=c2["value"], unit=UNIT, ms_per_step=c2["ms_per_step"],
                                e2e=c2["e2e"], workload=CONFIGS["c2"]["desc"],
                                clocks=c2["clocks"])
            c2_value = c2["value"]
        else:
            c2_value = main["value"]
        nested["ragged"] = measure_ragged(ctx, CONFIGS["c2r"], c2_value)
        torch.cuda.empty_cache()
        nested["c4_egnn"] = measure_egnn(ctx, CONFIGS["c4"])
    if ctx.rank == 0:
        cpu = None
        if ctx.world == 1:
            rate, cores, sample = cpu_oracle_rate(args.cpu_sample_s, W)
            cpu = dict(value=rate, unit=UNIT, kind="port", sample=sample, **host_info())
        B = main["per_gpu_batch"]
        line = dict(
            metric=METRIC, value=main["value"], unit=UNIT, n_gpus=ctx.world, steps=args.steps,
            warmup=args.warmup, ms_per_step=main["ms_per_step"], higher_is_better=True,
            scaling="weak", vs_baseline=None, dtype=GEMM_MODES[args.gemm][1], data="synthetic",
            config=dict(workload=W["desc"], global_batch=B * ctx.world, per_gpu_batch=B,
                        nodes_per_gpu=main["nodes_per_gpu"], edges_per_gpu=main["edges_per_gpu"],
                        parallelism=f"dp{ctx.world}", cuda_graph=main["cuda_graph"],
                        gemm_engine=args.gemm,
                        l2=("step working set (activations, E x H workspaces) > 126 MB L2; "
                            "8-batch input pool cycled")),
            e2e=main["e2e"], e2e_device_store=main["e2e_device_store"],
            roofline=main["roofline"], roofline_agg_fwd=main["roofline_agg_fwd"],
            roofline_gemm=main["roofline_gemm"], neighbour_list=main["neighbour_list"],
            sharded_store_fetch=main.get("sharded_store_fetch"),
            load_balance=main["load_balance"], cpu_baseline=cpu, clocks=main["clocks"],
            gpu_launches=main["gpu_launches"], launches_per_step=main.get("launches_per_step"),
            **nested)
        print(json.dumps(line), flush=True)
    if ctx.world > 1:
        # A communicator captured inside a CUDA graph can block NCCL teardown;
        # every rank is done and rank 0 has printed, so leave without it.
        torch.cuda.synchronize()
        ctx.comm.barrier()
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args, CONFIGS[args.config])
    else:
        run_native(args)


if __name__ == "__main__":
    main()
