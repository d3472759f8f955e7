"""aggregation microbenchmark (fused mode: h[N,H] + src + w).

E in {1, 4, 16}M edges (python tools/agg_micro.py --max-e 64 adds 64M),
H in {64, 128, 256, 512}, N = E/16; dst uniform then sorted (Poisson(16)
degrees), src uniform ("random") or within +-64 of dst ("block-local");
values N(0,1) fp32, seed 0.  Times gfm_agg_fwd and gfm_agg_bwd (prep +
CSC gather) with CUDA events, L2 flushed before every launch, and reports
GB/s by the SURVEY 8(d) formulas (algorithmic bytes; the per-edge row
gathers are mostly L2 hits, so the fraction of HBM peak can exceed 1).
The materialised-msg mode (i) is not implemented: the kernels never form
E x H messages.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_12909_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-e", type=int, default=16, help="largest E in millions")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--json", default=None)
a = ap.parse_args()
_lib.load(require_device=True)
dev = torch.device("cuda")
P = _lib.ptr
sh = _lib.stream_handle()
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6540.8
flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)


def timeit(fn):
    fn()
    tot = 0.0
    for _ in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / a.reps / 1e3  # seconds


def graph(E, pattern, rng):
    N = max(E // 16, 1)
    dst = np.sort(rng.integers(0, N, E)).astype(np.int64)
    if pattern == "random":
        src = rng.integers(0, N, E)
    else:
        src = np.clip(dst + rng.integers(-64, 65, E), 0, N - 1)
    rowptr = np.zeros(N + 1, np.int64)
    np.add.at(rowptr, dst + 1, 1)
    rowptr = np.cumsum(rowptr)
    w = (1.0 / (1.0 + rng.uniform(0.5, 5.0, E))).astype(np.float32)
    csc = np.argsort(src, kind="stable")
    csc_ptr = np.zeros(N + 1, np.int64)
    np.add.at(csc_ptr, src + 1, 1)
    csc_ptr = np.cumsum(csc_ptr)
    t = lambda x, dt=torch.int32: torch.as_tensor(np.ascontiguousarray(x)).to(dtype=dt, device=dev)
    return N, dict(rowptr=t(rowptr), col_src=t(src), w=t(w, torch.float32), csc_ptr=t(csc_ptr),
                   csc_eid=t(csc), csc_dst=t(dst[csc]), max_deg=int(np.diff(rowptr).max()))


rows = []
rng = np.random.default_rng(0)
for Em in [m for m in (1, 4, 16, 64) if m <= a.max_e]:
    E = Em * 1_000_000
    for pattern in ("random", "block-local"):
        N, g = graph(E, pattern, rng)
        for H in (64, 128, 256, 512):
            if E * H * 4 > 40e9:
                continue
            for kind, parts in (("sum", _lib.PART_SUM), ("pna", 15)):
                K = bin(parts).count("1")
                u8 = _lib.FLAG_ARGMAX_U8 if g["max_deg"] <= 256 else 0
                h = torch.randn(N, H, device=dev)
                agg = torch.empty(N, K * H, device=dev)
                am = torch.empty(N, H, dtype=torch.uint8 if u8 else torch.int32, device=dev) \
                    if parts & _lib.PART_MAX else None
                sm = torch.empty(N, H, device=dev) if parts & _lib.PART_STD else None
                dagg = torch.randn(N, K * H, device=dev)
                dh = torch.randn(N, H, device=dev)
                out = torch.empty(N, H, device=dev)
                ws = torch.empty(_lib.query("gfm_agg_bwd_workspace_bytes", N, H, parts, _lib.F32),
                                 dtype=torch.uint8, device=dev)

                def fwd():
                    _lib.call("gfm_agg_fwd", P(h), N, H, P(g["rowptr"]), P(g["col_src"]),
                              P(g["w"]), parts, P(agg), P(am), P(sm), _lib.F32, u8, sh)

                def bwd():
                    _lib.call("gfm_agg_bwd", P(dagg), P(agg), P(sm), P(am), P(h), P(g["rowptr"]),
                              P(g["csc_ptr"]), P(g["csc_eid"]), P(g["csc_dst"]), P(g["w"]), N, H,
                              parts, P(dh), None, P(out), P(ws), _lib.F32, u8, sh)

                tf, tb = timeit(fwd), timeit(bwd)
                # SURVEY 8(d) C5 formulas (s = 4)
                fb = E * H * 4 + 8 * E + 4 * (N + 1) + K * N * H * 4
                if parts & _lib.PART_MAX:
                    fb += 4 * N * H
                if parts & _lib.PART_STD:
                    fb += 4 * N * H
                bb = E * H * 4 + 8 * E + 4 * (N + 1) + N * H * 4
                if parts & _lib.PART_MAX:
                    bb += E * H * (1 if u8 else 4)
                if parts & _lib.PART_STD:
                    bb += E * H * 4
                r = dict(E=E, H=H, src=pattern, kind=kind, fwd_us=tf * 1e6, bwd_us=tb * 1e6,
                         fwd_gbs=fb / tf / 1e9, bwd_gbs=bb / tb / 1e9,
                         fwd_frac=fb / tf / 1e9 / peak, bwd_frac=bb / tb / 1e9 / peak)
                rows.append(r)
                print(f"E={Em:3d}M H={H:3d} {pattern:11s} {kind:3s}  fwd {tf * 1e6:9.1f} us "
                      f"{r['fwd_gbs']:7.0f} GB/s ({r['fwd_frac']:.2f})  bwd {tb * 1e6:9.1f} us "
                      f"{r['bwd_gbs']:7.0f} GB/s ({r['bwd_frac']:.2f})", flush=True)
                del h, agg, am, sm, dagg, dh, out, ws
        del g
        torch.cuda.empty_cache()
if a.json:
    json.dump(dict(peak_gbs=peak, rows=rows), open(a.json, "w"), indent=1)
