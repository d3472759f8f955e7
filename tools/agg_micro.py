"""aggregation microbenchmark.

E in {1, 4, 16, 64, 100}M edges (--max-e), H in {64, 128, 256, 512},
N = E/16; dst uniform then sorted (Poisson(16) degrees), src uniform
("random") or within +-64 of dst ("block-local"); values N(0,1) fp32,
seed 0.  Times gfm_agg_fwd and gfm_agg_bwd (prep + CSC gather) with CUDA
events, L2 flushed before every launch, and reports GB/s by the SURVEY 8(d)
formulas (algorithmic bytes) against MEASURED_PEAKS.json's HBM copy rate.

Two modes:
 (ii) fused  -- h[N, H] + src + w: the step's kernels gather h[src] rows;
 (i)  materialised -- msg[E, H] already formed (PyG scatter style, sum): the
      same kernels with every edge its own source row (col_src = identity,
      w = 1), so the forward streams msg once in CSR order and the backward
      writes dmsg[E, H] (one row per edge).
Configurations whose buffers would exceed --mem-gb are skipped (e.g. mode
(i) at 100M x 512: msg alone is 205 GB).
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
ap.add_argument("--max-e", type=int, default=100, help="largest E in millions")
ap.add_argument("--mem-gb", type=float, default=120.0, help="skip configs above this footprint")
ap.add_argument("--modes", default="fused,materialised")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--e-list", default=None, help="comma list of E in millions (default: all <= --max-e)")
ap.add_argument("--patterns", default="random,block-local")
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
    # the backward reads the weights in CSC order as the step does
    # (GFM_FLAG_W_CSC; GFM_W_CSC=0: w[eid] gathers)
    w_csc = os.environ.get("GFM_W_CSC", "1") != "0"
    return N, dict(rowptr=t(rowptr), col_src=t(src), w=t(w, torch.float32), csc_ptr=t(csc_ptr),
                   csc_eid=t(csc), csc_dst=t(dst[csc]), max_deg=int(np.diff(rowptr).max()),
                   w_bwd=t(w[csc] if w_csc else w, torch.float32),
                   w_flag=_lib.FLAG_W_CSC if w_csc else 0)


def identity_graph(E, g):
    """mode (i): node e = edge e's message row (CSR order), w = 1"""
    rowptr = g["rowptr"]
    N = rowptr.shape[0] - 1
    iota = torch.arange(E, dtype=torch.int32, device=dev)
    dst = torch.repeat_interleave(torch.arange(N, device=dev, dtype=torch.int32),
                                  (rowptr[1:] - rowptr[:-1]).long())
    return dict(rowptr=rowptr, col_src=iota, w=torch.ones(E, device=dev),
                csc_ptr=torch.arange(E + 1, dtype=torch.int32, device=dev), csc_eid=iota,
                csc_dst=dst, max_deg=g["max_deg"], n_rows=E, n_dst=N)


def materialised(E, H, g, kind, parts, K, u8):
    """mode (i): aggregate E precomputed message rows (fwd) and write the
    E dmsg rows (bwd) -- one streaming pass each"""
    ig = identity_graph(E, g)
    N = ig["n_dst"]
    msg = torch.randn(E, H, device=dev)
    agg = torch.empty(N, K * H, device=dev)
    am = torch.empty(N, H, dtype=torch.uint8 if u8 else torch.int32, device=dev) \
        if parts & _lib.PART_MAX else None
    sm = torch.empty(N, H, device=dev) if parts & _lib.PART_STD else None
    dagg = torch.randn(N, K * H, device=dev)
    dmsg = torch.zeros(E, H, device=dev)
    out = torch.empty(E, H, device=dev)
    ws = torch.empty(_lib.query("gfm_agg_bwd_workspace_bytes", N, H, parts, _lib.F32),
                     dtype=torch.uint8, device=dev)

    def fwd():
        _lib.call("gfm_agg_fwd", P(msg), N, H, P(ig["rowptr"]), P(ig["col_src"]), P(ig["w"]),
                  parts, P(agg), P(am), P(sm), _lib.F32, u8, sh)

    def bwd():
        _lib.call("gfm_agg_bwd", P(dagg), P(agg), P(sm), P(am), P(msg), P(ig["rowptr"]),
                  P(ig["csc_ptr"]), P(ig["csc_eid"]), P(ig["csc_dst"]), P(ig["w"]), E, H, parts,
                  P(dmsg), None, P(out), P(ws), _lib.F32, u8, sh)

    tf, tb = timeit(fwd), timeit(bwd)
    # (i): fwd reads msg (E H s) + rowptr + K N H s out; bwd reads the dst
    # rows of G (+ coef, argmax) per edge and writes E H s dmsg
    fb = E * H * 4 + 4 * (N + 1) + K * N * H * 4
    bb = E * H * 4 + E * H * 4 + 8 * E
    if parts & _lib.PART_STD:
        bb += E * H * 4 * 2  # coef rows + the msg values
    if parts & _lib.PART_MAX:
        bb += E * H * (1 if u8 else 4)
    r = dict(E=E, H=H, src="materialised", kind=kind, fwd_us=tf * 1e6, bwd_us=tb * 1e6,
             fwd_gbs=fb / tf / 1e9, bwd_gbs=bb / tb / 1e9, fwd_frac=fb / tf / 1e9 / peak,
             bwd_frac=bb / tb / 1e9 / peak, mode="materialised")
    print(f"E={E // 1000000:3d}M H={H:3d} {'(i) msg[E,H]':11s} {kind:3s}  fwd {tf * 1e6:9.1f} us "
          f"{r['fwd_gbs']:7.0f} GB/s ({r['fwd_frac']:.2f})  bwd {tb * 1e6:9.1f} us "
          f"{r['bwd_gbs']:7.0f} GB/s ({r['bwd_frac']:.2f})", flush=True)
    del msg, agg, am, sm, dagg, dmsg, out, ws, ig
    torch.cuda.empty_cache()
    return r


rows = []
rng = np.random.default_rng(0)
modes = a.modes.split(",")
E_LIST = [int(x) for x in a.e_list.split(",")] if a.e_list else \
    [m for m in (1, 4, 16, 64, 100) if m <= a.max_e]
for Em in E_LIST:
    E = Em * 1_000_000
    for pattern in a.patterns.split(","):
        N, g = graph(E, pattern, rng)
        for H in (64, 128, 256, 512):
            for kind, parts in (("sum", _lib.PART_SUM), ("pna", 15)):
                K = bin(parts).count("1")
                u8 = _lib.FLAG_ARGMAX_U8 if g["max_deg"] <= 256 else 0
                # footprint: h, agg, dagg, dh, out, argmax, std mean, G + coef
                fp = 4 * N * H * (1 + K + K + 2 + 1 + 2) + N * H
                # (i) is the PyG scatter-sum baseline: one message row per edge,
                # sum only (the kernels' node count is the source count, so the
                # dst-side prep of mean/std/max needs the fused layout)
                if "materialised" in modes and pattern == "random" and kind == "sum" and \
                        E * H * 4 * 3 + 4 * N * H * (2 * K + 3) < a.mem_gb * 1e9:
                    rows.append(materialised(E, H, g, kind, parts, K, u8))
                if "fused" not in modes or fp > a.mem_gb * 1e9:
                    continue
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
                              P(g["csc_ptr"]), P(g["csc_eid"]), P(g["csc_dst"]), P(g["w_bwd"]), N,
                              H, parts, P(dh), None, P(out), P(ws), _lib.F32, u8 | g["w_flag"],
                              sh)

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
                r = dict(E=E, H=H, src=pattern, kind=kind, mode="fused", fwd_us=tf * 1e6,
                         bwd_us=tb * 1e6,
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
