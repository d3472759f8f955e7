"""Event-timed (CUDA-graph replay) sweep of the tcgen05 linear forward over (M, K) at N = 64 / 128
(warm L2, 20 reps) -- separates per-launch overhead from per-k-block cost.
python tools/gemm_sweep.py [mode]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_12909_b200 import _lib  # noqa: E402
from paper_2406_12909_b200._lib import call, ptr, stream_handle  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
_lib.load(require_device=True)
call("gfm_set_gemm_mode", mode)
dev = torch.device("cuda")
s = stream_handle()
for N in (64, 128):
    for M in (4096, 32768, 131072):
        for K in (32, 64, 320, 1024):
            X = torch.randn(M, K, device=dev)
            W = torch.randn(N, K, device=dev)
            Y = torch.empty(M, N, device=dev)

            def run():
                call("gfm_linear_fwd", ptr(X), K, K, None, 0, 0, ptr(W), K, None, 0, None, M,
                     None, N, 0, ptr(Y), N, _lib.F32, stream_handle())
            for _ in range(3):
                run()
            torch.cuda.synchronize()
            # graph-captured so host launch cost does not leak into the timing
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(20):
                    run()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            print(f"N={N:4d} M={M:7d} K={K:5d}  {us:8.1f} us  {M * K * 4 / us / 1e3:7.0f} GB/s(A)")
