"""Accuracy + speed probe of the float32 GEMM engines (SIMT, tcgen05 3xTF32,
tcgen05 1xTF32) on the step's GEMM shapes, against a float64 torch reference.

    python tools/gemm_probe.py
"""

import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_12909_b200 import _lib  # noqa: E402
from paper_2406_12909_b200._lib import call, ptr, query, stream_handle  # noqa: E402

MODES = {"simt": 0, "tc3": 1, "tc1": 2}


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def rel_err(got, ref):
    return float((got.double() - ref).abs().max() / ref.abs().max())


def main():
    _lib.load(require_device=True)
    dev = torch.device("cuda")
    s = stream_handle()
    g = torch.Generator(device=dev).manual_seed(0)
    rows = []
    for (M, K1, K2, N) in [(32768, 64, 256, 64), (442390, 64, 0, 64), (51200, 512, 2048, 512)]:
        X1 = torch.randn(M, K1, device=dev, generator=g)
        X2 = torch.randn(M, K2, device=dev, generator=g) if K2 else None
        W1 = torch.randn(N, K1, device=dev, generator=g) / K1 ** 0.5
        W2 = torch.randn(N, K2, device=dev, generator=g) / max(K2, 1) ** 0.5 if K2 else None
        bias = torch.randn(N, device=dev, generator=g)
        Y = torch.empty(M, N, device=dev)
        Xc = X1.double() if X2 is None else torch.cat([X1, X2], 1).double()
        Wc = W1.double() if W2 is None else torch.cat([W1, W2], 1).double()
        ref = Xc @ Wc.T + bias.double()
        flops = 2.0 * M * N * (K1 + K2)
        for name, mode in MODES.items():
            call("gfm_set_gemm_mode", mode)

            def run():
                call("gfm_linear_fwd", ptr(X1), K1, K1, ptr(X2), K2, K2, ptr(W1), K1, ptr(W2), K2,
                     ptr(bias), M, None, N, 0, ptr(Y), N, _lib.F32, s)
            us = timeit(run)
            err = rel_err(Y, ref)
            rows.append((f"fwd M={M} K={K1 + K2} N={N}", name, us, flops / us / 1e6, err))
        # weight grad dW = dY^T X
        dY = torch.randn(M, N, device=dev, generator=g)
        g1 = torch.empty(N, K1, device=dev)
        g2 = torch.empty(N, K2, device=dev) if K2 else None
        gb = torch.empty(N, device=dev)
        ref1 = dY.double().T @ X1.double()
        for name, mode in MODES.items():
            call("gfm_set_gemm_mode", mode)
            ws = torch.empty(query("gfm_linear_bwd_weight_workspace_bytes", M, N, K1, K2, 1, _lib.F32),
                             dtype=torch.uint8, device=dev)

            def runw():
                call("gfm_linear_bwd_weight", ptr(dY), N, M, None, N, ptr(X1), K1, K1, ptr(X2), K2,
                     K2, 1, ptr(g1), ptr(g2), ptr(gb), ptr(ws), _lib.F32, s)
            us = timeit(runw, 5)
            rows.append((f"wgrad M={M} K={K1 + K2} N={N}", name, us, flops / us / 1e6,
                         rel_err(g1, ref1)))
    call("gfm_set_gemm_mode", 1)
    print(f"{'shape':40s} {'engine':6s} {'us':>9s} {'TFLOP/s':>8s} {'max rel err':>12s}")
    for r in rows:
        print(f"{r[0]:40s} {r[1]:6s} {r[2]:9.1f} {r[3]:8.1f} {r[4]:12.3e}")


if __name__ == "__main__":
    main()
