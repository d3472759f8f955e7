"""Does the tcgen05 kind::tf32 MMA truncate or round its fp32 smem operands?

Y = X W^T on the 3xTF32 engine, against float64, for (a) random fp32 inputs,
(b) the same inputs with the WEIGHT operand (B, read raw from shared memory)
pre-truncated to tf32 (low 13 bits zero: hi = x, lo = 0 exactly), (c) with
X (A, split in registers) pre-truncated, (d) both.  If the hardware
truncates, (a) is as accurate as (b); if it rounds, (a) carries an extra
~2^-12 relative bias from B.

    python tools/tf32_probe.py
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2406_12909_b200 import _lib  # noqa: E402
from paper_2406_12909_b200._lib import call, ptr, stream_handle  # noqa: E402


def trunc(t):
    return (t.view(torch.int32) & -8192).view(torch.float32)


def rn(t):  # round to nearest (ties away) to tf32
    i = t.view(torch.int32)
    return ((i + 4096) & -8192).view(torch.float32)


def main():
    _lib.load(require_device=True)
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    M, K, N = 8192, 2560, 512
    X = torch.randn(M, K, device=dev, generator=g)
    W = torch.randn(N, K, device=dev, generator=g) / K ** 0.5
    s = stream_handle()
    for mode, mname in ((1, "tc3"), (0, "simt"), (2, "tc1")):
        call("gfm_set_gemm_mode", mode)
        for xa, wa, label in ((X, W, "raw A, raw B"), (X, trunc(W), "raw A, trunc B"),
                              (trunc(X), W, "trunc A, raw B"), (X, rn(W), "raw A, rn B"),
                              (trunc(X), trunc(W), "trunc A, trunc B")):
            Y = torch.empty(M, N, device=dev)
            call("gfm_linear_fwd", ptr(xa), K, K, None, 0, 0, ptr(wa), K, None, 0, None, M, None,
                 N, 0, ptr(Y), N, _lib.F32, s)
            ref = xa.double() @ wa.double().T
            err = (Y.double() - ref)
            print(f"{mname:5s} {label:18s} max|err|/max|ref| {err.abs().max() / ref.abs().max():.3e}"
                  f"  mean(err)/rms(ref) {err.mean() / ref.pow(2).mean().sqrt():+.3e}"
                  f"  rms(err)/rms(ref) {err.pow(2).mean().sqrt() / ref.pow(2).mean().sqrt():.3e}")
    call("gfm_set_gemm_mode", 1)
    # bias check in the other role: W^T-shaped op (weight gradient, both MN-major)
    dY = torch.randn(M, N, device=dev, generator=g)
    for xa, label in ((X[:, :512].contiguous(), "raw"), (trunc(X[:, :512].contiguous()), "trunc X")):
        g1 = torch.empty(N, 512, device=dev)
        ws = torch.empty(_lib.query("gfm_linear_bwd_weight_workspace_bytes", M, N, 512, 0, 0,
                                    _lib.F32), dtype=torch.uint8, device=dev)
        call("gfm_linear_bwd_weight", ptr(dY), N, M, None, N, ptr(xa), 512, 512, None, 1, 0, 0,
             ptr(g1), None, None, ptr(ws), _lib.F32, s)
        ref = dY.double().T @ xa.double()
        err = g1.double() - ref
        print(f"wgrad {label:8s} max|err|/max|ref| {err.abs().max() / ref.abs().max():.3e}  "
              f"rms(err)/rms(ref) {err.pow(2).mean().sqrt() / ref.pow(2).mean().sqrt():.3e}")


if __name__ == "__main__" and len(sys.argv) == 1:
    main()


def k_scan():
    """relative error of exact-tf32 inputs vs K (accumulator precision)"""
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1)
    s = stream_handle()
    M, N = 8192, 256
    for K in (32, 64, 128, 256, 512, 1024, 2560, 8192):
        X = trunc(torch.randn(M, K, device=dev, generator=g))
        W = trunc(torch.randn(N, K, device=dev, generator=g) / K ** 0.5)
        ref = X.double() @ W.double().T
        for mode, mname in ((1, "tc3"), (0, "simt")):
            call("gfm_set_gemm_mode", mode)
            Y = torch.empty(M, N, device=dev)
            call("gfm_linear_fwd", ptr(X), K, K, None, 0, 0, ptr(W), K, None, 0, None, M, None,
                 N, 0, ptr(Y), N, _lib.F32, s)
            err = Y.double() - ref
            rr = ref.pow(2).mean().sqrt()
            print(f"K={K:5d} {mname:5s} rms(err)/rms(ref) {err.pow(2).mean().sqrt() / rr:.3e} "
                  f"bias toward zero {-(err * ref.sign()).mean() / rr:+.3e}")
    call("gfm_set_gemm_mode", 1)


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "k":
    k_scan()
