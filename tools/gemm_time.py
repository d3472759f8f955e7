"""Time the C3 step's GEMM shapes on the tensor-core engine (CUDA events,
mean of 20 launches after warm-up) and report useful TFLOP/s.

    python tools/gemm_time.py            (GFM_TC_FLUSH_KB selects the flush depth)
"""

import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_12909_b200 import _lib  # noqa: E402
from paper_2406_12909_b200._lib import call, ptr, query, stream_handle  # noqa: E402


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
    return a.elapsed_time(b) / reps


def main():
    _lib.load(require_device=True)
    dev = torch.device("cuda")
    s = stream_handle()
    M, H, K = 51200, 512, 4
    h = torch.randn(M, H, device=dev)
    agg = torch.randn(M, K * H, device=dev)
    W, U = torch.randn(H, H, device=dev) * 0.04, torch.randn(H, K * H, device=dev) * 0.02
    b = torch.zeros(H, device=dev)
    Y = torch.empty(M, H, device=dev)
    dz = torch.randn(M, H, device=dev)
    dh, dagg = torch.empty(M, H, device=dev), torch.empty(M, K * H, device=dev)
    g1, g2, gb = torch.empty(H, H, device=dev), torch.empty(H, K * H, device=dev), torch.empty(H, device=dev)
    ws = torch.empty(query("gfm_linear_bwd_weight_workspace_bytes", M, H, H, K * H, 1, _lib.F32),
                     dtype=torch.uint8, device=dev)
    fl = 2.0 * M * H * (H + K * H)
    rows = {
        "fwd [h|agg] -> h (tanh)": (lambda: call(
            "gfm_linear_fwd", ptr(h), H, H, ptr(agg), K * H, K * H, ptr(W), H, ptr(U), K * H,
            ptr(b), M, None, H, 1, ptr(Y), H, _lib.F32, s), fl),
        "bwd-data dz -> [dh|dagg]": (lambda: call(
            "gfm_linear_bwd_data", ptr(dz), H, M, None, H, ptr(W), H, H, ptr(U), K * H, K * H,
            ptr(dh), H, ptr(dagg), K * H, None, 0, _lib.F32, s), fl),
        "wgrad dz^T [h|agg|1]": (lambda: call(
            "gfm_linear_bwd_weight", ptr(dz), H, M, None, H, ptr(h), H, H, ptr(agg), K * H, K * H,
            1, ptr(g1), ptr(g2), ptr(gb), ptr(ws), _lib.F32, s), fl + 2.0 * M * H),
    }
    print(f"GFM_TC_FLUSH_KB={os.environ.get('GFM_TC_FLUSH_KB', 'default')}")
    for name, (fn, flops) in rows.items():
        ms = timeit(fn)
        print(f"{name:28s} {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TF/s useful")


if __name__ == "__main__":
    main()
