"""Run one GEMM shape/engine a few times (ncu target).
python tools/gemm_one.py fwd|wgrad|bwd MODE M K1 K2 N"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_12909_b200 import _lib  # noqa: E402
from paper_2406_12909_b200._lib import call, ptr, query, stream_handle  # noqa: E402

kind = sys.argv[1]
mode, M, K1, K2, N = (int(x) for x in sys.argv[2:7])
_lib.load(require_device=True)
call("gfm_set_gemm_mode", mode)
dev = torch.device("cuda")
X1 = torch.randn(M, K1, device=dev)
X2 = torch.randn(M, K2, device=dev) if K2 else None
W1 = torch.randn(N, K1, device=dev)
W2 = torch.randn(N, K2, device=dev) if K2 else None
dY = torch.randn(M, N, device=dev)
Y = torch.empty(M, N, device=dev)
s = stream_handle()
ws = torch.empty(query("gfm_linear_bwd_weight_workspace_bytes", M, N, K1, K2, 1, _lib.F32),
                 dtype=torch.uint8, device=dev)
g1, g2, gb = torch.empty(N, K1, device=dev), torch.empty(N, max(K2, 1), device=dev), torch.empty(N, device=dev)
o1, o2 = torch.empty(M, K1, device=dev), torch.empty(M, max(K2, 1), device=dev)
for _ in range(3):
    if kind == "fwd":
        call("gfm_linear_fwd", ptr(X1), K1, K1, ptr(X2), K2, K2, ptr(W1), K1, ptr(W2), K2, None, M,
             None, N, 0, ptr(Y), N, _lib.F32, s)
    elif kind == "wgrad":
        call("gfm_linear_bwd_weight", ptr(dY), N, M, None, N, ptr(X1), K1, K1, ptr(X2), K2, K2, 1,
             ptr(g1), ptr(g2), ptr(gb), ptr(ws), _lib.F32, s)
    else:
        call("gfm_linear_bwd_data", ptr(dY), N, M, None, N, ptr(W1), K1 + K2, K1, ptr(W2), K1 + K2, K2,
             ptr(o1), K1, ptr(o2), max(K2, 1), None, 0, _lib.F32, s)
torch.cuda.synchronize()
print("ok")
