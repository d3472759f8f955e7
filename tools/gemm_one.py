"""Run one GEMM shape/engine a few times (ncu target).
python tools/gemm_one.py MODE M K1 K2 N [pair]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_12909_b200 import _lib  # noqa: E402
from paper_2406_12909_b200._lib import call, ptr, stream_handle  # noqa: E402

mode, M, K1, K2, N = (int(x) for x in sys.argv[1:6])
_lib.load(require_device=True)
call("gfm_set_gemm_mode", mode)
dev = torch.device("cuda")
X1 = torch.randn(M, K1, device=dev)
X2 = torch.randn(M, K2, device=dev) if K2 else None
W1 = torch.randn(N, K1, device=dev)
W2 = torch.randn(N, K2, device=dev) if K2 else None
Y = torch.empty(M, N, device=dev)
for _ in range(3):
    call("gfm_linear_fwd", ptr(X1), K1, K1, ptr(X2), K2, K2, ptr(W1), K1, ptr(W2), K2, None, M, None,
         N, 0, ptr(Y), N, _lib.F32, stream_handle())
torch.cuda.synchronize()
print("ok")
