"""CTA-pair (cta_group::2) tcgen05 GEMMs == the single-CTA kernels, bitwise:
an M = 256 pair MMA accumulates every output element over the same k-steps
in the same order as two M = 128 MMAs.  Covers K-major operands (forward),
MN-major B (backward-data), MN-major A in TMEM (weight gradient, split-K),
odd M-tile counts (the pair's second CTA past the end), several column tiles,
and flushed accumulation (K > 512)."""

import numpy as np
import pytest
import torch

from paper_2406_12909_b200 import _lib

pytestmark = pytest.mark.gpu
P = _lib.ptr


def _rand(*shape, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.randn(*shape, device="cuda", generator=g)


def _both(fn, pairs_expected=None):
    """fn() with the single-CTA kernels, then with CTA pairs (asserting
    whether the pair kernel ran)"""
    outs = []
    for on in (0, 1):
        prev = _lib.query("gfm_set_tc_pairs", on)
        n0 = _lib.query("gfm_tc_pair_launches")
        try:
            outs.append([t.cpu().numpy() for t in fn()])
        finally:
            _lib.query("gfm_set_tc_pairs", prev)
        ran = _lib.query("gfm_tc_pair_launches") > n0
        assert ran == (bool(on) and bool(pairs_expected)) or pairs_expected is None, (on, ran)
    return outs


# (pairs run for K >= 512: the shallower shapes check the single-CTA path is
# still chosen and unchanged)
@pytest.mark.parametrize("M,K1,K2,N", [(1000, 96, 0, 128), (300, 512, 2048, 512), (129, 64, 448, 64),
                                       (4096, 640, 0, 96), (1000, 512, 0, 128)])
def test_pair_forward_bitwise(M, K1, K2, N):
    X1, X2 = _rand(M, K1, seed=1), _rand(M, max(K2, 1), seed=2)
    W1, W2 = _rand(N, K1, seed=3), _rand(N, max(K2, 1), seed=4)
    b = _rand(N, seed=5)
    s = _lib.stream_handle()

    def run():
        Y = torch.empty(M, N, device="cuda")
        _lib.call("gfm_linear_fwd", P(X1), K1, K1, P(X2) if K2 else None, K2, K2, P(W1), K1,
                  P(W2) if K2 else None, K2, P(b), M, None, N, 1, P(Y), N, _lib.F32, s)
        torch.cuda.synchronize()
        return [Y]

    (a,), (c,) = _both(run, pairs_expected=K1 + K2 >= 512 and M > 128)
    np.testing.assert_array_equal(a, c)


@pytest.mark.parametrize("M,N,K1,K2", [(1000, 512, 128, 512), (333, 640, 64, 0), (300, 128, 64, 64)])
def test_pair_backward_data_bitwise(M, N, K1, K2):
    dY = _rand(M, N, seed=6)
    W1, W2 = _rand(N, K1, seed=7), _rand(N, max(K2, 1), seed=8)
    gate = torch.tanh(_rand(M, K1, seed=9))
    s = _lib.stream_handle()

    def run():
        o1, o2 = torch.empty(M, K1, device="cuda"), torch.empty(M, max(K2, 1), device="cuda")
        _lib.call("gfm_linear_bwd_data", P(dY), N, M, None, N, P(W1), K1, K1,
                  P(W2) if K2 else None, K2, K2, P(o1), K1, P(o2) if K2 else None, K2, P(gate),
                  K1, _lib.F32, s)
        torch.cuda.synchronize()
        return [o1, o2] if K2 else [o1]

    a, c = _both(run, pairs_expected=N >= 512 and M > 128)
    for x, y in zip(a, c):
        np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("M,N,K1,K2,bias", [(5000, 128, 128, 512, 1), (2000, 64, 64, 0, 0)])
def test_pair_weight_gradient_bitwise(M, N, K1, K2, bias):
    dY = _rand(M, N, seed=10)
    X1, X2 = _rand(M, K1, seed=11), _rand(M, max(K2, 1), seed=12)
    s = _lib.stream_handle()
    ws = torch.empty(_lib.query("gfm_linear_bwd_weight_workspace_bytes", M, N, K1, K2, bias,
                                _lib.F32), dtype=torch.uint8, device="cuda")

    def run():
        g1, g2 = torch.empty(N, K1, device="cuda"), torch.empty(N, max(K2, 1), device="cuda")
        gb = torch.empty(N, device="cuda")
        _lib.call("gfm_linear_bwd_weight", P(dY), N, M, None, N, P(X1), K1, K1,
                  P(X2) if K2 else None, K2, K2, bias, P(g1), P(g2) if K2 else None,
                  P(gb) if bias else None, P(ws), _lib.F32, s)
        torch.cuda.synchronize()
        return [g1] + ([g2] if K2 else []) + ([gb] if bias else [])

    a, c = _both(run, pairs_expected=False)  # weight gradients stay single-CTA
    for x, y in zip(a, c):
        np.testing.assert_array_equal(x, y)
    ref = dY.double().T @ X1.double()
    assert float((torch.as_tensor(c[0], device="cuda").double() - ref).abs().max()
                 / ref.abs().max()) < 1e-5
