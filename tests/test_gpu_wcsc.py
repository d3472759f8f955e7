"""GFM_FLAG_W_CSC: the aggregation backward reading the edge weights in CSC
order (w_csc = edge_w[csc_eid], gfm_permute) is bitwise the same as reading
w[eid] through the CSC edge ids -- every kernel family (scalar fp64, float4
rows, column slabs, smem tiles), u8 and int32 argmax."""

import numpy as np
import pytest
import torch

from test_gpu_parity import F32, F64, _wide_batch

from paper_2406_12909_b200 import _lib, model as M

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tile", [False, True])
@pytest.mark.parametrize("u8", [False, True])
@pytest.mark.parametrize("kind", ["pna-agg", "sum-agg", "mean-agg"])
@pytest.mark.parametrize("H,dtype", [(16, F32), (64, F32), (512, F32), (64, F64)])
def test_w_csc_bitwise(H, dtype, kind, u8, tile, monkeypatch):
    if tile:
        monkeypatch.setenv("GFM_AGG_TILE", "1")
    parts, K = M.KIND_PARTS[kind], M._n_parts(kind)
    code = _lib.F64 if dtype == F64 else _lib.F32
    flags = (_lib.FLAG_ARGMAX_U8 if u8 else 0) | (_lib.FLAG_SCALAR if dtype == F64 else 0)
    _, b = _wide_batch(H, dtype, 3, True)
    N, E = b.n_nodes, b.n_edges
    rg = np.random.default_rng(H)
    t = lambda *shape: torch.as_tensor(rg.normal(size=shape), dtype=dtype, device="cuda")
    h, dagg, dh, gate = t(N, H), t(N, K * H), t(N, H), t(N, H)
    agg = torch.empty(N, K * H, dtype=dtype, device="cuda")
    am = torch.empty(N, H, dtype=torch.uint8 if u8 else torch.int32, device="cuda")
    sm = torch.empty(N, H, dtype=dtype, device="cuda")
    s = _lib.stream_handle()
    P = _lib.ptr
    _lib.call("gfm_agg_fwd", P(h), N, H, P(b.rowptr), P(b.col_src), P(b.edge_w), parts, P(agg),
              P(am), P(sm), code, flags, s)
    w_csc = torch.full_like(b.edge_w, float("nan"))
    _lib.call("gfm_permute", P(b.csc_eid), E, P(b.rowptr) + 4 * N, P(b.edge_w), P(w_csc), code, s)
    np.testing.assert_array_equal(w_csc.cpu().numpy(),
                                  b.edge_w[b.csc_eid.long()].cpu().numpy())
    ws = torch.empty(_lib.query("gfm_agg_bwd_workspace_bytes", N, H, parts, code),
                     dtype=torch.uint8, device="cuda")
    outs = []
    for w, extra in ((b.edge_w, 0), (w_csc, _lib.FLAG_W_CSC)):
        out = torch.empty(N, H, dtype=dtype, device="cuda")
        _lib.call("gfm_agg_bwd", P(dagg), P(agg), P(sm), P(am), P(h), P(b.rowptr), P(b.csc_ptr),
                  P(b.csc_eid), P(b.csc_dst), P(w), N, H, parts, P(dh), P(gate), P(out), P(ws),
                  code, flags | extra, s)
        outs.append(out.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
