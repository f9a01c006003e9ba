"""tcgen05 GEMM + SIMT GEMM numerics vs a plain torch fp32 reference (GPU)."""

import ctypes as C

import pytest
import torch

from paper_2605_29233_b200 import _lib

pytestmark = pytest.mark.gpu


def _ptr(t):
    return C.c_void_p(t.data_ptr())


@pytest.mark.parametrize("n_out,K,rows,BN", [
    (256, 128, 64, 64), (768, 256, 64, 64), (4096, 4096, 56, 64), (12288, 4096, 64, 64),
    (1000, 320, 120, 128), (4097, 256, 192, 256), (4608, 3584, 320, 256), (4096, 12288, 64, 64)])
def test_tc_gemm_partials(n_out, K, rows, BN):
    torch.manual_seed(0)
    W = (torch.randn(n_out, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    rows_alloc = ((rows + BN - 1) // BN) * BN
    X = torch.zeros(rows_alloc, K, device="cuda", dtype=torch.bfloat16)
    X[:rows] = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    L = _lib.lib()
    need = C.c_longlong(0)
    rc = L.bb_debug_gemm_tc(_ptr(W), _ptr(X), None, n_out, K, rows_alloc, BN, 0, 0, None, C.byref(need),
                            None, None, 0.0, 0.0, 0.0, None)
    assert rc == 0
    work = torch.zeros(need.value, device="cuda")
    out = torch.zeros(rows_alloc, n_out, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    rc = L.bb_debug_gemm_tc(_ptr(W), _ptr(X), _ptr(out), n_out, K, rows_alloc, BN, 0, 0, _ptr(work), None,
                            None, None, 0.0, 0.0, 0.0, C.c_void_p(s))
    assert rc == 0
    torch.cuda.synchronize()
    ref = X.float() @ W.float().T
    err = (out - ref).abs().max().item()
    assert err < 2e-3 * max(1.0, ref.abs().max().item()), err


@pytest.mark.parametrize("n_out,K,rows,BN", [(4097, 256, 56, 64), (126463, 4096, 56, 64), (33, 256, 200, 256)])
def test_tc_gemm_head_epilogue(n_out, K, rows, BN):
    torch.manual_seed(1)
    W = (torch.randn(n_out, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    rows_alloc = ((rows + BN - 1) // BN) * BN
    X = torch.randn(rows_alloc, K, device="cuda").to(torch.bfloat16)
    tgt = torch.randint(0, n_out, (rows_alloc,), device="cuda", dtype=torch.int32)
    boost = torch.rand(rows_alloc, device="cuda") * 8
    hs, sc, sg = 0.5, 0.72, 33.0
    nt = (n_out + 127) // 128
    out = torch.zeros(rows_alloc, nt, 4, device="cuda")
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    rc = L.bb_debug_gemm_tc(_ptr(W), _ptr(X), _ptr(out), n_out, K, rows_alloc, BN, 1, 0, None, None,
                            _ptr(tgt), _ptr(boost), hs, sc, sg, C.c_void_p(s))
    assert rc == 0
    torch.cuda.synchronize()
    raw = (X.float() @ W.float().T) * hs
    lg = raw + sg * torch.clamp(raw - sc, min=0)
    lg[torch.arange(rows_alloc, device="cuda"), tgt.long()] += boost
    m = out[..., 0].max(1).values
    lse = m + torch.log((out[..., 2] * torch.exp(out[..., 0] - m[:, None])).sum(1))
    ref_lse = torch.logsumexp(lg, 1)
    assert (lse - ref_lse).abs().max().item() < 1e-2
    tile_best = out[..., 0].argmax(1)
    am = out[..., 1].contiguous().view(torch.int32)[torch.arange(rows_alloc), tile_best]
    ref_am = lg.argmax(1)
    agree = (am.long() == ref_am).float().mean().item()
    assert agree > 0.97, agree


def test_simt_gemm():
    torch.manual_seed(2)
    W = torch.randn(300, 200, device="cuda")
    X = torch.randn(70, 200, device="cuda")
    out = torch.zeros(70, 300, device="cuda")
    rc = _lib.lib().bb_debug_gemm_simt(_ptr(W), _ptr(X), _ptr(out), 300, 200, 70,
                                       C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    ref = X.double() @ W.double().T
    assert (out.double() - ref).abs().max().item() < 1e-3
