"""Does an L2 prefetch of a GEMM's weights make the GEMM faster?  O-proj /
QKV shapes: cold (L2 flushed), warm (second back-to-back run), and after a
tensor-tile or bulk prefetch (issued on the same stream, then a short spin)."""
import ctypes as C, sys, json
import torch
sys.path.insert(0, '.')
from paper_2605_29233_b200 import _lib

L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def timed(fn):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); fn(); b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3


for n_out, K in [(4096, 4096), (12288, 4096), (24576, 4096)]:
    rows, BN = 64, 64
    W = (torch.randn(n_out, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    X = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    need = C.c_longlong(0)
    L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), None, n_out, K, rows, BN, 0, 0, None,
                       C.byref(need), None, None, 0.0, 0.0, 0.0, None)
    work = torch.zeros(max(need.value, 1), device="cuda")
    out = torch.zeros(rows, n_out, device="cuda")

    def gemm():
        assert L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(out.data_ptr()),
                                  n_out, K, rows, BN, 0, 0, C.c_void_p(work.data_ptr()), None, None, None,
                                  0.5, 0.72, 33.0, C.c_void_p(s)) == 0

    def pf(kind):
        assert L.bb_debug_l2_prefetch(C.c_void_p(W.data_ptr()), n_out, K, kind, C.c_void_p(s)) == 0

    for _ in range(3):
        gemm()
    res = {"n_out": n_out, "K": K, "MB": n_out * K * 2 / 2**20}
    for name, prep in [("cold", lambda: flush.zero_()),
                       ("warm", lambda: gemm()),
                       ("pf_tile", lambda: (flush.zero_(), pf(0), torch.cuda._sleep(200000))),
                       ("pf_bulk", lambda: (flush.zero_(), pf(1), torch.cuda._sleep(200000))),
                       ("sleep_only", lambda: (flush.zero_(), torch.cuda._sleep(200000)))]:
        ts = []
        for _ in range(9):
            prep()
            torch.cuda.synchronize()
            ts.append(timed(gemm))
        res[name] = round(sorted(ts)[4], 2)
    print(json.dumps(res))
