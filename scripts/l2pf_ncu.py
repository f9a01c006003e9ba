"""ncu target: flush, tile-prefetch a weight into L2, sleep, run the GEMM
(profile the GEMM's dram bytes).  argv[1] = prefetch kind (-1 = none)."""
import ctypes as C, sys
import torch
sys.path.insert(0, '.')
from paper_2605_29233_b200 import _lib
L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
kind = int(sys.argv[1])
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for n_out, K in [(4096, 4096), (24576, 4096)]:
    rows, BN = 64, 64
    W = (torch.randn(n_out, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    X = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    need = C.c_longlong(0)
    L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), None, n_out, K, rows, BN, 0, 0, None,
                       C.byref(need), None, None, 0.0, 0.0, 0.0, None)
    work = torch.zeros(max(need.value, 1), device="cuda")
    out = torch.zeros(rows, n_out, device="cuda")
    flush.zero_()
    torch.cuda._sleep(400000)
    if kind >= 0:
        assert L.bb_debug_l2_prefetch(C.c_void_p(W.data_ptr()), n_out, K, kind, C.c_void_p(s)) == 0
        torch.cuda._sleep(400000)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    assert L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(out.data_ptr()),
                              n_out, K, rows, BN, 0, 0, C.c_void_p(work.data_ptr()), None, None, None,
                              0.5, 0.72, 33.0, C.c_void_p(s)) == 0
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
