"""HBM bandwidth of the tcgen05 weight-streaming GEMM vs number of CTAs."""
import ctypes as C, sys, json
import torch
sys.path.insert(0, '.')
from paper_2605_29233_b200 import _lib
L = _lib.lib()
def run(n_out, K, rows, grid, iters=20):
    W = (torch.randn(n_out, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    X = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    need = C.c_longlong(0)
    L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), None, n_out, K, rows, 64, 0, grid, None, C.byref(need), None, None, 0.0, 0.0, 0.0, None)
    work = torch.zeros(max(need.value, 1), device="cuda"); out = torch.zeros(rows, n_out, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    def call():
        return L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(out.data_ptr()), n_out, K, rows, 64, 0, grid, C.c_void_p(work.data_ptr()), None, None, None, 0.0, 0.0, 0.0, C.c_void_p(s))
    for _ in range(3): call()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(iters):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); call(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts) // 2]
    return n_out * K * 2 / 1e9 / (t / 1e3)
for g in (32, 64, 96, 128, 148):
    print(json.dumps({"grid": g, "GBps_gu": round(run(24576, 4096, 64, g)), "GBps_down": round(run(4096, 12288, 64, g))}), flush=True)
