"""Time the tcgen05 stream-K GEMM on the LLaDA-8B layer shapes (bandwidth)."""
import ctypes as C, sys, json
import torch
sys.path.insert(0, '.')
from paper_2605_29233_b200 import _lib

def run(n_out, K, rows, BN, mode=0, iters=20):
    W = (torch.randn(n_out, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    X = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
    L = _lib.lib(); need = C.c_longlong(0)
    L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), None, n_out, K, rows, BN, mode, 0, None, C.byref(need), None, None, 0.0, 0.0, 0.0, None)
    work = torch.zeros(max(need.value, 1), device="cuda")
    nt = (n_out + 127)//128
    out = torch.zeros(rows, n_out if mode == 0 else nt*4, device="cuda")
    tgt = torch.zeros(rows, dtype=torch.int32, device="cuda"); boost = torch.zeros(rows, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    def call():
        return L.bb_debug_gemm_tc(C.c_void_p(W.data_ptr()), C.c_void_p(X.data_ptr()), C.c_void_p(out.data_ptr()), n_out, K, rows, BN, mode, 0, C.c_void_p(work.data_ptr()), None, C.c_void_p(tgt.data_ptr()), C.c_void_p(boost.data_ptr()), 0.5, 0.72, 33.0, C.c_void_p(s))
    for _ in range(3): assert call() == 0
    ts = []
    for _ in range(iters):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); call(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts)//2]
    gb = n_out*K*2/1e9
    return {"n_out": n_out, "K": K, "rows": rows, "BN": BN, "mode": mode, "ms": t, "GBps": gb/(t/1e3)}

res = []
for shp in [(12288, 4096, 64, 64), (4096, 4096, 64, 64), (24576, 4096, 64, 64), (4096, 12288, 64, 64), (126464, 4096, 64, 64), (12288, 4096, 320, 256), (24576, 4096, 320, 256)]:
    res.append(run(*shp))
    if shp[0] == 126464: res.append(run(*shp, mode=1))
for r in res: print(json.dumps(r))
