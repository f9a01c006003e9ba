"""Real (graph + PDL) per-kernel timeline of one request of a bench config
(BB_TL_CFG = c2 | c3 | c5, BB_TL_DTYPE = bf16 | bf16x2) from the device kernel
log (BB_KLOG=1): each kernel's slot = time from its predecessor's completion
to its own completion (next kernel's stamp)."""
import collections, json, os, sys
os.environ["BB_KLOG"] = "1"
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2605_29233_b200 as bb
from paper_2605_29233_b200.scheduler import get_session

# the bench's workload table (c2 / c3 / c5): same shapes, scheduler config, head_scale
import bench  # noqa: E402
_cfgd = bench.CONFIGS[os.environ.get("BB_TL_CFG", "c2")]
bb, params, cfg = bench.make_model(_cfgd, os.environ.get("BB_TL_DTYPE", "bf16"))
P, G = _cfgd["P"], _cfgd["G"]
vocab = params.vocab
R = int(os.environ.get("BB_TL_R", "1"))  # requests per session (multi-request batching)
if os.environ.get("BB_TL_TFLAGS"):  # session test flags (A/B: attention kernel / cluster size)
    from paper_2605_29233_b200.engine import Session
    s = Session(params, cfg, P, R, trace=False, test_flags=int(os.environ["BB_TL_TFLAGS"]))
else:
    s = get_session(params, cfg, P, R, trace=False)


def inputs(seed0):
    ts = [bb.make_task(seed0 + i, P, G, vocab) for i in range(R)]
    return np.stack([t.prompt for t in ts]), np.stack([t.target for t in ts])


for seed in (1000, 1001):
    s.set_inputs(*inputs(seed * 100)); s.launch()
s.stream.synchronize()
s.klog(reset=True); s.gemm_stats(reset=True)
import ctypes as _C; from paper_2605_29233_b200 import _lib as _L; _L.lib().bb_session_phase_stats(s.h, (_C.c_ulonglong * 16)(), 1, _C.c_void_p(s.stream.cuda_stream))
s.set_inputs(*inputs(100200))
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record(s.stream); it = s.launch(); ev1.record(s.stream); ev1.synchronize()
log = s.klog()
c = s.v_ctrl[0].cpu().numpy()
nfe = int(c[5] + c[6] + c[7])
nfe = max(nfe, it)  # (R > 1: iterations of the batch)
names = [n for n, _ in log]
ts = np.array([t for _, t in log], dtype=np.int64)
agg = collections.defaultdict(lambda: [0, 0])
for i in range(len(log) - 1):
    agg[names[i]][0] += 1
    agg[names[i]][1] += int(ts[i + 1] - ts[i])
tot = ts[-1] - ts[0]
print(f"request: {ev0.elapsed_time(ev1):.2f} ms event-timed, {tot/1e6:.2f} ms logged span, {len(log)} kernels, "
      f"{it} iterations, nfe {nfe} (split {c[5]},{c[6]},{c[7]})")
rows = sorted(agg.items(), key=lambda x: -x[1][1])
print(f"{'kernel':22s} {'n':>6s} {'total ms':>9s} {'per NFE us':>10s} {'avg us':>8s} {'share':>6s}")
for k, (n, ns) in rows:
    print(f"{k:22s} {n:6d} {ns/1e6:9.3f} {ns/1e3/nfe:10.1f} {ns/1e3/n:8.2f} {100*ns/tot:5.1f}%")
# largest gaps (host/graph boundaries)
d = np.diff(ts)
big = np.argsort(-d)[:8]
print("largest slots:", [(names[i], round(d[i] / 1e3, 1)) for i in big])
json.dump({"kernels": {k: {"n": n, "ns": ns} for k, (n, ns) in rows}, "nfe": nfe, "span_ns": int(tot)},
          open("gpurun_out/timeline_c2.json", "w"))
gs = s.gemm_stats()
for k, name in ((5, "attn block: duration after PDL wait"), (6, "attn block: CTA start spread"),
                (13, "attn full: duration after PDL wait"),
                (0, "gemm qkv"), (1, "gemm o"), (2, "gemm gate_up"), (3, "gemm down")):
    if gs[k][4]:
        print(f"live {name:40s} {gs[k][3] / gs[k][4] / 1e3:8.2f} us avg over {gs[k][4]} launches")
import ctypes as C
from paper_2605_29233_b200 import _lib
ph = (C.c_ulonglong * 16)()
_lib.lib().bb_session_phase_stats(s.h, ph, 0, C.c_void_p(s.stream.cuda_stream))
if ph[0]:
    names_ph = ["rows+keys loaded", "merge copies issued", "merge blocks received",
                "outputs stored", "chunk0 landed", "chunk loop done", "end"]
    print("attention phase offsets (avg us from PDL release): " +
          ", ".join(f"{n} {ph[i + 1] / ph[0] / 1e3:.2f}" for i, n in enumerate(names_ph)))

