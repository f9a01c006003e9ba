"""Run the C2 workload (LLaDA-8B shape, B={8,16,32}, P64, G256) and profile a
window of block-step iterations (cudaProfilerStart/Stop around them) so that
`ncu --profile-from-start off` captures exactly those kernels."""
import os, sys
sys.path.insert(0, '.')
import torch
import paper_2605_29233_b200 as bb
from paper_2605_29233_b200.scheduler import get_session

HS, GAMMA = float(os.environ.get("BB_HS", 0.4)), float(os.environ.get("BB_GAMMA", 8.0))
N_PROF = int(os.environ.get("BB_PROF_ITERS", 2))
_CFG = {"c2": (64, 256, (8, 16, 32)), "c5": (2048, 1024, (8, 16, 32, 64))}[os.environ.get("BB_TL_CFG", "c2")]
P, G = _CFG[0], _CFG[1]
vocab = bb.Vocab(size=bb.LLADA_8B_VOCAB)
cfg = bb.SchedulerConfig(block_sizes=_CFG[2], gen_len=G)
params = bb.build_model(0, vocab, bb.LLADA_8B, head_scale=HS, gamma=GAMMA, dtype=os.environ.get("BB_DTYPE", "bf16x2"),
                         init="hash")
task = bb.make_task(2, P, G, vocab)
s = get_session(params, cfg, P, 1)
s.set_inputs(task.prompt[None], task.target[None])
s.prefill()
use_graph = os.environ.get("BB_GRAPH", "0") == "1"
N_SKIP = int(os.environ.get("BB_PROF_SKIP", 5))  # iterations run before the profiled window
for it in range(1, N_SKIP + 1):
    s.iteration(it % cfg.refresh_interval == 0, use_graph)
s.stream.synchronize()
torch.cuda.profiler.start()
for it in range(N_SKIP + 1, N_SKIP + 1 + N_PROF):
    s.iteration(it % cfg.refresh_interval == 0, use_graph)
s.stream.synchronize()
torch.cuda.profiler.stop()
print("ctrl", s.v_ctrl[0, :24].tolist())
