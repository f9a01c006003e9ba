"""Profile one prefill (full pass) of an R-request LLaDA-8B-shape session so that
`ncu --profile-from-start off` captures exactly its kernels (BB_DTYPE, BB_R)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_2605_29233_b200 as bb
from paper_2605_29233_b200.scheduler import get_session

R = int(os.environ.get("BB_R", 1))
vocab = bb.Vocab(size=bb.LLADA_8B_VOCAB)
cfg = bb.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=256)
params = bb.build_model(0, vocab, bb.LLADA_8B, head_scale=0.4, gamma=8.0, dtype=os.environ.get("BB_DTYPE", "bf16x2"),
                         init="hash")
tasks = [bb.make_task(2 + i, 64, 256, vocab) for i in range(R)]
s = get_session(params, cfg, 64, R)
s.set_inputs(np.stack([t.prompt for t in tasks]), np.stack([t.target for t in tasks]))
s.prefill()
s.stream.synchronize()
torch.cuda.profiler.start()
s.prefill()
s.stream.synchronize()
torch.cuda.profiler.stop()
print("ok")
