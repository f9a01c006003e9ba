"""Multi-request batching on one GPU (SURVEY 8(f1), config C4's per-GPU shard):
R requests of the LLaDA-8B-shape model stacked into one device session, every
iteration one forward over all live requests' branch windows.  Prints one JSON
line per R: decoded tokens/s (device time, inputs resident), NFE/request and
ms per iteration.

    python scripts/batch_bench.py [R ...]      (default: 1 4 8 16 32)
"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_29233_b200 as bb  # noqa: E402
from paper_2605_29233_b200.scheduler import get_session  # noqa: E402

P, G = 64, 256
Rs = [int(a) for a in sys.argv[1:]] or [1, 4, 8, 16, 32]
vocab = bb.Vocab(size=bb.LLADA_8B_VOCAB)
cfg = bb.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=G)
params = bb.build_model(0, vocab, bb.LLADA_8B, head_scale=0.4, gamma=8.0, dtype="bf16")
for R in Rs:
    s = get_session(params, cfg, P, R, trace=False)
    tasks = [bb.make_task(5000 + i, P, G, vocab) for i in range(R)]
    prompts = torch.tensor(np.stack([t.prompt for t in tasks]).astype(np.int32), device="cuda")
    targets = torch.tensor(np.stack([t.target for t in tasks]).astype(np.int32), device="cuda")
    s.set_inputs(prompts, targets)
    s.launch()  # warmup (graph capture)
    s.stream.synchronize()
    tasks = [bb.make_task(7000 + i, P, G, vocab) for i in range(R)]
    prompts = torch.tensor(np.stack([t.prompt for t in tasks]).astype(np.int32), device="cuda")
    targets = torch.tensor(np.stack([t.target for t in tasks]).astype(np.int32), device="cuda")
    s.set_inputs(prompts, targets)
    s.stream.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(s.stream)
    it = s.launch()
    e1.record(s.stream)
    e1.synchronize()
    wall = time.perf_counter() - t0
    ms = e0.elapsed_time(e1)
    res = s.results(tasks, vocab)
    tok = sum(r.tokens_decoded for r in res)
    nfe = [r.nfe.total for r in res]
    print(json.dumps({"requests": R, "decoded_tokens": tok, "device_ms": round(ms, 2), "wall_s": round(wall, 3),
                      "tokens_per_s": round(tok / (ms / 1e3), 1), "iterations": it,
                      "ms_per_iteration": round(ms / it, 3), "nfe_per_request_mean": float(np.mean(nfe)),
                      "block_rows_per_step": R * 56}), flush=True)
