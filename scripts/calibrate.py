"""Calibrate head_scale / gamma of the random-init LLaDA-8B-shape model so the
BlockBatch dynamics are non-degenerate (multi-token commits, merges, syncs) —
SURVEY §7 hard part 2.  Prints one JSON line per setting."""
import json, sys, time
sys.path.insert(0, '.')
import torch
import paper_2605_29233_b200 as bb

P, G = 64, 256
vocab = bb.Vocab(size=bb.LLADA_8B_VOCAB)
cfg = bb.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=G)
settings = [(float(a), float(b)) for a, b in (x.split(":") for x in sys.argv[1:])] or \
    [(0.05, 8.0), (0.1, 8.0), (0.2, 8.0), (0.3, 8.0), (0.5, 8.0), (1.0, 8.0)]
base = None
for hs, gamma in settings:
    t0 = time.time()
    params = bb.build_model(0, vocab, bb.LLADA_8B, head_scale=hs, gamma=gamma, dtype="bf16", init="hash")
    torch.cuda.synchronize()
    tb = time.time() - t0
    tasks = [bb.make_task(s, P, G, vocab) for s in range(4)]
    bb.run_batch(params, tasks[:1], cfg)  # warm (graph capture)
    res = []
    t1 = time.time()
    for t in tasks:
        res.append(bb.run_blockbatch(params, t, cfg))
    torch.cuda.synchronize()
    dt = time.time() - t1
    rec = {"head_scale": hs, "gamma": gamma, "build_s": round(tb, 2), "wall_s": round(dt, 3),
           "nfe": [list(r.nfe.snapshot()) for r in res], "tokens": [r.tokens_decoded for r in res],
           "merges": sum(r.stats["merges"] for r in res), "syncs": sum(r.stats["syncs"] for r in res),
           "commits": sum(r.stats["commits"] for r in res), "correct": sum(r.correct for r in res),
           "winner_bs": [r.block_size for r in res],
           "tok_per_s": round(sum(r.tokens_decoded for r in res) / dt, 1),
           "ms_per_nfe": round(1000 * dt / sum(r.nfe.total for r in res), 3)}
    print(json.dumps(rec), flush=True)
    del params
    torch.cuda.empty_cache()
