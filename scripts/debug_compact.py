"""A/B of block-pass compaction in batched sessions (tiny model): test flags
0 (compaction, fixed-piece GEMMs over the live row chunks), 256 (same pieces,
every chunk: must be bitwise equal to 0), 8 (static layout, classic
stream-K: equal up to summation order); per-request NFE."""
import sys
sys.path.insert(0, '.')
import paper_2605_29233_b200 as bb
from paper_2605_29233_b200.engine import Session
from paper_2605_29233_b200.scheduler import _cfg_key
dims = bb.ModelDims(layers=2, d_model=256, max_len=192, arch="llada", n_heads=2, n_kv_heads=2, head_dim=128,
                    d_ff=512, rope_theta=500000.0)
vocab = bb.Vocab(size=1000)
cfg = bb.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=64)
for R in (4, 8):
    tasks = [bb.make_task(s, 32, 64, vocab) for s in range(R)]
    for dt in ("bf16x2", "bf16"):
        for flags in (0, 256, 8):
            p = bb.build_model(0, vocab, dims, head_scale=0.25, dtype=dt)
            p._sessions[_cfg_key(cfg, 32, R, True)] = Session(p, cfg, 32, R, test_flags=flags)
            rs = bb.run_batch(p, tasks, cfg)
            print(R, dt, flags, [sum(r.nfe.snapshot()) for r in rs], flush=True)
