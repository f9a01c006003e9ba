"""N>1 request-parallel host logic over torch.distributed (gloo, world size 2, CPU)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2605_29233_b200 import dp


class _R:
    def __init__(self, seed, L):
        rng = np.random.default_rng(seed)
        self.row = type("Row", (), {"tokens": rng.integers(0, 50, size=L)})()
        self.nfe = type("N", (), {"snapshot": lambda s, v=seed: (1, 10 + v, v % 3)})()
        self.branch_index = seed % 3
        self.tokens_decoded = 100 + seed
        self.eos_position = None if seed % 2 else seed + 5


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, L, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = dp.shard(n, rank, world)
    local = dp.pack_results([_R(i, L) for i in mine], L)
    allr = dp.gather_results(local, n, rank, world)
    if rank == 0:
        q.put(allr)
    dist.barrier()
    dist.destroy_process_group()


def test_shard_balanced_and_complete():
    for n in (1, 7, 8, 256):
        for w in (1, 2, 3, 8):
            parts = [dp.shard(n, r, w) for r in range(w)]
            assert sorted(i for p in parts for i in p) == list(range(n))
            assert max(map(len, parts)) - min(map(len, parts)) <= 1


def test_gather_results_world2_gloo():
    n, L, world = 7, 12, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = dp.pack_results([_R(i, L) for i in range(n)], L)
    np.testing.assert_array_equal(got, want)
