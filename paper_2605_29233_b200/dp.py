"""Request-level data parallelism over GPUs (one process per GPU).

BlockBatch requests are independent: prompts are sharded
round-robin over ranks, every rank runs its shard with its own replica of the
weights, and there is no collective on the per-step path.  The only exchange
is one all-gather of the per-request results at the end (tokens, NFE triple,
winner, decoded count) so rank 0 can report — a few KB regardless of model
size.  Works with any torch.distributed backend (NCCL on the GPUs, gloo in the
CPU tests).
"""

from __future__ import annotations

import numpy as np


def shard(n_items: int, rank: int, world: int) -> list[int]:
    """Round-robin request indices owned by `rank` (deterministic, balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return list(range(rank, n_items, world))


def pack_results(results, L: int) -> np.ndarray:
    """[n, L + 6] int64 rows: tokens | nfe0 nfe1 nfe2 | winner | tokens_decoded | eos (-1 = None)."""
    out = np.full((len(results), L + 6), -1, dtype=np.int64)
    for i, r in enumerate(results):
        out[i, :L] = r.row.tokens[:L]
        out[i, L:L + 3] = r.nfe.snapshot()
        out[i, L + 3] = r.branch_index
        out[i, L + 4] = r.tokens_decoded
        out[i, L + 5] = -1 if r.eos_position is None else r.eos_position
    return out


def gather_results(local: np.ndarray, n_items: int, rank: int, world: int, device="cpu") -> np.ndarray:
    """All-gather the packed per-request rows of every rank and put them back in
    request order (one collective, end of run)."""
    import torch
    import torch.distributed as dist
    width = local.shape[1]
    per = (n_items + world - 1) // world
    buf = torch.full((per, width), -2, dtype=torch.int64, device=device)
    if len(local):
        buf[:len(local)] = torch.from_numpy(local).to(device)
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf)
    out = np.empty((n_items, width), dtype=np.int64)
    for r in range(world):
        g = gathered[r].cpu().numpy()
        for j, idx in enumerate(shard(n_items, r, world)):
            out[idx] = g[j]
    return out
