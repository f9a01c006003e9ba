"""Step-operator seams of the reference API, on the device.

The reference exposes its forward as module-level functions that the
scheduler (and user code, and its tests) call directly:
``full_forward`` / ``block_forward`` (model.py:322-343),
``init_full_forward`` (scheduler.py:80-89) and ``batched_block_forward``
(scheduler.py:116-131).  Here each is one call into the C-ABI library on a
*seam session*: one request whose branches own private KV pages and whose
head slots can hold a whole row, so any window fits.  Caches move in and out
as ``KvCache`` objects backed by CUDA fp32 vectors (bb_kv_scatter /
bb_kv_gather), logits are materialised by the LM head (bb_head_logits) --
the only place full logits exist; the fused step never writes them.
"""

from __future__ import annotations

import numpy as np

from .errors import ContractError, StateError


def _torch():
    import torch
    return torch


def _seam_session(params, L: int, P: int, nb: int):
    from .engine import Session
    from .scheduler import SchedulerConfig
    key = ("seam", L, P, nb)
    s = params._sessions.get(key)
    if s is None:
        if L - P < 1:
            raise ContractError("a row needs a non-empty generation region")
        cfg = SchedulerConfig(block_sizes=tuple(L + i for i in range(nb)), gen_len=L - P)
        s = Session(params, cfg, P, 1, trace=False, seam=True)
        s.seam_init()
        params._sessions[key] = s
    return s


def _check_len(params, row):
    if len(row) > params.dims.max_len:  # model.py:286-287
        raise ContractError(f"sequence length {len(row)} exceeds max_len {params.dims.max_len}")


def _check_target(row, target):
    if target is not None and len(target) != len(row) - row.prompt_len:  # model.py:249-253
        raise ContractError("target length does not match the generation region")


def _check_block(row, cache, window):
    L = len(row)
    if window.start < 0 or window.end > L:  # model.py:336-337
        raise ContractError(f"window {window} out of bounds for length {L}")
    outside = np.ones(L, dtype=bool)
    outside[window.start:window.end] = False
    if not np.asarray(cache.valid)[outside].all():  # model.py:339-342
        raise StateError("cache invalid outside the active window")


def _load_row(s, k: int, row, start: int, end: int):
    torch = _torch()
    with torch.cuda.stream(s.stream):
        s.v_tokens[0, k].copy_(torch.from_numpy(np.asarray(row.tokens, dtype=np.int32)), non_blocking=False)
        s.v_branch[0, k, 0] = int(start)
        s.v_branch[0, k, 1] = int(end)


def _load_target(s, target):
    torch = _torch()
    if target is not None:
        with torch.cuda.stream(s.stream):
            s.v_target[0].copy_(torch.from_numpy(np.asarray(target, dtype=np.int32)), non_blocking=False)


def _load_cache(s, k: int, cache, params):
    d = params.dims
    want = (d.layers, s.Lseq, d.n_kv_heads * d.hd)
    if tuple(cache.shape) != want:
        raise ContractError(f"cache shape {tuple(cache.shape)} does not match the model {want}")
    torch = _torch()
    vec = cache.device_vec()
    s.stream.wait_stream(torch.cuda.current_stream())
    s.kv_scatter(0, k, vec)


def _cache_out(s, k: int, valid, params):
    from .model import KvCache
    d = params.dims
    return KvCache(vec=s.kv_vec(0, k), shape=(d.layers, s.Lseq, d.n_kv_heads * d.hd), valid=valid)


def full_forward(params, row, target):
    """model.py:322-328."""
    _check_len(params, row)
    _check_target(row, target)
    L = len(row)
    s = _seam_session(params, L, row.prompt_len, 1)
    _load_row(s, 0, row, 0, L)
    _load_target(s, target)
    s.seam_forward(True, 1, target is not None)
    out = s.head_outputs([0])[0]
    return out, _cache_out(s, 0, np.ones(L, dtype=bool), params)


def block_forward(params, row, cache, window, target):
    """model.py:331-343.  A window covering the whole row is a full forward
    (nothing of the cache is read), computed by the full pass."""
    _check_block(row, cache, window)
    _check_len(params, row)
    _check_target(row, target)
    L = len(row)
    if window.start == 0 and window.end == L:
        return full_forward(params, row, target)
    s = _seam_session(params, L, row.prompt_len, 1)
    _load_row(s, 0, row, window.start, window.end)
    _load_target(s, target)
    _load_cache(s, 0, cache, params)
    s.seam_forward(False, 1, target is not None)
    out = s.head_outputs([0])[0]
    valid = np.asarray(cache.valid, dtype=bool).copy()
    valid[window.start:window.end] = True
    return out, _cache_out(s, 0, valid, params)


def batched_block_forward(params, packed, rows, caches, branches, target) -> dict:
    """scheduler.py:116-131 as ONE device pass: every packed branch's window
    rows stacked into the GEMMs, each attending to its own cache.  Mutates
    ``caches[k]`` (replaced by the new cache) like the reference."""
    order = list(packed.branch_order)
    if not order:
        raise ContractError("pack_active_blocks requires a non-empty active set")
    row0 = rows[order[0]]
    L, P = len(row0), row0.prompt_len
    for k in order:
        _check_block(rows[k], caches[k], branches[k].window)
        _check_len(params, rows[k])
        _check_target(rows[k], target)
        if len(rows[k]) != L or rows[k].prompt_len != P:
            raise ContractError("batched rows must share length and prompt length")
    full = [i for i, k in enumerate(order) if branches[k].window.start == 0 and branches[k].window.end == L]
    if full:  # whole-row windows: the full pass (block_forward's rule), one branch at a time
        outputs = {}
        for k in order:
            out, caches[k] = block_forward(params, rows[k], caches[k], branches[k].window, target)
            if not np.array_equal(out.positions, packed.slice_for(k)):
                raise ContractError("forward output does not cover the packed query")
            outputs[k] = out
        return outputs
    s = _seam_session(params, L, P, len(order))
    _load_target(s, target)
    for i, k in enumerate(order):
        w = branches[k].window
        _load_row(s, i, rows[k], w.start, w.end)
        _load_cache(s, i, caches[k], params)
    s.seam_forward(False, (1 << len(order)) - 1, target is not None)
    outs = s.head_outputs(range(len(order)))
    outputs = {}
    for i, k in enumerate(order):
        out = outs[i]
        if not np.array_equal(out.positions, packed.slice_for(k)):
            raise ContractError("forward output does not cover the packed query")
        w = branches[k].window
        valid = np.asarray(caches[k].valid, dtype=bool).copy()
        valid[w.start:w.end] = True
        caches[k] = _cache_out(s, i, valid, params)
        outputs[k] = out
    return outputs


def init_full_forward(params, rows, target):
    """scheduler.py:80-89: one prefill over the shared initial row; the cache
    is broadcast to every branch."""
    base = rows[0]
    for row in rows[1:]:
        if not np.array_equal(row.tokens, base.tokens) or row.prompt_len != base.prompt_len:
            raise ContractError("initial branch rows differ")
    out, cache = full_forward(params, base, target)
    return out, [cache.copy() for _ in rows]
