"""Branch-parallel decoding on the B200 (reference ``scheduler.py``).

``run_blockbatch`` keeps the reference signature and result type.  The whole
Alg. 1 loop runs on the device: one batched forward over every active
branch's window rows per iteration (tcgen05 GEMMs with all windows stacked
into the GEMM N dimension, paged shared-prefix attention, fused LM head +
confidence), Eq. 1 commits, EOS cycle, Alg. 2 merge / leader sync and the
periodic refresh — see csrc/bb_control.cu.  ``run_batch`` runs many
requests in one session (request-level batching on one GPU).
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

import numpy as np

from . import _lib
from .decoding import (BranchState, GenerationResult, TraceEvent, check_eos, EOS_READY)
from .engine import Session
from .errors import ConfigError, ContractError
from .model import ModelParams, SequenceRow, Task, Vocab

TRACE_SCHEMA = "blockbatch-trace-v1"
DEFAULT_BLOCK_SIZES = (4, 8, 16, 32, 64, 128)
HARD_CAP_FACTOR = 4


@dataclass
class SchedulerConfig:
    """scheduler.py:32-63.  ``log_kv`` ("norms" | "full") / ``log_consistency``
    switch ``run_blockbatch`` to the diagnostics mode (the step in parts with
    device KV gathers and side-effect-free fresh forwards between them)."""

    block_sizes: tuple = DEFAULT_BLOCK_SIZES
    tau_conf: float = 0.9
    tau_merge: float = 0.5
    tau_sync: int = 8
    refresh_interval: int = 32
    gen_len: int = 256
    merge_enabled: bool = True
    sync_enabled: bool = True
    log_kv: str = "none"
    log_consistency: bool = False

    def validate(self) -> None:
        if not self.block_sizes:
            raise ConfigError("block_sizes must be non-empty")
        if len(set(self.block_sizes)) != len(self.block_sizes):
            raise ConfigError("block_sizes must be distinct")
        if any(b < 1 for b in self.block_sizes):
            raise ConfigError("block sizes must be positive")
        if not 0.0 <= self.tau_conf <= 1.0:
            raise ConfigError("tau_conf outside [0, 1]")
        if not 0.0 <= self.tau_merge <= 1.0:
            raise ConfigError("tau_merge outside [0, 1]")
        if self.tau_sync < 0:
            raise ConfigError("tau_sync must be non-negative")
        if self.refresh_interval < 1:
            raise ConfigError("refresh_interval must be >= 1")
        if self.gen_len < 1:
            raise ConfigError("gen_len must be >= 1")
        if self.log_kv not in ("none", "norms", "full"):
            raise ConfigError(f"unknown log_kv mode {self.log_kv!r}")


@dataclass(frozen=True)
class PackedQuery:
    """scheduler.py:66-77 (the host view of a step's packed masked positions)."""
    branch_order: tuple
    positions: np.ndarray
    offsets: tuple

    def slice_for(self, branch_index: int) -> np.ndarray:
        i = self.branch_order.index(branch_index)
        return self.positions[self.offsets[i]:self.offsets[i + 1]]


def get_active_branches(branches, rows, mask_id) -> list[int]:
    """scheduler.py:92-100"""
    return [b.index for b in branches
            if not b.done and len(rows[b.index].masked_positions(mask_id, b.window))]


def pack_active_blocks(rows, branches, active, mask_id) -> PackedQuery:
    """scheduler.py:103-113"""
    if not active:
        raise ContractError("pack_active_blocks requires a non-empty active set")
    chunks, offsets = [], [0]
    for k in active:
        pos = rows[k].masked_positions(mask_id, branches[k].window)
        chunks.append(pos)
        offsets.append(offsets[-1] + len(pos))
    return PackedQuery(tuple(active), np.concatenate(chunks), tuple(offsets))


def init_full_forward(params: ModelParams, rows: list, target):
    """scheduler.py:80-89 on the device (seams.init_full_forward)."""
    from . import seams
    return seams.init_full_forward(params, rows, target)


def batched_block_forward(params: ModelParams, packed: PackedQuery, rows: list, caches: list, branches: list,
                          target) -> dict:
    """scheduler.py:116-131: one fused device pass over every packed branch's
    window (seams.batched_block_forward); replaces ``caches[k]``."""
    from . import seams
    return seams.batched_block_forward(params, packed, rows, caches, branches, target)


def select_eos_winner(branches, rows, vocab: Vocab) -> BranchState:
    """scheduler.py:216-222"""
    ready = [b for b in branches if check_eos(b, rows[b.index], vocab) == EOS_READY]
    if not ready:
        raise ContractError("select_eos_winner requires an eos-ready branch")
    return max(ready, key=lambda b: (b.tokens_decoded, -b.block_size))


# -------------------------------------------------------------- sessions
def _cfg_key(cfg: SchedulerConfig, P: int, R: int, trace: bool):
    return (tuple(cfg.block_sizes), float(cfg.tau_conf), float(cfg.tau_merge), float(cfg.tau_sync),
            int(cfg.refresh_interval), int(cfg.gen_len), bool(cfg.merge_enabled), bool(cfg.sync_enabled),
            P, R, bool(trace))


def get_session(params: ModelParams, cfg: SchedulerConfig, prompt_len: int, n_requests: int = 1,
                trace: bool = True) -> Session:
    """Cached device session for (params, cfg, prompt_len, n_requests); the
    cache lives on the model (freed with it, or by params.clear_sessions())."""
    cache = params._sessions
    key = _cfg_key(cfg, prompt_len, n_requests, trace)
    s = cache.get(key)
    if s is None:
        if len(cache) >= 4:
            cache.pop(next(iter(cache)))
        s = Session(params, cfg, prompt_len, n_requests, trace=trace)
        cache[key] = s
    return s


def _check_call(params, cfg, tasks, diagnostics: bool = False):
    cfg.validate()
    if (cfg.log_kv != "none" or cfg.log_consistency) and not diagnostics:
        raise ConfigError("KV-space logging (log_kv / log_consistency) is per request: use run_blockbatch")
    P = tasks[0].prompt_len
    for t in tasks:
        if t.gen_len != cfg.gen_len:
            raise ConfigError("cfg.gen_len does not match the task")
        if t.prompt_len != P:
            raise ConfigError("all tasks of a batch must share the prompt length")
    if P + cfg.gen_len > params.dims.max_len:
        raise ContractError(f"sequence length {P + cfg.gen_len} exceeds max_len {params.dims.max_len}")
    return P


def run_blockbatch(params: ModelParams, task: Task, cfg: SchedulerConfig, forward_hook=None,
                   forward_observer=None, _single: bool = False, _hard_cap: int = 0) -> GenerationResult:
    """scheduler.py:225-394 on the device: prefill, batched block denoising,
    merge/sync, periodic refresh, early EOS return, final selection.

    ``forward_hook(kind)`` fires once per charged NFE, as the forward is
    charged (the host waits for each iteration's status); an exception from
    the hook aborts the run like the reference's.  ``forward_observer(kind,
    active, pre_rows, pre_caches, windows, outputs, post_caches)`` fires after
    every batched block forward with host rows, device-backed ``KvCache``
    snapshots before/after and the step's materialised ``DenoiseOutput``s
    (scheduler.py:339-342) -- the replay harness of test_acceptance.py:183-204.
    KV logging (``cfg.log_kv`` / ``cfg.log_consistency``) runs the step in
    parts the same way."""
    cfg.validate()
    if forward_observer is not None or cfg.log_kv != "none" or cfg.log_consistency:
        return _run_stepped(params, task, cfg, forward_hook, forward_observer, _hard_cap)
    return run_batch(params, [task], cfg, forward_hook=forward_hook, _single=_single, _hard_cap=_hard_cap)[0]


def _hook_deltas(forward_hook, prev, ctrl_row):
    """Fire forward_hook for each NFE charged since ``prev`` (init, block, refresh order)."""
    now = [int(ctrl_row[_lib.C_NFE0]), int(ctrl_row[_lib.C_NFE1]), int(ctrl_row[_lib.C_NFE2])]
    for i, kind in enumerate(("init", "block", "refresh")):
        for _ in range(now[i] - prev[i]):
            forward_hook(kind)
    prev[:] = now


def _run_stepped(params: ModelParams, task: Task, cfg: SchedulerConfig, forward_hook=None, forward_observer=None,
                 hard_cap: int = 0):
    """run_blockbatch with the step in parts (bb_prefill_part /
    bb_block_step_part) so host callbacks see the state between the forward
    and the commit/merge/sync that follows it: the forward observer
    (scheduler.py:326-342) and the KV-space logging of scheduler.py:268-281,
    288-294, 332-347 and 376-390 -- per block_forward / refresh event the
    ``kv_delta`` norm of each touched branch's cache change (log_kv), its
    vectorized cache ("full"), and ``E_before`` / ``E_after`` =
    ||kv_vectorize(cache) - kv_vectorize(full_forward(row).cache)|| around the
    forward (log_consistency); the init event carries each branch's cache norm.
    Caches are gathered on the device (bb_kv_gather), fresh forwards run into
    reserved scratch pages without changing the session (bb_fresh_kv), norms
    are fp64 device reductions (bb_sqdiff_norm).  Decisions, tokens, NFE and
    the rest of the trace are those of the plain run."""
    import torch
    from .model import KvCache
    P = _check_call(params, cfg, [task], diagnostics=True)
    diag = cfg.log_kv != "none" or cfg.log_consistency
    s = Session(params, cfg, P, 1, trace=True, diagnostics=diag, logits=forward_observer is not None,
                hard_cap=hard_cap)
    s.set_inputs(task.prompt[None], task.target[None])
    B = len(cfg.block_sizes)
    n = s.kv_numel()
    d = params.dims
    kv_shape = (d.layers, s.Lseq, d.n_kv_heads * d.hd)
    snap = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in range(B)] if diag else []
    cur = torch.empty(n, dtype=torch.float32, device="cuda") if diag else None
    fresh = torch.empty(n, dtype=torch.float32, device="cuda") if cfg.log_consistency else None
    norms, full = cfg.log_kv != "none", cfg.log_kv == "full"
    charged = [0, 0, 0]

    def hooks():
        if forward_hook is not None:
            _hook_deltas(forward_hook, charged, s.ctrl_now()[0])

    def consistency(ks):
        out = {}
        for k in ks:
            s.kv_gather(0, k, cur)
            s.fresh_kv(0, k, fresh)
            out[k] = s.sqdiff_norm(cur, fresh)
        return out

    def before(ks):
        e = consistency(ks) if cfg.log_consistency else None
        if norms:
            for k in ks:
                s.kv_gather(0, k, snap[k])
        return e

    def after(ks, e_before):
        extra = {}
        if norms:
            dl = {}
            for k in ks:
                s.kv_gather(0, k, cur)
                dl[k] = s.sqdiff_norm(cur, snap[k])
            extra["kv_delta"] = dl
        if full:
            kv = {}
            for k in ks:
                s.kv_gather(0, k, cur)
                s.stream.synchronize()
                kv[k] = cur.cpu().numpy().astype(np.float64).tolist()
            extra["kv"] = kv
        if cfg.log_consistency:
            extra["E_before"] = e_before
            extra["E_after"] = consistency(ks)
        return _jsonify(extra)

    def mask_list(m):
        return [k for k in range(B) if (m >> k) & 1]

    # prefill: the init event's kv_delta is each branch's cache norm (delta from empty)
    s.prefill_part(0)
    hooks()
    init_extra = {}
    if norms:
        init_extra["kv_delta"] = {}
        for k in range(B):
            s.kv_gather(0, k, cur)
            init_extra["kv_delta"][k] = s.sqdiff_norm(cur)
    if full:
        s.stream.synchronize()
        init_extra["kv"] = {}
        for k in range(B):
            s.kv_gather(0, k, cur)
            s.stream.synchronize()
            init_extra["kv"][k] = cur.cpu().numpy().astype(np.float64).tolist()
    init_extra = _jsonify(init_extra)
    s.prefill_part(1)
    block_extras, refresh_extras = [], []
    it = 0
    while it < s.max_iterations():
        c = s.ctrl_now()[0]
        if c[_lib.C_STATUS] != 0:
            break
        it += 1
        s.block_step_part(0)
        c = s.ctrl_now()[0]
        active = mask_list(int(c[_lib.C_ACTIVE_MASK])) if c[_lib.C_STATUS] == 0 else []
        eb = before(active) if (active and diag) else None
        if active and forward_observer is not None:
            toks = s.v_tokens[0].cpu().numpy()
            brs = s.v_branch[0].cpu().numpy()
            pre_rows = [SequenceRow(toks[k].astype(np.int64), P) for k in active]
            pre_caches = [KvCache(vec=s.kv_vec(0, k), shape=kv_shape, valid=np.ones(s.Lseq, dtype=bool))
                          for k in active]
            from .model import BlockWindow
            windows = [BlockWindow(int(brs[k, 0]), int(brs[k, 1])) for k in active]
        s.block_step_part(1)
        hooks()
        if active and forward_observer is not None:
            outputs = s.head_outputs(active)
            post = [KvCache(vec=s.kv_vec(0, k), shape=kv_shape, valid=np.ones(s.Lseq, dtype=bool)) for k in active]
            forward_observer("block", list(active), pre_rows, pre_caches, windows, outputs, post)
        if active and diag:
            block_extras.append(after(active, eb))
        s.block_step_part(2)
        if it % cfg.refresh_interval == 0:
            c = s.ctrl_now()[0]
            todo = mask_list(int(c[_lib.C_REFRESH_MASK])) if (c[_lib.C_STATUS] == 0 and c[_lib.C_REFRESH_DUE]) else []
            eb = before(todo) if (todo and diag) else None
            s.refresh()
            hooks()
            if todo and diag:
                refresh_extras.append(after(todo, eb))
    s.stream.synchronize()
    res = s.results([task], params.vocab)[0]
    if diag:
        bi = ri = 0
        for ev in res.trace:
            if ev.kind == "init":
                ev.extra.update(init_extra)
            elif ev.kind == "block_forward":
                ev.extra.update(block_extras[bi])
                bi += 1
            elif ev.kind == "refresh":
                ev.extra.update(refresh_extras[ri])
                ri += 1
        if bi != len(block_extras) or ri != len(refresh_extras):
            raise ContractError("diagnostics out of step with the device trace")
    return res


def run_batch(params: ModelParams, tasks: list, cfg: SchedulerConfig, forward_hook=None, trace: bool = True,
              use_graph: bool = True, _single: bool = False, _hard_cap: int = 0, _init_gen=None) -> list:
    """Many independent requests (same P, G) in one device session: every
    iteration runs one forward over all live requests' branch windows;
    NFE, trace and termination stay per request.  With ``forward_hook`` the
    host waits for each iteration (graph replay, then a status read) and fires
    the hook for every NFE charged, request by request."""
    P = _check_call(params, cfg, tasks)
    if _hard_cap:
        s = Session(params, cfg, P, len(tasks), trace=trace or forward_hook is not None, hard_cap=_hard_cap)
    else:
        s = get_session(params, cfg, P, len(tasks), trace=trace or forward_hook is not None)
    s.set_inputs(np.stack([t.prompt for t in tasks]), np.stack([t.target for t in tasks]), init_gen=_init_gen)
    if forward_hook is None:
        s.launch(use_graph=use_graph)
    else:
        charged = [[0, 0, 0] for _ in tasks]

        def fire():
            c = s.ctrl_now()
            for r in range(len(tasks)):
                _hook_deltas(forward_hook, charged[r], c[r])
            return c
        s.prefill()
        c = fire()
        it = 0
        while it < s.max_iterations() and (c[:, _lib.C_STATUS] == 0).any():
            it += 1
            s.iteration(with_refresh=it % cfg.refresh_interval == 0, use_graph=use_graph)
            c = fire()
    return s.results(tasks, params.vocab, single=_single)


# -------------------------------------------------------------- merge/sync seam
def merge_sync(rows: list, caches: list, branches: list, tau_merge: float, tau_sync: float, vocab: Vocab,
               merge_enabled: bool = True, sync_enabled: bool = True) -> list[dict]:
    """Alg. 2 (scheduler.py:144-209) on the GPU — the production merge/sync
    core (csrc/bb_control.cu: merge_sync_core) fed with the caller's host
    state; decisions are bit-exact given identical probabilities (fp32).
    Mutates rows, caches (``.copy()`` on sync), branches like the reference."""
    import torch
    B = len(branches)
    if B > _lib.MAXB:
        raise ConfigError(f"at most {_lib.MAXB} branches")
    L = len(rows[0])
    P = rows[0].prompt_len
    n_out = vocab.n_out
    rt = torch.tensor(np.stack([r.tokens for r in rows]).astype(np.int32), device="cuda")
    br = np.zeros((B, _lib.B_WORDS), np.int32)
    for b in branches:
        br[b.index] = [b.window.start, b.window.end, int(b.done), b.tokens_decoded, b.tokens_merged,
                       b.block_size, 0, 0]
    brt = torch.tensor(br, device="cuda")
    cov = torch.tensor(np.stack([b.prob_covered for b in branches]).astype(np.uint8), device="cuda")
    pm = torch.tensor(np.stack([b.prob_map for b in branches]).astype(np.float32), device="cuda")
    cap = 8 * B * L + 64
    ev = torch.zeros(cap, _lib.EVW, dtype=torch.int32, device="cuda")
    ctrl = torch.zeros(_lib.C_WORDS, dtype=torch.int32, device="cuda")
    ptab = torch.zeros(B * L * B, dtype=torch.float32, device="cuda")
    pok = torch.zeros(B * L, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib.lib().bb_merge_sync_maps(B, L, P, vocab.size, p(rt), p(brt), p(cov), p(pm), n_out,
                                             float(tau_merge), float(tau_sync), int(merge_enabled),
                                             int(sync_enabled), p(ev), cap, p(ctrl), p(ptab), p(pok),
                                             C.c_void_p(s)), "bb_merge_sync_maps")
    c = ctrl.cpu().numpy()
    if c[_lib.C_STATUS] != 0:
        raise ContractError(f"merge_sync device error {int(c[_lib.C_STATUS])}")
    rows_out = rt.cpu().numpy()
    br_out = brt.cpu().numpy()
    cov_out = cov.cpu().numpy().astype(bool)
    events = []
    from .model import BlockWindow
    for e in ev[:int(c[_lib.C_NEV])].cpu().numpy():
        kind = _lib.EV_KINDS[int(e[_lib.E_KIND])]
        d = int(e[_lib.E_BRANCH])
        if kind == "merge":
            prob = float(branches[d].prob_map[int(e[_lib.E_A1]), int(e[_lib.E_A2])])
            events.append({"kind": "merge", "dest": d, "source": int(e[_lib.E_A0]), "pos": int(e[_lib.E_A1]),
                           "token": int(e[_lib.E_A2]), "prob": prob})
        else:
            lead = int(e[_lib.E_A0])
            rows[d] = rows[lead].copy()
            caches[d] = caches[lead].copy()
            branches[d].prob_map = branches[lead].prob_map.copy()
            events.append({"kind": "sync", "dest": d, "leader": lead, "gap": int(e[_lib.E_A1])})
    for b in branches:
        k = b.index
        rows[k].tokens[:] = rows_out[k]
        b.window = BlockWindow(int(br_out[k, 0]), int(br_out[k, 1]))
        b.done = bool(br_out[k, 2])
        b.tokens_decoded = int(br_out[k, 3])
        b.tokens_merged = int(br_out[k, 4])
        b.prob_covered = cov_out[k].copy()
    return events


# -------------------------------------------------------------- trace IO
def _jsonify(obj):
    """scheduler.py:397-406"""
    if isinstance(obj, dict):
        return {str(k): _jsonify(v) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_jsonify(v) for v in obj]
    if isinstance(obj, np.generic):
        return obj.item()
    if isinstance(obj, np.ndarray):
        return obj.tolist()
    return obj


def write_trace(path, trace: list) -> None:
    """scheduler.py:409-414: JSONL with a schema header line."""
    with open(path, "w") as fh:
        fh.write(json.dumps({"schema": TRACE_SCHEMA}) + "\n")
        for event in trace:
            fh.write(json.dumps(_jsonify(event.to_record())) + "\n")


def read_trace(path) -> list[dict]:
    """scheduler.py:417-422"""
    with open(path) as fh:
        header = json.loads(fh.readline())
        if header.get("schema") != TRACE_SCHEMA:
            raise ContractError(f"unknown trace schema: {header}")
        return [json.loads(line) for line in fh if line.strip()]


# --------------------------------------------------------------------------
# run summary CSV (the reference CLI's per-run table, cli.py:147-165)
# --------------------------------------------------------------------------
SUMMARY_FIELDS = ["task_seed", "mode", "block_size", "correct", "tokens_decoded", "eos_position", "nfe_init",
                  "nfe_block", "nfe_refresh", "nfe_total", "tokens"]


def generated_tokens(result, vocab) -> list[int]:
    """analysis.py:160-171: generated tokens up to and including the first eos, masks excluded."""
    out = []
    for t in result.row.tokens[result.row.prompt_len:]:
        t = int(t)
        if t == vocab.mask_id:
            break
        out.append(t)
        if t == vocab.eos_id:
            break
    return out


def summary_row(seed: int, mode: str, result, vocab) -> dict:
    """cli.py:157-165"""
    return {"task_seed": seed, "mode": mode, "block_size": result.block_size, "correct": int(result.correct),
            "tokens_decoded": result.tokens_decoded,
            "eos_position": "" if result.eos_position is None else result.eos_position,
            "nfe_init": result.nfe.nfe_init, "nfe_block": result.nfe.nfe_block,
            "nfe_refresh": result.nfe.nfe_refresh, "nfe_total": result.nfe.total,
            "tokens": " ".join(str(t) for t in generated_tokens(result, vocab))}


def write_summary(path, rows: list[dict]) -> None:
    """cli.py:147-154: the summary table as CSV (header + one row per run)."""
    import csv
    with open(path, "w", newline="") as fh:
        w = csv.DictWriter(fh, fieldnames=SUMMARY_FIELDS)
        w.writeheader()
        w.writerows(rows)
