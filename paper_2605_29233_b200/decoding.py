"""Decoding-rule types and seams of the blockbatch API (reference ``decoding.py``).

``confidence_transition`` (Eq. 1) runs on the GPU through the C-ABI
(``bb_commit_probs``), the same device rule the fused step applies.  The
window-lifecycle helpers are small host utilities over host ``SequenceRow``
objects kept for API compatibility; inside ``run_blockbatch`` the identical
rules run on the device (csrc/bb_control.cu).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, ContractError
from .model import BlockWindow, DenoiseOutput, SequenceRow, Vocab

EOS_NONE = "none"
EOS_PENDING = "pending"
EOS_READY = "ready"
HARD_CAP_FACTOR = 4


@dataclass
class DecodeConfig:
    """decoding.py:29-44"""
    block_size: int
    gen_len: int = 256
    tau_conf: float = 0.9
    refresh_interval: int = 32

    def validate(self) -> None:
        if not 0.0 <= self.tau_conf <= 1.0:
            raise ConfigError(f"tau_conf {self.tau_conf} outside [0, 1]")
        if self.gen_len < 1:
            raise ConfigError("gen_len must be >= 1")
        if self.refresh_interval < 1:
            raise ConfigError("refresh_interval must be >= 1")
        if self.block_size < 1:
            raise ConfigError("block_size must be >= 1")


@dataclass
class NfeCounter:
    """decoding.py:47-58"""
    nfe_init: int = 0
    nfe_block: int = 0
    nfe_refresh: int = 0

    @property
    def total(self) -> int:
        return self.nfe_init + self.nfe_block + self.nfe_refresh

    def snapshot(self) -> tuple[int, int, int]:
        return (self.nfe_init, self.nfe_block, self.nfe_refresh)


@dataclass
class TraceEvent:
    """decoding.py:61-75"""
    step: int
    kind: str
    branch: int | None
    decoded: tuple
    nfe: tuple
    extra: dict = field(default_factory=dict)

    def to_record(self) -> dict:
        rec = {"step": self.step, "kind": self.kind, "branch": self.branch,
               "decoded": list(self.decoded), "nfe": list(self.nfe)}
        if self.extra:
            rec["extra"] = self.extra
        return rec


@dataclass
class BranchState:
    """decoding.py:78-93"""
    index: int
    block_size: int
    window: BlockWindow
    done: bool = False
    tokens_decoded: int = 0
    tokens_merged: int = 0
    prob_map: np.ndarray | None = None
    prob_covered: np.ndarray | None = None

    def refresh_decoded(self, row: SequenceRow, mask_id: int) -> None:
        gen = row.tokens[row.prompt_len:]
        self.tokens_decoded = int(np.count_nonzero(gen != mask_id))


@dataclass
class GenerationResult:
    """decoding.py:96-105 (+ ``stats``: device counters of the run)."""
    row: SequenceRow
    branch_index: int
    block_size: int
    nfe: NfeCounter
    trace: list
    correct: bool
    tokens_decoded: int
    eos_position: int | None
    stats: dict = field(default_factory=dict)


def confidence_transition(output: DenoiseOutput, row: SequenceRow, window: BlockWindow,
                          tau_conf: float) -> list[tuple[int, int]]:
    """Eq. 1 (decoding.py:108-129) on the GPU (bb_commit_probs): conf = max
    prob, choice = lowest-id argmax, i* = lowest-position max conf; commit iff
    conf >= tau or i == i*.  Mutates ``row.tokens``; returns sorted pairs."""
    import torch
    mask_id = output.probs.shape[1]
    masked = np.flatnonzero(row.tokens == mask_id)
    masked = masked[(masked >= window.start) & (masked < window.end)]
    if sorted(int(p) for p in output.positions) != [int(p) for p in masked]:
        raise ContractError("output positions do not match the masked window positions")
    if len(masked) == 0:
        return []
    out = output.restrict(masked)
    n, n_out = out.probs.shape
    probs = torch.from_numpy(np.ascontiguousarray(out.probs, dtype=np.float32)).cuda()
    pos = torch.from_numpy(masked.astype(np.int32)).cuda()
    dev_row = torch.from_numpy(row.tokens.astype(np.int32)).cuda()
    pairs = torch.zeros(n, 2, dtype=torch.int32, device="cuda")
    count = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().bb_commit_probs(C.c_void_p(probs.data_ptr()), n, n_out, C.c_void_p(pos.data_ptr()),
                                          C.c_void_p(dev_row.data_ptr()), float(tau_conf),
                                          C.c_void_p(pairs.data_ptr()), C.c_void_p(count.data_ptr()),
                                          C.c_void_p(s)), "bb_commit_probs")
    k = int(count.item())
    commits = [(int(p), int(t)) for p, t in pairs[:k].cpu().tolist()]
    for p, t in commits:
        row.tokens[p] = t
    return commits


def window_complete(row: SequenceRow, window: BlockWindow, mask_id: int) -> bool:
    """decoding.py:137-140"""
    if window.empty:
        return True
    return not (row.tokens[window.start:window.end] == mask_id).any()


def advance_block(branch: BranchState, row: SequenceRow, mask_id: int) -> BranchState:
    """decoding.py:143-154"""
    if not window_complete(row, branch.window, mask_id):
        raise ContractError("advance_block called with an incomplete window")
    length = len(row)
    start = branch.window.end
    if start >= length:
        branch.window = BlockWindow(length, length)
        branch.done = True
    else:
        branch.window = BlockWindow(start, min(start + branch.block_size, length))
    return branch


def earliest_eos(row: SequenceRow, vocab: Vocab) -> int | None:
    """decoding.py:157-160"""
    hits = np.flatnonzero(row.tokens[row.prompt_len:] == vocab.eos_id)
    return int(hits[0]) + row.prompt_len if len(hits) else None


def check_eos(branch: BranchState, row: SequenceRow, vocab: Vocab) -> str:
    """decoding.py:163-168"""
    eos = earliest_eos(row, vocab)
    if eos is None:
        return EOS_NONE
    return EOS_PENDING if (row.tokens[row.prompt_len:eos] == vocab.mask_id).any() else EOS_READY


def realign_for_eos(branch: BranchState, row: SequenceRow, vocab: Vocab) -> None:
    """decoding.py:171-180"""
    eos = earliest_eos(row, vocab)
    if eos is None:
        return
    masked = np.flatnonzero(row.tokens[:eos] == vocab.mask_id)
    if len(masked) == 0:
        return
    first = int(masked[0])
    branch.window = BlockWindow(first, min(first + branch.block_size, eos))


def realign_to_first_mask(branch: BranchState, row: SequenceRow, mask_id: int) -> None:
    """decoding.py:183-191"""
    masked = np.flatnonzero(row.tokens == mask_id)
    length = len(row)
    if len(masked) == 0:
        branch.window = BlockWindow(length, length)
        branch.done = True
        return
    first = int(masked[0])
    branch.window = BlockWindow(first, min(first + branch.block_size, length))


def single_branch_decode(params, task, cfg: DecodeConfig, preset=None):
    """decoding.py:203-276 — one branch, no merge/sync, its own refresh counter.

    Runs on the device as a singleton BlockBatch session: with one branch,
    merge and sync disabled, the loops are identical (criterion 04,
    test_acceptance.py:164-180)."""
    from .scheduler import SchedulerConfig, run_batch, run_blockbatch
    cfg.validate()
    scfg = SchedulerConfig(block_sizes=(cfg.block_size,), tau_conf=cfg.tau_conf,
                           refresh_interval=cfg.refresh_interval, gen_len=cfg.gen_len, merge_enabled=False,
                           sync_enabled=False)
    if not preset:
        return run_blockbatch(params, task, scfg, _single=True)
    # apply_preset (decoding.py:194-200): committed tokens placed before the prefill
    if cfg.gen_len != task.gen_len:
        raise ConfigError("cfg.gen_len does not match the task")
    P = task.prompt_len
    init_gen = np.full((1, task.gen_len), -1, dtype=np.int64)
    for pos, tok in preset:
        if pos < P or pos >= P + task.gen_len:
            raise ContractError(f"preset position {pos} outside the generation region")
        init_gen[0, pos - P] = tok
    return run_batch(params, [task], scfg, _single=True, _init_gen=init_gen)[0]


def vanilla_decode(params, task, cfg: DecodeConfig):
    """decoding.py:279-321 — the reference's baseline decoder: one full forward
    per round over the whole row (no cache reuse) and exactly one committed
    token per round (Eq. 1 with tau 1.0 over the masked positions before the
    first eos), so a generation costs about gen_len forwards.

    Runs on the device (bb_run_vanilla: full pass + LM head + commit kernels,
    one captured graph per round) in a one-branch session of block size
    gen_len; returns the reference's GenerationResult and trace records."""
    from .scheduler import SchedulerConfig, _check_call, get_session
    cfg.validate()
    if cfg.gen_len != task.gen_len:
        raise ConfigError("cfg.gen_len does not match the task")
    scfg = SchedulerConfig(block_sizes=(cfg.gen_len,), gen_len=cfg.gen_len, tau_conf=1.0,
                           merge_enabled=False, sync_enabled=False)
    P = _check_call(params, scfg, [task])
    s = get_session(params, scfg, P, 1, trace=True)
    s.set_inputs(task.prompt[None], task.target[None])
    s.launch_vanilla()
    return s.results([task], params.vocab, single=True)[0]
