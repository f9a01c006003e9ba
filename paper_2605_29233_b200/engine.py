"""Device sessions: one workspace per (model, scheduler config, request count).

A session owns a single caller-allocated device workspace (a torch uint8
tensor — torch is only the allocator here) carved by the C library into the
device state of R requests x B branches (rows, branch windows, paged KV,
probability maps, trace ring) and the two forward passes.  ``run`` uploads
prompts/targets, calls ``bb_run`` (prefill + the captured per-iteration
CUDA graph until every request finished) and decodes the results.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from . import _lib
from .errors import ConfigError, ContractError, RunawayError, StateError


def _torch():
    import torch
    return torch


class Session:
    def __init__(self, params, cfg, prompt_len: int, n_requests: int = 1, trace: bool = True,
                 page_size: int = 16, pages_per_item: int = 4, event_capacity: int | None = None,
                 diagnostics: bool = False, test_flags: int = 0, logits: bool = False, seam: bool = False,
                 hard_cap: int = 0):
        torch = _torch()
        # no reference to `params` itself: the model's session cache
        # (ModelParams._sessions) owns its sessions, so a session must not keep
        # the model alive (the cache would never be collected)
        self.dims, self.vocab = params.dims, params.vocab
        self.cfg = cfg
        self.P, self.G, self.R = prompt_len, cfg.gen_len, n_requests
        self.B = len(cfg.block_sizes)
        if self.B > _lib.MAXB:
            raise ConfigError(f"at most {_lib.MAXB} block sizes per request")
        L = _lib.lib()
        bs = (C.c_int * 8)(*(list(cfg.block_sizes) + [0] * (8 - self.B)))
        if event_capacity is None:
            event_capacity = 64 + 24 * (self.G + 4) * self.B
        self.desc = _lib.SessionDesc(
            n_requests=n_requests, n_branches=self.B, block_sizes=bs, prompt_len=prompt_len, gen_len=cfg.gen_len,
            tau_conf=cfg.tau_conf, tau_merge=cfg.tau_merge, tau_sync=float(cfg.tau_sync),
            refresh_interval=cfg.refresh_interval, merge_enabled=int(cfg.merge_enabled),
            sync_enabled=int(cfg.sync_enabled), page_size=page_size, pages_per_item=pages_per_item,
            trace=int(trace), event_capacity=event_capacity, diagnostics=int(diagnostics),
            test_flags=int(test_flags), logits=int(logits), seam=int(seam), hard_cap=int(hard_cap))
        nbytes = C.c_size_t(0)
        model = params.handle()
        _lib.check(L.bb_session_workspace_bytes(model, C.byref(self.desc), C.byref(nbytes)),
                   "bb_session_workspace_bytes")
        self.ws = torch.zeros(nbytes.value + 2048, dtype=torch.uint8, device="cuda")
        h = C.c_void_p()
        _lib.check(L.bb_session_create(model, C.byref(self.desc), C.c_void_p(self.ws.data_ptr()),
                                       self.ws.numel(), C.byref(h)), "bb_session_create")
        self.h = h
        info = (C.c_int * 16)()
        L.bb_session_info(h, info, 16)
        self.info = list(info)
        self.Lseq = self.info[2]
        self.ev_cap = self.info[3]
        self.stream = torch.cuda.Stream()
        self.v_tokens = self._view(_lib.VIEW_TOKENS, torch.int32, (self.R, self.B, self.Lseq))
        self.v_target = self._view(_lib.VIEW_TARGET, torch.int32, (self.R, self.G))
        self.v_prompt = self._view(_lib.VIEW_PROMPT, torch.int32, (self.R, self.P))
        self.v_init_gen = self._view(_lib.VIEW_INIT_GEN, torch.int32, (self.R, self.G))
        self._preset_dirty = False
        self.v_ctrl = self._view(_lib.VIEW_CTRL, torch.int32, (self.R, _lib.C_WORDS))
        self.v_branch = self._view(_lib.VIEW_BRANCH, torch.int32, (self.R, self.B, _lib.B_WORDS))
        self.v_events = self._view(_lib.VIEW_EVENTS, torch.int32, (self.R, self.ev_cap, _lib.EVW))
        self.v_pages = self._view(_lib.VIEW_PAGES, torch.int32, (self.R, self.B, self.info[7]))
        self.v_refc = self._view(_lib.VIEW_REFC, torch.int32, (self.R, self.info[8]))
        nr = self.info[9]
        self.v_head = {name: self._view(vid, dt, (nr,)) for name, vid, dt in (
            ("masked", _lib.VIEW_HEAD_MASKED, torch.int32), ("m", _lib.VIEW_HEAD_M, torch.float32),
            ("s", _lib.VIEW_HEAD_S, torch.float32), ("arg", _lib.VIEW_HEAD_ARG, torch.int32),
            ("pos", _lib.VIEW_SLOT_POS, torch.int32), ("branch", _lib.VIEW_SLOT_BR, torch.int32))}
        self.h2d_bytes = self.d2h_bytes = 0

    def _view(self, which, dtype, shape):
        off, nb = C.c_longlong(0), C.c_longlong(0)
        _lib.check(_lib.lib().bb_session_view(self.h, which, C.byref(off), C.byref(nb)), "bb_session_view")
        n = int(np.prod(shape))
        return self.ws[off.value:off.value + nb.value].view(dtype)[:n].view(*shape)

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and _lib._lib is not None:
                _lib._lib.bb_session_destroy(self.h)
        except Exception:
            pass

    # ---------------------------------------------------------------- inputs
    def set_inputs(self, prompts, targets, init_gen=None):
        """prompts [R, P], targets [R, G]: host arrays (copied H2D on the session
        stream) or CUDA tensors (copied D2D after the producing stream's work).
        init_gen [R, G] (optional): the initial generation row, token or -1 =
        mask (single_branch_decode presets)."""
        torch = _torch()
        self.stream.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.stream):
            if init_gen is not None or self._preset_dirty:
                g = np.full((self.R, self.G), -1, dtype=np.int32) if init_gen is None else \
                    np.ascontiguousarray(np.asarray(init_gen), dtype=np.int32)
                t = torch.from_numpy(g).pin_memory()
                self.v_init_gen.copy_(t, non_blocking=True)
                self.h2d_bytes += t.numel() * 4
                self._preset_dirty = init_gen is not None
            for dst, src in ((self.v_prompt, prompts), (self.v_target, targets)):
                if isinstance(src, torch.Tensor) and src.is_cuda:
                    t = src if src.dtype == torch.int32 else src.to(torch.int32)
                    dst.copy_(t, non_blocking=True)
                    t.record_stream(self.stream)
                else:
                    t = torch.from_numpy(np.ascontiguousarray(np.asarray(src), dtype=np.int32)).pin_memory()
                    dst.copy_(t, non_blocking=True)
                    self.h2d_bytes += t.numel() * 4

    def max_iterations(self) -> int:
        hard_cap = 4 * self.G * self.B + 16
        return 10 * hard_cap + 4

    def launch(self, use_graph: bool = True) -> int:
        """Enqueue the whole run (bb_run) on the session stream; returns #iterations."""
        it = C.c_int(0)
        _lib.check(_lib.lib().bb_run(self.h, self.max_iterations(), int(use_graph),
                                     C.c_void_p(self.stream.cuda_stream), C.byref(it)), "bb_run")
        return it.value

    def launch_vanilla(self, use_graph: bool = True) -> int:
        """vanilla_decode rounds (bb_run_vanilla) on the session stream; the
        session must have one branch of block size gen_len."""
        it = C.c_int(0)
        _lib.check(_lib.lib().bb_run_vanilla(self.h, self.max_iterations(), int(use_graph),
                                             C.c_void_p(self.stream.cuda_stream), C.byref(it)), "bb_run_vanilla")
        return it.value

    # ---------------------------------------------------------------- diagnostics
    # (log_kv / log_consistency: the step in parts, KV gathers, fresh forwards)
    def prefill_part(self, part: int):
        _lib.check(_lib.lib().bb_prefill_part(self.h, part, C.c_void_p(self.stream.cuda_stream)), "bb_prefill_part")

    def block_step_part(self, part: int):
        _lib.check(_lib.lib().bb_block_step_part(self.h, part, C.c_void_p(self.stream.cuda_stream)),
                   "bb_block_step_part")

    def refresh(self):
        _lib.check(_lib.lib().bb_refresh(self.h, C.c_void_p(self.stream.cuda_stream)), "bb_refresh")

    def kv_numel(self) -> int:
        d = self.dims
        return d.layers * self.Lseq * 2 * d.n_kv_heads * d.hd

    def kv_gather(self, r: int, k: int, dst):
        _lib.check(_lib.lib().bb_kv_gather(self.h, r, k, C.c_void_p(dst.data_ptr()),
                                           C.c_void_p(self.stream.cuda_stream)), "bb_kv_gather")

    def fresh_kv(self, r: int, k: int, dst):
        _lib.check(_lib.lib().bb_fresh_kv(self.h, r, k, C.c_void_p(dst.data_ptr()),
                                          C.c_void_p(self.stream.cuda_stream)), "bb_fresh_kv")

    def sqdiff_norm(self, a, b=None) -> float:
        torch = _torch()
        out = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().bb_sqdiff_norm(self.h, C.c_void_p(a.data_ptr()), None if b is None else C.c_void_p(b.data_ptr()),
                                             a.numel(), C.c_void_p(out.data_ptr()),
                                             C.c_void_p(self.stream.cuda_stream)), "bb_sqdiff_norm")
        self.stream.synchronize()
        return float(out.item())

    # ---------------------------------------------------------------- seams
    def seam_init(self):
        _lib.check(_lib.lib().bb_seam_init(self.h, C.c_void_p(self.stream.cuda_stream)), "bb_seam_init")

    def seam_forward(self, full: bool, mask: int, use_target: bool):
        _lib.check(_lib.lib().bb_seam_forward(self.h, int(full), int(mask), int(use_target),
                                              C.c_void_p(self.stream.cuda_stream)), "bb_seam_forward")

    def kv_scatter(self, r: int, k: int, src):
        _lib.check(_lib.lib().bb_kv_scatter(self.h, r, k, C.c_void_p(src.data_ptr()),
                                            C.c_void_p(self.stream.cuda_stream)), "bb_kv_scatter")

    def head_outputs(self, branches, r: int = 0) -> dict:
        """DenoiseOutput per branch of the last head pass (masked head slots
        of request r, in position order): materialised logits and probs."""
        torch = _torch()
        from .model import DenoiseOutput
        rows = self.info[9]
        n_out = self.vocab.n_out
        if getattr(self, "_lbuf", None) is None:
            self._lbuf = torch.empty(rows, n_out, dtype=torch.float32, device="cuda")
            self._pbuf = torch.empty(rows, n_out, dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().bb_head_logits(self.h, C.c_void_p(self._lbuf.data_ptr()),
                                             C.c_void_p(self._pbuf.data_ptr()),
                                             C.c_void_p(self.stream.cuda_stream)), "bb_head_logits")
        self.stream.synchronize()
        masked = self.v_head["masked"].cpu().numpy()
        pos = self.v_head["pos"].cpu().numpy()
        br = self.v_head["branch"].cpu().numpy()
        nrq = self.info[14]
        out = {}
        for k in branches:
            sl = np.flatnonzero((masked != 0) & (br == k) & (pos >= 0))
            sl = sl[(sl >= r * nrq) & (sl < (r + 1) * nrq)]
            sl = sl[np.argsort(pos[sl], kind="stable")]
            idx = torch.from_numpy(sl.astype(np.int64)).to("cuda")
            lg = self._lbuf.index_select(0, idx).double().cpu().numpy()
            pr = self._pbuf.index_select(0, idx).double().cpu().numpy()
            out[k] = DenoiseOutput(pos[sl].astype(int), lg, pr)
        return out

    def kv_vec(self, r: int, k: int):
        """Branch k's cache of request r as a new CUDA fp32 kv_vectorize vector."""
        torch = _torch()
        v = torch.empty(self.kv_numel(), dtype=torch.float32, device="cuda")
        self.kv_gather(r, k, v)
        self.stream.synchronize()
        return v

    def ctrl_now(self) -> np.ndarray:
        self.stream.synchronize()
        return self.v_ctrl.cpu().numpy()

    def prefill(self):
        _lib.check(_lib.lib().bb_prefill(self.h, C.c_void_p(self.stream.cuda_stream)), "bb_prefill")

    def iteration(self, with_refresh: bool, use_graph: bool = True):
        _lib.check(_lib.lib().bb_iteration(self.h, int(with_refresh), int(use_graph),
                                           C.c_void_p(self.stream.cuda_stream)), "bb_iteration")

    # ---------------------------------------------------------------- results
    def fetch(self, trace: bool = True) -> dict:
        """D2H of the run's results on the session stream (ctrl words, branch
        rows, branch states and — if traced — the event records)."""
        torch = _torch()
        with torch.cuda.stream(self.stream):
            ctrl = self.v_ctrl.to("cpu", non_blocking=False)
            out = {"ctrl": ctrl.numpy(), "tokens": self.v_tokens.cpu().numpy(),
                   "branch": self.v_branch.cpu().numpy()}
            self.d2h_bytes += out["ctrl"].nbytes + out["tokens"].nbytes + out["branch"].nbytes
            if trace:
                nmax = int(out["ctrl"][:, _lib.C_NEV].max())
                out["events"] = self.v_events[:, :nmax].cpu().numpy()
                self.d2h_bytes += out["events"].nbytes
        return out

    def head_results(self) -> dict:
        """Per head slot of the last head pass: masked flag, max logit m, sum
        exp s, argmax, position, branch (numerics tests)."""
        self.stream.synchronize()
        return {k: v.cpu().numpy() for k, v in self.v_head.items()}

    def snapshot(self, dst_ctrl, dst_branch):
        """Device-side copy of the result words (ctrl, branch state) into
        caller buffers — no host sync (used inside timed regions)."""
        torch = _torch()
        with torch.cuda.stream(self.stream):
            dst_ctrl.copy_(self.v_ctrl, non_blocking=True)
            dst_branch.copy_(self.v_branch, non_blocking=True)

    def gemm_stats(self, reset: bool = False):
        buf = (C.c_ulonglong * 80)()
        _lib.check(_lib.lib().bb_session_gemm_stats(self.h, buf, int(reset), C.c_void_p(self.stream.cuda_stream)),
                   "bb_session_gemm_stats")
        return [[int(buf[k * 5 + j]) for j in range(5)] for k in range(16)]

    KLOG_NAMES = {1: "embed", 2: "post_qkv", 3: "attn_seg", 4: "post_residual", 5: "post_gu", 6: "norm",
                  7: "gather_head", 8: "head_tiles_f32", 9: "head_reduce", 10: "prefill_init", 11: "prefill_post",
                  12: "block_pack", 13: "step_commit", 14: "merge_prep", 15: "merge_sync", 16: "refresh_pack",
                  17: "refresh_end", 18: "copy_pages", 20: "gemm_simt", 21: "attn_simt", 22: "attn_combine", 23: "layer_stream", 24: "attn_seg_pre",
                  100: "gemm_qkv", 101: "gemm_o", 102: "gemm_gate_up", 103: "gemm_down", 104: "gemm_head", 151: "gemm_o_pre",
                  108: "gemm_qkv_full", 109: "gemm_o_full", 110: "gemm_gate_up_full", 111: "gemm_down_full"}

    def klog(self, reset: bool = False):
        """Kernel timeline of a BB_KLOG=1 session: list of (name, t_ns)."""
        cap = 1 << 20
        buf = (C.c_ulonglong * (2 * cap))()
        n = C.c_longlong(0)
        _lib.check(_lib.lib().bb_session_klog(self.h, buf, cap, int(reset), C.byref(n),
                                              C.c_void_p(self.stream.cuda_stream)), "bb_session_klog")
        return [(self.KLOG_NAMES.get(int(buf[2 * i]), str(int(buf[2 * i]))), int(buf[2 * i + 1]))
                for i in range(n.value)]

    def counters(self):
        buf = (C.c_longlong * 5)()
        _lib.check(_lib.lib().bb_session_counters(self.h, buf), "bb_session_counters")
        return {"kernel_launches": buf[0], "graph_launches": buf[1], "kernels_per_step": buf[2],
                "kernels_per_step_refresh": buf[3], "kernels_prefill": buf[4]}

    def results(self, tasks, vocab, single=False, fetched=None):
        from .decoding import GenerationResult, NfeCounter
        from .model import SequenceRow, exact_match
        f = fetched if fetched is not None else self.fetch()
        res = []
        for r, task in enumerate(tasks):
            c = f["ctrl"][r]
            st = int(c[_lib.C_STATUS])
            if st < 0:
                if st == _lib.BB_ERR_RUNAWAY:
                    raise RunawayError(f"blockbatch run exceeded the hard cap ({4 * self.G * self.B + 16})")
                raise StateError(f"device session error {st} (request {r})")
            if st != 1:
                raise StateError(f"request {r} did not finish (status {st})")
            if c[_lib.C_EV_OVERFLOW]:
                raise StateError("trace event capacity exceeded")
            w = int(c[_lib.C_WINNER])
            eos = int(c[_lib.C_EOS])
            row = SequenceRow(f["tokens"][r, w].astype(np.int64), self.P)
            trace = decode_events(f["events"][r, :int(c[_lib.C_NEV])], self.B, single) if "events" in f else []
            nfe = NfeCounter(int(c[_lib.C_NFE0]), int(c[_lib.C_NFE1]), int(c[_lib.C_NFE2]))
            stats = {"iterations": int(c[_lib.C_ITER]), "merges": int(c[_lib.C_MERGES]),
                     "syncs": int(c[_lib.C_SYNCS]), "commits": int(c[_lib.C_COMMITS]),
                     "refreshes": int(c[_lib.C_REFRESHES]), "cow_pages": int(c[_lib.C_COW_PAGES])}
            res.append(GenerationResult(row=row, branch_index=w, block_size=int(self.cfg.block_sizes[w]), nfe=nfe,
                                        trace=trace, correct=exact_match(row, task, vocab),
                                        tokens_decoded=int(f["branch"][r, w, _lib.B_DEC]),
                                        eos_position=None if eos < 0 else eos, stats=stats))
        return res


def decode_events(ev: np.ndarray, n_branches: int, single: bool = False) -> list:
    """Device trace records -> TraceEvent list (decoding.py:61-75 / scheduler.py emit order)."""
    from .decoding import TraceEvent
    out = []
    for i, e in enumerate(ev):
        kind = _lib.EV_KINDS[int(e[_lib.E_KIND])]
        br = int(e[_lib.E_BRANCH])
        branch = None if br < 0 else br
        dec = tuple(int(x) for x in e[_lib.E_DEC:_lib.E_DEC + n_branches])
        nfe = (int(e[_lib.E_NFE0]), int(e[_lib.E_NFE1]), int(e[_lib.E_NFE2]))
        a0, a1, a2 = int(e[_lib.E_A0]), int(e[_lib.E_A1]), int(e[_lib.E_A2])
        if kind == "init":
            extra = {"extra_nfe": None}
        elif kind in ("block_forward", "refresh"):
            extra = {"active": [k for k in range(n_branches) if (a0 >> k) & 1]}
        elif kind == "decode":
            extra = {"commits": a0}
        elif kind == "merge":
            prob = float(np.array([e[_lib.E_PROB]], dtype=np.int32).view(np.float32)[0])
            extra = {"source": a0, "pos": a1, "token": a2, "prob": prob}
        elif kind == "sync":
            extra = {"leader": a0, "gap": a1}
        elif kind in ("eos_ready", "finish"):
            extra = {"eos": None if a0 < 0 else a0}
        else:
            extra = {}
        if single:  # single_branch_decode's record shapes (decoding.py:222-271)
            branch = 0
            if kind in ("init", "block_forward", "refresh", "finish"):
                extra = {}
        out.append(TraceEvent(i, kind, branch, dec, nfe, extra))
    return out
