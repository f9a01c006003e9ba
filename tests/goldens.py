"""Loading and comparison helpers for the golden fixtures (tests only)."""

from __future__ import annotations

import json
import math
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
_cache = {}


def load(name):
    if name not in _cache:
        with open(os.path.join(GOLDEN, name)) as fh:
            _cache[name] = json.load(fh)
    return _cache[name]


def _close(a, b, tol):
    if isinstance(a, float) or isinstance(b, float):
        return a is not None and b is not None and math.isclose(float(a), float(b),
                                                                rel_tol=tol, abs_tol=tol)
    return a == b


def diff_trace(got: list, want: list, prob_tol=1e-9, kv_tol=1e-4):
    """First mismatch between two trace record lists, or None.  Discrete
    fields must be equal; merge-event probabilities within ``prob_tol``."""
    for i, (g, w) in enumerate(zip(got, want)):
        for key in ("step", "kind", "branch", "decoded", "nfe"):
            if g.get(key) != w.get(key):
                return f"event {i} field {key}: got {g.get(key)} want {w.get(key)} ({w})"
        ge, we = g.get("extra", {}), w.get("extra", {})
        if set(ge) != set(we):
            return f"event {i} extra keys: got {sorted(ge)} want {sorted(we)}"
        for k in we:
            if k == "prob":
                if not _close(ge[k], we[k], prob_tol):
                    return f"event {i} prob: got {ge[k]} want {we[k]}"
            elif k in ("kv_delta", "E_before", "E_after"):
                # KV-space norms (scheduler.py:268-281): float64 reference vs the
                # device's fp32 caches (fp64 reductions)
                if set(ge[k]) != set(we[k]):
                    return f"event {i} {k} branches: got {sorted(ge[k])} want {sorted(we[k])}"
                for b in we[k]:
                    if not math.isclose(float(ge[k][b]), float(we[k][b]), rel_tol=kv_tol, abs_tol=kv_tol):
                        return f"event {i} {k}[{b}]: got {ge[k][b]} want {we[k][b]}"
            elif ge[k] != we[k]:
                return f"event {i} extra {k}: got {ge[k]} want {we[k]}"
    if len(got) != len(want):
        return f"trace length: got {len(got)} want {len(want)}"
    return None


def compare_run(got: dict, want: dict, prob_tol=1e-9, trace=True, kv_tol=1e-4):
    for key in ("tokens", "nfe", "branch_index", "block_size", "tokens_decoded",
                "eos_position", "correct"):
        g, w = got[key], want[key]
        if isinstance(w, list):
            g = [int(x) for x in g]
        if g != w:
            return f"{key}: got {g} want {w}"
    if trace:
        return diff_trace(got["trace"], want["trace"], prob_tol, kv_tol)
    return None
