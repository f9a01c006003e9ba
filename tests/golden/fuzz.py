"""Deterministic input generators for the commit / merge-sync fixtures.

Shared by ``make_golden.py`` (which runs the reference on these inputs) and
the tests (which rebuild the same inputs from the stored seeds and run the
device kernels).  numpy's PCG64 ``default_rng`` streams are version-stable.

The generators follow the reference's own fuzzers
(``pkg/tests/test_decoding.py:45-59`` build_instance,
``pkg/tests/test_scheduler.py:94-121`` _fuzz_state); probabilities are
rounded to float32 so the device (fp32) sees exactly the values the
reference (float64) decided on.
"""

from __future__ import annotations

import numpy as np


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def transition_instance(seed: int, vocab_size: int = 32, length: int = 48):
    """-> tokens, prompt_len, start, end, masked, probs(f32-exact), tau"""
    rng = np.random.default_rng(seed)
    mask_id = vocab_size + 1
    n_out = vocab_size + 1
    tokens = np.full(length, mask_id, dtype=np.int64)
    committed = rng.random(length) < rng.uniform(0.0, 0.8)
    tokens[committed] = rng.integers(0, vocab_size, size=committed.sum())
    prompt_len = int(rng.integers(1, 8))
    tokens[:prompt_len] = rng.integers(0, vocab_size, size=prompt_len)
    start = int(rng.integers(prompt_len, length - 1))
    end = int(rng.integers(start + 1, length + 1))
    pos = np.flatnonzero(tokens == mask_id)
    masked = pos[(pos >= start) & (pos < end)]
    logits = rng.standard_normal((len(masked), n_out)) * 3.0
    # occasional exact ties in confidence and in argmax
    if len(masked) >= 2 and rng.random() < 0.2:
        logits[1] = logits[0]
    if len(masked) >= 1 and rng.random() < 0.2:
        logits[0, 3] = logits[0].max()
    e = np.exp(logits - logits.max(axis=1, keepdims=True))
    probs = f32(e / e.sum(axis=1, keepdims=True))
    tau = float(np.float32(rng.uniform(0.0, 1.05)))
    return tokens, prompt_len, start, end, masked, probs, tau


def merge_state(seed: int, n_branches: int = 4, vocab_size: int = 32, length: int = 40,
                prompt_len: int = 6):
    """-> dict(rows[B,L], block_sizes, starts, ends, done, prob_maps[B,L,n_out] (f32-exact),
    covered[B,L])"""
    rng = np.random.default_rng(seed)
    mask_id = vocab_size + 1
    n_out = vocab_size + 1
    rows, bs, st, en, dn, pm, cv = [], [], [], [], [], [], []
    for _ in range(n_branches):
        t = np.full(length, mask_id, dtype=np.int64)
        t[:prompt_len] = 1
        nd = int(rng.integers(0, length - prompt_len + 1))
        t[prompt_len:prompt_len + nd] = rng.integers(0, vocab_size, size=nd)
        sc = rng.random(length) < 0.1
        sc[:prompt_len] = False
        t[sc] = rng.integers(0, vocab_size, size=sc.sum())
        b = int(rng.choice([4, 8, 16]))
        fm = np.flatnonzero(t == mask_id)
        s = int(fm[0]) if len(fm) else length
        p = rng.random((length, n_out))
        rows.append(t)
        bs.append(b)
        st.append(s)
        en.append(min(s + b, length))
        dn.append(bool(s >= length))
        pm.append(f32(p / p.sum(axis=1, keepdims=True)))
        cv.append(rng.random(length) < 0.8)
    # distinct block sizes are not required by merge_sync itself
    return {"rows": np.stack(rows), "block_sizes": np.array(bs), "starts": np.array(st),
            "ends": np.array(en), "done": np.array(dn), "prob_maps": np.stack(pm),
            "covered": np.stack(cv), "prompt_len": prompt_len, "mask_id": mask_id}
