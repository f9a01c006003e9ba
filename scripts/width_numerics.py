"""bf16 product-path numerics at the benchmarked WIDTHS vs the oracle.

    python scripts/width_numerics.py [--shapes c2w,c3w,c5w] [--layers 2] [--seeds 2] [--out F]

The full-width model of each benchmarked config (C2 LLaDA-8B: d4096, 32x128
heads, SwiGLU 12288, V 126463; C3 Dream-7B: d3584, GQA 28:4, bias, V 152063;
C5: C2 at P=2048, G=1024, 4 branches) truncated to ``--layers`` layers, run
through the product session (prefill, then one batched block step over every
active branch on the shared-prefix aliased pages) with logits materialised
(Session(logits=True): the LM-head epilogue also writes the raw tile), and
compared per masked window position with the oracle forward (oracle/bb_oracle
.py, model.py:278-343) on the same bf16 weights:

  * ``exact``: the oracle in fp32 with NO activation rounding (the model the
    bf16 weights define),
  * ``emul``:  the oracle rounding at the device's bf16 storage points.

Reported per shape and spike gain: max |delta| of the normalised logits
(log-softmax, every vocabulary column), max |delta conf| (max prob), top-1
agreement.  North-star bar: max-abs <= 2e-2 on normalised logits."""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

SHAPES = {
    "c2w": dict(dims="LLADA_8B", V="LLADA_8B_VOCAB", P=64, G=256, bs=(8, 16, 32)),
    "c3w": dict(dims="DREAM_7B", V="DREAM_7B_VOCAB", P=64, G=512, bs=(4, 16, 32)),
    "c5w": dict(dims="LLADA_8B", V="LLADA_8B_VOCAB", P=2048, G=1024, bs=(8, 16, 32, 64)),
}


def lognorm(x):
    x = np.asarray(x, dtype=np.float64)
    m = x.max(-1, keepdims=True)
    return x - (m + np.log(np.exp(x - m).sum(-1, keepdims=True)))


def compare(dev, ref):
    """dev/ref: DenoiseOutput-like (positions, logits); per-position stats."""
    idx = {int(p): i for i, p in enumerate(ref.positions)}
    rows = np.array([idx[int(p)] for p in dev.positions], dtype=int)
    a = lognorm(dev.logits)
    b = lognorm(ref.logits[rows])
    return {"n": len(rows), "max_abs": float(np.abs(a - b).max()) if len(rows) else 0.0,
            "max_dconf": float(np.abs(np.exp(a.max(1)) - np.exp(b.max(1))).max()) if len(rows) else 0.0,
            "top1": int((a.argmax(1) == b.argmax(1)).sum())}


def merge(acc, s):
    if acc is None:
        return dict(s)
    return {"n": acc["n"] + s["n"], "max_abs": max(acc["max_abs"], s["max_abs"]),
            "max_dconf": max(acc["max_dconf"], s["max_dconf"]), "top1": acc["top1"] + s["top1"]}


def run_shape(name, layers, n_seeds, gains, head_scale=0.4, dtype="bf16"):
    import torch
    import paper_2605_29233_b200 as bb
    from paper_2605_29233_b200.engine import Session
    from oracle import bb_oracle as O
    sh = SHAPES[name]
    P, G = sh["P"], sh["G"]
    L = P + G
    dims = dataclasses.replace(getattr(bb, sh["dims"]), layers=layers, max_len=L)
    V = getattr(bb, sh["V"])
    vocab = bb.Vocab(size=V)
    cfg = bb.SchedulerConfig(block_sizes=sh["bs"], gen_len=G)
    t0 = time.time()
    arch0 = O.OArch(kind="llada", vocab_size=V, layers=layers, d_model=dims.d_model, n_heads=dims.n_heads,
                    n_kv_heads=dims.n_kv_heads, head_dim=dims.hd, d_ff=dims.d_ff, max_len=L,
                    rope_theta=dims.rope_theta, norm_eps=dims.norm_eps, qkv_bias=dims.qkv_bias,
                    head_scale=head_scale)
    W32 = O.hash_weights(arch0, 0)
    for k in list(W32):  # the device's bf16 weights (norm gains / bias stay fp32), held as fp32
        if k not in ("ln1", "ln2", "lnf", "bqkv"):
            W32[k] = O.bf16_round(W32[k]).astype(np.float32)
    t_w = time.time() - t0
    out = {}
    for gain in gains:
        params = bb.build_model(0, vocab, dims, head_scale=head_scale, spike_gain=gain, dtype=dtype)
        arch = dataclasses.replace(arch0, spike_gain=gain)
        acc = {"prefill_exact": None, "prefill_emul": None, "block_exact": None, "block_emul": None}
        for seed in range(n_seeds):
            task = bb.make_task(seed, P, G, vocab)
            s = Session(params, cfg, P, 1, trace=False, logits=True)
            s.set_inputs(task.prompt[None], task.target[None])
            s.prefill()
            pre = s.head_outputs([0])[0]
            st = s.fetch(trace=False)
            row0 = np.full(L, arch.mask_id, dtype=np.int64)
            row0[:P] = task.prompt
            ref_x, cache = O.full_forward(arch, W32, row0, P, task.target, None, np.float32)
            ref_e, _ = O.full_forward(arch, W32, row0, P, task.target, O.bf16_round, np.float32)
            acc["prefill_exact"] = merge(acc["prefill_exact"], compare(pre, ref_x))
            acc["prefill_emul"] = merge(acc["prefill_emul"], compare(pre, ref_e))
            if st["ctrl"][0, 0] != 0:
                continue
            s.iteration(with_refresh=False)
            outs = s.head_outputs(range(len(sh["bs"])))
            for k, dev in outs.items():
                if len(dev.positions) == 0:
                    continue
                tok = st["tokens"][0, k].astype(np.int64)
                a, b = int(st["branch"][0, k, 0]), int(st["branch"][0, k, 1])
                rx, _ = O.block_forward(arch, W32, tok, P, cache, a, b, task.target, None, np.float32)
                re_, _ = O.block_forward(arch, W32, tok, P, cache, a, b, task.target, O.bf16_round, np.float32)
                acc["block_exact"] = merge(acc["block_exact"], compare(dev, rx))
                acc["block_emul"] = merge(acc["block_emul"], compare(dev, re_))
            del s
        out[f"gain{gain:g}"] = acc
        print(f"[width] {name} {dtype} L{layers} gain {gain:g}: " + json.dumps(acc), file=sys.stderr, flush=True)
        del params
        torch.cuda.empty_cache()
    return {"shape": name, "dtype": dtype, "layers": layers, "P": P, "G": G, "block_sizes": list(sh["bs"]), "d_model": dims.d_model,
            "vocab_n_out": vocab.n_out, "head_scale": head_scale, "weights_s": round(t_w, 1), "results": out}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="c2w,c3w,c5w")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--seeds", type=int, default=2)
    ap.add_argument("--gains", default="0,33")
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "bf16x2"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = [run_shape(n, args.layers, args.seeds, [float(g) for g in args.gains.split(",")], dtype=args.dtype)
           for n in args.shapes.split(",")]
    js = json.dumps(res)
    if args.out:
        os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
        with open(args.out, "w") as f:
            f.write(js + "\n")
    print(js)


if __name__ == "__main__":
    main()
