"""bf16 product path vs the fp32 verification path at the benchmarked shapes.

    python scripts/parity_bf16.py --config c2 --n 64 [--out profiles/r02/parity/c2.json]

Both runs use the SAME weights (the fp32 model is the exact upcast of the
bf16 model, ``model.verification_copy``), the same prompts (make_task seeds
0..n-1) and the same scheduler config as bench.py, so they differ only in
arithmetic: bf16 activations/KV + tcgen05 GEMMs and attention vs fp32 SIMT.
The fp32 path is the one that reproduces the reference's float64 run
bit-exactly on every fixture (tests/test_gpu_parity.py).

Per prompt: NFE triple, committed tokens, winner and the trace (every
record's kind, branch, decoded snapshot, NFE and payload; merge
probabilities compared to 1e-3 relative).  For a prompt whose traces differ
the first divergent record is reported (margin audit: which decision
flipped, at which step).  Also records merges / syncs / commits per request
(the head_scale calibration record, SURVEY §7 hard part 2)."""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import bench  # noqa: E402  (the bench's config table: same workload)


def rec(e):
    r = e.to_record()
    r.pop("step", None)
    return r


def same_event(a, b, prob_tol=1e-3):
    if {k: v for k, v in a.items() if k != "extra"} != {k: v for k, v in b.items() if k != "extra"}:
        return False
    xa, xb = a.get("extra") or {}, b.get("extra") or {}
    for k in set(xa) | set(xb):
        va, vb = xa.get(k), xb.get(k)
        if k == "prob" and va is not None and vb is not None:
            if abs(va - vb) > prob_tol * max(1.0, abs(vb)):
                return False
        elif va != vb:
            return False
    return True


def first_divergence(ta, tb):
    for i, (a, b) in enumerate(zip(ta, tb)):
        if not same_event(a, b):
            return i, a, b
    if len(ta) != len(tb):
        i = min(len(ta), len(tb))
        return i, ta[i] if i < len(ta) else None, tb[i] if i < len(tb) else None
    return None


def compare(seeds, prod, ref):
    rows, n_nfe, n_tok, n_trace = [], 0, 0, 0
    for seed, a, b in zip(seeds, prod, ref):
        ta, tb = [rec(e) for e in a.trace], [rec(e) for e in b.trace]
        div = first_divergence(ta, tb)
        same_nfe = a.nfe.snapshot() == b.nfe.snapshot()
        same_tok = bool(np.array_equal(a.row.tokens, b.row.tokens)) and a.branch_index == b.branch_index
        n_nfe += same_nfe
        n_tok += same_tok
        n_trace += div is None
        p = {"seed": seed, "nfe_prod": list(a.nfe.snapshot()), "nfe_f32": list(b.nfe.snapshot()),
             "same_nfe": same_nfe, "same_tokens": same_tok, "same_trace": div is None,
             "tokens_decoded": [a.tokens_decoded, b.tokens_decoded],
             "token_diffs": int((a.row.tokens != b.row.tokens).sum()),
             "stats_prod": a.stats, "stats_f32": b.stats}
        if div is not None:
            i, ea, eb = div
            p["first_divergence"] = {"index": i, "of": [len(ta), len(tb)], "prod": ea, "f32": eb}
        rows.append(p)
    n = len(seeds)
    summary = {"prompts": n, "same_nfe": n_nfe, "same_tokens": n_tok, "same_trace": n_trace,
               "frac_same_nfe": n_nfe / n, "frac_same_tokens": n_tok / n, "frac_same_trace": n_trace / n,
               "mean_nfe_prod": float(np.mean([r.nfe.total for r in prod])),
               "mean_nfe_f32": float(np.mean([r.nfe.total for r in ref])),
               "per_request_prod": {k: float(np.mean([r.stats[k] for r in prod]))
                                    for k in ("merges", "syncs", "commits", "refreshes")}}
    return rows, summary


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c5"])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--seed0", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--dtype", default="bf16x2", help="comma list of product numerics (bf16, bf16x2)")
    args = ap.parse_args()
    import torch
    from paper_2605_29233_b200.model import verification_copy
    cfgd = bench.CONFIGS[args.config]
    dtypes = args.dtype.split(",")
    bb, p0, cfg = bench.make_model(cfgd, dtypes[0])
    p32 = verification_copy(p0)
    models = {dtypes[0]: p0}
    for dt in dtypes[1:]:  # same bf16 weights, other activation numerics
        from dataclasses import replace
        models[dt] = replace(p0, dtype=dt, _handle=[None], _sessions={})
    torch.cuda.synchronize()
    seeds = list(range(args.seed0, args.seed0 + args.n))
    tasks = [bb.make_task(s, cfgd["P"], cfgd["G"], p0.vocab) for s in seeds]
    out = {"config": args.config, "workload": cfgd["workload"], "head_scale": cfgd["head_scale"],
           "gamma": cfgd["gamma"], "seeds": [seeds[0], seeds[-1]], "reference": "device fp32 verification path, same weights",
           "products": {}}
    t_run = {}
    res = {}
    for name, params in list(models.items()) + [("f32", p32)]:
        rr = []
        t0 = time.time()
        for t in tasks:
            rr.append(bb.run_blockbatch(params, t, cfg))
        torch.cuda.synchronize()
        t_run[name] = time.time() - t0
        res[name] = rr
        print(f"[parity] {name}: {len(rr)} prompts in {t_run[name]:.1f}s", file=sys.stderr, flush=True)
    for dt in dtypes:
        rows, summary = compare(seeds, res[dt], res["f32"])
        summary["wall_s"] = t_run[dt]
        out["products"][dt] = {"summary": summary, "prompts": rows}
        print(json.dumps({"dtype": dt, **summary}))
    out["wall_s_f32"] = t_run["f32"]
    if args.out:
        os.makedirs(os.path.dirname(args.out), exist_ok=True)
        with open(args.out, "w") as f:
            f.write(json.dumps(out) + "\n")


if __name__ == "__main__":
    main()
