"""Generate the golden fixtures from the REFERENCE itself.

Run in the build container (needs /root/reference; it does not travel to the
GPU box — the fixtures it writes do):

    python tests/golden/make_golden.py [--vanilla-only | --runaway-only]

Outputs (all under tests/golden/):
  runs_ref.json     full-run results (tokens, NFE, winner, complete trace) of
                    the reference's own run_blockbatch / single_branch_decode
                    on its own synthetic model: default dims and config C1
                    (4 layers, d256, V4096, P64, G128, B={8,16,32}).
  runs_llada.json   reference run_blockbatch (its scheduler, unmodified) with
                    the oracle's LLaDA/Dream-shape forward injected through
                    the scheduler's module-level forward seams
                    (scheduler.py:23-25) — pins the oracle's scheduler on a
                    second architecture; fp32-weight and bf16-emulating runs.
  runs_vanilla.json the reference's vanilla_decode baseline (decoding.py:279-321)
                    on its own model (default dims, and C1 at head_scale 2).
  runs_diag.json    reference run_blockbatch with log_kv="norms" and
                    log_consistency (KV-space logging).
  kernels.json      reference confidence_transition / merge_sync outputs on
                    the fuzzed inputs of fuzz.py (inputs rebuilt from seeds).
  forward_c1.npz    reference full_forward / block_forward numerics (C1, seed 0).
  summary_ref.csv   the reference CLI's run summary (cli.py:147-165,
                    summary_row / write_summary) of every runs_ref.json run of
                    the c1_hs2 and default_g4_eos configs (rebuilt as reference
                    GenerationResults; --summary-only regenerates just this).
  runs_preset.json  the reference's single_branch_decode with preset commits
                    (decoding.py:194-212): target tokens, a wrong token and an
                    eos placed before the prefill (--preset-only regenerates it).
  runs_runaway.json reference run_blockbatch with the hard cap lowered to 16
                    forwards (HARD_CAP_FACTOR = 0): forward_hook calls up to
                    the RunawayError (scheduler.py:310, 324-325).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import blockbatch as bb                       # noqa: E402  (the reference)
from blockbatch import decoding as bbd        # noqa: E402
from blockbatch import model as bbm           # noqa: E402
from blockbatch import scheduler as bbs       # noqa: E402

import fuzz                                   # noqa: E402
from oracle import bb_oracle as O             # noqa: E402


def result_record(r):
    return {"tokens": [int(t) for t in r.row.tokens], "nfe": list(r.nfe.snapshot()),
            "branch_index": int(r.branch_index), "block_size": int(r.block_size),
            "tokens_decoded": int(r.tokens_decoded),
            "eos_position": None if r.eos_position is None else int(r.eos_position),
            "correct": bool(r.correct),
            "trace": [bbs._jsonify(e.to_record()) for e in r.trace]}


REF_CONFIGS = [
    # name, model kwargs, P, G, seeds, scheduler kwargs
    ("default_b4_128_g64", dict(), 16, 64, range(10), dict(gen_len=64)),
    ("default_b8_32_g128", dict(), 16, 128, range(10), dict(block_sizes=(8, 16, 32), gen_len=128)),
    ("default_r4", dict(), 16, 64, range(6), dict(gen_len=64, refresh_interval=4)),
    ("default_r1_tau1", dict(), 16, 32, range(4), dict(gen_len=32, refresh_interval=1, tau_conf=1.0)),
    ("default_nomerge", dict(), 16, 64, range(5), dict(gen_len=64, merge_enabled=False)),
    ("default_nosync", dict(), 16, 64, range(5), dict(gen_len=64, sync_enabled=False)),
    ("default_sync0_merge0", dict(), 16, 64, range(5), dict(gen_len=64, tau_sync=0, tau_merge=0.0)),
    ("default_single8", dict(), 16, 64, range(5),
     dict(block_sizes=(8,), gen_len=64, merge_enabled=False, sync_enabled=False)),
    ("default_g3", dict(), 5, 3, range(6), dict(block_sizes=(1, 2, 4), gen_len=3)),
    ("default_g4_eos", dict(), 8, 4, range(8), dict(block_sizes=(2, 3), gen_len=4)),
    ("c1_hs2", dict(vocab=4096, layers=4, d_model=256, max_len=192, head_scale=2.0), 64, 128,
     range(4), dict(block_sizes=(8, 16, 32), gen_len=128)),
    ("c1_hs1", dict(vocab=4096, layers=4, d_model=256, max_len=192, head_scale=1.0), 64, 128,
     range(4), dict(block_sizes=(8, 16, 32), gen_len=128)),
]


def ref_params(mk):
    V = mk.get("vocab", 32)
    vocab = bbm.Vocab(size=V, category_of=bbm._default_categories(V))
    dims = bbm.ModelDims(layers=mk.get("layers", 2), d_model=mk.get("d_model", 32),
                         max_len=mk.get("max_len", 384))
    return bbm.build_model(0, vocab, dims, head_scale=mk.get("head_scale", 1.0)), vocab


def gen_ref_runs():
    out = {}
    for name, mk, P, G, seeds, sk in REF_CONFIGS:
        t0 = time.time()
        params, vocab = ref_params(mk)
        cfg = bbs.SchedulerConfig(**sk)
        runs = []
        for s in seeds:
            task = bbm.make_task(s, P, G, vocab)
            runs.append(result_record(bbs.run_blockbatch(params, task, cfg)))
        out[name] = {"model": {"vocab_size": vocab.size, "layers": params.dims.layers,
                               "d_model": params.dims.d_model, "max_len": params.dims.max_len,
                               "head_scale": params.head_scale, "gamma": params.gamma,
                               "radius": params.radius, "spike_cut": params.spike_cut,
                               "spike_gain": params.spike_gain, "seed": 0},
                     "prompt_len": P, "gen_len": G, "seeds": list(seeds),
                     "config": {k: (list(v) if isinstance(v, tuple) else v)
                                for k, v in cfg.__dict__.items()},
                     "runs": runs}
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)
    # single-branch decoder (equivalence oracle, decoding.py:203-276)
    params, vocab = ref_params({})
    sb = []
    for s in range(4):
        task = bbm.make_task(s, 16, 64, vocab)
        for b in (4, 32):
            r = bbd.single_branch_decode(params, task, bbd.DecodeConfig(block_size=b, gen_len=64))
            rec = result_record(r)
            rec.update(seed=s, block=b)
            sb.append(rec)
    out["single_branch_default"] = {"prompt_len": 16, "gen_len": 64, "runs": sb}
    return out


# ---- KV-space logging (row f(4)): run_blockbatch with log_kv / log_consistency --

DIAG_CONFIGS = [
    ("diag_default", dict(), 16, 64, range(4), dict(gen_len=64, log_kv="norms", log_consistency=True)),
    ("diag_r4", dict(), 16, 64, range(3), dict(gen_len=64, refresh_interval=4, log_kv="norms",
                                              log_consistency=True)),
    ("diag_b8_32", dict(), 16, 64, range(3), dict(block_sizes=(8, 16, 32), gen_len=64, refresh_interval=8,
                                                  log_kv="norms", log_consistency=True)),
]


def gen_diag_runs():
    out = {}
    for name, mk, P, G, seeds, sk in DIAG_CONFIGS:
        t0 = time.time()
        params, vocab = ref_params(mk)
        cfg = bbs.SchedulerConfig(**sk)
        runs = []
        for s in seeds:
            task = bbm.make_task(s, P, G, vocab)
            runs.append(result_record(bbs.run_blockbatch(params, task, cfg)))
        out[name] = {"model": {"vocab_size": vocab.size, "layers": params.dims.layers,
                               "d_model": params.dims.d_model, "max_len": params.dims.max_len,
                               "head_scale": params.head_scale, "gamma": params.gamma,
                               "radius": params.radius, "spike_cut": params.spike_cut,
                               "spike_gain": params.spike_gain, "seed": 0},
                     "prompt_len": P, "gen_len": G, "seeds": list(seeds),
                     "config": {k: (list(v) if isinstance(v, tuple) else v) for k, v in cfg.__dict__.items()},
                     "runs": runs}
        print(f"diag {name}: {time.time() - t0:.1f}s", flush=True)
    return out


# ---- vanilla_decode (decoding.py:279-321), the baseline decoder of row f(3) --

VANILLA_CONFIGS = [
    ("default_g32", dict(), 16, 32, range(6)),
    ("default_g64", dict(), 16, 64, range(4)),
    ("c1_hs2_g128", dict(vocab=4096, layers=4, d_model=256, max_len=192, head_scale=2.0), 64, 128, range(2)),
]


def gen_vanilla_runs():
    out = {}
    for name, mk, P, G, seeds in VANILLA_CONFIGS:
        t0 = time.time()
        params, vocab = ref_params(mk)
        runs = []
        for s in seeds:
            task = bbm.make_task(s, P, G, vocab)
            runs.append(result_record(bbd.vanilla_decode(params, task, bbd.DecodeConfig(block_size=G, gen_len=G))))
        out[name] = {"model": {"vocab_size": vocab.size, "layers": params.dims.layers,
                               "d_model": params.dims.d_model, "max_len": params.dims.max_len,
                               "head_scale": params.head_scale, "gamma": params.gamma,
                               "radius": params.radius, "spike_cut": params.spike_cut,
                               "spike_gain": params.spike_gain, "seed": 0},
                     "prompt_len": P, "gen_len": G, "seeds": list(seeds), "runs": runs}
        print(f"vanilla {name}: {time.time() - t0:.1f}s", flush=True)
    return out


# ---- LLaDA / Dream shape via the reference scheduler + oracle forward -------

LLADA_CONFIGS = [
    ("llada_tiny", dict(kind="llada", vocab_size=1000, layers=2, d_model=256, n_heads=4,
                        n_kv_heads=4, head_dim=64, d_ff=512, max_len=192, rope_theta=500000.0,
                        norm_eps=1e-5, head_scale=0.25), 32, 64, range(6),
     dict(block_sizes=(8, 16, 32), gen_len=64)),
    ("dream_tiny", dict(kind="llada", vocab_size=1000, layers=2, d_model=256, n_heads=4,
                        n_kv_heads=2, head_dim=64, d_ff=640, max_len=192, rope_theta=1e6,
                        norm_eps=1e-6, qkv_bias=True, head_scale=0.25), 32, 64, range(6),
     dict(block_sizes=(4, 16, 32), gen_len=64, refresh_interval=2)),
]


class _Params:
    def __init__(self, vocab):
        self.vocab = vocab


def injected(arch, W, rnd):
    def ff(params, row, target):
        o, c = O.full_forward(arch, W, row.tokens, row.prompt_len, target, rnd)
        return (bbm.DenoiseOutput(o.positions, o.logits, o.probs),
                bbm.KvCache(c["k"], c["v"], c["valid"]))

    def bf(params, row, cache, window, target):
        oc = {"k": cache.keys, "v": cache.values, "valid": cache.valid}
        o, c = O.block_forward(arch, W, row.tokens, row.prompt_len, oc, window.start,
                               window.end, target, rnd)
        return (bbm.DenoiseOutput(o.positions, o.logits, o.probs),
                bbm.KvCache(c["k"], c["v"], c["valid"]))
    return ff, bf


def gen_llada_runs():
    out = {}
    saved = (bbs.full_forward, bbs.block_forward)
    try:
        for name, ak, P, G, seeds, sk in LLADA_CONFIGS:
            arch = O.OArch(**ak)
            base = O.hash_weights(arch, 0)
            for mode in ("f32", "bf16"):
                t0 = time.time()
                W = O.weights_as(base, mode)
                rnd = O.bf16_round if mode == "bf16" else None
                bbs.full_forward, bbs.block_forward = injected(arch, W, rnd)
                vocab = bbm.Vocab(size=arch.vocab_size,
                                  category_of=bbm._default_categories(arch.vocab_size))
                cfg = bbs.SchedulerConfig(**sk)
                runs = []
                for s in seeds:
                    task = bbm.make_task(s, P, G, vocab)
                    runs.append(result_record(bbs.run_blockbatch(_Params(vocab), task, cfg)))
                out[f"{name}_{mode}"] = {
                    "arch": ak, "weights": {"kind": "hash", "seed": 0, "mode": mode},
                    "prompt_len": P, "gen_len": G, "seeds": list(seeds),
                    "config": {k: (list(v) if isinstance(v, tuple) else v)
                               for k, v in cfg.__dict__.items()},
                    "runs": runs}
                print(f"{name}_{mode}: {time.time() - t0:.1f}s", flush=True)
    finally:
        bbs.full_forward, bbs.block_forward = saved
    return out


# ---- kernel-level fixtures -------------------------------------------------

def gen_kernel_fixtures(n_trans=600, n_merge=400):
    vocab = bbm.Vocab()
    trans = []
    for seed in range(n_trans):
        tokens, P, s, e, masked, probs, tau = fuzz.transition_instance(seed)
        row = bbm.SequenceRow(tokens.copy(), P)
        outp = bbm.DenoiseOutput(masked, np.log(probs + 1e-300), probs)
        commits = bbd.confidence_transition(outp, row, bbm.BlockWindow(s, e), tau)
        trans.append({"seed": seed, "commits": [[int(p), int(t)] for p, t in commits]})
    merges = []
    for seed in range(n_merge):
        nb = 3 + seed % 3
        st = fuzz.merge_state(seed, n_branches=nb)
        rows = [bbm.SequenceRow(st["rows"][i].copy(), st["prompt_len"]) for i in range(nb)]
        branches = []
        for i in range(nb):
            b = bbd.BranchState(index=i, block_size=int(st["block_sizes"][i]),
                                window=bbm.BlockWindow(int(st["starts"][i]), int(st["ends"][i])),
                                done=bool(st["done"][i]),
                                prob_map=st["prob_maps"][i].copy(),
                                prob_covered=st["covered"][i].copy())
            b.refresh_decoded(rows[i], vocab.mask_id)
            branches.append(b)

        class FC:
            def __init__(self, tag):
                self.tag = tag

            def copy(self):
                return FC(self.tag)
        caches = [FC(i) for i in range(nb)]
        tau_merge = [0.03, 0.5, 0.0][seed % 3]
        tau_sync = [6, 8, 0][seed % 3]
        events = bbs.merge_sync(rows, caches, branches, tau_merge, tau_sync, vocab,
                                merge_enabled=(seed % 7 != 3), sync_enabled=(seed % 5 != 2))
        merges.append({
            "seed": seed, "n_branches": nb, "tau_merge": tau_merge, "tau_sync": tau_sync,
            "merge_enabled": seed % 7 != 3, "sync_enabled": seed % 5 != 2,
            "events": [bbs._jsonify(ev) for ev in events],
            "rows": [[int(t) for t in r.tokens] for r in rows],
            "cache_tags": [c.tag for c in caches],
            "branches": [{"start": b.window.start, "end": b.window.end, "done": b.done,
                          "tokens_decoded": b.tokens_decoded, "tokens_merged": b.tokens_merged,
                          "covered": [int(x) for x in b.prob_covered]} for b in branches]})
    return {"transition": trans, "merge": merges}


def gen_forward_c1():
    params, vocab = ref_params(dict(vocab=4096, layers=4, d_model=256, max_len=192, head_scale=2.0))
    task = bbm.make_task(0, 64, 128, vocab)
    row = task.fresh_row(vocab)
    out, cache = bbm.full_forward(params, row, task.target)
    row2 = row.copy()
    row2.tokens[64:70] = task.target[:6]
    out2, _ = bbm.block_forward(params, row2, cache, bbm.BlockWindow(64, 96), task.target)
    res = {}
    for tag, o in (("full", out), ("block", out2)):
        lse = o.logits.max(1) + np.log(np.exp(o.logits - o.logits.max(1, keepdims=True)).sum(1))
        res[f"{tag}_positions"] = o.positions
        res[f"{tag}_maxlogit"] = o.logits.max(1)
        res[f"{tag}_argmax"] = o.probs.argmax(1)
        res[f"{tag}_conf"] = o.probs.max(1)
        res[f"{tag}_lse"] = lse
        res[f"{tag}_logits_rows"] = o.logits[:4].astype(np.float32)
    res["block_tokens"] = row2.tokens
    return res


# ---- hard cap (scheduler.py:310, 324-325) and forward_hook order ------------

def gen_runaway_runs():
    """Reference runs with HARD_CAP_FACTOR = 0 (cap = 16 forwards): the
    forward_hook calls up to the RunawayError, or the full list if the run
    finishes under the cap."""
    params, vocab = ref_params({})
    cfg = bbs.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=128)
    saved = bbs.HARD_CAP_FACTOR
    runs = []
    try:
        bbs.HARD_CAP_FACTOR = 0
        for s in range(6):
            task = bbm.make_task(s, 16, 128, vocab)
            calls = []
            try:
                r = bbs.run_blockbatch(params, task, cfg, forward_hook=calls.append)
                runs.append({"seed": s, "raised": False, "calls": calls, "nfe": list(r.nfe.snapshot())})
            except bbs.RunawayError:
                runs.append({"seed": s, "raised": True, "calls": calls})
    finally:
        bbs.HARD_CAP_FACTOR = saved
    return {"hard_cap": 16, "prompt_len": 16, "gen_len": 128, "block_sizes": [8, 16, 32], "runs": runs}


def gen_preset_runs():
    """single_branch_decode(preset=...) on the default model: per seed a preset
    of two target tokens, one wrong token and (odd seeds) an eos."""
    params, vocab = ref_params({})
    P, G = 16, 64
    runs = []
    for s in range(4):
        task = bbm.make_task(s, P, G, vocab)
        preset = [(P + 1, int(task.target[1])), (P + 5, int(task.target[5])),
                  (P + 9, int((task.target[9] + 1) % vocab.size))]
        if s % 2:
            preset.append((P + 40, vocab.eos_id))
        for b in (4, 16):
            r = bbd.single_branch_decode(params, task, bbd.DecodeConfig(block_size=b, gen_len=G), preset=preset)
            rec = result_record(r)
            rec.update(seed=s, block=b, preset=preset)
            runs.append(rec)
    return {"prompt_len": P, "gen_len": G, "runs": runs}


SUMMARY_CONFIGS = ("c1_hs2", "default_g4_eos")


def gen_summary_csv(path):
    """The reference's own summary_row / write_summary over the golden runs."""
    from blockbatch import cli as bbc
    runs = json.load(open(os.path.join(HERE, "runs_ref.json")))
    rows = []
    for name in SUMMARY_CONFIGS:
        g = runs[name]
        vs = g["model"]["vocab_size"]
        vocab = bbm.Vocab(size=vs, category_of={t: f"c{t % 4}" for t in range(vs)}) if vs != 32 else bbm.Vocab()
        for seed, r in zip(g["seeds"], g["runs"]):
            res = bbd.GenerationResult(row=bbm.SequenceRow(np.array(r["tokens"], dtype=np.int64), g["prompt_len"]),
                                       branch_index=r["branch_index"], block_size=r["block_size"],
                                       nfe=bbd.NfeCounter(*r["nfe"]), trace=[], correct=r["correct"],
                                       tokens_decoded=r["tokens_decoded"], eos_position=r["eos_position"])
            rows.append(bbc.summary_row(seed, f"blockbatch:{name}", res, vocab))
    bbc.write_summary(path, rows)


def main():
    t0 = time.time()
    if "--preset-only" in sys.argv:
        with open(os.path.join(HERE, "runs_preset.json"), "w") as fh:
            json.dump(gen_preset_runs(), fh, separators=(",", ":"))
        print(f"done in {time.time() - t0:.1f}s")
        return
    if "--summary-only" in sys.argv:
        gen_summary_csv(os.path.join(HERE, "summary_ref.csv"))
        print(f"done in {time.time() - t0:.1f}s")
        return
    with open(os.path.join(HERE, "runs_runaway.json"), "w") as fh:
        json.dump(gen_runaway_runs(), fh, separators=(",", ":"))
    if "--runaway-only" in sys.argv:
        print(f"done in {time.time() - t0:.1f}s")
        return
    with open(os.path.join(HERE, "runs_vanilla.json"), "w") as fh:
        json.dump(gen_vanilla_runs(), fh, separators=(",", ":"))
    with open(os.path.join(HERE, "runs_diag.json"), "w") as fh:
        json.dump(gen_diag_runs(), fh, separators=(",", ":"))
    if "--vanilla-only" in sys.argv:
        print(f"done in {time.time() - t0:.1f}s")
        return
    with open(os.path.join(HERE, "runs_ref.json"), "w") as fh:
        json.dump(gen_ref_runs(), fh, separators=(",", ":"))
    with open(os.path.join(HERE, "runs_llada.json"), "w") as fh:
        json.dump(gen_llada_runs(), fh, separators=(",", ":"))
    with open(os.path.join(HERE, "kernels.json"), "w") as fh:
        json.dump(gen_kernel_fixtures(), fh, separators=(",", ":"))
    np.savez_compressed(os.path.join(HERE, "forward_c1.npz"), **gen_forward_c1())
    gen_summary_csv(os.path.join(HERE, "summary_ref.csv"))
    with open(os.path.join(HERE, "runs_preset.json"), "w") as fh:
        json.dump(gen_preset_runs(), fh, separators=(",", ":"))
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
