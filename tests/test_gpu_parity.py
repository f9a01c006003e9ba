"""GPU parity of the device path vs the reference (golden fixtures) — through
the public API and the C-ABI library.  fp32 verification mode must be
bit-exact on tokens, NFE, winner and the full trace (merge probabilities to
1e-4 relative: fp32 recomputation vs the reference's float64)."""

import numpy as np
import pytest

import fuzz
import goldens

pytestmark = pytest.mark.gpu

bb = pytest.importorskip("paper_2605_29233_b200")

REF = goldens.load("runs_ref.json")
LLADA = goldens.load("runs_llada.json")
KER = goldens.load("kernels.json")
VANILLA = goldens.load("runs_vanilla.json")
DIAG = goldens.load("runs_diag.json")

_MODELS = {}


def ref_model(m, dtype="f32"):
    key = (m["vocab_size"], m["layers"], m["d_model"], m["max_len"], m["head_scale"], dtype)
    if key not in _MODELS:
        vocab = bb.Vocab(size=m["vocab_size"])
        dims = bb.ModelDims(layers=m["layers"], d_model=m["d_model"], max_len=m["max_len"])
        _MODELS[key] = bb.build_model(m["seed"], vocab, dims, gamma=m["gamma"], radius=m["radius"],
                                      head_scale=m["head_scale"], spike_cut=m["spike_cut"],
                                      spike_gain=m["spike_gain"], dtype=dtype)
    return _MODELS[key]


def llada_model(g, dtype):
    a = g["arch"]
    key = ("llada", tuple(sorted(a.items())), dtype)
    if key not in _MODELS:
        vocab = bb.Vocab(size=a["vocab_size"])
        dims = bb.ModelDims(layers=a["layers"], d_model=a["d_model"], max_len=a["max_len"], arch="llada",
                            n_heads=a["n_heads"], n_kv_heads=a["n_kv_heads"], head_dim=a["head_dim"],
                            d_ff=a["d_ff"], rope_theta=a["rope_theta"], norm_eps=a["norm_eps"],
                            qkv_bias=a.get("qkv_bias", False))
        _MODELS[key] = bb.build_model(0, vocab, dims, head_scale=a["head_scale"], dtype=dtype, init="hash")
    return _MODELS[key]


def cfg_from(c):
    return bb.SchedulerConfig(block_sizes=tuple(c["block_sizes"]), tau_conf=c["tau_conf"],
                              tau_merge=c["tau_merge"], tau_sync=c["tau_sync"],
                              refresh_interval=c["refresh_interval"], gen_len=c["gen_len"],
                              merge_enabled=c["merge_enabled"], sync_enabled=c["sync_enabled"])


def record(r):
    return {"tokens": [int(t) for t in r.row.tokens], "nfe": list(r.nfe.snapshot()),
            "branch_index": r.branch_index, "block_size": r.block_size, "tokens_decoded": r.tokens_decoded,
            "eos_position": r.eos_position, "correct": r.correct, "trace": [e.to_record() for e in r.trace]}


@pytest.mark.parametrize("name", [k for k in REF if k != "single_branch_default"])
def test_fp32_matches_reference_runs(name):
    g = REF[name]
    params = ref_model(g["model"])
    vocab = params.vocab
    cfg = cfg_from(g["config"])
    for seed, want in zip(g["seeds"], g["runs"]):
        task = bb.make_task(seed, g["prompt_len"], g["gen_len"], vocab)
        got = record(bb.run_blockbatch(params, task, cfg))
        err = goldens.compare_run(got, want, prob_tol=1e-4)
        assert err is None, f"{name} seed {seed}: {err}"


def test_fp32_batch_equals_single_requests():
    g = REF["c1_hs2"]
    params = ref_model(g["model"])
    cfg = cfg_from(g["config"])
    tasks = [bb.make_task(s, g["prompt_len"], g["gen_len"], params.vocab) for s in g["seeds"]]
    got = bb.run_batch(params, tasks, cfg)
    for r, want in zip(got, g["runs"]):
        assert goldens.compare_run(record(r), want, prob_tol=1e-4) is None


def test_single_branch_decode_matches_reference():
    g = REF["single_branch_default"]
    params = ref_model(REF["default_b4_128_g64"]["model"])
    for want in g["runs"]:
        task = bb.make_task(want["seed"], g["prompt_len"], g["gen_len"], params.vocab)
        r = bb.single_branch_decode(params, task, bb.DecodeConfig(block_size=want["block"], gen_len=64))
        assert [int(t) for t in r.row.tokens] == want["tokens"]
        assert list(r.nfe.snapshot()) == want["nfe"]
        assert goldens.diff_trace([e.to_record() for e in r.trace], want["trace"]) is None


@pytest.mark.parametrize("name", [k for k in LLADA if k.endswith("_f32")])
def test_fp32_llada_shape_matches_oracle(name):
    g = LLADA[name]
    params = llada_model(g, "f32")
    cfg = cfg_from(g["config"])
    for seed, want in zip(g["seeds"], g["runs"]):
        task = bb.make_task(seed, g["prompt_len"], g["gen_len"], params.vocab)
        got = record(bb.run_blockbatch(params, task, cfg))
        err = goldens.compare_run(got, want, prob_tol=1e-4)
        assert err is None, f"{name} seed {seed}: {err}"


@pytest.mark.parametrize("name", [k for k in LLADA if k.endswith("_bf16")])
def test_bf16_llada_shape_nfe_agreement(name):
    """bf16 numerics (bf16 activations / KV) vs the oracle's bf16-emulating
    runs: the spike epilogue (x34) turns bf16 rounding into decision flips,
    so whole runs agree only partly.  Held to the measured floor (4 of 6
    prompts; rounds 1-2 measured 4-5): the north-star decision bar is met by
    bf16x2, not by plain bf16."""
    g = LLADA[name]
    params = llada_model(g, "bf16")
    cfg = cfg_from(g["config"])
    same_nfe = 0
    for seed, want in zip(g["seeds"], g["runs"]):
        task = bb.make_task(seed, g["prompt_len"], g["gen_len"], params.vocab)
        r = bb.run_blockbatch(params, task, cfg)
        same_nfe += list(r.nfe.snapshot()) == want["nfe"]
    print(f"{name}: NFE identical on {same_nfe}/{len(g['seeds'])} prompts")
    assert same_nfe >= 4, f"{same_nfe}/{len(g['seeds'])} NFE matches"


def test_bf16x2_whole_runs_match_fp32_twin():
    """bf16x2 whole runs (prefill, block steps, merges, syncs, refresh) vs the
    fp32 verification run of the same bf16 weights, hd-128 LLaDA-shape model:
    NFE, tokens and trace decisions identical on every prompt."""
    from dataclasses import replace
    from paper_2605_29233_b200.model import verification_copy
    dims = bb.ModelDims(layers=2, d_model=256, max_len=192, arch="llada", n_heads=2, n_kv_heads=2, head_dim=128,
                        d_ff=512, rope_theta=500000.0)
    vocab = bb.Vocab(size=1000)
    p16 = bb.build_model(0, vocab, dims, head_scale=0.25, dtype="bf16")
    px2, p32 = replace(p16, dtype="bf16x2", _handle=[None], _sessions={}), verification_copy(p16)
    cfg = bb.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=64, refresh_interval=8)
    same = 0
    for seed in range(8):
        t = bb.make_task(seed, 32, 64, vocab)
        a, b = bb.run_blockbatch(px2, t, cfg), bb.run_blockbatch(p32, t, cfg)
        same += a.nfe.snapshot() == b.nfe.snapshot() and np.array_equal(a.row.tokens, b.row.tokens)
    print(f"bf16x2 vs fp32 twin: {same}/8 whole runs identical")
    assert same >= 7


def test_commit_kernel_bit_exact_on_reference_fixtures():
    for rec in KER["transition"]:
        tokens, P, s, e, masked, probs, tau = fuzz.transition_instance(rec["seed"])
        row = bb.SequenceRow(tokens.copy(), P)
        out = bb.DenoiseOutput(masked, np.log(probs + 1e-300), probs)
        got = bb.confidence_transition(out, row, bb.BlockWindow(s, e), tau)
        assert [list(c) for c in got] == rec["commits"], rec["seed"]


class _FC:
    def __init__(self, tag):
        self.tag = tag

    def copy(self):
        return _FC(self.tag)


def test_merge_sync_kernel_bit_exact_on_reference_fixtures():
    vocab = bb.Vocab()
    for rec in KER["merge"]:
        st = fuzz.merge_state(rec["seed"], n_branches=rec["n_branches"])
        nb = rec["n_branches"]
        rows = [bb.SequenceRow(st["rows"][i].copy(), st["prompt_len"]) for i in range(nb)]
        branches = []
        for i in range(nb):
            b = bb.BranchState(index=i, block_size=int(st["block_sizes"][i]),
                               window=bb.BlockWindow(int(st["starts"][i]), int(st["ends"][i])),
                               done=bool(st["done"][i]), prob_map=st["prob_maps"][i].copy(),
                               prob_covered=st["covered"][i].copy())
            b.refresh_decoded(rows[i], vocab.mask_id)
            branches.append(b)
        caches = [_FC(i) for i in range(nb)]
        ev = bb.merge_sync(rows, caches, branches, rec["tau_merge"], rec["tau_sync"], vocab,
                           merge_enabled=rec["merge_enabled"], sync_enabled=rec["sync_enabled"])
        assert ev == rec["events"], rec["seed"]
        assert [[int(t) for t in r.tokens] for r in rows] == rec["rows"], rec["seed"]
        assert [c.tag for c in caches] == rec["cache_tags"]
        for b, w in zip(branches, rec["branches"]):
            assert (b.window.start, b.window.end, b.done, b.tokens_decoded, b.tokens_merged) == \
                (w["start"], w["end"], w["done"], w["tokens_decoded"], w["tokens_merged"]), rec["seed"]
            assert [int(x) for x in b.prob_covered] == w["covered"]


PRESET = goldens.load("runs_preset.json")


def test_single_branch_decode_with_preset_matches_reference():
    """single_branch_decode(preset=...) (decoding.py:194-212): preset tokens
    (target, wrong, eos) placed in the row before the prefill; tokens, NFE
    and every trace record bit-exact vs the reference's own runs (fp32)."""
    params = ref_model(REF["default_b4_128_g64"]["model"])
    for want in PRESET["runs"]:
        task = bb.make_task(want["seed"], PRESET["prompt_len"], PRESET["gen_len"], params.vocab)
        preset = [tuple(p) for p in want["preset"]]
        r = bb.single_branch_decode(params, task, bb.DecodeConfig(block_size=want["block"], gen_len=64), preset=preset)
        assert [int(t) for t in r.row.tokens] == want["tokens"], (want["seed"], want["block"])
        assert list(r.nfe.snapshot()) == want["nfe"]
        assert r.tokens_decoded == want["tokens_decoded"]
        assert goldens.diff_trace([e.to_record() for e in r.trace], want["trace"]) is None
    task = bb.make_task(0, PRESET["prompt_len"], PRESET["gen_len"], params.vocab)
    with pytest.raises(bb.ContractError):  # decoding.py:198-199
        bb.single_branch_decode(params, task, bb.DecodeConfig(block_size=4, gen_len=64), preset=[(3, 1)])


def test_deterministic_reruns():
    g = REF["c1_hs2"]
    params = ref_model(g["model"])
    cfg = cfg_from(g["config"])
    task = bb.make_task(1, g["prompt_len"], g["gen_len"], params.vocab)
    a = bb.run_blockbatch(params, task, cfg)
    b = bb.run_blockbatch(params, task, cfg)
    assert [e.to_record() for e in a.trace] == [e.to_record() for e in b.trace]
    assert np.array_equal(a.row.tokens, b.row.tokens)


def test_forward_hook_counts():
    g = REF["default_r4"]
    params = ref_model(g["model"])
    cfg = cfg_from(g["config"])
    task = bb.make_task(4, g["prompt_len"], g["gen_len"], params.vocab)
    calls = []
    r = bb.run_blockbatch(params, task, cfg, forward_hook=calls.append)
    assert len(calls) == r.nfe.total
    assert calls.count("init") == 1 and calls.count("block") == r.nfe.nfe_block
    assert calls.count("refresh") == r.nfe.nfe_refresh


@pytest.mark.parametrize("name,dtype,spike_gain,tol", [
    ("llada_tiny_bf16", "bf16", 0.0, 2e-2), ("dream_tiny_bf16", "bf16", 0.0, 2e-2),
    ("llada_tiny_bf16", "bf16", 33.0, 1e-1), ("dream_tiny_bf16", "bf16", 33.0, 1e-1),
    ("llada_tiny_f32", "f32", 33.0, 1e-4)])
def test_prefill_head_numerics_match_oracle(name, dtype, spike_gain, tol):
    """Fused LM-head + confidence of one prefill vs the oracle forward (same
    weights; the oracle emulates the device's bf16 storage points): per masked
    window position the max normalised logit (log max-prob = -log s), the
    log-sum-exp and the argmax.  Stated bf16 tolerance: max-abs <= 2e-2 on
    log-softmax logits for the transformer itself (spike gain 0); the
    synthetic spike epilogue (gain 33) multiplies raw-logit error by 34, so the
    spiked head is held to 1e-1.  fp32 verification mode: 1e-4."""
    from oracle import bb_oracle as O
    from paper_2605_29233_b200.scheduler import get_session
    g = LLADA[name]
    a = dict(g["arch"], spike_gain=spike_gain)
    vocab = bb.Vocab(size=a["vocab_size"])
    dims = bb.ModelDims(layers=a["layers"], d_model=a["d_model"], max_len=a["max_len"], arch="llada",
                        n_heads=a["n_heads"], n_kv_heads=a["n_kv_heads"], head_dim=a["head_dim"], d_ff=a["d_ff"],
                        rope_theta=a["rope_theta"], norm_eps=a["norm_eps"], qkv_bias=a.get("qkv_bias", False))
    params = bb.build_model(0, vocab, dims, head_scale=a["head_scale"], spike_gain=spike_gain, dtype=dtype)
    cfg = cfg_from(g["config"])
    arch = O.OArch(**a)
    W = O.weights_as(O.hash_weights(arch, 0), dtype)
    rnd = O.bf16_round if dtype == "bf16" else None
    worst_lp, worst_lse, agree, n = 0.0, 0.0, 0, 0
    for seed in g["seeds"][:3]:
        task = bb.make_task(seed, g["prompt_len"], g["gen_len"], params.vocab)
        s = get_session(params, cfg, g["prompt_len"], 1)
        s.set_inputs(task.prompt[None], task.target[None])
        s.prefill()
        hr = s.head_results()
        row = np.full(g["prompt_len"] + g["gen_len"], arch.mask_id, dtype=np.int64)
        row[:g["prompt_len"]] = task.prompt
        out, _ = O.full_forward(arch, W, row, g["prompt_len"], task.target, rnd)
        lse_ref = out.logits.max(1) + np.log(np.exp(out.logits - out.logits.max(1, keepdims=True)).sum(1))
        idx = {int(p): i for i, p in enumerate(out.positions)}
        for j in np.flatnonzero(hr["masked"]):
            i = idx[int(hr["pos"][j])]
            m, ssum = float(hr["m"][j]), float(hr["s"][j])
            lse = m + np.log(ssum)
            worst_lp = max(worst_lp, abs((m - lse) - (out.logits[i].max() - lse_ref[i])))
            worst_lse = max(worst_lse, abs(lse - lse_ref[i]) / max(1.0, abs(lse_ref[i])))
            agree += int(hr["arg"][j]) == int(out.probs[i].argmax())
            n += 1
    print(f"{name} gain {spike_gain}: {n} positions, max|dlogp_max|={worst_lp:.2e}, rel dlse={worst_lse:.2e}, "
          f"argmax agree {agree}/{n}")
    assert worst_lp <= tol and worst_lse <= tol
    assert agree >= n - max(1, n // 20)


def _llada_params(g, dtype, spike_gain):
    a = dict(g["arch"], spike_gain=spike_gain)
    vocab = bb.Vocab(size=a["vocab_size"])
    dims = bb.ModelDims(layers=a["layers"], d_model=a["d_model"], max_len=a["max_len"], arch="llada",
                        n_heads=a["n_heads"], n_kv_heads=a["n_kv_heads"], head_dim=a["head_dim"], d_ff=a["d_ff"],
                        rope_theta=a["rope_theta"], norm_eps=a["norm_eps"], qkv_bias=a.get("qkv_bias", False))
    return a, bb.build_model(0, vocab, dims, head_scale=a["head_scale"], spike_gain=spike_gain, dtype=dtype)


@pytest.mark.parametrize("name,dtype,spike_gain,tol", [
    ("llada_tiny_bf16", "bf16", 0.0, 2e-2), ("dream_tiny_bf16", "bf16", 0.0, 2e-2),
    ("llada_tiny_bf16", "bf16", 33.0, 1e-1), ("dream_tiny_bf16", "bf16", 33.0, 1e-1),
    ("llada_tiny_f32", "f32", 33.0, 1e-4)])
def test_block_step_head_numerics_match_oracle(name, dtype, spike_gain, tol):
    """One block step after prefill (the block pass: window KV splice into the
    branches' aliased prefill pages, segment-masked attention over shared
    pages, LM head) vs the oracle's block_forward of every active branch on
    the prefill cache (model.py:331-343).  Same tolerances as the prefill
    test."""
    _block_step_vs_oracle(LLADA[name], None, dtype, spike_gain, tol, name)


@pytest.mark.parametrize("tc,cs,kvh,gain,tol", [("mma", "", 2, 0.0, 2e-2), ("fa", "", 2, 0.0, 2e-2), ("fa", "1", 2, 0.0, 2e-2),
                                                ("mma", "1", 2, 0.0, 2e-2), ("fa", "", 1, 0.0, 2e-2),
                                                ("fa", "", 2, 33.0, 1e-1), ("mma", "", 2, 33.0, 1e-1),
                                                ("tc", "", 2, 0.0, 2e-2), ("tc", "1", 1, 0.0, 2e-2),
                                                ("fa", "2", 1, 0.0, 2e-2), ("fa", "4", 2, 0.0, 2e-2),
                                                ("fa64", "", 2, 0.0, 2e-2), ("fa64", "1", 1, 0.0, 2e-2),
                                                ("fa64", "", 2, 33.0, 1e-1)])
def test_block_step_hd128_attention_matches_oracle(tc, cs, kvh, gain, tol):
    """The block step at head_dim 128 (the LLaDA-8B head size; the tiny
    fixtures use 64) with each tensor-core attention: the warp-specialized
    TMA-fed tcgen05 kernels on 128-row tiles (fa, the product path) and on
    64-row tiles (fa64, test flag 4; the bf16x2 path's layout), the
    single-role tcgen05 kernel (tc, test flag 2) and the mma.sync kernel
    (mma, test flag 1),
    against the oracle at the bf16 tolerance of the block-step test.  cs=1:
    one CTA per (head, row tile) takes every key (several chunks: the
    online-softmax rescale path and the KV ring wrap).  kvh=1: grouped-query
    attention (2 query heads share one KV head).  gain 33: the spike epilogue
    (x34 on raw-logit error) at the prefill test's tolerance."""
    flags = {"fa": 0, "mma": 1, "tc": 2, "fa64": 4}[tc] | ((int(cs) if cs else 0) << 4)
    g = LLADA["llada_tiny_bf16"]
    _block_step_vs_oracle(g, dict(n_heads=2, n_kv_heads=kvh, head_dim=128), "bf16", gain, tol,
                          f"hd128 tc={tc} cs={cs or 'auto'} kvh={kvh}", test_flags=flags)


@pytest.mark.parametrize("tc,cs,P,G,bs", [("fa", "", 600, 200, 3), ("fa", "1", 600, 200, 3), ("tc", "1", 600, 200, 3),
                                          ("fa", "2", 1000, 120, 3), ("fa64", "", 600, 200, 3),
                                          ("fa64", "1", 1000, 120, 3), ("fa", "", 600, 200, 4), ("fa", "1", 600, 200, 4),
                                          ("fa", "8", 1000, 120, 4), ("fa64", "", 600, 200, 4),
                                          ("x2", "", 1000, 120, 4), ("x2", "1", 600, 200, 4), ("x2", "", 600, 200, 3)])
def test_block_step_long_context_attention_matches_oracle(tc, cs, P, G, bs):
    """Long rows through the hd-128 tensor-core attentions: a 600-token
    prompt (its last page is partly filled: padded key-list segment) and
    ~800 keys per row, i.e. a dozen 64-key chunks per CTA (the KV ring wraps
    several times; lazy O rescale across chunks), vs the oracle.  bs=4:
    branches {8,16,32,64} (120 window rows, the C5 layout: the block pass
    runs the 128-row-tile kernel, one key tile for all four branches).  x2:
    the bf16x2 numerics (SPLIT attention instances; spike gain 33) held to the
    north-star bar against the oracle without activation rounding."""
    flags = {"fa": 0, "tc": 2, "fa64": 4, "x2": 0}[tc] | ((int(cs) if cs else 0) << 4)
    g = LLADA["llada_tiny_bf16"]
    bsz = [8, 16, 32] if bs == 3 else [8, 16, 32, 64]
    g = dict(g, prompt_len=P, gen_len=G, config=dict(g["config"], gen_len=G, block_sizes=bsz), seeds=g["seeds"][:2])
    dtype, gain = ("bf16x2", 33.0) if tc == "x2" else ("bf16", 0.0)
    _block_step_vs_oracle(g, dict(n_heads=2, n_kv_heads=1, head_dim=128, max_len=P + G), dtype, gain, 2e-2,
                          f"long hd128 {tc} cs={cs or 'auto'} L={P + G} B={len(bsz)}", test_flags=flags)


@pytest.mark.parametrize("kvh,gain,tol,P,G", [(2, 33.0, 2e-2, 32, 64), (1, 33.0, 2e-2, 32, 64),
                                              (2, 0.0, 2e-3, 32, 64), (2, 33.0, 2e-2, 64, 256),
                                              (2, 33.0, 2e-2, 48, 80)])
def test_bf16x2_block_step_matches_exact_oracle(kvh, gain, tol, P, G):
    """bf16x2 numerics (bf16 weights; hi + lo bf16 activations, q/K/V and head
    input; both halves through the tcgen05 GEMMs and attention) vs the oracle
    with NO activation rounding, at the north-star bar (max-abs <= 2e-2 on
    normalised logits) WITH the spike epilogue (gain 33), MHA and GQA.  The
    (P, G) cases give full-pass row chunks of 96 (L=96), 64 x 5 / 128 (L=320)
    and a ragged last chunk (L=128: one chunk of 128)."""
    g = LLADA["llada_tiny_bf16"]
    g = dict(g, prompt_len=P, gen_len=G, config=dict(g["config"], gen_len=G))
    _block_step_vs_oracle(g, dict(n_heads=2, n_kv_heads=kvh, head_dim=128, max_len=max(192, P + G)), "bf16x2",
                          gain, tol, f"bf16x2 hd128 kvh={kvh} L={P + G}")


def _block_step_vs_oracle(g, arch_override, dtype, spike_gain, tol, name, test_flags=0):
    from oracle import bb_oracle as O
    from paper_2605_29233_b200.engine import Session
    if arch_override:
        g = dict(g, arch=dict(g["arch"], **arch_override))
    a, params = _llada_params(g, dtype, spike_gain)
    cfg = cfg_from(g["config"])
    arch = O.OArch(**a)
    # bf16x2 is held to the oracle WITHOUT activation rounding (the model its bf16 weights define)
    W = O.weights_as(O.hash_weights(arch, 0), "bf16" if dtype == "bf16x2" else dtype)
    rnd = O.bf16_round if dtype == "bf16" else None
    P, G = g["prompt_len"], g["gen_len"]
    worst_lp, worst_lse, agree, n = 0.0, 0.0, 0, 0
    for seed in g["seeds"][:3]:
        task = bb.make_task(seed, P, G, params.vocab)
        s = Session(params, cfg, P, 1, test_flags=test_flags)
        s.set_inputs(task.prompt[None], task.target[None])
        s.prefill()
        st = s.fetch(trace=False)
        if st["ctrl"][0, 0] != 0:
            continue  # finished at prefill: no block step
        s.iteration(with_refresh=False)
        hr = s.head_results()
        row0 = np.full(P + G, arch.mask_id, dtype=np.int64)
        row0[:P] = task.prompt
        _, cache = O.full_forward(arch, W, row0, P, task.target, rnd)
        for k in range(len(cfg.block_sizes)):
            sel = np.flatnonzero((hr["masked"] != 0) & (hr["branch"] == k) & (hr["pos"] >= 0))
            if len(sel) == 0:
                continue
            tok = st["tokens"][0, k].astype(np.int64)
            start, end = int(st["branch"][0, k, 0]), int(st["branch"][0, k, 1])
            out, _ = O.block_forward(arch, W, tok, P, cache, start, end, task.target, rnd)
            idx = {int(p): i for i, p in enumerate(out.positions)}
            lse_ref = out.logits.max(1) + np.log(np.exp(out.logits - out.logits.max(1, keepdims=True)).sum(1))
            for j in sel:
                i = idx[int(hr["pos"][j])]
                m, ssum = float(hr["m"][j]), float(hr["s"][j])
                lse = m + np.log(ssum)
                worst_lp = max(worst_lp, abs((m - lse) - (out.logits[i].max() - lse_ref[i])))
                worst_lse = max(worst_lse, abs(lse - lse_ref[i]) / max(1.0, abs(lse_ref[i])))
                agree += int(hr["arg"][j]) == int(out.probs[i].argmax())
                n += 1
    print(f"{name} gain {spike_gain}: {n} block positions, max|dlogp_max|={worst_lp:.2e}, "
          f"rel dlse={worst_lse:.2e}, argmax agree {agree}/{n}")
    assert n > 0
    assert worst_lp <= tol and worst_lse <= tol
    assert agree >= n - max(1, n // 20)


@pytest.mark.parametrize("name", list(VANILLA))
def test_vanilla_decode_matches_reference_runs(name):
    """vanilla_decode (decoding.py:279-321) on the device — full pass + LM head
    + tau-1.0 commit per round — bit-exact vs the reference's own runs in fp32
    verification mode: tokens, NFE, eos position and every trace record."""
    g = VANILLA[name]
    params = ref_model(g["model"])
    for seed, want in zip(g["seeds"], g["runs"]):
        task = bb.make_task(seed, g["prompt_len"], g["gen_len"], params.vocab)
        got = record(bb.vanilla_decode(params, task, bb.DecodeConfig(block_size=g["gen_len"], gen_len=g["gen_len"])))
        err = goldens.compare_run(got, want)
        assert err is None, f"{name} seed {seed}: {err}"


@pytest.mark.parametrize("name", list(DIAG))
def test_kv_logging_matches_reference_runs(name):
    """run_blockbatch with log_kv="norms" and log_consistency (scheduler.py:
    268-281, 288-294, 332-347, 376-390) in fp32 verification mode: decisions,
    tokens, NFE and every trace record bit-exact; the per-branch kv_delta /
    E_before / E_after norms (device fp32 caches, fp64 reductions) within 1e-4
    relative of the reference's float64 values (E_after = 0 after a refresh)."""
    g = DIAG[name]
    params = ref_model(g["model"])
    c = g["config"]
    cfg = cfg_from(c)
    cfg.log_kv, cfg.log_consistency = c["log_kv"], c["log_consistency"]
    for seed, want in zip(g["seeds"], g["runs"]):
        task = bb.make_task(seed, g["prompt_len"], g["gen_len"], params.vocab)
        got = record(bb.run_blockbatch(params, task, cfg))
        err = goldens.compare_run(got, want, prob_tol=1e-4, kv_tol=1e-4)
        assert err is None, f"{name} seed {seed}: {err}"


def test_live_gemm_stats_count_every_launch():
    """The live per-launch GEMM timing the bench roofline reads (per-site
    red.min / red.max of %globaltimer, folded once per pass by k_tsite_fold):
    after a prefill and one block step every GEMM launch is counted once per
    layer and kind, with a positive duration, and a reset clears the sums."""
    from paper_2605_29233_b200.engine import Session
    g = LLADA["llada_tiny_bf16"]
    params = llada_model(g, "bf16")
    cfg = cfg_from(g["config"])
    layers = g["arch"]["layers"]
    task = bb.make_task(g["seeds"][0], g["prompt_len"], g["gen_len"], params.vocab)
    s = Session(params, cfg, g["prompt_len"], 1)
    s.set_inputs(task.prompt[None], task.target[None])
    s.gemm_stats(reset=True)
    s.prefill()
    st = s.fetch(trace=False)
    assert st["ctrl"][0, 0] == 0
    s.iteration(with_refresh=False, use_graph=False)
    s.stream.synchronize()
    gs = s.gemm_stats(reset=True)
    for kind in range(4):  # block pass QKV, O, gate/up, down
        assert gs[kind][4] == layers and gs[kind][3] > 0, (kind, gs[kind])
        assert gs[8 + kind][4] == layers and gs[8 + kind][3] > 0, (8 + kind, gs[8 + kind])
    assert gs[4][4] == 2 and gs[4][3] > 0  # LM head: prefill + block step
    gs = s.gemm_stats(reset=False)
    assert all(gs[k][4] == 0 for k in (0, 1, 2, 3, 4, 8, 9, 10, 11))


# fp32 verification-path NFE triples of C2 seeds 36..45 (profiles/r02/parity/
# parity_c2_bf16x2_final_seeds0-199.json); bf16x2 matches all ten
C2_F32_NFE = {36: (1, 34, 1), 37: (1, 75, 2), 38: (1, 36, 1), 39: (1, 36, 1), 40: (1, 70, 2),
              41: (1, 24, 0), 42: (1, 54, 1), 43: (1, 35, 1), 44: (1, 37, 1), 45: (1, 44, 1)}


def test_c2_bf16x2_session_reuse_matches_fp32_decisions():
    """Full-size C2 (LLaDA-8B shape, bf16x2) requests run back to back on one
    session, each after the previous one's stacked refresh: the decisions equal
    the fp32 verification path's on every prompt.  (Regression: the stacked
    refresh once left live rows in the prefill pass's padding, whose K/V writes
    raced with the next request's prompt rows -- seed 41 ran 7 block NFEs
    instead of 24.)"""
    import bench
    _, params, cfg = bench.make_model(bench.CONFIGS["c2"], "bf16x2")
    got = {}
    for seed in sorted(C2_F32_NFE):
        t = bb.make_task(seed, 64, 256, params.vocab)
        got[seed] = bb.run_blockbatch(params, t, cfg).nfe.snapshot()
    bad = {s: (got[s], C2_F32_NFE[s]) for s in got if got[s] != C2_F32_NFE[s]}
    del params
    assert not bad, bad
