"""The step-operator seams of the reference API on the device, and the live
host callbacks of run_blockbatch.

GPU equivalents of the reference's own seam tests -- test_model.py:55-89
(full-window block == full forward, bounds / cache-validity errors),
test_scheduler.py:72-91 (batched == sequential, bitwise),
test_acceptance.py:183-204 (criterion 05: replay every branch step through
block_forward, bitwise), test_scheduler.py:207-219 (NFE hook exactness) and
test_scheduler.py:245-260 (trace round trip) -- in fp32 verification mode,
plus the reference's own full_forward / block_forward numerics
(tests/golden/forward_c1.npz) and its hard-cap behaviour
(tests/golden/runs_runaway.json, RunawayError at scheduler.py:324-325).
"""

import numpy as np
import pytest

import goldens

pytestmark = pytest.mark.gpu

bb = pytest.importorskip("paper_2605_29233_b200")

_M = {}


def default_params():
    if "default" not in _M:
        _M["default"] = bb.build_model(0, bb.Vocab(), dtype="f32")
    return _M["default"]


def c1_params():
    if "c1" not in _M:
        vocab = bb.Vocab(size=4096)
        dims = bb.ModelDims(layers=4, d_model=256, max_len=192)
        _M["c1"] = bb.build_model(0, vocab, dims, head_scale=2.0, dtype="f32")
    return _M["c1"]


def _branches(vocab, rows, sizes):
    P, L = rows[0].prompt_len, len(rows[0])
    out = []
    for i, b in enumerate(sizes):
        st = bb.BranchState(index=i, block_size=b, window=bb.BlockWindow(P, min(P + b, L)),
                            prob_map=np.zeros((L, vocab.n_out)), prob_covered=np.zeros(L, dtype=bool))
        out.append(st)
    return out


def _lse(logits):
    m = logits.max(1)
    return m + np.log(np.exp(logits - m[:, None]).sum(1))


def test_full_forward_matches_reference_numerics():
    """full_forward (model.py:322-328) vs the reference's own float64 output on C1."""
    F = np.load(goldens.GOLDEN + "/forward_c1.npz")
    params = c1_params()
    task = bb.make_task(0, 64, 128, params.vocab)
    out, cache = bb.full_forward(params, task.fresh_row(params.vocab), task.target)
    assert np.array_equal(out.positions, F["full_positions"])
    assert np.array_equal(out.probs.argmax(1), F["full_argmax"])
    np.testing.assert_allclose(out.probs.max(1), F["full_conf"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(_lse(out.logits), F["full_lse"], rtol=1e-5, atol=1e-4)
    np.testing.assert_allclose(out.logits[:4], F["full_logits_rows"], rtol=1e-5, atol=1e-4)
    assert cache.valid.all() and cache.keys.shape == (4, 192, 256)


def test_block_forward_matches_reference_numerics():
    """block_forward (model.py:331-343) over the prefill cache vs the reference."""
    F = np.load(goldens.GOLDEN + "/forward_c1.npz")
    params = c1_params()
    task = bb.make_task(0, 64, 128, params.vocab)
    _, cache = bb.full_forward(params, task.fresh_row(params.vocab), task.target)
    row2 = bb.SequenceRow(F["block_tokens"].astype(np.int64), 64)
    out, new = bb.block_forward(params, row2, cache, bb.BlockWindow(64, 96), task.target)
    assert np.array_equal(out.positions, F["block_positions"])
    assert np.array_equal(out.probs.argmax(1), F["block_argmax"])
    np.testing.assert_allclose(out.probs.max(1), F["block_conf"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(_lse(out.logits), F["block_lse"], rtol=1e-5, atol=1e-4)
    np.testing.assert_allclose(out.logits[:4], F["block_logits_rows"], rtol=1e-5, atol=1e-4)
    # copy-then-write: the input cache is unchanged, outside the window the new one equals it
    k0, k1 = cache.keys, new.keys
    assert np.array_equal(k0[:, :64], k1[:, :64]) and np.array_equal(k0[:, 96:], k1[:, 96:])
    assert not np.array_equal(k0[:, 64:96], k1[:, 64:96])


def test_full_forward_queries_masked_positions_only():
    """test_model.py:55-60"""
    params = default_params()
    task = bb.make_task(1, 16, 64, params.vocab)
    row = task.fresh_row(params.vocab)
    row.tokens[20:30] = 3
    out, _ = bb.full_forward(params, row, task.target)
    np.testing.assert_array_equal(out.positions, np.flatnonzero(row.tokens == params.vocab.mask_id))


def test_block_forward_full_window_matches_full_forward():
    """test_model.py:63-74: a block covering the whole row is bitwise a full forward."""
    params = default_params()
    task = bb.make_task(1, 16, 64, params.vocab)
    row = task.fresh_row(params.vocab)
    full_out, full_cache = bb.full_forward(params, row, task.target)
    empty = bb.KvCache.empty(params.dims.layers, len(row), params.dims.d_model)
    empty.valid[:] = True
    blk_out, blk_cache = bb.block_forward(params, row, empty, bb.BlockWindow(0, len(row)), task.target)
    assert np.array_equal(full_out.logits, blk_out.logits)
    assert np.array_equal(full_out.probs, blk_out.probs)
    assert np.array_equal(full_cache.keys, blk_cache.keys)
    assert np.array_equal(full_cache.values, blk_cache.values)


def test_block_forward_errors():
    """test_model.py:77-89: window bounds -> ContractError; invalid cache outside -> StateError."""
    params = default_params()
    task = bb.make_task(1, 16, 64, params.vocab)
    row = task.fresh_row(params.vocab)
    _, cache = bb.full_forward(params, row, task.target)
    with pytest.raises(bb.ContractError):
        bb.block_forward(params, row, cache, bb.BlockWindow(0, len(row) + 1), task.target)
    empty = bb.KvCache.empty(params.dims.layers, len(row), params.dims.d_model)
    with pytest.raises(bb.StateError):
        bb.block_forward(params, row, empty, bb.BlockWindow(16, 20), task.target)
    with pytest.raises(bb.StateError):
        bb.kv_vectorize(empty)


def test_batched_forward_equals_sequential():
    """test_scheduler.py:72-91: one fused device pass over every branch's window
    is bitwise the per-branch block_forward (logits, probs, keys, values)."""
    params = default_params()
    vocab = params.vocab
    task = bb.make_task(1, 16, 64, vocab)
    rows = [task.fresh_row(vocab) for _ in range(3)]
    branches = _branches(vocab, rows, (4, 8, 16))
    out0, caches = bb.init_full_forward(params, rows, task.target)
    packed = bb.pack_active_blocks(rows, branches, [0, 1, 2], vocab.mask_id)
    assert packed.offsets == (0, 4, 12, 28)
    ref_out, ref_cache = {}, {}
    for k in range(3):
        ref_out[k], ref_cache[k] = bb.block_forward(params, rows[k], caches[k].copy(), branches[k].window,
                                                    task.target)
    got = bb.batched_block_forward(params, packed, rows, caches, branches, task.target)
    for k in range(3):
        assert np.array_equal(got[k].logits, ref_out[k].logits)
        assert np.array_equal(got[k].probs, ref_out[k].probs)
        assert np.array_equal(caches[k].keys, ref_cache[k].keys)
        assert np.array_equal(caches[k].values, ref_cache[k].values)
    with pytest.raises(bb.ContractError):
        bb.init_full_forward(params, [rows[0], bb.SequenceRow(np.roll(rows[1].tokens, 1), 16)], task.target)


def test_observer_replay_is_bitwise():
    """Criterion 05 (test_acceptance.py:183-204): every batched block step of
    run_blockbatch, replayed branch by branch through block_forward on the
    observer's pre-step rows / caches / windows, is bitwise the fused step's
    output and post-step cache -- and observing does not change the run."""
    params = default_params()
    steps = [0]
    for seed in range(5):
        task = bb.make_task(seed, 16, 64, params.vocab)

        def observer(kind, active, pre_rows, pre_caches, windows, outputs, post_caches, _task=task):
            assert kind == "block"
            for idx, k in enumerate(active):
                out, cache = bb.block_forward(params, pre_rows[idx], pre_caches[idx], windows[idx], _task.target)
                assert np.array_equal(out.logits, outputs[k].logits)
                assert np.array_equal(out.probs, outputs[k].probs)
                assert np.array_equal(cache.keys, post_caches[idx].keys)
                assert np.array_equal(cache.values, post_caches[idx].values)
                steps[0] += 1

        cfg = bb.SchedulerConfig(gen_len=64)
        got = bb.run_blockbatch(params, task, cfg, forward_observer=observer)
        plain = bb.run_blockbatch(params, task, cfg)
        assert np.array_equal(got.row.tokens, plain.row.tokens)
        assert [e.to_record() for e in got.trace] == [e.to_record() for e in plain.trace]
    assert steps[0] > 60, steps[0]


def test_forward_hook_live_and_hard_cap_match_reference():
    """The hook fires once per charge as the forward happens, in the
    reference's order; with the cap lowered to 16 forwards the run raises
    RunawayError after exactly the reference's hook calls (scheduler.py:310,
    324-325; reference runs with HARD_CAP_FACTOR = 0)."""
    g = goldens.load("runs_runaway.json")
    params = default_params()
    cfg = bb.SchedulerConfig(block_sizes=tuple(g["block_sizes"]), gen_len=g["gen_len"])
    raised = 0
    for want in g["runs"]:
        task = bb.make_task(want["seed"], g["prompt_len"], g["gen_len"], params.vocab)
        calls = []
        if want["raised"]:
            with pytest.raises(bb.RunawayError):
                bb.run_blockbatch(params, task, cfg, forward_hook=calls.append, _hard_cap=g["hard_cap"])
            raised += 1
        else:
            r = bb.run_blockbatch(params, task, cfg, forward_hook=calls.append, _hard_cap=g["hard_cap"])
            assert list(r.nfe.snapshot()) == want["nfe"]
        assert calls == want["calls"], want["seed"]
    assert raised >= 2


def test_forward_hook_abort_stops_the_run():
    """An exception from the hook propagates mid-run (it fires live, not replayed)."""
    params = default_params()
    task = bb.make_task(3, 16, 64, params.vocab)

    class Stop(Exception):
        pass
    calls = []

    def hook(kind):
        calls.append(kind)
        if len(calls) == 3:
            raise Stop
    with pytest.raises(Stop):
        bb.run_blockbatch(params, task, bb.SchedulerConfig(gen_len=64), forward_hook=hook)
    assert calls == ["init", "block", "block"]


def test_forward_hook_counts_with_refresh():
    """test_scheduler.py:207-219."""
    params = default_params()
    task = bb.make_task(4, 16, 64, params.vocab)
    calls = []
    r = bb.run_blockbatch(params, task, bb.SchedulerConfig(gen_len=64, refresh_interval=8), forward_hook=calls.append)
    assert len(calls) == r.nfe.total
    assert calls.count("init") == r.nfe.nfe_init == 1
    assert calls.count("block") == r.nfe.nfe_block
    assert calls.count("refresh") == r.nfe.nfe_refresh
    for ev in r.trace:
        assert sum(ev.nfe) <= r.nfe.total


def test_trace_roundtrip(tmp_path):
    """test_scheduler.py:245-260 on a device run with log_kv="norms"."""
    params = default_params()
    task = bb.make_task(2, 16, 64, params.vocab)
    r = bb.run_blockbatch(params, task, bb.SchedulerConfig(gen_len=64, log_kv="norms"))
    path = tmp_path / "trace.jsonl"
    bb.write_trace(path, r.trace)
    records = bb.read_trace(path)
    assert len(records) == len(r.trace)
    assert records[0]["kind"] == "init" and records[-1]["kind"] == "finish"
    assert records == [bb.scheduler._jsonify(e.to_record()) for e in r.trace]
    with open(path) as fh:
        assert "schema" in fh.readline()
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"schema": "other"}\n')
    with pytest.raises(bb.ContractError):
        bb.read_trace(bad)


def test_log_kv_full_is_the_vectorized_cache():
    """log_kv="full" (scheduler.py:279-280): decisions identical to the plain
    run; the init event's per-branch vector is kv_vectorize of the prefill
    cache (= full_forward of the fresh row, bitwise) and its norm is the
    init kv_delta of log_kv="norms"."""
    params = default_params()
    task = bb.make_task(5, 16, 32, params.vocab)
    base = bb.SchedulerConfig(gen_len=32)
    full = bb.run_blockbatch(params, task, bb.SchedulerConfig(gen_len=32, log_kv="full"))
    norms = bb.run_blockbatch(params, task, bb.SchedulerConfig(gen_len=32, log_kv="norms"))
    plain = bb.run_blockbatch(params, task, base)
    assert np.array_equal(full.row.tokens, plain.row.tokens) and full.nfe.snapshot() == plain.nfe.snapshot()
    _, cache = bb.full_forward(params, task.fresh_row(params.vocab), task.target)
    want = bb.kv_vectorize(cache)
    init = full.trace[0]
    assert init.kind == "init"
    n_blocks = 0
    for k, vec in init.extra["kv"].items():
        v = np.asarray(vec)
        assert np.array_equal(v, want)
        assert np.isclose(np.linalg.norm(v), norms.trace[0].extra["kv_delta"][k], rtol=1e-6)
    for ev in full.trace:
        if ev.kind == "block_forward":
            n_blocks += 1
            assert set(ev.extra["kv"]) == set(ev.extra["kv_delta"]) == {str(k) for k in ev.extra["active"]}
            for vec in ev.extra["kv"].values():
                assert len(vec) == want.size
    assert n_blocks == full.nfe.nfe_block


def test_model_memory_is_released():
    """ModelParams owns its device sessions: dropping the model frees them."""
    import gc

    import torch
    gc.collect()
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    p = bb.build_model(1, bb.Vocab(), dtype="f32")
    task = bb.make_task(0, 16, 64, p.vocab)
    bb.run_blockbatch(p, task, bb.SchedulerConfig(gen_len=64))
    bb.full_forward(p, task.fresh_row(p.vocab), task.target)
    assert torch.cuda.memory_allocated() > before
    del p
    gc.collect()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() <= before


def test_batched_compaction_matches_static_layout():
    """Batched bf16x2 sessions compact the block pass to the live requests
    (finished requests cost no GEMM rows): the decisions equal those of the
    same batch with the static per-request layout (test flag 8) and of the
    requests run alone, on a 4-request batch whose requests finish at
    different iterations."""
    from paper_2605_29233_b200.engine import Session
    from paper_2605_29233_b200.scheduler import _cfg_key
    dims = bb.ModelDims(layers=2, d_model=256, max_len=192, arch="llada", n_heads=2, n_kv_heads=2, head_dim=128,
                        d_ff=512, rope_theta=500000.0)
    vocab = bb.Vocab(size=1000)
    cfg = bb.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=64)
    tasks = [bb.make_task(s, 32, 64, vocab) for s in range(4)]

    def run(flags):
        p = bb.build_model(0, vocab, dims, head_scale=0.25, dtype="bf16x2")
        if flags:
            p._sessions[_cfg_key(cfg, 32, len(tasks), True)] = Session(p, cfg, 32, len(tasks), test_flags=flags)
        return [(r.nfe.snapshot(), r.row.tokens.tolist()) for r in bb.run_batch(p, tasks, cfg)]
    compact, static = run(0), run(8)
    single = []
    p1 = bb.build_model(0, vocab, dims, head_scale=0.25, dtype="bf16x2")
    for t in tasks:
        r = bb.run_blockbatch(p1, t, cfg)
        single.append((r.nfe.snapshot(), r.row.tokens.tolist()))
    nfes = [c[0] for c in compact]
    assert len(set(n[1] for n in nfes)) > 1, "requests should finish at different iterations"
    same_static = sum(a == b for a, b in zip(compact, static))
    same_single = sum(a == b for a, b in zip(compact, single))
    print(f"compacted vs static: {same_static}/4, vs single requests: {same_single}/4, static vs single "
          f"{sum(a == b for a, b in zip(static, single))}/4; nfe {nfes} / {[x[0] for x in static]} / "
          f"{[x[0] for x in single]}")
    assert same_static >= 3 and same_single >= 3


def _refresh_model(dtype, max_len=192):
    dims = bb.ModelDims(layers=2, d_model=256, max_len=max_len, arch="llada", n_heads=2, n_kv_heads=2, head_dim=128,
                        d_ff=512, rope_theta=500000.0)
    return bb.build_model(0, bb.Vocab(size=1000), dims, head_scale=0.25, dtype=dtype)


@pytest.mark.parametrize("dtype,P,G,bsz", [("bf16", 32, 64, (8, 16, 32)), ("bf16x2", 32, 64, (8, 16, 32)),
                                           ("bf16", 1024, 64, (8, 16, 32, 64)),
                                           ("bf16x2", 1024, 64, (8, 16, 32, 64))])
def test_stacked_refresh_kv_matches_per_branch_passes(dtype, P, G, bsz):
    """The stacked refresh (every refreshing branch in one B x L full pass,
    own key list per (request, branch)) writes the same caches as one full
    pass per branch (test flag 2048; the reference's loop, scheduler.py:379-383):
    after prefill + one block step + refresh, every branch's kv_vectorize of
    both requests of a 2-request session agrees (the GEMM row chunking differs,
    so within bf16 rounding, not bitwise), and the page tables are identical.
    L = 1088 runs the full passes on the 128-row attention (C5's kernel) over
    4 branches' row groups."""
    import torch
    from paper_2605_29233_b200.engine import Session
    p = _refresh_model(dtype, max_len=max(192, P + G))
    vocab = p.vocab
    nb = len(bsz)
    cfg = bb.SchedulerConfig(block_sizes=bsz, gen_len=G, refresh_interval=1)
    tasks = [bb.make_task(s, P, G, vocab) for s in (3, 4)]
    prompts = np.stack([t.prompt for t in tasks])
    targets = np.stack([t.target for t in tasks])
    out = {}
    for flags in (0, 2048):
        s = Session(p, cfg, P, 2, test_flags=flags)
        s.set_inputs(prompts, targets)
        s.prefill()
        s.iteration(True, use_graph=False)
        ctrl = s.ctrl_now()
        assert (ctrl[:, 18] == 1).all(), ctrl[:, 18]  # C_REFRESHES: one refresh charged per request
        out[flags] = ([[s.kv_vec(r, k).cpu().numpy() for k in range(nb)] for r in range(2)],
                      s.v_pages.cpu().numpy().copy() if hasattr(s, "v_pages") else None, ctrl.copy())
        del s
        torch.cuda.synchronize()
    (kv_a, pt_a, c_a), (kv_b, pt_b, c_b) = out[0], out[2048]
    if pt_a is not None:
        assert np.array_equal(pt_a, pt_b)
    worst = 0.0
    for r in range(2):
        for k in range(nb):
            a, b = kv_a[r][k], kv_b[r][k]
            assert np.isfinite(a).all()
            worst = max(worst, float(np.abs(a - b).max() / (np.abs(b).max() + 1e-30)))
    tol = 2e-2 if dtype == "bf16" else 1e-4
    print(f"{dtype} L={P + G}: stacked vs per-branch refresh KV max rel diff {worst:.2e}")
    assert worst <= tol


def test_stacked_refresh_whole_runs_match_per_branch_passes():
    """Whole bf16x2 runs with a refresh every 4 iterations: stacked refresh vs
    one full pass per branch (test flag 2048) give the same NFE and tokens."""
    from paper_2605_29233_b200.engine import Session
    from paper_2605_29233_b200.scheduler import _cfg_key
    cfg = bb.SchedulerConfig(block_sizes=(8, 16, 32), gen_len=64, refresh_interval=4)
    tasks = [bb.make_task(s, 32, 64, bb.Vocab(size=1000)) for s in range(6)]

    def run(flags):
        p = _refresh_model("bf16x2")
        p._sessions[_cfg_key(cfg, 32, 1, True)] = Session(p, cfg, 32, 1, test_flags=flags)
        res = [bb.run_blockbatch(p, t, cfg) for t in tasks]
        return [(r.nfe.snapshot(), r.row.tokens.tolist()) for r in res]
    a, b = run(0), run(2048)
    assert all(x[0][2] > 0 for x in a), "every run should refresh"
    same = sum(x == y for x, y in zip(a, b))
    print(f"stacked vs per-branch refresh: {same}/6 identical runs; nfe {[x[0] for x in a]} / {[x[0] for x in b]}")
    assert same >= 5
