#!/usr/bin/env python
"""BlockBatch batched denoising step on B200 — benchmark (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c5|c1] [--impl ours|reference]

Metric (BASELINE.json): decoded tokens/s on the LLaDA-8B-shape random-init
bf16 model, 3 block-size branches {8,16,32}, gen 256, one prompt per GPU
(config[1] = "c2"); NFE/request reported beside it.

A *step* is one whole request through the hot path: prefill + batched block
denoising iterations (+ periodic refresh) until the request finishes — i.e.
one run_blockbatch of a fresh synthetic prompt.  K timed steps use K
distinct prompts per GPU (weak scaling over ranks: prompts are sharded,
no per-step collective; one NCCL all-gather of results at the end).

value : decoded tokens (winner's tokens_decoded) of all ranks / max-rank
        device time, inputs already resident in HBM (CUDA events on the
        session stream).
e2e   : same metric through the public API (run_blockbatch with host
        numpy prompt/target: pinned H2D, the run, D2H of results), CUDA
        events on the session stream around K calls.
roofline : the tcgen05 weight-streaming GEMM (QKV/O/gate-up/down of the
        block step), per-launch durations measured live inside the timed
        region (%globaltimer accounting in the kernel), algorithmic bytes =
        weights + activations per launch; peak = MEASURED_PEAKS.json hbm_gbs.
cpu_baseline : the oracle port (oracle/bb_oracle.py, NumPy fp32) on a
        bounded sample of the same workload, extrapolated per request.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

CONFIGS = {
    "c2": dict(workload="LLaDA-8B-shape random-init bf16, 1 prompt per GPU, branches {8,16,32}, gen 256",
               shape="llada", P=64, G=256, bs=(8, 16, 32), R=32, head_scale=0.4, gamma=8.0),
    "c3": dict(workload="Dream-7B-shape random-init bf16, branches {4,16,32}, gen 512, refresh every 2 blocks",
               shape="dream", P=64, G=512, bs=(4, 16, 32), R=2, head_scale=0.4, gamma=8.0),
    "c5": dict(workload="LLaDA-8B-shape long context: 2048-token prompt, branches {8,16,32,64}, gen 1024",
               shape="llada", P=2048, G=1024, bs=(8, 16, 32, 64), R=32, head_scale=0.4, gamma=8.0),
    "c4": dict(workload="LLaDA-8B-shape random-init, 256 synthetic prompts sharded request-parallel over the GPUs, "
                        "8 requests batched per device step, branches {8,16,32}, gen 256",
               shape="llada", P=64, G=256, bs=(8, 16, 32), R=32, head_scale=0.4, gamma=8.0, n_prompts=256, batch=8),
    "c1": dict(workload="reference synthetic model 4L d256 V4096, P64, branches {8,16,32}, gen 128 (bf16)",
               shape="ref", P=64, G=128, bs=(8, 16, 32), R=32, head_scale=2.0, gamma=8.0),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for i, n in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------- model / workload
def make_model(cfgd, dtype="bf16"):
    import paper_2605_29233_b200 as bb
    if cfgd["shape"] == "llada":
        vocab, dims = bb.Vocab(size=bb.LLADA_8B_VOCAB), bb.LLADA_8B
    elif cfgd["shape"] == "dream":
        vocab, dims = bb.Vocab(size=bb.DREAM_7B_VOCAB), bb.DREAM_7B
    else:
        vocab, dims = bb.Vocab(size=4096), bb.ModelDims(layers=4, d_model=256, max_len=192)
    needed = cfgd["P"] + cfgd["G"]
    if dims.max_len < needed:
        import dataclasses
        dims = dataclasses.replace(dims, max_len=needed)
    params = bb.build_model(0, vocab, dims, head_scale=cfgd["head_scale"], gamma=cfgd["gamma"], dtype=dtype)
    cfg = bb.SchedulerConfig(block_sizes=cfgd["bs"], gen_len=cfgd["G"], refresh_interval=cfgd["R"])
    return bb, params, cfg


def step_bytes_flops(params, cfgd, rows_block, kv_positions):
    """Algorithmic HBM bytes / FLOPs of one block step."""
    d = params.dims
    e = 2
    layer_w = (d.qkv_out * d.d_model + d.d_model * d.n_heads * d.hd + 2 * d.d_ff * d.d_model
               + d.d_model * d.d_ff)
    head_w = params.vocab.n_out * d.d_model
    kv = 2 * d.layers * kv_positions * d.n_kv_heads * d.hd * e
    byts = e * (d.layers * layer_w + head_w) + kv
    flops = 2 * rows_block * (d.layers * layer_w + head_w)
    return byts, flops, layer_w * e


def nfe_weighted_roofline(params, cfgd, rows_block, nfe_split, hbm_gbs, tflops, ms_per_nfe):
    """Roofline time per NFE weighted by NFE kind: a block step
    streams the weights once for its window rows; the prefill is one full pass
    of L rows (+ the LM head over the window rows); a refresh recomputes every
    non-done branch over all L rows (charged as one NFE; the minimum streams the
    weights once for B*L rows).  t = max(bytes / HBM, FLOPs / dense bf16 peak)."""
    d = params.dims
    e = 2
    L = cfgd["P"] + cfgd["G"]
    B = len(cfgd["bs"])
    layer_w = (d.qkv_out * d.d_model + d.d_model * d.n_heads * d.hd + 2 * d.d_ff * d.d_model
               + d.d_model * d.d_ff)
    head_w = params.vocab.n_out * d.d_model
    kv_pos = 2 * d.layers * d.n_kv_heads * d.hd * e  # bytes of K+V per position

    def t(byts, flops):
        return max(byts / (hbm_gbs * 1e6), flops / (tflops * 1e9))

    w = e * (d.layers * layer_w + head_w)
    t_block = t(w + kv_pos * L * B, 2 * rows_block * (d.layers * layer_w + head_w) + 4 * rows_block * L * d.n_heads * d.hd * d.layers)
    t_init = t(w + kv_pos * L, 2 * L * d.layers * layer_w + 2 * rows_block * head_w + 4 * L * L * d.n_heads * d.hd * d.layers)
    t_ref = t(w + kv_pos * L * B, 2 * B * L * d.layers * layer_w + 2 * rows_block * head_w
              + 4 * B * L * L * d.n_heads * d.hd * d.layers)
    n = [float(x) for x in nfe_split]
    t_avg = (n[0] * t_init + n[1] * t_block + n[2] * t_ref) / max(sum(n), 1e-9)
    return {"t_roof_ms": {"init": t_init, "block": t_block, "refresh": t_ref}, "nfe_split": n,
            "t_roof_per_nfe_ms": t_avg, "ms_per_nfe": ms_per_nfe, "frac": t_avg / ms_per_nfe,
            "peaks": {"hbm_gbs": hbm_gbs, "bf16_tflops": tflops}}


# ---------------------------------------------------------------- CPU baseline (oracle port)
def nfe_split_for(config):
    """The committed per-request NFE split + tokens/request (profiles/nfe_split.json)."""
    d = json.load(open(os.path.join(HERE, "profiles", "nfe_split.json")))[config]
    return tuple(d["nfe_split"]), float(d["tokens_per_request"]), d["source"]


class CpuSampler:
    """The oracle (oracle/bb_oracle.py, NumPy fp32, all host threads) on the
    bench workload at FULL depth and width.  Weights of two distinct layers
    are generated (counter hash, as on the device) and the model's layers
    cycle through them: a forward's cost does not depend on the values, and
    every layer still streams its ~0.9 GB of fp32 weights from DRAM (far
    larger than any host cache).  One sample = one full forward of the shared
    row (L rows: prefill / refresh) + one block step (every branch's window
    against the prefill cache); a request = the committed NFE split of those
    (a refresh is one full forward per non-done branch, as in
    scheduler.py:379-383)."""

    def __init__(self, cfgd, config):
        from oracle import bb_oracle as O
        import paper_2605_29233_b200.model as M
        self.O, self.cfgd = O, cfgd
        self.split, self.tok, self.src = nfe_split_for(config)
        dims = M.LLADA_8B if cfgd["shape"] == "llada" else M.DREAM_7B
        V = M.LLADA_8B_VOCAB if cfgd["shape"] == "llada" else M.DREAM_7B_VOCAB
        self.P, self.G = cfgd["P"], cfgd["G"]
        L = self.P + self.G
        mk = dict(kind="llada", vocab_size=V, d_model=dims.d_model, n_heads=dims.n_heads,
                  n_kv_heads=dims.n_kv_heads, head_dim=dims.hd, d_ff=dims.d_ff, max_len=L,
                  rope_theta=dims.rope_theta, norm_eps=dims.norm_eps, qkv_bias=dims.qkv_bias,
                  head_scale=cfgd["head_scale"], gamma=cfgd["gamma"])
        t = time.perf_counter()
        W2 = O.hash_weights(O.OArch(layers=2, **mk), 0)
        per_layer = ("wqkv", "wo", "wg", "wu", "wd", "ln1", "ln2", "bqkv")
        self.W = {k: ([v[l % 2] for l in range(dims.layers)] if k in per_layer else v) for k, v in W2.items()}
        self.t_gen = time.perf_counter() - t
        self.arch = O.OArch(layers=dims.layers, **mk)
        task = O.make_task(0, self.P, self.G, V)
        self.target = task.target
        self.row = np.full(L, V + 1, dtype=np.int64)
        self.row[:self.P] = task.prompt
        self.layers = dims.layers

    def sample(self):
        O, P, L = self.O, self.P, self.P + self.G
        t = time.perf_counter()
        _, cache = O.full_forward(self.arch, self.W, self.row, P, self.target, cdtype=np.float32)
        t_full = time.perf_counter() - t
        t = time.perf_counter()
        for b in self.cfgd["bs"]:
            O.block_forward(self.arch, self.W, self.row, P, cache, P, min(P + b, L), self.target, cdtype=np.float32)
        t_block = time.perf_counter() - t
        n0, n1, n2 = self.split
        t_req = n0 * t_full + n1 * t_block + n2 * len(self.cfgd["bs"]) * t_full
        return self.tok / t_req, t_full, t_block

    def describe(self, t_full, t_block, n):
        return (f"oracle NumPy fp32 at full depth ({self.layers} layers) and width, {n} sample(s): "
                f"full forward L={self.P + self.G} {t_full:.2f}s, block step over all {len(self.cfgd['bs'])} "
                f"branch windows {t_block:.2f}s (medians); request = committed NFE split "
                f"{tuple(round(x, 2) for x in self.split)} x those, {self.tok:.0f} tokens/request "
                f"({self.src}); weights generated in {self.t_gen:.1f}s, not timed")


def cpu_baseline(cfgd, config, samples=1):
    from oracle import bb_oracle as O
    if cfgd["shape"] == "ref":
        arch = O.ref_arch(vocab_size=4096, layers=4, d_model=256, max_len=192, head_scale=2.0)
        W = O.philox_ref_weights(arch, 0)
        task = O.make_task(0, cfgd["P"], cfgd["G"], arch.vocab_size)
        t0 = time.perf_counter()
        r = O.run_blockbatch(arch, W, task, O.OConfig(block_sizes=cfgd["bs"], gen_len=cfgd["G"],
                                                          refresh_interval=cfgd["R"]))
        dt = time.perf_counter() - t0
        return {"value": r.tokens_decoded / dt, "unit": "decoded tokens/s", "cores": os.cpu_count(),
                "kind": "port", "sample": f"one full run_blockbatch (seed 0) through the oracle, {dt:.1f}s"}
    cs = CpuSampler(cfgd, config)
    res = [cs.sample() for _ in range(samples)]
    v = statistics.median(r[0] for r in res)
    return {"value": v, "unit": "decoded tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": cs.describe(statistics.median(r[1] for r in res), statistics.median(r[2] for r in res),
                                  samples)}


# ---------------------------------------------------------------- C4: request-parallel, batched
def _session(params, cfg, P, R, args):
    """The device session of the timed runs; --test-flags (A/B measurements
    only, e.g. 2048 = per-branch refresh passes) builds it with those flags."""
    from paper_2605_29233_b200.scheduler import get_session, _cfg_key
    if args.test_flags:
        from paper_2605_29233_b200.engine import Session
        s = Session(params, cfg, P, R, trace=False, test_flags=args.test_flags)
        params._sessions[_cfg_key(cfg, P, R, False)] = s
        return s
    return get_session(params, cfg, P, R, trace=False)


def bench_c4(args, cfgd, bb, params, cfg, rank, world, dist, local):
    """BASELINE config C4: n_prompts prompts sharded round-robin over the ranks
    (dp.shard; no per-step collective), each rank running its share in device
    sessions of `batch` requests (every live request's branch windows stacked
    into one forward per iteration, scheduler.run_batch).  A step = one batch;
    all of a rank's batches are timed.  value = decoded tokens of all ranks /
    max-rank time; one all-gather of the results at the end."""
    import torch
    from paper_2605_29233_b200 import dp, _lib
    from paper_2605_29233_b200.scheduler import get_session
    P, G, Rb = cfgd["P"], cfgd["G"], cfgd["batch"]
    mine = dp.shard(cfgd["n_prompts"], rank, world)
    nbat = (len(mine) + Rb - 1) // Rb
    Wm = max(args.warmup, 1)
    s = _session(params, cfg, P, Rb, args)
    warm = [bb.make_task(900000 + rank * 1000 + i, P, G, params.vocab) for i in range(Rb)]
    batches = [[bb.make_task(1000 + g, P, G, params.vocab) for g in mine[b * Rb:(b + 1) * Rb]] for b in range(nbat)]
    while batches and len(batches[-1]) < Rb:  # pad the last batch with repeats (counted once)
        batches[-1].append(batches[-1][-1])
    n_real = [min(Rb, len(mine) - b * Rb) for b in range(nbat)]

    def dev(ts):
        return (torch.tensor(np.stack([t.prompt for t in ts]).astype(np.int32), device="cuda"),
                torch.tensor(np.stack([t.target for t in ts]).astype(np.int32), device="cuda"))
    wp, wt = dev(warm)
    inputs = [dev(b) for b in batches]
    for _ in range(Wm):
        s.set_inputs(wp, wt)
        s.launch()
    s.stream.synchronize()
    launches0 = s.counters()["kernel_launches"]
    snaps = [(torch.zeros(Rb, 32, dtype=torch.int32, device="cuda"),
              torch.zeros(Rb, len(cfgd["bs"]), 8, dtype=torch.int32, device="cuda")) for _ in range(nbat)]
    its = []
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(s.stream)
        for b in range(nbat):
            s.set_inputs(*inputs[b])
            its.append(s.launch())
            s.snapshot(*snaps[b])
        ev1.record(s.stream)
        ev1.synchronize()
    t_ms = ev0.elapsed_time(ev1)
    launches = s.counters()["kernel_launches"] - launches0
    tok = 0.0
    nfe = []
    dyn = {"merges": 0.0, "syncs": 0.0, "commits": 0.0}
    for b in range(nbat):
        c, br = snaps[b][0].cpu().numpy(), snaps[b][1].cpu().numpy()
        if not (c[:n_real[b], _lib.C_STATUS] == 1).all():
            raise RuntimeError("requests did not finish")
        for r in range(n_real[b]):
            tok += float(br[r, c[r, _lib.C_WINNER], _lib.B_DEC])
            nfe.append(c[r, _lib.C_NFE0:_lib.C_NFE2 + 1].astype(np.int64))
            for k, w in (("merges", _lib.C_MERGES), ("syncs", _lib.C_SYNCS), ("commits", _lib.C_COMMITS)):
                dyn[k] += float(c[r, w])
    # e2e: the same prompts through run_batch with host inputs (pinned H2D, D2H of the results)
    h2d0, d2h0 = s.h2d_bytes, s.d2h_bytes
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s.stream)
    e2e_tok = 0.0
    for b in range(nbat):
        rs = bb.run_batch(params, batches[b], cfg, trace=False)
        e2e_tok += sum(r.tokens_decoded for r in rs[:n_real[b]])
    e1.record(s.stream)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    loc = torch.tensor([tok, t_ms, e2e_tok, e2e_ms, float(len(nfe)), float(sum(x.sum() for x in nfe))],
                       dtype=torch.float64, device="cuda")
    if dist is not None:
        allv = [torch.zeros_like(loc) for _ in range(world)]
        dist.all_gather(allv, loc)
        allv = torch.stack(allv).cpu().numpy()
    else:
        allv = loc.cpu().numpy()[None]
    if rank == 0:
        t_max = allv[:, 1].max()
        n_req = allv[:, 4].sum()
        line = {"metric": "decoded tokens/s", "value": allv[:, 0].sum() / (t_max / 1e3), "unit": "decoded tokens/s",
                "n_gpus": world, "steps": nbat, "warmup": Wm, "ms_per_step": t_max / max(nbat, 1),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": args.precision,
                "data": "synthetic (random-init weights, make_task prompts)",
                "config": {"workload": cfgd["workload"], "branches": list(cfgd["bs"]), "prompt_len": P, "gen_len": G,
                           "prompts": cfgd["n_prompts"], "requests_per_session": Rb,
                           "parallelism": f"request-parallel dp{world}",
                           "l2": "inputs larger than L2 (16 GB of weights streamed per batched step)"},
                "requests": int(n_req), "nfe_per_request": allv[:, 5].sum() / max(n_req, 1),
                "ms_per_batched_iteration": float(t_ms / max(sum(its), 1)),
                "dynamics_per_request": {k: v / max(len(nfe), 1) for k, v in dyn.items()},
                "e2e": {"value": allv[:, 2].sum() / (allv[:, 3].max() / 1e3), "unit": "decoded tokens/s",
                        "h2d_bytes_per_step": (s.h2d_bytes - h2d0) / max(nbat, 1),
                        "d2h_bytes_per_step": (s.d2h_bytes - d2h0) / max(nbat, 1)},
                "roofline": None, "cpu_baseline": None, "clocks": clk.summary(),
                "gpu_launches": int(launches)}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ---------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--precision", default="bf16x2", choices=["bf16", "bf16x2"],
                    help="bf16x2 (default, the numerics that meet the north-star logit tolerance): bf16 weights "
                         "with hi+lo bf16 activations / KV; bf16: bf16 activations / KV")
    ap.add_argument("--batch", type=int, default=None,
                    help="c4: requests per device session (default 8: the best of 1-32 measured, "
                         "profiles/r02/c4_batch/)")
    ap.add_argument("--prompts", type=int, default=None, help="c4: total prompts (default 256)")
    ap.add_argument("--test-flags", type=int, default=0,
                    help="A/B only: session test flags of the timed runs (bb_session_desc.test_flags)")
    ap.add_argument("--no-variant", action="store_true",
                    help="skip the same-run device measurement of the other numerics mode")
    args = ap.parse_args()
    cfgd = dict(CONFIGS[args.config])
    if args.config == "c4":
        if args.batch:
            cfgd["batch"] = args.batch
        if args.prompts:
            cfgd["n_prompts"] = args.prompts
        cfgd["workload"] = (f"LLaDA-8B-shape random-init, {cfgd['n_prompts']} synthetic prompts sharded request-parallel "
                            f"over the GPUs, {cfgd['batch']} requests batched per device step, branches {{8,16,32}}, gen 256")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    metric = "decoded tokens/s"

    if args.impl == "reference":
        if rank != 0:
            return
        # reference arm: the oracle port of the reference's CPU path on the host
        # cores, full depth; W untimed samples, then K timed samples (median)
        if cfgd["shape"] == "ref":
            cb = cpu_baseline(cfgd, args.config)
        else:
            cs = CpuSampler(cfgd, args.config)
            for _ in range(args.warmup):
                cs.sample()
            res = [cs.sample() for _ in range(args.steps)]
            vals = [r[0] for r in res]
            cb = {"value": statistics.median(vals), "unit": "decoded tokens/s", "cores": os.cpu_count(),
                  "kind": "port", "samples": [round(x, 4) for x in vals],
                  "sample": cs.describe(statistics.median(r[1] for r in res), statistics.median(r[2] for r in res),
                                        len(res))}
        line = {"impl": "reference", "metric": metric, "value": cb["value"], "unit": cb["unit"],
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": {"workload": cfgd["workload"], "branches": list(cfgd["bs"]), "prompt_len": cfgd["P"],
                           "gen_len": cfgd["G"]},
                "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": cb["unit"], "h2d_bytes_per_step": 0,
                                            "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    bb, params, cfg = make_model(cfgd, args.precision)
    if args.config == "c4":
        return bench_c4(args, cfgd, bb, params, cfg, rank, world, dist, local)
    from paper_2605_29233_b200.scheduler import get_session
    P, G = cfgd["P"], cfgd["G"]
    vocab = params.vocab
    s = _session(params, cfg, P, 1, args)
    K, Wm = args.steps, max(args.warmup, 1)
    from paper_2605_29233_b200 import dp, _lib
    # prompts: global request g -> seed 1000 + g, sharded round-robin over ranks
    mine = dp.shard(K * world, rank, world)
    tasks = ([bb.make_task(900000 + rank * 1000 + i, P, G, vocab) for i in range(Wm)]
             + [bb.make_task(1000 + g, P, G, vocab) for g in mine])
    dev_p = torch.tensor(np.stack([t.prompt for t in tasks]).astype(np.int32), device="cuda")
    dev_t = torch.tensor(np.stack([t.target for t in tasks]).astype(np.int32), device="cuda")
    nb = len(cfgd["bs"])
    snap_c = torch.zeros(Wm + K, 1, 32, dtype=torch.int32, device="cuda")
    snap_b = torch.zeros(Wm + K, 1, nb, 8, dtype=torch.int32, device="cuda")
    snap_tok = torch.zeros(Wm + K, 1, nb, P + G, dtype=torch.int32, device="cuda")

    def one(i):
        s.set_inputs(dev_p[i:i + 1], dev_t[i:i + 1])
        s.launch(use_graph=True)
        s.snapshot(snap_c[i], snap_b[i])
        with torch.cuda.stream(s.stream):
            snap_tok[i].copy_(s.v_tokens, non_blocking=True)

    log(f"[bench] rank {rank}: warmup {Wm} requests")
    for i in range(Wm):
        one(i)
    s.stream.synchronize()
    s.gemm_stats(reset=True)
    c0 = s.counters()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(s.stream)
        for i in range(Wm, Wm + K):
            one(i)
        ev1.record(s.stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    t_ms = ev0.elapsed_time(ev1)
    c1 = s.counters()
    gst = s.gemm_stats(reset=False)
    ctrl = snap_c[Wm:].cpu().numpy()
    brs = snap_b[Wm:].cpu().numpy()
    toks = snap_tok[Wm:].cpu().numpy()
    status = ctrl[:, 0, 0]
    if not (status == 1).all():
        raise RuntimeError(f"requests did not finish: status {status.tolist()}")
    winners = ctrl[:, 0, 1]
    tokens = np.array([brs[i, 0, winners[i], 3] for i in range(K)], dtype=np.int64)
    nfe = ctrl[:, 0, 5:8].astype(np.int64)
    # one all-gather of the per-request results at the end (no per-step collective)
    L = P + G
    packed = np.full((K, L + 6), -1, dtype=np.int64)
    for i in range(K):
        packed[i, :L] = toks[i, 0, winners[i]]
        packed[i, L:L + 3] = nfe[i]
        packed[i, L + 3] = winners[i]
        packed[i, L + 4] = tokens[i]
        packed[i, L + 5] = ctrl[i, 0, 2]
    if dist is not None:
        all_res = dp.gather_results(packed, K * world, rank, world, device="cuda")
        tt = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
        allt = [torch.zeros_like(tt) for _ in range(world)]
        dist.all_gather(allt, tt)
        t_max_ms = max(float(x.item()) for x in allt)
    else:
        all_res = packed
        t_max_ms = t_ms
    tot_tokens = float(all_res[:, L + 4].sum())
    value = tot_tokens / (t_max_ms / 1e3)

    # ---- e2e through the public API (host buffers) ----
    e2e_tasks = tasks[Wm:Wm + K]  # same prompts as the device-resident run
    if dist is not None:
        dist.barrier()
    # the public call exactly as a user makes it: run_blockbatch with its default
    # trace on (the event records come back to the host every request)
    from paper_2605_29233_b200.scheduler import get_session as _gs
    s_e2e = _gs(params, cfg, P, 1, trace=True)
    bb.run_blockbatch(params, tasks[0], cfg)  # untimed: builds the traced session's graphs
    h2d0, d2h0 = s_e2e.h2d_bytes, s_e2e.d2h_bytes
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_e2e.stream)
    e2e_tok = 0
    for t in e2e_tasks:
        r = bb.run_blockbatch(params, t, cfg)
        e2e_tok += r.tokens_decoded
    e1.record(s_e2e.stream)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    h2d = (s_e2e.h2d_bytes - h2d0) / K
    d2h = (s_e2e.d2h_bytes - d2h0) / K
    e2e_local = torch.tensor([float(e2e_tok), e2e_ms], dtype=torch.float64, device="cuda")
    if dist is not None:
        alle = [torch.zeros_like(e2e_local) for _ in range(world)]
        dist.all_gather(alle, e2e_local)
        alle = torch.stack(alle).cpu().numpy()
    else:
        alle = e2e_local.cpu().numpy()[None]
    e2e_value = alle[:, 0].sum() / (alle[:, 1].max() / 1e3)

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (live per-launch timing) ----
    peaks = {}
    pk = os.path.join(HERE, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm = peaks.get("hbm_gbs", 6650.0)
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    tflops = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1350.0))  # dense bf16, long steps
    d = params.dims
    rows = sum(cfgd["bs"])
    kinds = {0: (d.qkv_out, d.d_model), 1: (d.d_model, d.n_heads * d.hd), 2: (2 * d.d_ff, d.d_model),
             3: (d.d_model, d.d_ff)}
    tot_bytes, tot_ns, tot_ns_w, launches = 0.0, 0.0, 0.0, 0
    per_kind = {}
    for k, (n_out, kk) in kinds.items():
        n_l, ns, ns_w = gst[k][4], gst[k][3], gst[k][2]
        if n_l == 0:
            continue
        byts = 2.0 * (n_out * kk + rows * kk + rows * n_out)  # weights + bf16 activations in/out
        tot_bytes += byts * n_l
        tot_ns += ns
        tot_ns_w += ns_w
        launches += n_l
        per_kind[["qkv", "o", "gate_up", "down"][k]] = {"avg_us": ns / n_l / 1e3, "GBps": byts * n_l / ns,
                                                         "avg_us_after_wait": ns_w / n_l / 1e3}
    # duration convention: min over CTAs of kernel ENTRY -> max over CTAs of exit,
    # so the weight tiles prefetched before the PDL dependency wait are inside
    # the window (and so is any overlap with the predecessor's tail)
    achieved = tot_bytes / tot_ns if tot_ns else 0.0   # bytes/ns == GB/s
    head_l, head_ns = gst[4][4], gst[4][3]
    nfe_mean = nfe.mean(axis=0)
    step_b, step_f, _ = step_bytes_flops(params, cfgd, rows, (P + G) * len(cfgd["bs"]))
    ms_per_nfe = t_ms / max(nfe.sum(), 1)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": None, "peak_source": peak_src,
            # (bf16x2: the MMA's N holds every row twice, hi and lo -> the <2 * rows-per-chunk> instance)
            "kernel": f"k_gemm_tc<{s.info[11] * (2 if args.precision == 'bf16x2' else 1)},0> tcgen05 "
                      "weight-streaming GEMM (block-step QKV/O/gate-up/down)",
            "launches_timed": launches, "per_kind": per_kind,
            "duration_convention": "kernel entry (before the pre-wait weight TMA) to last CTA exit, "
                                   "min/max over CTAs, every launch in the timed region",
            "frac_from_dependency_wait": (tot_bytes / tot_ns_w / hbm) if tot_ns_w else None,
            "head_gemm_GBps": (2.0 * params.vocab.n_out * d.d_model * head_l / head_ns) if head_ns else None,
            "step": {"bytes": step_b, "flops": step_f, "t_roof_ms": step_b / (hbm * 1e6),
                     "ms_per_nfe": ms_per_nfe, "frac": (step_b / (hbm * 1e6)) / ms_per_nfe},
            "step_nfe_weighted": nfe_weighted_roofline(params, cfgd, rows, nfe_mean, hbm, tflops, ms_per_nfe)}
    trf = os.path.join(HERE, "profiles", "gemm_traffic.json")
    if os.path.exists(trf):
        try:
            tj = json.load(open(trf))
            roof["traffic"] = tj.get("dram_bytes_per_launch")
            roof["traffic_algorithmic_bytes_per_launch"] = tot_bytes / launches if launches else None
            roof["traffic_source"] = tj.get("source")
        except Exception:
            pass
    cb = None
    if not args.no_cpu_baseline and world == 1:  # rank 0 at N = 1 only (the other ranks would idle in a barrier)
        try:
            cb = cpu_baseline(cfgd, args.config)
        except Exception as exc:  # never let the reported baseline sink the bench line
            cb = {"value": None, "unit": metric, "cores": os.cpu_count(), "kind": "port",
                  "sample": f"failed: {exc!r}"}
    counters = c1["kernel_launches"] - c0["kernel_launches"]
    variants = {}
    if not args.no_variant and dist is None:
        # the other numerics mode on the same weights and prompts, device-resident, same clock
        # protocol (a secondary number: the headline is --precision)
        from dataclasses import replace as _replace
        other = "bf16" if args.precision == "bf16x2" else "bf16x2"
        p2 = _replace(params, dtype=other, _handle=[None], _sessions={})
        s2 = get_session(p2, cfg, P, 1, trace=False)
        for i in range(Wm):
            s2.set_inputs(dev_p[i:i + 1], dev_t[i:i + 1])
            s2.launch(use_graph=True)
        s2.stream.synchronize()
        v0, v1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sc2 = torch.zeros(K, 1, 32, dtype=torch.int32, device="cuda")
        sb2 = torch.zeros(K, 1, nb, 8, dtype=torch.int32, device="cuda")
        v0.record(s2.stream)
        for i in range(Wm, Wm + K):
            s2.set_inputs(dev_p[i:i + 1], dev_t[i:i + 1])
            s2.launch(use_graph=True)
            s2.snapshot(sc2[i - Wm], sb2[i - Wm])
        v1.record(s2.stream)
        v1.synchronize()
        vms = v0.elapsed_time(v1)
        c2_, b2_ = sc2.cpu().numpy(), sb2.cpu().numpy()
        tok2 = float(sum(b2_[i, 0, c2_[i, 0, 1], 3] for i in range(K)))
        nfe2 = float(c2_[:, 0, 5:8].sum())
        variants[other] = {"value": tok2 / (vms / 1e3), "unit": "decoded tokens/s", "ms_per_nfe": vms / max(nfe2, 1),
                           "nfe_per_request": nfe2 / K, "note": "same prompts and weights, device-resident, same "
                           "timing protocol; decisions (and so NFE) differ with the numerics"}
        del s2, p2
    line = {
        "metric": metric, "value": value, "unit": "decoded tokens/s", "n_gpus": world, "steps": K,
        "warmup": Wm, "ms_per_step": t_max_ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.precision, "data": "synthetic (random-init weights, make_task prompts)",
        "config": {"workload": cfgd["workload"], "branches": list(cfgd["bs"]), "prompt_len": P, "gen_len": G,
                   "refresh_interval": cfgd["R"], "head_scale": cfgd["head_scale"], "gamma": cfgd["gamma"],
                   "requests_per_gpu_per_step": 1, "parallelism": f"request-parallel dp{world}",
                   "l2": "inputs larger than L2 (16 GB of weights streamed per block step)"},
        "nfe_per_request": float(all_res[:, L:L + 3].sum(axis=1).mean()), "nfe_split": nfe_mean.tolist(),
        "requests": int(len(all_res)),
        "tokens_per_request": float(tokens.mean()), "ms_per_nfe": ms_per_nfe,
        "dynamics_per_request": {k: float(ctrl[:, 0, w].mean()) for k, w in (
            ("merges", _lib.C_MERGES), ("syncs", _lib.C_SYNCS), ("commits", _lib.C_COMMITS),
            ("refreshes", _lib.C_REFRESHES), ("cow_pages", _lib.C_COW_PAGES))},
        "e2e": {"value": e2e_value, "unit": "decoded tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "roofline": roof, "cpu_baseline": cb, "clocks": clk.summary(), "gpu_launches": int(counters),
        "precision_variants": variants,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
