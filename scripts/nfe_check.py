"""Quick decision-parity check of a numerics build against stored fp32 NFE
triples (no fp32 rerun): runs the product numerics over the seeds of a
parity_bf16.py output and counts identical NFE triples.

    python scripts/nfe_check.py PARITY.json [--dtype bf16x2] [--test-flags N]

(bisecting numerics changes between builds; the fp32 verification path is the
reference the parity file recorded)."""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("parity")
    ap.add_argument("--dtype", default="bf16x2")
    ap.add_argument("--test-flags", type=int, default=0)
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    d = json.load(open(a.parity))
    recs = d["products"][a.dtype]["prompts"] if "products" in d else d["prompts"]
    cfgd = bench.CONFIGS[a.config]
    bb, params, cfg = bench.make_model(cfgd, a.dtype)
    if a.test_flags:
        from paper_2605_29233_b200.engine import Session
        from paper_2605_29233_b200.scheduler import _cfg_key
        params._sessions[_cfg_key(cfg, cfgd["P"], 1, True)] = Session(params, cfg, cfgd["P"], 1,
                                                                      test_flags=a.test_flags)
    same, bad = 0, []
    for p in recs:
        t = bb.make_task(p["seed"], cfgd["P"], cfgd["G"], params.vocab)
        r = bb.run_blockbatch(params, t, cfg)
        ok = list(r.nfe.snapshot()) == p["nfe_f32"]
        same += ok
        if not ok:
            bad.append(p["seed"])
    print(json.dumps({"dtype": a.dtype, "test_flags": a.test_flags, "prompts": len(recs), "same_nfe": same,
                      "mismatch_seeds": bad}))


if __name__ == "__main__":
    main()
