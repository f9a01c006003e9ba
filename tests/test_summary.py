"""Run-summary CSV parity (reference cli.py:147-165,
analysis.py:160-171): ``summary_row`` / ``write_summary`` produce the
reference CLI's table byte for byte.  The golden CSV was written by the
reference's own functions (tests/golden/make_golden.py --summary-only)."""

import os

import numpy as np
import pytest

import goldens

bb = pytest.importorskip("paper_2605_29233_b200")

CONFIGS = ("c1_hs2", "default_g4_eos")  # make_golden.SUMMARY_CONFIGS


def _want():
    with open(os.path.join(goldens.GOLDEN, "summary_ref.csv"), "rb") as fh:
        return fh.read()


def _vocab(g):
    return bb.Vocab(size=g["model"]["vocab_size"])


def test_summary_csv_matches_reference_from_golden_runs(tmp_path):
    runs = goldens.load("runs_ref.json")
    rows = []
    for name in CONFIGS:
        g = runs[name]
        for seed, r in zip(g["seeds"], g["runs"]):
            res = bb.GenerationResult(row=bb.SequenceRow(np.array(r["tokens"], dtype=np.int64), g["prompt_len"]),
                                      branch_index=r["branch_index"], block_size=r["block_size"],
                                      nfe=bb.NfeCounter(*r["nfe"]), trace=[], correct=r["correct"],
                                      tokens_decoded=r["tokens_decoded"], eos_position=r["eos_position"])
            rows.append(bb.summary_row(seed, f"blockbatch:{name}", res, _vocab(g)))
    path = tmp_path / "summary.csv"
    bb.write_summary(path, rows)
    assert path.read_bytes() == _want()


@pytest.mark.gpu
def test_summary_csv_of_device_runs_matches_reference(tmp_path):
    """fp32 verification mode: the device runs' summary table is the reference's."""
    from test_gpu_parity import cfg_from, ref_model
    runs = goldens.load("runs_ref.json")
    rows = []
    for name in CONFIGS:
        g = runs[name]
        params = ref_model(g["model"])
        cfg = cfg_from(g["config"])
        for seed in g["seeds"]:
            task = bb.make_task(seed, g["prompt_len"], g["gen_len"], params.vocab)
            rows.append(bb.summary_row(seed, f"blockbatch:{name}", bb.run_blockbatch(params, task, cfg), params.vocab))
    path = tmp_path / "summary.csv"
    bb.write_summary(path, rows)
    assert path.read_bytes() == _want()
