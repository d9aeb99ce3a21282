"""The decoder harness (paper_2602_11470_b200/harness.py, SURVEY.md §8(f)
rank 1) against the reference's own harness: the golden fixture
tests/golden/ref_harness.json.gz is emitted by the UNMODIFIED reference
(oracle/ref_golden.cpp `harness` set: make_weights, seeded_prompt,
plaintext_reference, plan_decode, run_generation). On CPU the harness runs over
the slot-simulator oracle, so its level trace, per-phase ledger, bootstrap
count and generated tokens must equal the reference report exactly."""
import gzip
import json
import os

import numpy as np
import pytest

from harness_sim_ops import SimOps
from oracle.slot_sim import SimBackend
from paper_2602_11470_b200 import harness as Hn

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_harness.json.gz")


def cases():
    with gzip.open(GOLD, "rt") as f:
        return json.load(f)["cases"]


def _seq_sum(a):
    s = 0.0
    for v in np.ravel(a):
        s += float(v)
    return s


@pytest.mark.parametrize("ci", range(5))
def test_weights_prompt_and_plaintext_reference(ci):
    c = cases()[ci]
    cfg = Hn.ModelConfig.from_json(c["config"])
    w = Hn.make_weights(cfg)
    mats = [("embedding", w.embedding, c["weights"]["embedding"])]
    for b, blk in enumerate(w.blocks):
        for name in ("wq", "wk", "wv", "wo", "w_gate", "w_up", "w_down", "gamma1", "beta1", "gamma2", "beta2"):
            mats.append((f"{b}.{name}", getattr(blk, name), c["weights"]["blocks"][b][name]))
    for name, m, want in mats:  # bit-exact draws (seeded mt19937_64 + libstdc++ normal_distribution)
        flat = np.ravel(m)
        assert list(flat[:len(want["head"])]) == want["head"], name
        assert _seq_sum(flat) == want["sum"], name
        if "last" in want:
            assert flat[-1] == want["last"], name
    prompt = Hn.seeded_prompt(cfg, c["n0"])
    assert prompt == c["prompt"]
    ref = Hn.plaintext_reference(cfg, w, prompt, c["gen_len"])
    assert ref.tokens == c["ref_tokens"]
    for got, want in zip(ref.final_states, c["ref_final_states"]):
        np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


@pytest.mark.parametrize("ci", range(5))
def test_generation_matches_reference_report(ci):
    c = cases()[ci]
    cfg = Hn.ModelConfig.from_json(c["config"])
    w = Hn.make_weights(cfg)
    plan = Hn.PlacementPlan.from_json(c["plan"])
    be = SimBackend(cfg.N, cfg.L)
    rep = Hn.run_generation(be, SimOps(be), cfg, w, c["prompt"], c["gen_len"], plan)
    want = c["report"]
    assert rep.generated == want["generated"]
    assert rep.bootstrap_count == want["bootstrap_count"]
    got_trace = [(e.step, e.block, e.phase, e.level_in, e.level_out, e.bootstrap_to) for e in rep.level_trace]
    want_trace = [(e["step"], e["block"], e["phase"], e["level_in"], e["level_out"], e["bootstrap_to"])
                  for e in want["level_trace"]]
    assert got_trace == want_trace
    assert [p for p in rep.phase_rows()] == want["phases"]
    assert rep.to_csv() == c["report_csv"]
    if cfg.mode == "exact":
        assert rep.max_abs_error < 1e-9
    else:  # approx mode: the approximation error itself, as the reference measured it
        assert abs(rep.max_abs_error - want["max_abs_error"]) <= 1e-6 * max(1.0, want["max_abs_error"])


def test_plan_levels_and_block_budget():
    """test_harness.cpp:433-447: the five projection/rotary stages consume
    exactly five levels per block instance; rope-and-cache exactly one; the
    exact-mode nonlinear stages are level-free."""
    c = cases()[0]
    cfg = Hn.ModelConfig.from_json(c["config"])
    w = Hn.make_weights(cfg)
    be = SimBackend(cfg.N, cfg.L)
    rep = Hn.run_generation(be, SimOps(be), cfg, w, c["prompt"], c["gen_len"], Hn.PlacementPlan.from_json(c["plan"]))
    lv = {}
    for e in rep.level_trace:
        if e.phase == "RoPE & Cache":
            assert e.level_in - e.level_out == 1
        if e.phase in ("Q, K, V", "RoPE & Cache", "Output projection", "Up & Gate projection", "Down projection"):
            lv[(e.step, e.block)] = lv.get((e.step, e.block), 0) + e.level_in - e.level_out
        if e.phase in ("Softmax", "Add & Norm"):
            assert e.level_in == e.level_out
    assert len(lv) == 8 * 2 and set(lv.values()) == {5}


@pytest.mark.parametrize("ci", range(5))
def test_generation_over_ckks_oracle(ci):
    """The same harness over the bit-exact CPU CKKS twin (real RNS-CKKS): the
    reference's tokens, level trace and ledger, within CKKS precision."""
    from oracle.ckks import CkksOracle
    c = cases()[ci]
    cfg = Hn.ModelConfig.from_json(c["config"])
    w = Hn.make_weights(cfg)
    be = CkksOracle(cfg.N, cfg.L, alpha=2, seed=5)
    rep = Hn.run_generation(be, SimOps(be), cfg, w, c["prompt"], c["gen_len"], Hn.PlacementPlan.from_json(c["plan"]))
    assert rep.generated == c["report"]["generated"]
    assert rep.phase_rows() == c["report"]["phases"]
    if cfg.mode == "exact":
        assert rep.max_abs_error < 1e-6, rep.max_abs_error
    else:  # CKKS noise on top of the approximation error the reference measured
        ref_err = c["report"]["max_abs_error"]
        assert abs(rep.max_abs_error - ref_err) <= 1e-4 * max(1.0, ref_err)
