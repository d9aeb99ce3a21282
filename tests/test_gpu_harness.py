"""The decoder harness end to end on the GPU backend (
test_harness.cpp:406-453, 508-520): every homomorphic stage of prefill and of
each decode step runs through the CUDA library; exact-mode softmax / norm /
SiLU and the plan's bootstraps are client round trips. The generated tokens,
level trace and per-phase ledger must equal the reference's own report
(tests/golden/ref_harness.json.gz) and the hidden states must stay within
CKKS precision of the plaintext model."""
import gzip
import json
import os

import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_harness.json.gz")


@pytest.mark.parametrize("ci", [0, 1, 2, 3, 4])
def test_gpu_generation_matches_reference(ci):
    import paper_2602_11470_b200 as sf
    from paper_2602_11470_b200 import harness as Hn
    with gzip.open(GOLD, "rt") as f:
        c = json.load(f)["cases"][ci]
    cfg = Hn.ModelConfig.from_json(c["config"])
    w = Hn.make_weights(cfg)
    be = sf.Backend(cfg.N, cfg.L, alpha=2, seed=5)
    rep = Hn.run_generation(be, Hn.GpuOps(be), cfg, w, c["prompt"], c["gen_len"],
                            Hn.PlacementPlan.from_json(c["plan"]))
    want = c["report"]
    assert rep.generated == want["generated"]
    assert rep.bootstrap_count == want["bootstrap_count"]
    assert [(e.step, e.block, e.phase, e.level_in, e.level_out, e.bootstrap_to) for e in rep.level_trace] == \
        [(e["step"], e["block"], e["phase"], e["level_in"], e["level_out"], e["bootstrap_to"])
         for e in want["level_trace"]]
    assert rep.phase_rows() == want["phases"]
    if cfg.mode == "exact":
        # CKKS at scale 2^40: states and logits of the whole generation within
        # 1e-6 of the exact double-precision model (the reference's own bound)
        assert rep.max_abs_error < 1e-6, rep.max_abs_error
    else:  # approx mode: the reference's approximation error, plus CKKS noise
        ref_err = want["max_abs_error"]
        assert abs(rep.max_abs_error - ref_err) <= 1e-4 * max(1.0, ref_err)
    # and word-for-word the CPU CKKS twin (same keys and encryption seeds):
    # every decrypted hidden state identical to the last bit
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from harness_sim_ops import SimOps
    from oracle.ckks import CkksOracle
    ob = CkksOracle(cfg.N, cfg.L, alpha=2, seed=5)
    orep = Hn.run_generation(ob, SimOps(ob), cfg, w, c["prompt"], c["gen_len"], Hn.PlacementPlan.from_json(c["plan"]))
    assert orep.generated == rep.generated
    for a, b in zip(rep.hidden, orep.hidden):
        assert (a == b).all()
    assert rep.max_abs_error == orep.max_abs_error
