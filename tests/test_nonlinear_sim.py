"""Homomorphic nonlinearities (paper_2602_11470_b200/nonlinear.py, SURVEY.md
§8(f) rank 3) against the reference's own outputs: every case of
tests/golden/ref_nonlinear.json.gz (emitted by the unmodified nonlinear.cpp)
replayed over the slot-simulator oracle must give the same slots (to float64
round-off: the least-squares fits are solved by different routines), the same
output levels and the same ledger counts; then over the CKKS oracle within
CKKS precision."""
import numpy as np
import pytest

from nonlinear_cases import cases, run_case
from oracle.layout import Layout
from oracle.slot_sim import SimBackend
from paper_2602_11470_b200 import nonlinear as NL

CASES = cases()


class _SeededSim(SimBackend):
    def encrypt(self, slots, level=-1, layout=None, seed=None):
        return super().encrypt(slots, level, layout)


def _layout(d, N, off, heads, deferred):
    return Layout("interleaved", d, N // d, off, heads, deferred)


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_nonlinear_matches_reference(ci):
    c = CASES[ci]
    be = _SeededSim(c["N"], c["L"])
    be.ledger.reset()
    outs = run_case(c, be, _layout)
    assert [o.level for o in outs] == c["out_levels"]
    assert be.ledger.totals().asdict() == c["counts"]
    for o, want in zip(outs, c["outputs"]):
        np.testing.assert_allclose(o.slots, want, rtol=0, atol=1e-9 * max(1.0, np.max(np.abs(want))))


def test_specs_traces_and_budget():
    sm = NL.desk_spec("desk-default", "softmax")
    assert NL.softmax_depth(sm) == sm.depth_budget == 6 + 1 + 14 + 1
    back = NL.ApproxSpec.from_json(sm.to_json())
    assert back == sm
    tr = NL.sublayer_trace("softmax", sm)
    assert sum(p.depth for p in tr) == NL.softmax_depth(sm)
    assert NL.sublayer_trace("softmax", NL.ApproxSpec(function="softmax", exact=True)) == []
    nm = NL.desk_spec("desk-default", "norm")
    assert sum(p.depth for p in NL.sublayer_trace("norm", nm)) == NL.norm_depth(nm)
    be = SimBackend(16, 30)
    spec = NL.desk_spec("desk-default", "silu")
    spec.depth_budget = 3
    with pytest.raises(NL.InfeasibleLayer):
        NL.approx_silu(be, be.encrypt(np.zeros(16)), spec)


def test_domain_strict_or_clamp():
    """test_nonlinear.cpp:160-171."""
    be = SimBackend(16, 20)
    spec = NL.desk_spec("desk-default", "inverse")
    x = be.encrypt(np.full(16, 0.5) - np.eye(16)[3] * 0.499)  # one slot below 1/64
    with pytest.raises(NL.DomainViolation):
        NL.goldschmidt(be, x, NL.INVERSE, spec)
    spec.strict_domain = False
    y = NL.goldschmidt(be, x, NL.INVERSE, spec)
    assert abs(y.slots[3] - 64.0) < 1.0 and abs(y.slots[0] - 2.0) < 1e-3


@pytest.mark.parametrize("ci", [i for i, c in enumerate(CASES) if c["op"] != "eval_cheb" or c["extra"]["deg"] in (5, 31)])
def test_nonlinear_over_ckks_oracle(ci):
    """Real RNS-CKKS (the bit-exact CPU twin): same levels and ledger, outputs
    within CKKS precision of the reference's float64 slots."""
    from oracle.ckks import CkksOracle
    c = CASES[ci]
    be = CkksOracle(c["N"], c["L"], alpha=2, seed=9)
    be.ledger.reset()
    outs = run_case(c, be, _layout)
    assert [o.level for o in outs] == c["out_levels"]
    assert be.ledger.totals().asdict() == c["counts"]
    for o, want in zip(outs, c["outputs"]):
        want = np.array(want)
        np.testing.assert_allclose(be.decrypt(o), want, rtol=0, atol=1e-5 * max(1.0, np.max(np.abs(want))))
