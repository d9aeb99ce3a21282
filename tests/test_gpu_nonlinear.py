"""Homomorphic nonlinearities on the GPU backend:
every reference golden case (tests/golden/ref_nonlinear.json.gz) runs through
the CUDA library -- polynomial evaluation, Goldschmidt, exponential, softmax,
layer norm, SiLU/GeLU -- with the reference's output levels and ledger counts,
outputs word-identical to the bit-exact CPU CKKS twin (same keys and seeds)
and within CKKS precision of the reference's float64 slots."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.dirname(__file__))

from nonlinear_cases import cases, run_case  # noqa: E402

CASES = cases()


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_gpu_nonlinear(ci):
    import paper_2602_11470_b200 as sf
    from oracle.ckks import CkksOracle
    from oracle.layout import Layout as OLayout
    c = CASES[ci]
    be = sf.Backend(c["N"], c["L"], alpha=2, seed=9)
    be.ledger.reset()
    outs = run_case(c, be, lambda d, N, o, h, df: sf.Layout("interleaved", d, N // d, o, h, df))
    assert [o.level for o in outs] == c["out_levels"]
    assert be.ledger.totals().asdict() == c["counts"]
    ob = CkksOracle(c["N"], c["L"], alpha=2, seed=9)
    oouts = run_case(c, ob, lambda d, N, o, h, df: OLayout("interleaved", d, N // d, o, h, df))
    for o, oo, want in zip(outs, oouts, c["outputs"]):
        assert np.array_equal(o.data(), oo.data())  # word for word
        want = np.array(want)
        np.testing.assert_allclose(be.decrypt(o), want, rtol=0, atol=1e-5 * max(1.0, np.max(np.abs(want))))
