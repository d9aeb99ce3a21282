"""Ring 2^17 (the largest fused-path ring: 256 x 512, C = 512 row kernels): an
HE-VMM whose giant sums are two-digit rotation sums (ks_sum_kernel with the
digit-aware high-word fold cadence), plus a rotation, word for word against the
CPU twin."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_vmm_and_rotation_at_ring_2_17_match_the_twin():
    import paper_2602_11470_b200 as sf
    from oracle import protocols as P
    from oracle.ckks import CkksOracle
    from oracle.layout import make_interleaved
    N, L, rows, cols = 65536, 3, 64, 64  # 4 limbs at alpha = 2: two digits
    rng = np.random.default_rng(17)
    W = rng.normal(size=(rows, cols)) / 8
    x = rng.normal(size=rows)
    g, o = sf.Backend(N, L, alpha=2), CkksOracle(N, L, alpha=2)
    ly = make_interleaved(rows, N, 0)
    slots = np.zeros(N)
    slots[np.arange(rows) * ly.t] = x
    xg, xo = g.encrypt(slots, L, ly, seed=5), o.encrypt(slots, L, ly, seed=5)
    assert np.array_equal(xg.data(), xo.data())
    yg = sf.vmm_interleaved(g, xg, W, bsgs=True, mask_output=True)
    yo = P.vmm_interleaved(o, xo, W, bsgs=True, mask_output=True)
    assert np.array_equal(yg.data(), yo.data())
    got = g.decrypt(yg)[np.arange(cols) * (N // cols)]
    assert np.max(np.abs(got - x @ W)) < 1e-4
    assert np.array_equal(g.rotate(xg, 7).data(), o.rotate(xo, 7).data())
