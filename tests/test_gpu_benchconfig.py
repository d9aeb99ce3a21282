"""Word-exact parity at the bench's OWN configuration (VERDICT r1 "Next" #1).

bench.py times ring 2^16 (2^15 slots), L = 7, alpha = 2, key seed 1, the
reference bench weights sin(0.001(31r+c)+0.25) (W = None plans,
slotforge_cli.cpp:88-92) and the Table-4 stage levels. Those parameters select
the production kernel instantiations (fused_col_kernel<8,8,...>,
ks_row_kernel<8,8>, ks_sum_kernel<8,8,...>, ntt_row_epi<8,8,...> with the
fused head-mask epilogue, vmm_mac_kernel at 2^16) that the golden-size tests
never reach. Every test here runs one bench operator on the GPU and the same
operator on the CPU CKKS twin (oracle/ckks_oracle.cpp via oracle/ckks.py,
OpenMP on the host cores) and compares every ciphertext word.

Operators (reference lines): vmm_interleaved (vmm.cpp:179-236) at level 4 and
its sharded multi-VMM partial at level 3; rope_apply / make_v_pieces /
v_append / k_append at position 2047 (kv_attention.cpp:111-182); qk_dot over
16 K-cts at level 2 (kv_attention.cpp:184-214); softmax_times_v over one group
(kv_attention.cpp:216-241). Sizes are bounded so the twin finishes in tens of
seconds; the kernels and parameters are the bench's.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SLOTS, L, ALPHA, SEED = 32768, 7, 2, 1
D, H, NP = 4096, 32, 2048


def bench_weight(rows, cols):
    """The reference bench weight, with the same libm sin the C++ plan uses
    (numpy's vectorised sin may differ by an ulp, which would change the
    rounded plaintext words)."""
    from oracle.ckks import bench_weight as bw
    return bw(rows, cols)


@pytest.fixture(scope="module")
def pair():
    import paper_2602_11470_b200 as sf
    from oracle.ckks import CkksOracle
    return sf.Backend(SLOTS, L, alpha=ALPHA, seed=SEED), CkksOracle(SLOTS, L, alpha=ALPHA, seed=SEED)


def _eq(a, b, what):
    da, db = a.data(), b.data()
    assert da.shape == db.shape, (what, da.shape, db.shape)
    bad = int(np.count_nonzero(da != db))
    assert bad == 0, f"{what}: {bad} of {da.size} words differ"
    assert a.level == b.level and abs(a.scale - b.scale) <= 1e-9 * abs(b.scale), what


def _activation(d, seed, level, g, o, sf, offset=0, deferred=False):
    """A fresh client encryption in the interleaved layout; deferred=True tags
    it like a VMM output whose mask is deferred (the bench's q / k / v)."""
    from oracle.layout import make_interleaved
    s = np.zeros(SLOTS)
    t = SLOTS // d
    s[np.arange(d) * t + offset] = np.random.default_rng(seed).normal(size=d)
    ly_g, ly_o = sf.make_interleaved(d, SLOTS, offset), make_interleaved(d, SLOTS, offset)
    if deferred:
        ly_g, ly_o = ly_g.with_(deferred_mask=True), ly_o.with_(deferred_mask=True)
    return g.encrypt(s, level, ly_g, seed=seed), o.encrypt(s, level, ly_o, seed=seed), s


def test_bench_vmm_4096_level4_bench_weights(pair):
    """Q-projection shape: 4096 x 4096 BSGS VMM at level 4 with the W = None
    bench-weight plan (vmm_mac_kernel, hoisted babies, giant rotation sums,
    reduce ladder), and the multi-VMM path the bench uses for Q/K (shared
    ladder + babies, K plan at output offset 2047 mod t = 7)."""
    import paper_2602_11470_b200 as sf
    from oracle import protocols as P
    g, o = pair
    W = bench_weight(D, D)
    xg, xo, xs = _activation(D, 42, 4, g, o, sf)
    wq = sf.VmmPlan(g, None, D, D, 4, 0, 0, True)
    wk = sf.VmmPlan(g, None, D, D, 4, 0, (NP - 1) % 8, True)
    q_g, k_g = sf.vmm_interleaved_multi(g, xg, [wq, wk])
    q_o = P.vmm_interleaved(o, xo, W, bsgs=True, out_offset=0)
    _eq(q_g, q_o, "Q = x W (4096^2, level 4)")
    # decrypted against float64 on the valid lanes (deferred garbage elsewhere)
    t = SLOTS // D
    want = xs[np.arange(D) * t] @ W
    assert np.max(np.abs(g.decrypt(q_g)[np.arange(D) * t] - want)) < 1e-3
    k_o = P.vmm_interleaved(o, xo, W, bsgs=True, out_offset=(NP - 1) % 8)
    _eq(k_g, k_o, "K = x W (output offset 7)")


def test_bench_multi_vmm_partial_4096_to_14336(pair):
    """Up/gate shape 4096 -> 14336 at level 3 (d_out padded to 16384): the
    rank-0 partial of a world of 8 (one giant group of the multi-VMM over the
    gate and up plans) against the twin's partial of the same giant subset."""
    import paper_2602_11470_b200 as sf
    from paper_2602_11470_b200 import shard
    from oracle import shard_ref
    g, o = pair
    FF = 14336
    xg, xo, _ = _activation(D, 44, 3, g, o, sf)
    wg = sf.VmmPlan(g, None, D, FF, 3, 0, 0, True)
    wu = sf.VmmPlan(g, None, D, FF, 3, 0, 0, True)
    parts = shard.vmm_multi_partial(g, xg, [wg, wu], 0, 8)
    want = shard_ref.vmm_partial(o, xo, bench_weight(D, FF), True, 0, 0, 8)
    _eq(parts[0], want, "gate partial (rank 0 of 8)")
    _eq(parts[1], want, "up partial (same weights)")


def _bench_cache(g, o, sf, P, n_prime, level=2, distinct_k=2):
    """A cache at the bench's n' with the bench's shapes. Untouched ciphertexts
    may share one encryption (values are immutable), which keeps the twin small."""
    from oracle.layout import make_interleaved
    cfg_g = sf.AttentionConfig(SLOTS, D, H, 0, NP)
    cfg_o = P.AttentionConfig(SLOTS, D, H, 0, NP)
    t, gt, dh = cfg_g.t, cfg_g.group_tokens, cfg_g.d_head
    rng = np.random.default_rng(7)
    n_k = (n_prime + t - 1) // t
    kg, ko = [], []
    for j in range(n_k):
        if j < distinct_k or j == n_k - 1:
            s = np.zeros(SLOTS)
            for tau in range(min(t, n_prime - j * t)):
                s[np.arange(D) * t + tau] = rng.normal(size=D)
            ly_g, ly_o = sf.make_interleaved(D, SLOTS, 0, H), make_interleaved(D, SLOTS, 0, H)
            cur = (g.encrypt(s, level, ly_g, seed=1000 + j), o.encrypt(s, level, ly_o, seed=1000 + j))
        kg.append(cur[0])
        ko.append(cur[1])
    n_groups = (n_prime + gt - 1) // gt
    vg, vo = [], []
    for gi in range(n_groups):
        s = rng.normal(size=SLOTS)
        a, b = g.encrypt(s, level, seed=2000 + gi), o.encrypt(s, level, seed=2000 + gi)
        vg.append([a] * (2 * dh - 1))
        vo.append([b] * (2 * dh - 1))
    cache_g = sf.kv_from_cts(g, cfg_g, n_prime, kg, vg)
    cache_o = P.KVCache(n_prime, ko, vo)
    return cfg_g, cfg_o, cache_g, cache_o


def test_bench_rope_and_appends_at_position_2047(pair):
    """RoPE & Cache stage of the bench token (position n' = 2047): rope_apply of
    q and k (level 3 -> 2), make_v_pieces (128 masked pieces), v_append into
    group 1 and k_append into the partially filled last K-ct (offset 7)."""
    import paper_2602_11470_b200 as sf
    from oracle import protocols as P
    g, o = pair
    cfg_g, cfg_o, cache_g, cache_o = _bench_cache(g, o, sf, P, NP - 1)
    pos = NP - 1
    off = pos % cfg_g.t
    qg, qo, _ = _activation(D, 50, 3, g, o, sf, deferred=True)
    kg, ko, _ = _activation(D, 51, 3, g, o, sf, offset=off, deferred=True)
    vg, vo, _ = _activation(D, 52, 3, g, o, sf, offset=off, deferred=True)
    qr_g, kr_g = sf.rope_apply(g, qg, cfg_g, pos), sf.rope_apply(g, kg, cfg_g, pos)
    qr_o, kr_o = P.rope_apply(o, qo, cfg_o, pos), P.rope_apply(o, ko, cfg_o, pos)
    _eq(qr_g, qr_o, "rope(q)")
    _eq(kr_g, kr_o, "rope(k)")
    pieces_g = sf.make_v_pieces(g, cache_g, vg, pos)
    pieces_o = P.make_v_pieces(o, vo, cfg_o, pos)
    for e in (0, 1, 63, 127):
        _eq(pieces_g[e], pieces_o[e], f"v piece {e}")
    c2_g = sf.k_append(g, sf.v_append(g, cache_g, pieces_g), kr_g)
    c2_o = P.k_append(o, P.v_append(o, cache_o, pieces_o, cfg_o), kr_o, cfg_o)
    assert c2_g.n_prime == c2_o.n_prime == NP
    _eq(c2_g.k_cts[-1], c2_o.k_cts[-1], "last K-ct after k_append")
    for idx in (0, 127, 254):
        _eq(c2_g.v_cts[1][idx], c2_o.v_cts[1][idx], f"group-1 V variant {idx} after v_append")


def test_bench_qk_dot_16_kcts_level2(pair):
    """QK^T at the bench's levels over 16 K-cts (two per pack group): replicate,
    ct x ct + relinearise/rescale, radix fold rotation sums, the ReplicateExtract
    head mask fused into the fold's last ModDown epilogue, pack rotation sums."""
    import paper_2602_11470_b200 as sf
    from oracle import protocols as P
    g, o = pair
    cfg_g, cfg_o, cache_g, cache_o = _bench_cache(g, o, sf, P, 16 * 8, distinct_k=16)
    from oracle.layout import make_interleaved
    ly_g, ly_o = sf.make_interleaved(D, SLOTS, 0, H), make_interleaved(D, SLOTS, 0, H)
    s = np.zeros(SLOTS)
    s[np.arange(D) * 8] = np.random.default_rng(60).normal(size=D)
    qg, qo = g.encrypt(s, 2, ly_g, seed=61), o.encrypt(s, 2, ly_o, seed=61)
    maps_g = sf.qk_dot(g, qg, cache_g)
    maps_o = P.qk_dot(o, qo, cache_o, cfg_o)
    assert len(maps_g) == len(maps_o) == 1
    _eq(maps_g[0], maps_o[0], "QK^T score map")


def test_bench_softmax_times_v_one_group(pair):
    """Score*V over one group at the bench's levels (probabilities and V at
    level 2): the probability rotations, the lazily relinearised product sum
    (one relinearisation), the lane fold and the output mask."""
    import paper_2602_11470_b200 as sf
    from oracle import protocols as P
    g, o = pair
    cfg_g, cfg_o, cache_g, cache_o = _bench_cache(g, o, sf, P, 40)
    p = np.zeros(SLOTS)
    gt = cfg_g.group_tokens
    for h in range(H):
        p[h * gt:h * gt + 40] = 1.0 / 40
    pg, po = g.encrypt(p, 2, seed=70), o.encrypt(p, 2, seed=70)
    att_g = sf.softmax_times_v(g, [pg], cache_g)
    att_o = P.softmax_times_v(o, [po], cache_o, cfg_o)
    _eq(att_g, att_o, "Score*V output")
