"""GPU parity: the product (sm_100a kernels via include/sf_b200.h) against the
CPU CKKS oracle, word for word, and against the reference's golden slots.

Bar (ROUND-1 spec): every ciphertext the GPU produces is
bit-identical to the oracle's for the same keys / seeds / inputs; decrypted
slots match the reference golden vectors within TOL (CKKS precision at
scale 2^40); ledger counts and levels equal the reference's exactly.
"""
import numpy as np
import pytest

from golden_util import cases, counts_dict, layout_from

pytestmark = pytest.mark.gpu

TOL = 1e-6


def _pair(N, L, **kw):
    import paper_2602_11470_b200 as sf
    from oracle.ckks import CkksOracle
    return sf.Backend(N, L, **kw), CkksOracle(N, L, **kw)


def _eq(g, o):
    gd, od = g.data(), o.data()
    assert gd.shape == od.shape, (gd.shape, od.shape)
    bad = np.argwhere(gd != od)
    assert bad.size == 0, f"{len(bad)} words differ, first at {bad[:3].tolist()}"


@pytest.mark.parametrize("N,L,alpha,log_n", [(8, 3, 2, None), (512, 4, 2, None), (2048, 5, 3, None),
                                             (16, 2, 3, 8), (4096, 3, 2, None), (32768, 4, 5, None)])
def test_keys_and_encryption_bit_exact(N, L, alpha, log_n):
    kw = dict(alpha=alpha, log_n=log_n) if log_n else dict(alpha=alpha)
    g, o = _pair(N, L, **kw)
    assert np.array_equal(g.primes, o.primes)
    from oracle.ckks import _u64, lib
    sk = np.empty((len(o.primes), o.n), dtype=np.uint64)
    lib().ock_secret_key(o.ptr, _u64(sk))
    assert np.array_equal(g.secret_key(), sk)
    for r in (1, -3):
        ge = g.galois_elt(r)
        assert ge == lib().ock_galois_elt(o.ptr, r)
        kk = np.empty_like(g.switching_key(ge))
        lib().ock_key(o.ptr, ge, _u64(kk))
        assert np.array_equal(g.switching_key(ge), kk)
    rng = np.random.default_rng(N)
    x = rng.normal(size=N)
    import ctypes as C
    enc_o = np.empty((L + 1, o.n), dtype=np.uint64)
    lib().ock_encode(o.ptr, x.ctypes.data_as(C.POINTER(C.c_double)), 2.0 ** 40, L + 1, _u64(enc_o))
    assert np.array_equal(g.encode(x, 2.0 ** 40, L + 1), enc_o)
    cg, co = g.encrypt(x, L, seed=77), o.encrypt(x, L, seed=77)
    _eq(cg, co)
    assert np.max(np.abs(g.decrypt(cg) - x)) < TOL


@pytest.mark.parametrize("N,L,alpha", [(64, 4, 2), (2048, 5, 2), (2048, 6, 7)])
def test_every_evaluator_op_bit_exact(N, L, alpha):
    g, o = _pair(N, L, alpha=alpha)
    rng = np.random.default_rng(5)
    a, b, p = rng.normal(size=N), rng.normal(size=N), rng.normal(size=N)
    ga, oa = g.encrypt(a, L, seed=1), o.encrypt(a, L, seed=1)
    gb, ob = g.encrypt(b, L - 1, seed=2), o.encrypt(b, L - 1, seed=2)
    steps = [
        ("add", lambda be, x, y: be.add(x, y)),
        ("sub", lambda be, x, y: be.sub(x, y)),
        ("add_plain", lambda be, x, y: be.add_plain(x, p)),
        ("mul_plain", lambda be, x, y: be.mul_plain(x, p)),
        ("mac_plain", lambda be, x, y: be.mac_plain([(be.level_drop(x, y.level), p), (y, -p)])),
        ("mul", lambda be, x, y: be.mul(x, y)),
        ("rotate", lambda be, x, y: be.rotate(x, 3)),
        ("rotate_neg", lambda be, x, y: be.rotate(x, -N // 2 + 1)),
        ("level_drop", lambda be, x, y: be.level_drop(x, 1)),
        ("chain", lambda be, x, y: be.rotate(be.mul(be.mul_plain(x, p), y), 5)),
    ]
    for name, f in steps:
        rg, ro = f(g, ga, gb), f(o, oa, ob)
        assert rg.level == ro.level, name
        _eq(rg, ro)
        assert abs(rg.scale - ro.scale) <= 1e-9 * abs(ro.scale), name
        assert np.max(np.abs(g.decrypt(rg) - o.decrypt(ro))) < 1e-12, name
    hs = g.rotate_hoisted(ga, [1, 2, 7])
    for r, h in zip([1, 2, 7], hs):
        _eq(h, o.rotate(oa, r))
    assert g.ledger.totals().hoisted_rotations == 3


def test_zero_ciphertext_semantics():
    import paper_2602_11470_b200 as sf
    g, o = _pair(16, 3, alpha=2)
    z = g.zeros()
    x = g.encrypt(np.arange(16.0), 2, seed=3)
    y = g.add(z, x)
    assert y.level == 2
    _eq(y, o.add(o.zeros(), o.encrypt(np.arange(16.0), 2, seed=3)))
    assert g.ledger.totals().additions == 1
    with pytest.raises(sf.LevelUnderflow):
        g.mul_plain(g.level_drop(x, 0), 1.0)


def test_level_rules_and_errors():
    import paper_2602_11470_b200 as sf
    be = sf.Backend(8, 5)
    a = be.encrypt(np.full(8, 3.0), 5)
    b = be.encrypt(np.full(8, 2.0), 3)
    m = be.mul(a, b)
    assert m.level == 2 and np.allclose(be.decrypt(m), 6.0, atol=TOL)
    mp = be.mul_plain(m, 0.5)
    assert mp.level == 1 and np.allclose(be.decrypt(mp), 3.0, atol=TOL)
    fl = be.mul_plain(mp, 2.0)
    assert fl.level == 0
    with pytest.raises(sf.LevelUnderflow):
        be.mul(fl, fl)
    with pytest.raises(sf.LevelUnderflow):
        be.mul_plain(fl, 2.0)
    assert be.add(fl, fl).level == 0 and be.rotate(fl, 1).level == 0
    with pytest.raises(sf.InvalidTarget):
        be.bootstrap(a, 0)
    with pytest.raises(sf.InvalidTarget):
        be.level_drop(b, 4)
    with pytest.raises(sf.ShapeMismatch):
        be.encrypt(np.zeros(16))
    with pytest.raises(sf.ShapeMismatch):
        sf.Backend(10, 3)
    t = be.ledger.totals()
    assert (t.ct_ct_mults, t.ct_pt_mults) == (1, 2)
    r = be.rotate(be.encrypt(np.arange(1.0, 9.0), 3), 1)
    assert np.allclose(be.decrypt(r), np.roll(np.arange(1.0, 9.0), -1), atol=TOL)
    assert be.rotate(a, 8) is not None and be.ledger.totals().rotations == 2


@pytest.mark.parametrize("which,stride", [("small", 2), ("medium", 1)])
def test_vmm_fused_driver_bit_exact_and_matches_reference(which, stride):
    import paper_2602_11470_b200 as sf
    from oracle import protocols as P
    from oracle.layout import make_interleaved
    for c in cases(which, "vmm")[::stride]:
        N, L = c["N"], c["L"]
        W = np.array(c["W"]).reshape(c["rows"], c["cols"])
        g, o = _pair(N, L, alpha=3)
        lin = make_interleaved(P.padded_dim(c["rows"]), N, c["tau_in"])
        xg = g.encrypt(np.array(c["x_slots"]), L, lin, seed=11)
        xo = o.encrypt(np.array(c["x_slots"]), L, lin, seed=11)
        yg = sf.vmm_interleaved(g, xg, W, bsgs=c["bsgs"], out_offset=c["tau_out"], mask_output=c["mask_output"])
        yo = P.vmm_interleaved(o, xo, W, bsgs=c["bsgs"], out_offset=c["tau_out"], mask_output=c["mask_output"])
        _eq(yg, yo)
        want_y = np.array(c["y_slots"])  # CKKS precision relative to the output's magnitude
        assert np.max(np.abs(g.decrypt(yg) - want_y)) < TOL * max(1.0, np.max(np.abs(want_y)))
        assert g.ledger.totals().asdict() == c["counts"]
        assert yg.level == c["level"]
        ly = yg.layout
        want = layout_from(c["layout"])
        assert (ly.kind, ly.d, ly.t, ly.offset, ly.deferred_mask) == (want.kind, want.d, want.t, want.offset,
                                                                        want.deferred_mask)


def _replay_attention_gpu(be, c):
    """Same sequence as tests/test_oracle_golden.py:replay_attention, through
    the product's C++ protocol entry points."""
    import paper_2602_11470_b200 as sf
    N, L, d, H, np_ = c["N"], c["L"], c["d"], c["H"], c["n_prime"]
    cfg = sf.AttentionConfig(N, d, H, 0, np_)
    t = cfg.t
    K = np.array(c["K"]).reshape(np_, d)
    V = np.array(c["V"]).reshape(np_, d)
    cache = sf.KVCache(be, cfg)
    counts = []
    for u in range(np_):
        vly = sf.make_interleaved(d, N, u % t, H).with_(deferred_mask=True)
        open_ = np.full(N, 7.5)
        open_[np.arange(d) * t + u % t] = V[u]
        v_open = be.encrypt(open_, L - 1, vly)
        c0 = be.ledger.totals()
        parts = sf.make_v_pieces(be, cache, v_open, u)
        cache = sf.v_append(be, cache, parts)
        kly = sf.make_interleaved(d, N, u % t, H)
        ks = np.zeros(N)
        ks[np.arange(d) * t + u % t] = K[u]
        cache = sf.k_append(be, cache, be.encrypt(ks, L - 2, kly))
        counts.append((be.ledger.totals() - c0).asdict())
    be.ledger.reset()
    qs = np.zeros(N)
    qs[np.arange(d) * t] = np.array(c["q"])
    qc = be.encrypt(qs, L - 2, sf.make_interleaved(d, N, 0, H))
    with be.phase("QK^T"):
        maps = sf.qk_dot(be, qc, cache)
    probs = sf.exact_softmax_maps(be, maps, cfg, cache.n_prime)
    with be.phase("Score*V"):
        out = sf.softmax_times_v(be, probs, cache)
    return dict(cache=cache, maps=maps, probs=probs, out=out, append_counts=counts)


@pytest.mark.parametrize("which,stride", [("small", 3), ("medium", 1)])
def test_attention_protocol_bit_exact_and_matches_reference(which, stride):
    from oracle.ckks import CkksOracle
    from test_oracle_golden import replay_attention
    import paper_2602_11470_b200 as sf
    for c in cases(which, "attn")[::stride]:
        g = sf.Backend(c["N"], c["L"], alpha=4)
        o = CkksOracle(c["N"], c["L"], alpha=4)
        rg = _replay_attention_gpu(g, c)
        ro = replay_attention(o, c)
        assert rg["append_counts"] == [dict(x) for x in c["append_counts"]]
        for a, b in zip(rg["cache"].k_cts, ro["cache"].k_cts):
            _eq(a, b)
        for ga, oa in zip(rg["cache"].v_cts, ro["cache"].v_cts):
            for a, b in zip(ga, oa):
                _eq(a, b)
        for a, b in zip(rg["maps"], ro["maps"]):
            _eq(a, b)
        _eq(rg["out"], ro["out"])
        # the attention chain stacks ~10 key switches: its decryption error depends on the
        # key draw (heavy-tailed over seeds), hence a 4x looser bar than one VMM
        assert np.max(np.abs(g.decrypt(rg["out"]) - np.array(c["out_slots"]))) < 4 * TOL
        assert rg["out"].level == c["out_level"]
        assert g.ledger.phase_totals("QK^T").asdict() == c["qk_counts"]
        assert g.ledger.phase_totals("Score*V").asdict() == c["sv_counts"]


def test_rope_bit_exact_and_matches_reference():
    from oracle import protocols as P
    from oracle.layout import make_interleaved
    import paper_2602_11470_b200 as sf
    for c in cases("small", "rope") + cases("medium", "rope"):
        N, L = c["N"], c["L"]
        g, o = _pair(N, L)
        ly = make_interleaved(c["d"], N, c["offset"]).with_(deferred_mask=True)
        xg = g.encrypt(np.array(c["x_slots"]), L, ly, seed=5)
        xo = o.encrypt(np.array(c["x_slots"]), L, ly, seed=5)
        cfg = sf.AttentionConfig(N, c["d"], c["d"] // c["d_head"], 0, 1)
        yg = sf.rope_apply(g, xg, cfg, c["pos"])
        yo = P.fused_extract(o, xo, "rope", dict(n=c["pos"], d_head=c["d_head"], s=ly.t))
        _eq(yg, yo)
        assert np.max(np.abs(g.decrypt(yg) - np.array(c["y_slots"]))) < 1e-5
        assert g.ledger.totals().asdict() == c["counts"]


def test_rope_prepare_then_apply_is_identical():
    """sf_rope_prepare encodes the plaintexts ahead of time (stream-ordered, no
    host wait); the following rope_apply must produce the same words as a cold
    one and charge the same ledger (prepare itself charges nothing)."""
    from oracle import protocols as P
    from oracle.layout import make_interleaved
    import paper_2602_11470_b200 as sf
    c = cases("medium", "rope")[0]
    N, L = c["N"], c["L"]
    g, o = _pair(N, L)
    ly = make_interleaved(c["d"], N, c["offset"]).with_(deferred_mask=True)
    xg = g.encrypt(np.array(c["x_slots"]), L, ly, seed=5)
    xo = o.encrypt(np.array(c["x_slots"]), L, ly, seed=5)
    cfg = sf.AttentionConfig(N, c["d"], c["d"] // c["d_head"], 0, 1)
    sf.rope_prepare(g, cfg, c["pos"], L, c["offset"])
    assert g.ledger.totals().asdict() == sf.OpCounts().asdict()
    yg = sf.rope_apply(g, xg, cfg, c["pos"])
    yo = P.fused_extract(o, xo, "rope", dict(n=c["pos"], d_head=c["d_head"], s=ly.t))
    _eq(yg, yo)
    assert g.ledger.totals().asdict() == c["counts"]
    # a stream of positions: the cache of old positions is pruned, results stay exact
    for pos in range(c["pos"] + 1, c["pos"] + 12):
        sf.rope_prepare(g, cfg, pos, L, c["offset"])
        _eq(sf.rope_apply(g, xg, cfg, pos), P.fused_extract(o, xo, "rope", dict(n=pos, d_head=c["d_head"], s=ly.t)))


def test_full_ring_ntt_and_rotation_parity():
    # ring 2^16 (the north-star N): encryption, mul_plain (rescale) and a
    # rotation (ModUp / key switch / ModDown) word-identical to the oracle
    g, o = _pair(32768, 4, alpha=5)
    rng = np.random.default_rng(9)
    x, p = rng.normal(size=32768), rng.normal(size=32768)
    cg, co = g.encrypt(x, 4, seed=21), o.encrypt(x, 4, seed=21)
    _eq(cg, co)
    _eq(g.mul_plain(cg, p), o.mul_plain(co, p))
    rg, ro = g.rotate(cg, 5), o.rotate(co, 5)
    _eq(rg, ro)
    # one hybrid key switch at ring 2^16 with a dense ternary secret: the
    # ModDown rounding term dominates; its max over 2^15 slots is heavy-tailed
    # over key draws (2^-15 .. 2^-18 for key seeds 1..3, both PRNGs of
    # DESIGN.md §3.4); precision bar 14 bits
    err = np.max(np.abs(g.decrypt(rg) - np.roll(x, -5)))
    assert -np.log2(err) > 14.0, err


@pytest.mark.parametrize("which", ["small", "medium"])
def test_prefill_bit_exact_and_matches_reference(which):
    # kv_attention.cpp:245-376 through the C ABI (sf_prefill_scores / _attend
    # around the exact softmax hook) vs the oracle restatement on CKKS
    import paper_2602_11470_b200 as sf
    from oracle import protocols as P
    from oracle.layout import make_interleaved
    for c in cases(which, "prefill"):
        N, L, d, H, n0 = c["N"], c["L"], c["d"], c["H"], c["n0"]
        g, o = _pair(N, L, alpha=3)
        W = [np.array(c[k]).reshape(d, d) for k in ("Wq", "Wk", "Wv")]
        ocfg = P.AttentionConfig(N, d, H, n0, max(n0, 16))
        gcfg = sf.AttentionConfig(N, d, H, n0, max(n0, 16))
        xo = [o.encrypt(np.array(s), L, make_interleaved(d, N, 0, H), seed=50 + i) for i, s in enumerate(c["x_prompt"])]
        xg = [g.encrypt(np.array(s), L, make_interleaved(d, N, 0, H), seed=50 + i) for i, s in enumerate(c["x_prompt"])]
        att_o, cache_o = P.prefill(o, xo, W[0], W[1], W[2], ocfg, P.exact_softmax_prefill_maps)
        att_g, cache_g = sf.prefill(g, xg, W[0], W[1], W[2], gcfg, sf.exact_softmax_prefill_maps)
        assert cache_g.n_prime == n0
        for a, b in zip(cache_g.k_cts, cache_o.k_cts):
            _eq(a, b)
        for ga, gb in zip(cache_g.v_cts, cache_o.v_cts):
            for a, b in zip(ga, gb):
                _eq(a, b)
        assert len(att_g) == len(c["attention"])
        for a, b, want in zip(att_g, att_o, c["attention"]):
            _eq(a, b)
            ws = np.array(want["slots"])  # relative to the output's magnitude (|slots| ~ 25)
            assert np.max(np.abs(g.decrypt(a) - ws)) < 1e-6 * max(1.0, np.max(np.abs(ws)))
            lw = layout_from(want["layout"])
            assert a.level == want["level"] and (a.layout.kind, a.layout.d, a.layout.t, a.layout.offset,
                                                  a.layout.heads, a.layout.deferred_mask) == (
                lw.kind, lw.d, lw.t, lw.offset, lw.heads, lw.deferred_mask)
        assert counts_dict(g.ledger.totals()) == c["counts"] == counts_dict(o.ledger.totals())
