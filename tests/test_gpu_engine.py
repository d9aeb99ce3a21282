"""The reference's engine contract (tests/test_engine.cpp) on the GPU backend:
level rules, ledger counting and phases, rotation semantics, layout
propagation, error types. Values are compared at CKKS precision instead of
exactly (the reference backend is a cleartext simulator)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-6


def test_add_sub_add_plain_values_levels_counts():  # test_engine.cpp:19-38
    import paper_2602_11470_b200 as sf
    be = sf.Backend(8, 5)
    a = be.encrypt(np.full(8, 1.5), 2)
    b = be.encrypt(np.full(8, 2.0), 4)
    s = be.add(a, b)
    assert s.level == 2 and np.allclose(be.decrypt(s), 3.5, atol=TOL)
    d = be.sub(b, a)
    assert d.level == 2 and np.allclose(be.decrypt(d), 0.5, atol=TOL)
    p = be.add_plain(b, 1.0)
    assert p.level == 4 and np.allclose(be.decrypt(p), 3.0, atol=TOL)
    t = be.ledger.totals()
    assert t.additions == 3 and t.ct_ct_mults == 0


def test_rotate_semantics_group_law_and_counts():  # test_engine.cpp:64-94
    import paper_2602_11470_b200 as sf
    be = sf.Backend(4, 3)
    a = be.encrypt(np.array([1.0, 2, 3, 4]), 3)
    assert np.allclose(be.decrypt(be.rotate(a, 1)), [2, 3, 4, 1], atol=TOL)
    assert np.allclose(be.decrypt(be.rotate(a, -1)), [4, 1, 2, 3], atol=TOL)
    assert np.allclose(be.decrypt(be.rotate(a, 0)), [1, 2, 3, 4], atol=TOL)
    assert np.allclose(be.decrypt(be.rotate(a, 4)), [1, 2, 3, 4], atol=TOL)
    assert be.ledger.totals().rotations == 2
    lhs = be.rotate(be.rotate(a, 3), 2)
    assert np.allclose(be.decrypt(lhs), be.decrypt(be.rotate(a, 5)), atol=TOL) and lhs.level == 3
    be2 = sf.Backend(8, 2)
    z = be2.zeros()
    be2.rotate(z, 1, hoisted=True)
    be2.rotate(z, 2, hoisted=True)
    be2.rotate(z, 3)
    t = be2.ledger.totals()
    assert (t.rotations, t.hoisted_rotations) == (3, 2)


def test_bootstrap_and_level_drop():  # test_engine.cpp:96-112
    import paper_2602_11470_b200 as sf
    be = sf.Backend(8, 6)
    a = be.encrypt(np.full(8, 7.0), 1)
    up = be.bootstrap(a, 5)
    assert up.level == 5 and np.allclose(be.decrypt(up), 7.0, atol=TOL)
    assert be.ledger.totals().bootstraps == 1
    with pytest.raises(sf.InvalidTarget):
        be.bootstrap(a, 0)
    with pytest.raises(sf.InvalidTarget):
        be.bootstrap(a, 7)
    down = be.level_drop(up, 2)
    assert down.level == 2
    with pytest.raises(sf.InvalidTarget):
        be.level_drop(down, 3)
    with pytest.raises(sf.InvalidTarget):
        be.level_drop(down, -1)
    assert be.ledger.totals().bootstraps == 1


def test_exact_transform_is_free_and_level_neutral():  # test_engine.cpp:114-121
    import paper_2602_11470_b200 as sf
    be = sf.Backend(8, 3)
    x = np.linspace(-2.0, 5.0, 8)
    a = be.encrypt(x, 1)
    y = be.exact_transform(a, np.exp)
    assert y.level == 1 and np.allclose(be.decrypt(y), np.exp(x), rtol=1e-6, atol=1e-6)
    assert be.ledger.totals() == sf.OpCounts()


def test_ledger_phases_nesting_conservation():  # test_engine.cpp:131-166
    import paper_2602_11470_b200 as sf
    be = sf.Backend(8, 9)
    a = be.encrypt(np.ones(8))
    be.add(a, a)
    with be.phase("alpha"):
        be.mul(a, a)
        be.rotate(a, 1)
        with be.phase("beta"):
            be.rotate(a, 2, hoisted=True)
        be.mul_plain(a, 2.0)
    be.add(a, a)
    L = be.ledger
    al, bt, dflt = L.phase_totals("alpha"), L.phase_totals("beta"), L.phase_totals("(unphased)")
    assert (al.ct_ct_mults, al.ct_pt_mults, al.rotations) == (1, 1, 1)
    assert (bt.rotations, bt.hoisted_rotations) == (1, 1)
    assert dflt.additions == 2
    tot = L.totals()
    for f in ("rotations", "hoisted_rotations", "ct_pt_mults", "ct_ct_mults", "additions"):
        assert getattr(tot, f) == getattr(al, f) + getattr(bt, f) + getattr(dflt, f)
    L.reset()
    assert L.totals() == sf.OpCounts()


def test_layout_propagation():  # test_engine.cpp:168-181
    import paper_2602_11470_b200 as sf
    be = sf.Backend(8, 4)
    ly = sf.make_interleaved(4, 8, 1)
    a = be.encrypt(np.ones(8), 4, ly)
    b = be.encrypt(np.full(8, 2.0), 4, ly)
    assert be.add(a, b).layout == ly
    assert be.mul(a, b).layout == ly
    assert be.mul_plain(a, 2.0).layout == ly
    assert be.bootstrap(be.level_drop(a, 1), 3).layout == ly
    assert be.rotate(a, 1).layout is None
    c = be.encrypt(np.full(8, 3.0), 4, sf.Layout("replicated", 4, 2, 0, 1, False))
    assert be.add(a, c).layout is None


def test_full_ring_fused_and_chained_ops_track_oracle():
    # ring 2^16 exercises the fused ModUp / ModDown / rescale kernels on every
    # op class; the chain must stay word-identical to the CPU oracle
    import paper_2602_11470_b200 as sf
    from oracle.ckks import CkksOracle
    g, o = sf.Backend(32768, 5, alpha=2), CkksOracle(32768, 5, alpha=2)
    rng = np.random.default_rng(1)
    x, y, p = rng.normal(size=32768), rng.normal(size=32768), rng.normal(size=32768)
    cg, co = g.encrypt(x, 5, seed=1), o.encrypt(x, 5, seed=1)
    dg, do = g.encrypt(y, 4, seed=2), o.encrypt(y, 4, seed=2)
    rg = g.rotate(g.mul(g.mul_plain(cg, p), dg), 7)
    ro = o.rotate(o.mul(o.mul_plain(co, p), do), 7)
    assert np.array_equal(rg.data(), ro.data())
    want = np.roll(x * p * y, -7)
    assert np.max(np.abs(g.decrypt(rg) - want)) < 1e-4


def test_graph_capture_replays_the_step_bit_exactly():
    # a captured step (VMM + attention-style ops on a 2^13 ring) replayed with
    # refilled inputs must reproduce the eager ciphertexts word for word
    import paper_2602_11470_b200 as sf
    from oracle.layout import make_interleaved
    N, L = 4096, 4
    be = sf.Backend(N, L, alpha=2)
    rng = np.random.default_rng(5)
    W = rng.normal(size=(64, 64)) / 8
    ly = make_interleaved(64, N, 0)

    def enc(seed):
        s = np.zeros(N)
        s[np.arange(64) * ly.t] = np.random.default_rng(seed).normal(size=64)
        return be.encrypt(s, L, ly, seed=seed)

    plan = sf.VmmPlan(be, W, 64, 64, L, 0, 0, True)  # offline encode: outside any capture

    def step(x, y):
        v = sf.vmm_interleaved(be, x, None, mask_output=True, plan=plan)
        m = be.mul(v, be.level_drop(y, v.level))
        return [v, be.rotate(m, 5)]

    xa, ya, xb, yb = enc(1), enc(2), enc(3), enc(4)
    want_a = [c.data() for c in step(xa, ya)]
    want_b = [c.data() for c in step(xb, yb)]
    x_slot, y_slot = be.import_ct(xa.data(), xa.level, xa.scale, xa.layout), be.import_ct(ya.data(), ya.level,
                                                                                             ya.scale, ya.layout)
    l0 = be.kernel_launches()
    graph, outs = be.capture(step, x_slot, y_slot)
    assert be.kernel_launches() - l0 == graph.kernel_launches > 0
    for words_x, words_y, want in ((xb.data(), yb.data(), want_b), (xa.data(), ya.data(), want_a)):
        be.refill(x_slot, words_x)
        be.refill(y_slot, words_y)
        graph.launch()
        got = [c.data() for c in outs]
        assert all(np.array_equal(g_, w_) for g_, w_ in zip(got, want))


def test_staged_uploads_inside_a_captured_step():
    # sf_ct_stage: the inputs' uploads as a parallel graph branch re-reading
    # pinned host words on every replay, each joined right before its first use;
    # replays with new host words reproduce the eager ciphertexts word for word
    import torch
    import paper_2602_11470_b200 as sf
    from oracle.layout import make_interleaved
    N, L = 4096, 4
    be = sf.Backend(N, L, alpha=2)
    W = np.random.default_rng(6).normal(size=(64, 64)) / 8
    ly = make_interleaved(64, N, 0)

    def enc(seed):
        s = np.zeros(N)
        s[np.arange(64) * ly.t] = np.random.default_rng(seed).normal(size=64)
        return be.encrypt(s, L, ly, seed=seed)

    plan = sf.VmmPlan(be, W, 64, 64, L, 0, 0, True)

    def step(x, y, staged=None, out=None):
        if staged:
            be.stage(x, staged[0], 0)
            be.stage(y, staged[1], 1)
            be.stage_wait(0)
        v = sf.vmm_interleaved(be, x, None, mask_output=True, plan=plan)
        if out is not None:
            be.stage_out(v, out, 2)  # read-back overlapping the rest of the step
        if staged:
            be.stage_wait(1)
        m = be.mul(v, be.level_drop(y, v.level))
        if out is not None:
            be.stage_wait(2)
        return [v, be.rotate(m, 5)]

    xa, ya, xb, yb = enc(1), enc(2), enc(3), enc(4)
    want_a = [c.data() for c in step(xa, ya)]
    want_b = [c.data() for c in step(xb, yb)]
    x_slot = be.import_ct(xa.data(), xa.level, xa.scale, xa.layout)
    y_slot = be.import_ct(ya.data(), ya.level, ya.scale, ya.layout)
    dt = torch.uint64 if hasattr(torch, "uint64") else torch.int64
    pin = [torch.empty(xa.data().shape, dtype=dt, pin_memory=True).numpy().view(np.uint64) for _ in range(2)]
    # eager staging first (overlap on the side stream, joined before use)
    pin[0][...], pin[1][...] = xb.data(), yb.data()
    got = [c.data() for c in step(x_slot, y_slot, staged=pin)]
    assert all(np.array_equal(g_, w_) for g_, w_ in zip(got, want_b))
    out = torch.empty(want_a[0].shape, dtype=dt, pin_memory=True).numpy().view(np.uint64)
    graph, outs = be.capture(step, x_slot, y_slot, staged=pin, out=out)
    for wx, wy, want in ((xa.data(), ya.data(), want_a), (xb.data(), yb.data(), want_b)):
        pin[0][...], pin[1][...] = wx, wy  # the graph re-reads the pinned words on replay
        graph.launch()
        be.synchronize()
        assert np.array_equal(out, want[0])  # staged read-back (sf_ct_stage_out)
        got = [c.data() for c in outs]
        assert all(np.array_equal(g_, w_) for g_, w_ in zip(got, want))
    with pytest.raises(TypeError):
        be.stage(x_slot, xa.data().astype(np.int64), 0)


def test_capture_cold_caches_and_graph_memory_is_released():
    """(1) Capturing a step whose lazy tables / keys are still cold: the capture
    is retried after one eager warm-up run and replays bit-exactly. (2) Graph-
    owned step outputs are freed when the graph and its handles are gone:
    repeated capture / launch / destroy cycles do not grow device memory."""
    import gc
    import paper_2602_11470_b200 as sf
    from oracle.layout import make_interleaved
    N, L = 4096, 4
    be = sf.Backend(N, L, alpha=2, seed=11)
    ly = make_interleaved(64, N, 0)
    s = np.zeros(N)
    s[np.arange(64) * ly.t] = np.random.default_rng(0).normal(size=64)
    x = be.encrypt(s, L, ly, seed=1)
    plan = sf.VmmPlan(be, np.random.default_rng(1).normal(size=(64, 64)) / 8, 64, 64, L, 0, 0, True)

    def step():
        return [be.rotate(sf.vmm_interleaved(be, x, None, mask_output=True, plan=plan), 7)]

    graph, outs = be.capture(step)  # cold: rotation key for 7, plan plaintexts, conversion tables
    graph.launch()
    want = step()[0].data()
    assert np.array_equal(outs[0].data(), want)
    del graph, outs
    gc.collect()
    # graph memory is reserved in 64 MiB chunks: make every capture's outputs
    # ~32 MiB so six leaked generations would be visible
    y = sf.vmm_interleaved(be, x, None, mask_output=True, plan=plan)

    def big_step():
        return [be.add(y, y) for _ in range(64)]

    big_step()
    g_base = be.mem_stats()[0]
    for i in range(6):
        g, o = be.capture(big_step)
        g.launch()
        assert np.array_equal(o[0].data(), o[63].data())
        del g, o
        gc.collect()
    assert be.mem_stats()[0] <= g_base + (64 << 20)  # released with the graphs and their handles


def test_vmm_multi_equals_separate_calls_and_ledger():
    # Q/K/V-style: three plans on one input (different output offsets) must give
    # the separate calls' ciphertexts word for word and the same ledger totals
    import paper_2602_11470_b200 as sf
    from oracle.layout import make_interleaved
    N, L = 4096, 4
    rng = np.random.default_rng(11)
    Ws = [rng.normal(size=(128, 128)) / 12 for _ in range(3)]
    s = np.zeros(N)
    ly = make_interleaved(128, N, 0)
    s[np.arange(128) * ly.t] = rng.normal(size=128)
    res = []
    for multi in (False, True):
        be = sf.Backend(N, L, alpha=2, seed=3)
        x = be.encrypt(s, L, ly, seed=8)
        plans = [sf.VmmPlan(be, W, 128, 128, L, 0, off, True) for W, off in zip(Ws, (0, 3, 5))]
        be.ledger.reset()
        if multi:
            ys = sf.vmm_interleaved_multi(be, x, plans, mask_output=True)
        else:
            ys = [sf.vmm_interleaved(be, x, None, mask_output=True, plan=p) for p in plans]
        res.append(([y.data() for y in ys], be.ledger.totals().asdict(), [y.layout for y in ys]))
    (d0, l0, y0), (d1, l1, y1) = res
    assert all(np.array_equal(a, b) for a, b in zip(d0, d1))
    assert l0 == l1 and y0 == y1


def test_wire_formats_round_trip(tmp_path):
    # reference weight files -> plan, encoded-plan cache, ciphertext wire format
    import paper_2602_11470_b200 as sf
    from oracle.layout import make_interleaved
    N, L = 4096, 3
    be = sf.Backend(N, L, alpha=2)
    rng = np.random.default_rng(2)
    W = rng.normal(size=(100, 60)) / 10
    sf.save_weight(str(tmp_path), "w_test", W)
    assert np.array_equal(np.fromfile(tmp_path / "w_test.bin").reshape(100, 60), W)
    ly = make_interleaved(128, N, 0)
    s = np.zeros(N)
    s[np.arange(100) * ly.t] = rng.normal(size=100)
    x = be.encrypt(s, L, ly, seed=4)
    p_mem = sf.VmmPlan(be, W, 100, 60, L, 0, 0, True)
    p_file = sf.vmm_plan_from_file(be, str(tmp_path), "w_test", L)
    y0 = sf.vmm_interleaved(be, x, None, plan=p_mem, mask_output=True)
    y1 = sf.vmm_interleaved(be, x, None, plan=p_file, mask_output=True)
    assert np.array_equal(y0.data(), y1.data())
    p_mem.save(str(tmp_path / "plan.sfvp"))
    p_back = sf.vmm_plan_load(be, str(tmp_path / "plan.sfvp"))
    y2 = sf.vmm_interleaved(be, x, None, plan=p_back, mask_output=True)
    assert np.array_equal(y0.data(), y2.data())
    wire = be.serialize(y0)
    z = be.deserialize(wire)
    assert np.array_equal(z.data(), y0.data()) and z.level == y0.level and z.layout == y0.layout
    assert abs(z.scale - y0.scale) == 0.0
    zero = be.zeros(2)
    zz = be.deserialize(be.serialize(zero))
    assert zz.level == 2
    with pytest.raises(sf.ShapeMismatch):
        be.deserialize(wire[:-8])
    other = sf.Backend(N, L + 1, alpha=2)
    with pytest.raises(sf.ShapeMismatch):
        other.deserialize(wire)
    # same shape, different scale primes / different keys: rejected (full-chain + key-id fingerprint)
    with pytest.raises(sf.ShapeMismatch):
        sf.Backend(N, L, alpha=2, scale_bits=39).deserialize(wire)
    with pytest.raises(sf.ShapeMismatch):
        sf.Backend(N, L, alpha=2, seed=99).deserialize(wire)
    # plans are key-independent: a plan saved under one key seed loads under another
    p_other = sf.vmm_plan_load(sf.Backend(N, L, alpha=2, seed=99), str(tmp_path / "plan.sfvp"))
    assert p_other is not None
    # non-canonical residue (word >= q) in an otherwise valid buffer: rejected
    bad = bytearray(wire)
    bad[-8:] = (2**64 - 1).to_bytes(8, "little")
    with pytest.raises(sf.DomainViolation):
        be.deserialize(bytes(bad))


def test_prime_bits_clamped_to_60():
    """The lazy kernels need q < 2^60 (8 lazy Shoup products per u64 in the
    fused column stage); 61-bit primes are rejected up front."""
    import paper_2602_11470_b200 as sf
    with pytest.raises(sf.DomainViolation):
        sf.Backend(1024, 2, q0_bits=61)
    with pytest.raises(sf.DomainViolation):
        sf.Backend(1024, 2, special_bits=61)


@pytest.mark.parametrize("mask", [False, True])
def test_vmm_many_matches_separate_calls(mask):
    """vmm_interleaved_many (one plan, several independent inputs, every stage
    batched) == separate vmm_interleaved calls, word for word and in the ledger."""
    import paper_2602_11470_b200 as sf
    N, L = 2048, 4
    rng = np.random.default_rng(21)
    be = sf.Backend(N, L, alpha=2)
    W = rng.normal(size=(192, 160)) / 16
    ly = sf.make_interleaved(256, N, 0)
    plan = sf.VmmPlan(be, W, 192, 160, L, 0, 2, True)
    xs = []
    for i in range(5):
        v = np.zeros(N)
        v[np.arange(192) * ly.t] = rng.normal(size=192)
        xs.append(be.encrypt(v, L, ly, seed=30 + i))
    be.ledger.reset()
    want = [sf.vmm_interleaved(be, x, None, plan=plan, mask_output=mask) for x in xs]
    counts = be.ledger.totals()
    be.ledger.reset()
    got = sf.vmm_interleaved_many(be, xs, plan, mask_output=mask)
    assert be.ledger.totals() == counts
    for a, b in zip(got, want):
        assert np.array_equal(a.data(), b.data())
        assert a.layout == b.layout


def test_vmm_many_fallback_paths():
    """vmm_interleaved_many with a non-BSGS plan, and with a trivial-zero input
    among the inputs, takes the per-input path and still equals separate calls."""
    import paper_2602_11470_b200 as sf
    N, L = 2048, 4
    rng = np.random.default_rng(23)
    be = sf.Backend(N, L, alpha=2)
    W = rng.normal(size=(64, 96)) / 8
    ly = sf.make_interleaved(64, N, 0)
    plan = sf.VmmPlan(be, W, 64, 96, L, 0, 1, False)
    xs = []
    for i in range(3):
        v = np.zeros(N)
        v[np.arange(64) * ly.t] = rng.normal(size=64)
        xs.append(be.encrypt(v, L, ly, seed=60 + i))
    want = [sf.vmm_interleaved(be, x, None, plan=plan) for x in xs]
    got = sf.vmm_interleaved_many(be, xs, plan)
    for a, b in zip(got, want):
        assert np.array_equal(a.data(), b.data())
    bplan = sf.VmmPlan(be, W, 64, 96, L, 0, 1, True)
    z = be.with_layout(be.zeros(L), ly)
    got = sf.vmm_interleaved_many(be, [xs[0], z], bplan)
    assert np.array_equal(got[0].data(), sf.vmm_interleaved(be, xs[0], None, plan=bplan).data())
