"""GPU check of the product's sharded entry points on one device: the partials
of every rank of a world of W, summed with sf_sum_partials and finished, must
give the single-GPU ciphertexts word for word, and the per-rank ledgers must
add up to the reference's counts (replicated work is charged on rank 0)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 3, 8])
def test_sharded_vmm_emulated(world):
    import paper_2602_11470_b200 as sf
    from paper_2602_11470_b200 import shard
    N, L = 2048, 5
    rng = np.random.default_rng(world)
    W = rng.normal(size=(256, 128)) / 16
    xs = np.zeros(N)
    xs[np.arange(256) * 8] = rng.normal(size=256)
    be = sf.Backend(N, L, alpha=2)
    x = be.encrypt(xs, L, sf.make_interleaved(256, N, 0), seed=5)
    plan = sf.VmmPlan(be, W, 256, 128, L, 0, 3, True)
    full = sf.vmm_interleaved(be, x, None, plan=plan)
    want = be.ledger.totals()
    be.ledger.reset()
    parts = [shard.vmm_partial(be, x, plan, r, world) for r in range(world)]
    y = shard.vmm_finish(be, shard.sum_partials(be, parts), plan)
    assert np.array_equal(y.data(), full.data())
    assert be.ledger.totals() == want
    assert y.layout == full.layout


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_sharded_vmm_multi_emulated(world):
    """Q/K/V-style multi-VMM of one input: shared ladder + babies, per-rank giant groups."""
    import paper_2602_11470_b200 as sf
    from paper_2602_11470_b200 import shard
    N, L = 2048, 5
    rng = np.random.default_rng(40 + world)
    xs = np.zeros(N)
    xs[np.arange(256) * 8] = rng.normal(size=256)
    be = sf.Backend(N, L, alpha=2)
    x = be.encrypt(xs, L, sf.make_interleaved(256, N, 0), seed=5)
    plans = [sf.VmmPlan(be, rng.normal(size=(256, 128)) / 16, 256, 128, L, 0, 3, True) for _ in range(3)]
    be.ledger.reset()
    full = sf.vmm_interleaved_multi(be, x, plans)
    want = be.ledger.totals()
    be.ledger.reset()
    parts = [shard.vmm_multi_partial(be, x, plans, r, world) for r in range(world)]
    accs = [shard.sum_partials(be, [parts[r][i] for r in range(world)]) for i in range(3)]
    ys = shard.vmm_multi_finish(be, accs, plans)
    for y, f in zip(ys, full):
        assert np.array_equal(y.data(), f.data())
        assert y.layout == f.layout
    assert be.ledger.totals() == want


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_attention_emulated(world):
    import paper_2602_11470_b200 as sf
    from paper_2602_11470_b200 import shard
    N, L, d, H, n = 2048, 6, 128, 4, 40
    cfg = sf.AttentionConfig(N, d, H, 0, 64)
    be = sf.Backend(N, L, alpha=2)
    rng = np.random.default_rng(11)
    t = cfg.t
    cache = sf.KVCache(be, cfg)
    for u in range(n):
        vs = np.full(N, 0.25)
        vs[np.arange(d) * t + u % t] = rng.normal(size=d)
        vly = sf.make_interleaved(d, N, u % t, H).with_(deferred_mask=True)
        cache = sf.v_append(be, cache, sf.make_v_pieces(be, cache, be.encrypt(vs, L - 1, vly, seed=100 + u), u))
        ks = np.zeros(N)
        ks[np.arange(d) * t + u % t] = rng.normal(size=d)
        cache = sf.k_append(be, cache, be.encrypt(ks, L - 2, sf.make_interleaved(d, N, u % t, H), seed=200 + u))
    qs = np.zeros(N)
    qs[np.arange(d) * t] = rng.normal(size=d)
    q = be.encrypt(qs, L - 2, sf.make_interleaved(d, N, 0, H), seed=7)
    be.ledger.reset()
    maps_full = sf.qk_dot(be, q, cache)
    want_qk = be.ledger.totals()
    be.ledger.reset()
    parts = [shard.qk_dot_partial(be, q, cache, r, world) for r in range(world)]
    maps = [shard.sum_partials(be, [parts[r][m] for r in range(world)]) for m in range(len(maps_full))]
    for a, b in zip(maps, maps_full):
        assert np.array_equal(a.data(), b.data())
    assert be.ledger.totals() == want_qk
    probs = [be.encrypt(np.full(N, 1.0 / n), L - 2, seed=50 + i) for i in range(len(maps_full))]
    be.ledger.reset()
    full = sf.softmax_times_v(be, probs, cache)
    want_sv = be.ledger.totals()
    be.ledger.reset()
    sp = [shard.softmax_times_v_partial(be, probs, cache, r, world) for r in range(world)]
    out = shard.softmax_times_v_finish(be, sp, cache)
    assert np.array_equal(out.data(), full.data())
    assert be.ledger.totals() == want_sv
