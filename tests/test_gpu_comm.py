"""GPU check of the library-stream sharded operators (csrc/comm.cpp) in a
world of one: NCCL's all-gather runs on the context stream, the exchanged
partials are mod-added and finished; results must equal the unsharded
operators word for word, eagerly and replayed from a captured CUDA graph
(the sharded step has no host synchronisation once its metadata is cached)."""
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def world1():
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    yield dist
    dist.destroy_process_group()


def _cache(sf, be, cfg, n, L, rng):
    N, d, t, H = cfg.N, cfg.d, cfg.t, cfg.H
    cache = sf.KVCache(be, cfg)
    for u in range(n):
        vs = np.full(N, 0.25)
        vs[np.arange(d) * t + u % t] = rng.normal(size=d)
        vly = sf.make_interleaved(d, N, u % t, H).with_(deferred_mask=True)
        cache = sf.v_append(be, cache, sf.make_v_pieces(be, cache, be.encrypt(vs, L - 1, vly, seed=100 + u), u))
        ks = np.zeros(N)
        ks[np.arange(d) * t + u % t] = rng.normal(size=d)
        cache = sf.k_append(be, cache, be.encrypt(ks, L - 2, sf.make_interleaved(d, N, u % t, H), seed=200 + u))
    return cache


@pytest.mark.parametrize("kind", ["nccl", "peer"])
def test_stream_sharded_ops_world1(world1, kind):
    """kind "nccl": NCCL all-gather on the library stream; "peer": the fused
    peer-memory exchange (csrc/p2p.cu; with one rank the peer is itself)."""
    import paper_2602_11470_b200 as sf
    from paper_2602_11470_b200 import shard
    N, L, d, H, n = 2048, 6, 128, 4, 40
    rng = np.random.default_rng(5)
    be = sf.Backend(N, L, alpha=2)
    sh = shard.StreamSharded(be) if kind == "nccl" else shard.PeerSharded(be, cap_words=1 << 17)
    try:
        # VMM
        W = rng.normal(size=(256, 128)) / 16
        xs = np.zeros(N)
        xs[np.arange(256) * 8] = rng.normal(size=256)
        x = be.encrypt(xs, L, sf.make_interleaved(256, N, 0), seed=5)
        plan = sf.VmmPlan(be, W, 256, 128, L, 0, 3, True)
        full = sf.vmm_interleaved(be, x, None, plan=plan)
        y = sh.vmm(x, plan)
        assert np.array_equal(y.data(), full.data())
        assert y.layout == full.layout
        plans = [plan, sf.VmmPlan(be, rng.normal(size=(256, 128)) / 16, 256, 128, L, 0, 3, True)]
        for a, b in zip(sh.vmm_multi(x, plans), sf.vmm_interleaved_multi(be, x, plans)):
            assert np.array_equal(a.data(), b.data())
        # attention
        cfg = sf.AttentionConfig(N, d, H, 0, 64)
        cache = _cache(sf, be, cfg, n, L, rng)
        qs = np.zeros(N)
        qs[np.arange(d) * cfg.t] = rng.normal(size=d)
        q = be.encrypt(qs, L - 2, sf.make_interleaved(d, N, 0, H), seed=7)
        maps_full = sf.qk_dot(be, q, cache)
        maps = sh.qk_dot(q, cache)
        assert len(maps) == len(maps_full)
        for a, b in zip(maps, maps_full):
            assert np.array_equal(a.data(), b.data())
        probs = [be.encrypt(np.full(N, 1.0 / n), L - 2, seed=50 + i) for i in range(len(maps_full))]
        att_full = sf.softmax_times_v(be, probs, cache)
        att = sh.softmax_times_v(probs, cache)
        assert np.array_equal(att.data(), att_full.data())

        # the same three operators captured into one graph and replayed on new inputs
        def step():
            return [sh.vmm(x, plan)] + sh.qk_dot(q, cache) + [sh.softmax_times_v(probs, cache)] + \
                sh.vmm_multi(x, plans)

        graph, outs = be.capture(step)
        xs2 = np.zeros(N)
        xs2[np.arange(256) * 8] = rng.normal(size=256)
        x2 = be.encrypt(xs2, L, sf.make_interleaved(256, N, 0), seed=6)
        be.refill(x, x2.data())
        graph.launch()
        be.synchronize()
        assert np.array_equal(outs[0].data(), sf.vmm_interleaved(be, x2, None, plan=plan).data())
        nm = len(maps_full)
        for a, b in zip(outs[1:1 + nm], maps_full):
            assert np.array_equal(a.data(), b.data())
        assert np.array_equal(outs[1 + nm].data(), att_full.data())
        for a, b in zip(outs[2 + nm:], sf.vmm_interleaved_multi(be, x2, plans)):
            assert np.array_equal(a.data(), b.data())
    finally:
        sh.close()
