"""The fused peer-memory exchange (csrc/p2p.cu) with TWO ranks: two processes
share the one GPU of this run (CUDA IPC works between processes on the same
device), exchange their symmetric-buffer handles over gloo, and run the
sharded VMM / multi-VMM / QK^T / Score*V -- eagerly and replayed from a
captured CUDA graph, several exchanges in a row so both data slots, the
flags and the acknowledgements cycle. Every result must equal the
single-device operator word for word (each rank computes the reference
itself). On a multi-GPU node the same code runs one rank per GPU over NVLink."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2602_11470_b200 as sf
        from paper_2602_11470_b200 import shard
        N, L, d, H, n = 2048, 6, 128, 4, 40
        rng = np.random.default_rng(5)
        be = sf.Backend(N, L, alpha=2, seed=3)
        W = rng.normal(size=(256, 128)) / 16
        xs = np.zeros(N)
        xs[np.arange(256) * 8] = rng.normal(size=256)
        x = be.encrypt(xs, L, sf.make_interleaved(256, N, 0), seed=5)
        plan = sf.VmmPlan(be, W, 256, 128, L, 0, 3, True)
        plans = [plan, sf.VmmPlan(be, rng.normal(size=(256, 128)) / 16, 256, 128, L, 0, 3, True)]
        cfg = sf.AttentionConfig(N, d, H, 0, 64)
        cache = sf.KVCache(be, cfg)
        for u in range(n):
            vs = np.full(N, 0.25)
            vs[np.arange(d) * cfg.t + u % cfg.t] = rng.normal(size=d)
            vly = sf.make_interleaved(d, N, u % cfg.t, H).with_(deferred_mask=True)
            cache = sf.v_append(be, cache, sf.make_v_pieces(be, cache, be.encrypt(vs, L - 1, vly, seed=100 + u), u))
            ks = np.zeros(N)
            ks[np.arange(d) * cfg.t + u % cfg.t] = rng.normal(size=d)
            cache = sf.k_append(be, cache, be.encrypt(ks, L - 2, sf.make_interleaved(d, N, u % cfg.t, H),
                                                     seed=200 + u))
        qs = np.zeros(N)
        qs[np.arange(d) * cfg.t] = rng.normal(size=d)
        qv = be.encrypt(qs, L - 2, sf.make_interleaved(d, N, 0, H), seed=7)
        n_maps = len(sf.qk_dot(be, qv, cache))
        probs = [be.encrypt(np.full(N, 1.0 / n), L - 2, seed=50 + i) for i in range(n_maps)]
        want = [sf.vmm_interleaved(be, x, None, plan=plan)] + sf.vmm_interleaved_multi(be, x, plans) + \
            sf.qk_dot(be, qv, cache) + [sf.softmax_times_v(be, probs, cache)]
        sh = shard.PeerSharded(be, cap_words=1 << 17)

        def step():
            return [sh.vmm(x, plan)] + sh.vmm_multi(x, plans) + sh.qk_dot(qv, cache) + \
                [sh.softmax_times_v(probs, cache)]

        ok = []
        for _ in range(2):  # eager, twice (both slots)
            ok.append(all(np.array_equal(a.data(), b.data()) for a, b in zip(step(), want)))
        graph, outs = be.capture(step)
        for _ in range(3):  # graph replays: the device-side epochs keep advancing
            graph.launch()
            be.synchronize()
            ok.append(all(np.array_equal(a.data(), b.data()) for a, b in zip(outs, want)))
        sh.close()
        dist.destroy_process_group()
        q.put((rank, ok))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


@pytest.mark.timeout(600)
def test_peer_exchange_two_ranks_one_gpu():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(2):
            r, v = q.get(timeout=540)
            res[r] = v
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(2):
        assert isinstance(res.get(r), list), res
        assert all(res[r]), res
