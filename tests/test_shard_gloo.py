"""Multi-process (world_size 2, gloo, CPU) check of the sharded hot path.

Each rank computes its partial VMM / QK^T / Score*V with the oracle restatement
of the sharding rules (oracle/shard_ref.py, mirroring csrc/protocols.cpp), the
partial ciphertext words are all-gathered over gloo, summed mod q and
finished; the result must equal the single-process ciphertexts word for word.
The same ownership rules are imported from the product (paper_2602_11470_b200.shard).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(be, cts):
    """all-gather of oracle ciphertexts: words + (level, scale, zero) metadata."""
    mine = [(c.data(), c.level, c.scale, c.is_zero) for c in cts]
    got = [None] * dist.get_world_size()
    dist.all_gather_object(got, mine)
    return [[be.import_ct(w.reshape(-1), lvl, sc, zero=z) for (w, lvl, sc, z) in r] for r in got]


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import protocols as P
        from oracle import shard_ref as S
        from oracle.ckks import CkksOracle
        from oracle.layout import make_interleaved

        res = {}
        # --- VMM: 64 -> 32 at 256 slots, BSGS (k = 8: babies 3, giants 3)
        N, L = 256, 5
        rng = np.random.default_rng(3)
        W = rng.normal(size=(64, 32)) / 8
        xs = np.zeros(N)
        xs[np.arange(64) * 4] = rng.normal(size=64)
        be = CkksOracle(N, L, alpha=2)
        x = be.encrypt(xs, L, make_interleaved(64, N, 0), seed=9)
        full = P.vmm_interleaved(be, x, W, bsgs=True, out_offset=3)
        part = S.vmm_partial(be, x, W, True, 3, rank, world)
        parts = [r[0] for r in _exchange(be, [part])]
        y = S.vmm_finish(be, S.sum_partials(be, parts), W, 0, 3)
        res["vmm"] = bool(np.array_equal(y.data(), full.data()))
        # --- attention over a 13-token cache at 64 slots, d 16, 2 heads
        N, L, d, H, n = 64, 6, 16, 2, 13
        cfg = P.AttentionConfig(N, d, H, 0, 16)
        be = CkksOracle(N, L, alpha=2)
        K, V = rng.normal(size=(n, d)), rng.normal(size=(n, d))
        cache = P.KVCache()
        for u in range(n):
            vly = make_interleaved(d, N, u % cfg.t, H).with_(deferred_mask=True)
            vs = np.full(N, 0.5)
            vs[np.arange(d) * cfg.t + u % cfg.t] = V[u]
            cache = P.v_append(be, cache, P.make_v_pieces(be, be.encrypt(vs, L - 1, vly, seed=100 + u), cfg, u), cfg)
            ks = np.zeros(N)
            ks[np.arange(d) * cfg.t + u % cfg.t] = K[u]
            cache = P.k_append(be, cache, be.encrypt(ks, L - 2, make_interleaved(d, N, u % cfg.t, H), seed=200 + u),
                               cfg)
        qs = np.zeros(N)
        qs[np.arange(d) * cfg.t] = rng.normal(size=d)
        q = be.encrypt(qs, L - 2, make_interleaved(d, N, 0, H), seed=300)
        maps_full = P.qk_dot(be, q, cache, cfg)
        mp_ = S.qk_dot_partial(be, q, cache, cfg, rank, world)
        got = _exchange(be, mp_)
        maps = [S.sum_partials(be, [got[r][m] for r in range(world)]) for m in range(len(mp_))]
        res["qk"] = all(np.array_equal(a.data(), b.data()) for a, b in zip(maps, maps_full))
        probs = [be.encrypt(np.full(N, 1.0 / n), L - 2, seed=400 + i) for i in range(len(maps_full))]
        sv_full = P.softmax_times_v(be, probs, cache, cfg)
        sp = S.softmax_times_v_partial(be, probs, cache, cfg, rank, world)
        parts = [r[0] for r in _exchange(be, [sp])]
        sv = S.softmax_times_v_finish(be, parts, cfg)
        res["sv"] = bool(np.array_equal(sv.data(), sv_full.data()))
        # --- ownership rules of the product partition the work exactly
        from paper_2602_11470_b200 import shard
        res["own"] = all(
            sorted(sum((f(m, r, world) for r in range(world)), [])) == list(range(m))
            for f in (shard.own_giants, shard.own_keys) for m in (1, 7, 45, 256)) and all(
            sorted(sum((shard.own_variants(nv, lo, dh, r, world) for r in range(world)), [])) == list(range(lo, dh))
            for nv, lo, dh in ((255, -127, 128), (255, -3, 128), (127, -63, 64), (8, 0, 8), (3, -1, 2)))
        out.put((rank, res))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        out.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


def test_sharded_hot_path_bit_exact_world2_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert "error" not in results[r], results[r]
        assert results[r] == {"vmm": True, "qk": True, "sv": True, "own": True}, results[r]
