"""Pins the numpy restatement of the reference (oracle/slot_sim.py +
oracle/protocols.py) against golden vectors emitted by the reference itself.
CPU only. Tolerances follow the reference tests: 1e-9 on values,
exact on counts, levels, layouts and on masked (exact-zero) slots."""
import numpy as np
import pytest

from golden_util import cases, counts_dict, layout_from
from oracle import protocols as P
from oracle.layout import Layout, make_interleaved
from oracle.slot_sim import SimBackend


@pytest.mark.parametrize("which", ["small", "medium"])
def test_vmm_cases_match_reference(which):
    cs = cases(which, "vmm")
    assert len(cs) >= (100 if which == "small" else 4)
    for c in cs:
        N, L = c["N"], c["L"]
        W = np.array(c["W"]).reshape(c["rows"], c["cols"])
        be = SimBackend(N, L)
        d_in = P.padded_dim(c["rows"])
        x = be.encrypt(np.array(c["x_slots"]), L, make_interleaved(d_in, N, c["tau_in"]))
        y = P.vmm_interleaved(be, x, W, bsgs=c["bsgs"], out_offset=c["tau_out"],
                              mask_output=c["mask_output"])
        want = np.array(c["y_slots"])
        assert np.max(np.abs(y.slots - want)) < 1e-9, c["N"]
        assert np.all(y.slots[want == 0.0] == 0.0) or not c["mask_output"]
        assert counts_dict(be.ledger.totals()) == c["counts"]
        assert y.level == c["level"]
        assert y.layout == layout_from(c["layout"])
        rot, ctpt, depth = P.predict_interleaved_cost(N, c["rows"], c["cols"], c["bsgs"], c["mask_output"])
        assert (rot, ctpt, depth) == (c["predicted"]["rotations"], c["predicted"]["ct_pt_mults"],
                                      c["predicted"]["depth"])
        assert c["counts"]["rotations"] == rot and c["counts"]["ct_pt_mults"] == ctpt
        assert L - y.level == depth


@pytest.mark.parametrize("which", ["small", "medium"])
def test_rope_cases_match_reference(which):
    for c in cases(which, "rope"):
        N, L = c["N"], c["L"]
        be = SimBackend(N, L)
        ly = make_interleaved(c["d"], N, c["offset"]).with_(deferred_mask=True)
        x = be.encrypt(np.array(c["x_slots"]), L, ly)
        p = P.rope_plaintexts(c["pos"], c["d_head"], ly, N)
        for k in range(3):
            assert np.max(np.abs(p[k] - np.array(c[f"p{k}"]))) < 1e-15
        y = P.fused_extract(be, x, "rope", dict(n=c["pos"], d_head=c["d_head"], s=ly.t))
        assert np.max(np.abs(y.slots - np.array(c["y_slots"]))) < 1e-9
        assert counts_dict(be.ledger.totals()) == c["counts"]
        assert y.level == c["level"] and y.layout == layout_from(c["layout"])


def replay_attention(be, c):
    """Rebuilds the golden attention case through the append protocol and one
    decode query, exactly as oracle/ref_golden.cpp:attn_case does."""
    N, L, d, H, np_ = c["N"], c["L"], c["d"], c["H"], c["n_prime"]
    cfg = P.AttentionConfig(N, d, H, 0, np_)
    P.validate_attention_config(cfg, N)
    t = cfg.t
    K = np.array(c["K"]).reshape(np_, d)
    V = np.array(c["V"]).reshape(np_, d)
    cache = P.KVCache()
    append_counts = []
    for u in range(np_):
        vly = make_interleaved(d, N, u % t, H).with_(deferred_mask=True)
        open_ = np.full(N, 7.5)
        open_[np.arange(d) * t + u % t] = V[u]
        v_open = be.encrypt(open_, L - 1, vly)
        c0 = be.ledger.totals()
        parts = P.make_v_pieces(be, v_open, cfg, u)
        cache = P.v_append(be, cache, parts, cfg)
        kly = make_interleaved(d, N, u % t, H)
        from oracle.layout import encode
        cache = P.k_append(be, cache, be.encrypt(encode(K[u], kly, N), L - 2, kly), cfg)
        append_counts.append(counts_dict(be.ledger.totals() - c0))
    be.ledger.reset()
    qly = make_interleaved(d, N, 0, H)
    from oracle.layout import encode
    qc = be.encrypt(encode(np.array(c["q"]), qly, N), L - 2, qly)
    with be.phase("QK^T"):
        maps = P.qk_dot(be, qc, cache, cfg)
    probs = P.exact_softmax_maps(be, maps, cfg, cache.n_prime)
    with be.phase("Score*V"):
        out = P.softmax_times_v(be, probs, cache, cfg)
    return dict(cfg=cfg, cache=cache, maps=maps, probs=probs, out=out, append_counts=append_counts)


@pytest.mark.parametrize("which", ["small", "medium"])
def test_attention_cases_match_reference(which):
    cs = cases(which, "attn")
    assert cs
    for c in cs:
        be = SimBackend(c["N"], c["L"])
        r = replay_attention(be, c)
        assert r["append_counts"] == [dict(x) for x in c["append_counts"]]
        for got, want in zip(r["cache"].k_cts, c["k_cts"]):
            assert np.array_equal(got.slots, np.array(want["slots"])) and got.level == want["level"]
        for g, grp in enumerate(c["v_cts"]):
            for i, want in enumerate(grp):
                got = r["cache"].v_cts[g][i]
                assert np.array_equal(got.slots, np.array(want["slots"])) and got.level == want["level"]
        for got, want in zip(r["maps"], c["maps"]):
            assert np.max(np.abs(got.slots - np.array(want))) < 1e-9
        assert r["maps"][0].level == c["map_level"]
        for got, want in zip(r["probs"], c["probs"]):
            assert np.max(np.abs(got.slots - np.array(want))) < 1e-12
        assert np.max(np.abs(r["out"].slots - np.array(c["out_slots"]))) < 1e-9
        assert r["out"].level == c["out_level"]
        assert r["out"].layout == layout_from(c["out_layout"])
        assert counts_dict(be.ledger.phase_totals("QK^T")) == c["qk_counts"]
        assert counts_dict(be.ledger.phase_totals("Score*V")) == c["sv_counts"]


def test_engine_rotation_golden():
    (c,) = cases("small", "engine_rotate")
    be = SimBackend(4, 3)
    a = be.encrypt(np.array(c["input"]), 3)
    for r in c["rotations"]:
        assert np.array_equal(be.rotate(a, r["r"]).slots, np.array(r["slots"]))
    assert be.ledger.totals().rotations == c["counted"]


def test_paper_scale_counts():
    # reference closed form (vmm.cpp:473-488) at the survey's appendix-A shapes
    assert P.predict_interleaved_cost(32768, 4096, 4096, True) == (50, 512, 1)
    assert P.predict_interleaved_cost(32768, 4096, 14336, True) == (93, 2048, 1)
    assert P.predict_interleaved_cost(32768, 14336, 4096, True) == (93, 2048, 1)
    assert P.predict_interleaved_cost(16384, 768, 768, True) == (22, 64, 1)
    for k, bg in {1: (1, 1), 2: (2, 1), 4: (2, 2), 5: (3, 2), 128: (12, 11), 512: (23, 23),
                  4096: (64, 64)}.items():
        assert P.bsgs_split(k) == bg


def replay_prefill(be, c):
    """oracle/ref_golden.cpp:prefill_case through the restated prefill."""
    N, L, d, H, n0 = c["N"], c["L"], c["d"], c["H"], c["n0"]
    cfg = P.AttentionConfig(N, d, H, n0, max(n0, 16))
    P.validate_attention_config(cfg, N)
    W = [np.array(c[k]).reshape(d, d) for k in ("Wq", "Wk", "Wv")]
    xs = [be.encrypt(np.array(s), L, make_interleaved(d, N, 0, H)) for s in c["x_prompt"]]
    att, cache = P.prefill(be, xs, W[0], W[1], W[2], cfg, P.exact_softmax_prefill_maps)
    return att, cache


@pytest.mark.parametrize("which", ["small", "medium"])
def test_prefill_cases_match_reference(which):
    cs = cases(which, "prefill")
    assert len(cs) >= (4 if which == "small" else 1)
    for c in cs:
        be = SimBackend(c["N"], c["L"])
        att, cache = replay_prefill(be, c)
        assert cache.n_prime == c["n_prime"]
        assert len(cache.k_cts) == len(c["k_cts"])
        for got, want in zip(cache.k_cts, c["k_cts"]):
            assert np.max(np.abs(got.slots - np.array(want["slots"]))) < 1e-9 and got.level == want["level"]
        assert [len(g) for g in cache.v_cts] == [len(g) for g in c["v_cts"]]
        for gg, gw in zip(cache.v_cts, c["v_cts"]):
            for got, want in zip(gg, gw):
                assert np.max(np.abs(got.slots - np.array(want["slots"]))) < 1e-9
        assert len(att) == len(c["attention"])
        for got, want in zip(att, c["attention"]):
            w = np.array(want["slots"])
            assert np.max(np.abs(got.slots - w)) < 1e-9
            assert np.all(got.slots[w == 0.0] == 0.0)
            assert got.level == want["level"] and got.layout == layout_from(want["layout"])
        assert counts_dict(be.ledger.totals()) == c["counts"]
