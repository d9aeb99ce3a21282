"""The CPU CKKS oracle against first principles and against the reference's
golden slot vectors (CPU only). The oracle is what the GPU product is held to
bit for bit, so these tests pin its own correctness:
  * NTT == the definitional evaluation at psi^(2 br(i) + 1)
  * encoder == the canonical-embedding inverse
  * every op decrypts to the slot-simulator result (reference semantics)
  * protocol replays decrypt to the reference golden vectors with exact counts
"""
import numpy as np
import pytest

from golden_util import cases, counts_dict, layout_from
from oracle import protocols as P
from oracle.ckks import CkksOracle, _u64, lib
from oracle.errors import LevelUnderflow
from oracle.layout import make_interleaved
from oracle.slot_sim import SimBackend

TOL = 1e-6  # CKKS at scale 2^40: observed errors are ~1e-9..1e-8 at these sizes


def _bitrev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2)


def _min_psi(q, n):
    m = 2 * n
    for g in range(2, 1000):
        c = pow(g, (q - 1) // m, q)
        if pow(c, n, q) == q - 1:
            return min(pow(c, k, q) for k in range(1, m, 2))


def test_chacha20_block_matches_cryptography():
    """keys and encryption randomness are a ChaCha20 counter
    stream. The twin's block function (the same definition the GPU product
    implements, csrc/common.h) is pinned to an independent implementation:
    the `cryptography` package (OpenSSL) keystream for the same key, 64-bit
    block counter and 64-bit nonce (IV = counter || nonce, little-endian)."""
    import ctypes as C
    import struct
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    from oracle.ckks import lib
    f = lib().ock_chacha20_block
    f.argtypes = [C.POINTER(C.c_uint32), C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32)]
    rng = np.random.default_rng(2026)
    for _ in range(16):
        key = rng.integers(0, 2**32, size=8, dtype=np.uint64).astype(np.uint32)
        ctr, nonce = (int(v) for v in rng.integers(0, 2**63, size=2))
        out = np.zeros(16, dtype=np.uint32)
        f(key.ctypes.data_as(C.POINTER(C.c_uint32)), ctr, nonce, out.ctypes.data_as(C.POINTER(C.c_uint32)))
        ks = Cipher(algorithms.ChaCha20(key.tobytes(), struct.pack("<QQ", ctr, nonce)), mode=None).encryptor()
        assert np.array_equal(np.frombuffer(ks.update(bytes(64)), dtype=np.uint32), out)


def test_key_stream_words_are_chacha20():
    """Word i of stream (seed, id) = 64-bit word i mod 8 of block i / 8 under the
    documented key layout (seed || "sf_b200 ckks rng" || 1 || 0), nonce = id."""
    import ctypes as C
    import struct
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    from oracle.ckks import lib
    f = lib().ock_rand64
    f.argtypes, f.restype = [C.c_uint64, C.c_uint64, C.c_uint64], C.c_uint64
    seed, stream = 0x0123456789ABCDEF, (4 << 56) | 3
    key = struct.pack("<Q", seed) + b"sf_b200 ckks rng" + struct.pack("<II", 1, 0)
    ks = Cipher(algorithms.ChaCha20(key, struct.pack("<QQ", 5, stream)), mode=None).encryptor().update(bytes(64))
    want = np.frombuffer(ks, dtype=np.uint64)
    got = np.array([f(seed, stream, 5 * 8 + w) for w in range(8)], dtype=np.uint64)
    assert np.array_equal(got, want)


def test_ntt_matches_definition():
    be = CkksOracle(8, 2)  # ring 16
    n, logn = be.n, be.log_n
    rng = np.random.default_rng(0)
    for pi, q in enumerate(int(x) for x in be.primes):
        assert (q - 1) % (2 * n) == 0
        psi = _min_psi(q, n)
        a = [int(v) for v in rng.integers(0, q, n, dtype=np.uint64)]
        want = [sum(a[j] * pow(psi, (2 * _bitrev(i, logn) + 1) * j, q) for j in range(n)) % q for i in range(n)]
        buf = np.array(a, dtype=np.uint64)
        lib().ock_ntt(be.ptr, pi, _u64(buf), 0)
        assert [int(x) for x in buf] == want
        lib().ock_ntt(be.ptr, pi, _u64(buf), 1)
        assert [int(x) for x in buf] == a


def test_encoder_matches_canonical_embedding():
    be = CkksOracle(16, 2)
    n = be.n
    rng = np.random.default_rng(1)
    z = rng.normal(size=16)
    co = np.empty(n, dtype=np.int64)
    import ctypes as C
    assert lib().ock_encode_coeffs(be.ptr, z.ctypes.data_as(C.POINTER(C.c_double)), 2.0 ** 30,
                                   co.ctypes.data_as(C.POINTER(C.c_int64))) == 0
    zeta = np.exp(1j * np.pi / n)
    k = np.arange(n)
    want = np.zeros(n)
    for j in range(n // 2):
        w = zeta ** pow(5, j, 2 * n)
        want += 2.0 / n * np.real(z[j] * w ** (-k))
    assert np.max(np.abs(co - np.round(want * 2.0 ** 30))) <= 1


def test_ops_decrypt_to_slot_semantics():
    N, L = 32, 4
    ck, sim = CkksOracle(N, L, alpha=2), SimBackend(N, L)
    rng = np.random.default_rng(2)
    a, b, p = rng.normal(size=N), rng.normal(size=N), rng.normal(size=N)
    ca, cb = ck.encrypt(a, 4), ck.encrypt(b, 3)
    sa, sb = sim.encrypt(a, 4), sim.encrypt(b, 3)
    for name, f in [("add", lambda be, x, y: be.add(x, y)), ("sub", lambda be, x, y: be.sub(x, y)),
                    ("mul", lambda be, x, y: be.mul(x, y)),
                    ("mul_plain", lambda be, x, y: be.mul_plain(x, p)),
                    ("add_plain", lambda be, x, y: be.add_plain(x, p)),
                    ("rot3", lambda be, x, y: be.rotate(x, 3)), ("rot-7", lambda be, x, y: be.rotate(x, -7)),
                    ("chain", lambda be, x, y: be.rotate(be.mul(be.mul_plain(x, p), y), 5))]:
        got, want = f(ck, ca, cb), f(sim, sa, sb)
        assert got.level == want.level, name
        assert np.max(np.abs(ck.decrypt(got) - want.slots)) < TOL, name
    assert counts_dict(ck.ledger.totals()) == counts_dict(sim.ledger.totals())
    z = ck.mul_plain(ck.mul_plain(ca, p), p)
    z = ck.level_drop(ck.mul_plain(z, p), 0)
    with pytest.raises(LevelUnderflow):
        ck.mul(z, z)
    with pytest.raises(LevelUnderflow):
        ck.mul_plain(z, p)


def test_rotation_group_law_and_free_zero_shift():
    ck = CkksOracle(16, 3)
    x = np.arange(16, dtype=float)
    c = ck.encrypt(x)
    assert ck.rotate(c, 16) is c and ck.rotate(c, 0) is c
    lhs = ck.decrypt(ck.rotate(ck.rotate(c, 3), 2))
    assert np.max(np.abs(lhs - np.roll(x, -5))) < TOL
    assert ck.ledger.totals().rotations == 2


def test_sparse_packing_rotation():
    # 8 logical slots in a ring of 64 (32 slots): data replicated 4x, rotations mod 8
    ck = CkksOracle(8, 2, log_n=6)
    x = np.arange(8, dtype=float) + 1
    y = ck.decrypt(ck.rotate(ck.encrypt(x), 3))
    assert np.max(np.abs(y - np.roll(x, -3))) < TOL


def test_double_hoisted_fold_matches_the_doubling_chain():
    # fold_steps' two radix sums with the first sum's b part kept extended
    # (fold2): on a fused ring (2^12) it decrypts to the
    # rotate/add chain; below the fused range it is the plain two-sum path word
    # for word; the ledger is the chain's either way
    for log_n, hoisted in ((12, True), (11, False)):
        n = 1 << (log_n - 1)
        rots = [1, 2, 4, 8, 16]  # 5 doublings: radix 8 then 4
        x = np.sin(np.arange(n) * 0.37)
        want = sum(np.roll(x, -k) for k in range(32))
        out = {}
        for dh in (True, False):
            ck = CkksOracle(n, 3, alpha=2)
            ck.fold_dh = dh
            y = ck.fold_steps(ck.encrypt(x), rots)
            assert np.max(np.abs(ck.decrypt(y) - want)) < 32 * TOL
            assert ck.ledger.totals().rotations == 5 and ck.ledger.totals().additions == 5
            out[dh] = y.data()
        assert np.array_equal(out[True], out[False]) != hoisted


@pytest.mark.parametrize("which", ["small"])
def test_vmm_protocol_decrypts_to_reference(which):
    for c in cases(which, "vmm")[::3]:
        N, L = c["N"], c["L"]
        W = np.array(c["W"]).reshape(c["rows"], c["cols"])
        be = CkksOracle(N, L, alpha=3)
        x = be.encrypt(np.array(c["x_slots"]), L, make_interleaved(P.padded_dim(c["rows"]), N, c["tau_in"]))
        y = P.vmm_interleaved(be, x, W, bsgs=c["bsgs"], out_offset=c["tau_out"], mask_output=c["mask_output"])
        assert np.max(np.abs(be.decrypt(y) - np.array(c["y_slots"]))) < TOL
        assert counts_dict(be.ledger.totals()) == c["counts"]
        assert y.level == c["level"] and y.layout == layout_from(c["layout"])


def test_attention_protocol_decrypts_to_reference():
    from test_oracle_golden import replay_attention
    for c in cases("small", "attn")[::4]:
        be = CkksOracle(c["N"], c["L"], alpha=4)
        r = replay_attention(be, c)
        assert r["append_counts"] == [dict(x) for x in c["append_counts"]]
        for got, want in zip(r["maps"], c["maps"]):
            assert np.max(np.abs(be.decrypt(got) - np.array(want))) < TOL
        assert np.max(np.abs(be.decrypt(r["out"]) - np.array(c["out_slots"]))) < TOL
        assert r["out"].level == c["out_level"]
        assert counts_dict(be.ledger.phase_totals("QK^T")) == c["qk_counts"]
        assert counts_dict(be.ledger.phase_totals("Score*V")) == c["sv_counts"]


def test_rope_protocol_decrypts_to_reference():
    for c in cases("small", "rope"):
        N, L = c["N"], c["L"]
        be = CkksOracle(N, L)
        ly = make_interleaved(c["d"], N, c["offset"]).with_(deferred_mask=True)
        x = be.encrypt(np.array(c["x_slots"]), L, ly)
        y = P.fused_extract(be, x, "rope", dict(n=c["pos"], d_head=c["d_head"], s=ly.t))
        assert np.max(np.abs(be.decrypt(y) - np.array(c["y_slots"]))) < 1e-5
        assert counts_dict(be.ledger.totals()) == c["counts"]


def test_prefill_replays_decrypt_to_reference_goldens():
    # kv_attention.cpp:245-376 on real CKKS: cache entries and attention outputs
    # decrypt to the reference's slot vectors, counts and levels exact
    from test_oracle_golden import replay_prefill
    for c in cases("small", "prefill"):
        be = CkksOracle(c["N"], c["L"], alpha=3)
        att, cache = replay_prefill(be, c)
        for got, want in zip(cache.k_cts, c["k_cts"]):
            assert np.max(np.abs(be.decrypt(got) - np.array(want["slots"]))) < TOL and got.level == want["level"]
        for gg, gw in zip(cache.v_cts, c["v_cts"]):
            for got, want in zip(gg, gw):
                assert np.max(np.abs(be.decrypt(got) - np.array(want["slots"]))) < TOL
        for got, want in zip(att, c["attention"]):
            assert np.max(np.abs(be.decrypt(got) - np.array(want["slots"]))) < 1e-5
            assert got.level == want["level"] and got.layout == layout_from(want["layout"])
        assert counts_dict(be.ledger.totals()) == c["counts"]
