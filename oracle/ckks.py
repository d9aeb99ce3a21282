"""ctypes wrapper around oracle/ckks_oracle.cpp (the CPU RNS-CKKS oracle) plus a
slotforge-shaped backend over it. TEST INFRASTRUCTURE ONLY.

The backend enforces the reference's level rules and ledger accounting
(engine.hpp:102-111, engine.cpp:143-214) exactly like oracle/slot_sim.py, but
the arithmetic is real CKKS, so (a) its decrypted outputs are compared with the
reference's golden slot vectors at CKKS precision and (b) its ciphertext words
are the bit-exact expectation for the GPU product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import DomainViolation, Error, InvalidTarget, LevelUnderflow, ShapeMismatch
from .layout import Layout, is_pow2, validate_layout
from .slot_sim import CostLedger

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_bin", "libsf_oracle.so")

_lib = None
U64P = C.POINTER(C.c_uint64)
DP = C.POINTER(C.c_double)


def build():
    subprocess.run(["make", "-s", "-f", os.path.join("oracle", "oracle.mk")], cwd=os.path.dirname(HERE),
                   check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        sig = {
            "ock_last_error": (C.c_char_p, []),
            "ock_context_new": (vp, [C.c_int] * 7 + [C.c_uint64]),
            "ock_context_free": (None, [vp]),
            "ock_num_primes": (C.c_int, [vp]),
            "ock_primes": (None, [vp, U64P]),
            "ock_secret_key": (None, [vp, U64P]),
            "ock_key": (None, [vp, C.c_uint64, U64P]),
            "ock_galois_elt": (C.c_uint64, [vp, C.c_int]),
            "ock_ntt": (None, [vp, C.c_int, U64P, C.c_int]),
            "ock_automorph": (None, [vp, U64P, U64P, C.c_uint64]),
            "ock_encode": (C.c_int, [vp, DP, C.c_double, C.c_int, U64P]),
            "ock_encode_coeffs": (C.c_int, [vp, DP, C.c_double, C.POINTER(C.c_int64)]),
            "ock_encrypt": (vp, [vp, DP, C.c_int, C.c_double, C.c_uint64]),
            "ock_zero": (vp, [vp, C.c_int]),
            "ock_import": (vp, [vp, U64P, C.c_int, C.c_double, C.c_int]),
            "ock_ct_free": (None, [vp]),
            "ock_ct_info": (None, [vp, C.POINTER(C.c_int), DP, C.POINTER(C.c_int)]),
            "ock_ct_data": (None, [vp, U64P]),
            "ock_decrypt": (None, [vp, vp, DP]),
            "ock_add": (vp, [vp, vp, vp]),
            "ock_sub": (vp, [vp, vp, vp]),
            "ock_add_plain": (vp, [vp, vp, DP]),
            "ock_mac_plain": (vp, [vp, C.POINTER(vp), DP, C.c_int]),
            "ock_mul": (vp, [vp, vp, vp]),
            "ock_rotate": (vp, [vp, vp, C.c_int]),
            "ock_rescale": (vp, [vp, vp]),
            "ock_tensor_sum": (vp, [vp, C.POINTER(vp), C.POINTER(vp), C.c_int]),
            "ock_rot_sum": (vp, [vp, C.POINTER(vp), C.POINTER(C.c_int), C.c_int]),
            "ock_rot_sum_rescale": (vp, [vp, C.POINTER(vp), C.POINTER(C.c_int), C.c_int]),
            "ock_rot_sum_rescale_scaled": (vp, [vp, C.POINTER(vp), C.POINTER(C.c_int), C.c_int]),
            "ock_rot_sum_scaled": (vp, [vp, C.POINTER(vp), C.POINTER(C.c_int), C.c_int]),
            "ock_fold2": (vp, [vp, vp, C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int), C.c_int]),
            "ock_mac_plain_lazy": (vp, [vp, C.POINTER(vp), DP, C.c_int]),
            "ock_relin_rescale": (vp, [vp, vp]),
            "ock_relin": (vp, [vp, vp]),
            "ock_ct_is_three": (C.c_int, [vp]),
            "ock_ct_d2": (None, [vp, U64P]),
            "ock_ct_set_d2": (None, [vp, U64P]),
            "ock_level_drop": (vp, [vp, vp, C.c_int]),
            "ock_bench_weight": (None, [C.c_int, C.c_int, DP]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def _u64(a: np.ndarray):
    return a.ctypes.data_as(U64P)


def _dp(a: np.ndarray):
    return a.ctypes.data_as(DP)


def bench_weight(rows: int, cols: int) -> np.ndarray:
    """The reference bench weight sin(0.001(31r+c)+0.25) (slotforge_cli.cpp:88-92),
    computed in C with libm exactly as the product's W = NULL plans are."""
    out = np.empty((rows, cols))
    lib().ock_bench_weight(rows, cols, _dp(out))
    return out


def fold_radix(d_head: int):
    """Radix split of the head fold: log2(d_head) = D bits as
    one rotation sum when D <= 3, else two sums of ceil(D/2) and floor(D/2) bits."""
    D = d_head.bit_length() - 1
    if D <= 0:
        return []
    return [D] if D <= 3 else [(D + 1) // 2, D // 2]


def fmix(z: int) -> int:
    M = (1 << 64) - 1
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & M
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & M
    z ^= z >> 31
    return z


def auto_seed(key_seed: int, k: int) -> int:
    """seed of the k-th encryption a context makes without an
    explicit seed (client-side re-encryptions inside exact_transform/bootstrap)."""
    return fmix(key_seed ^ ((0xE1C0000000000000 + k) & ((1 << 64) - 1)))


def _raise(msg: str):
    for cls in (LevelUnderflow, InvalidTarget, ShapeMismatch, DomainViolation):
        if msg.startswith(cls.__name__):
            raise cls(msg)
    raise Error(msg)


class OCt:
    """Oracle ciphertext: C handle + level + layout tag."""

    def __init__(self, ctx, ptr, level: int, layout: Optional[Layout]):
        if not ptr:
            _raise(lib().ock_last_error().decode())
        self.ctx, self.ptr, self.level, self.layout = ctx, ptr, level, layout

    def __del__(self):
        if self.ptr and lib is not None and _lib is not None:
            _lib.ock_ct_free(self.ptr)
            self.ptr = None

    def info(self):
        limbs, scale, zero = C.c_int(), C.c_double(), C.c_int()
        lib().ock_ct_info(self.ptr, C.byref(limbs), C.byref(scale), C.byref(zero))
        return limbs.value, scale.value, bool(zero.value)

    @property
    def scale(self):
        return self.info()[1]

    @property
    def is_zero(self):
        return self.info()[2]

    def data(self) -> np.ndarray:
        """[2][limbs][n] words, or [3][limbs][n] for a degree-2 (lazily
        relinearised) ciphertext."""
        limbs, _, _ = self.info()
        out = np.empty(2 * limbs * self.ctx.n, dtype=np.uint64)
        lib().ock_ct_data(self.ptr, _u64(out))
        out = out.reshape(2, limbs, self.ctx.n)
        if lib().ock_ct_is_three(self.ptr):
            d2 = np.empty(limbs * self.ctx.n, dtype=np.uint64)
            lib().ock_ct_d2(self.ptr, _u64(d2))
            out = np.concatenate([out, d2.reshape(1, limbs, self.ctx.n)])
        return out


@dataclass
class CkksParams:
    """DESIGN.md §3.1. slots = the reference engine's N (power of two <= n/2)."""
    slots: int
    L: int
    log_n: Optional[int] = None
    alpha: Optional[int] = None
    q0_bits: int = 60
    scale_bits: int = 40
    special_bits: int = 60
    seed: int = 1

    def resolved(self):
        log_n = self.log_n if self.log_n is not None else max(2, (2 * self.slots).bit_length() - 1)
        alpha = self.alpha if self.alpha is not None else min(self.L + 1, 5)
        return log_n, alpha


class CkksOracle:
    """slotforge-shaped backend over the CPU CKKS oracle."""

    sv_bsgs = True  # Score*V as the product's baby-step / giant-step sum
    qk_shift_fold = True  # the QK^T pack rotation rides the fold
    rope_fused = True  # RoPE as one rotation sum with a merged rescale
    vmm_scaled_giants = True  # HE-VMM giants rotated before their rescale, wider digits
    fold_dh = True  # two-step folds double-hoisted: the first sum's b part stays extended

    def __init__(self, N: int, L: int, **kw):
        if not is_pow2(N):
            raise ShapeMismatch("engine: N must be a power of two")
        if L < 1:
            raise InvalidTarget("engine: level budget L must be >= 1")
        self.params = CkksParams(N, L, **kw)
        self.log_n, self.alpha = self.params.resolved()
        self.n = 1 << self.log_n
        if 2 * N > self.n:
            raise ShapeMismatch("ckks: slot count exceeds ring degree / 2")
        self.N, self.L = N, L
        p = self.params
        self.ptr = lib().ock_context_new(self.log_n, N, L, p.q0_bits, p.scale_bits, self.alpha, p.special_bits,
                                         p.seed)
        if not self.ptr:
            _raise(lib().ock_last_error().decode())
        self.delta = float(2 ** p.scale_bits)
        self.ledger = CostLedger()
        self.enc_counter = 0
        np_ = lib().ock_num_primes(self.ptr)
        self.primes = np.empty(np_, dtype=np.uint64)
        lib().ock_primes(self.ptr, _u64(self.primes))

    def __del__(self):
        if getattr(self, "ptr", None) and _lib is not None:
            _lib.ock_context_free(self.ptr)
            self.ptr = None

    def phase(self, name):
        return self.ledger.phase(name)

    # --- helpers
    def _slots(self, s, what):
        s = np.ascontiguousarray(np.broadcast_to(np.asarray(s, dtype=np.float64), (self.N,)))
        return s

    def _check(self, c: OCt, what):
        if c.level < 0 or c.level > self.L:
            raise InvalidTarget(f"{what}: ciphertext level {c.level} out of [0, L]")

    def next_seed(self):
        s = auto_seed(self.params.seed, self.enc_counter)
        self.enc_counter += 1
        return s

    def _merge(self, a, b):
        return a.layout if (a.layout is not None and a.layout == b.layout) else None

    # --- client ops (off-ledger)
    def encrypt(self, slots, level: int = -1, layout: Optional[Layout] = None, seed: Optional[int] = None,
                scale: Optional[float] = None) -> OCt:
        if level < 0:
            level = self.L
        slots = np.asarray(slots, dtype=np.float64)
        if len(slots) != self.N:
            raise ShapeMismatch(f"encrypt: expected {self.N} slots, got {len(slots)}")
        if level > self.L:
            raise InvalidTarget("encrypt: level exceeds budget L")
        if layout is not None:
            validate_layout(layout, self.N)
        seed = self.next_seed() if seed is None else seed
        s = np.ascontiguousarray(slots)
        ptr = lib().ock_encrypt(self.ptr, _dp(s), level + 1, scale or self.delta, seed)
        return OCt(self, ptr, level, layout)

    def zeros(self, level: int = -1) -> OCt:
        if level < 0:
            level = self.L
        return OCt(self, lib().ock_zero(self.ptr, level + 1), level, None)

    def decrypt(self, c: OCt) -> np.ndarray:
        out = np.empty(self.N)
        lib().ock_decrypt(self.ptr, c.ptr, _dp(out))
        return out

    def import_ct(self, data: np.ndarray, level: int, scale: float, layout=None, zero=False) -> OCt:
        """Words [2|3][level+1][n] (3 = degree-2 ciphertext)."""
        d = np.ascontiguousarray(data, dtype=np.uint64).reshape(-1)
        w = (level + 1) * self.n
        ct = OCt(self, lib().ock_import(self.ptr, _u64(d[:2 * w].copy()), level + 1, scale, int(zero)), level,
                 layout)
        if d.size == 3 * w:
            lib().ock_ct_set_d2(ct.ptr, _u64(d[2 * w:].copy()))
        return ct

    # --- lazily relinearised products (Score*V)
    def tensor_sum(self, pairs) -> OCt:
        """sum of ct x ct products kept as a degree-2 ciphertext (no relin);
        charged k ct-ct mults and k-1 additions like the reference chain."""
        for a, b in pairs:
            self._check(a, "mul"), self._check(b, "mul")
            if min(a.level, b.level) <= 0:
                raise LevelUnderflow("mul: no multiplicative level left")
        for i, _ in enumerate(pairs):
            self.ledger.count_ct_ct()
            if i:
                self.ledger.count_add()
        aa = (C.c_void_p * len(pairs))(*[a.ptr for a, _ in pairs])
        bb = (C.c_void_p * len(pairs))(*[b.ptr for _, b in pairs])
        lvl = min(min(a.level, b.level) for a, b in pairs)
        return OCt(self, lib().ock_tensor_sum(self.ptr, aa, bb, len(pairs)), lvl, None)

    def relin_rescale(self, x) -> OCt:
        return OCt(self, lib().ock_relin_rescale(self.ptr, x.ptr), x.level - 1, None)

    def relin(self, x) -> OCt:
        """Relinearise a degree-2 ciphertext without rescaling."""
        return OCt(self, lib().ock_relin(self.ptr, x.ptr), x.level, None)

    def rescale(self, x) -> OCt:
        """Rescale by the top prime (off-ledger)."""
        if x.level <= 0:
            raise LevelUnderflow("rescale: no level left")
        return OCt(self, lib().ock_rescale(self.ptr, x.ptr), x.level - 1, x.layout)

    def mul_sum(self, pairs) -> OCt:
        return self.relin_rescale(self.tensor_sum(pairs))

    # --- evaluator ops (ledger-charged)
    def add(self, a, b):
        self._check(a, "add"), self._check(b, "add")
        self.ledger.count_add()
        return OCt(self, lib().ock_add(self.ptr, a.ptr, b.ptr), min(a.level, b.level), self._merge(a, b))

    def sub(self, a, b):
        self._check(a, "sub"), self._check(b, "sub")
        self.ledger.count_add()
        return OCt(self, lib().ock_sub(self.ptr, a.ptr, b.ptr), min(a.level, b.level), self._merge(a, b))

    def add_plain(self, a, p):
        self._check(a, "add_plain")
        p = self._slots(p, "add_plain")
        self.ledger.count_add()
        return OCt(self, lib().ock_add_plain(self.ptr, a.ptr, _dp(p)), a.level, a.layout)

    def mul(self, a, b):
        self._check(a, "mul"), self._check(b, "mul")
        lvl = min(a.level, b.level)
        if lvl <= 0:
            raise LevelUnderflow("mul: no multiplicative level left")
        self.ledger.count_ct_ct()
        return OCt(self, lib().ock_mul(self.ptr, a.ptr, b.ptr), lvl - 1, self._merge(a, b))

    def mul_plain(self, a, p):
        return self.mac_plain([(a, p)], _layout=a.layout)

    def mac_plain(self, terms, _layout="__first__"):
        """sum_k ct_k * p_k with one rescale (fused MAC); charged as k ct-pt
        mults and k-1 additions like the reference's mul_plain/add chain."""
        for c, _ in terms:
            self._check(c, "mul_plain")
            if c.level <= 0:
                raise LevelUnderflow("mul_plain: no multiplicative level left")
        for i, _ in enumerate(terms):
            self.ledger.count_ct_pt()
            if i:
                self.ledger.count_add()
        lvl = min(c.level for c, _ in terms)
        pts = np.ascontiguousarray(np.stack([self._slots(p, "mul_plain") for _, p in terms]))
        arr = (C.c_void_p * len(terms))(*[c.ptr for c, _ in terms])
        layout = terms[0][0].layout if _layout == "__first__" else _layout
        if _layout == "__first__":
            for c, _ in terms[1:]:
                if c.layout != layout:
                    layout = None
        return OCt(self, lib().ock_mac_plain(self.ptr, arr, _dp(pts), len(terms)), lvl - 1, layout)

    def mac_plain_lazy(self, terms):
        """sum_k ct_k * p_k WITHOUT the rescale (scale * q_top, same limbs), charged
        as the reference's k mul_plain + k - 1 additions (the HE-VMM giants, whose
        rescale is merged into their rotation sum)."""
        for c, _ in terms:
            self._check(c, "mul_plain")
            if c.level <= 0:
                raise LevelUnderflow("mul_plain: no multiplicative level left")
        for i, _ in enumerate(terms):
            self.ledger.count_ct_pt()
            if i:
                self.ledger.count_add()
        lvl = min(c.level for c, _ in terms)
        pts = np.ascontiguousarray(np.stack([self._slots(p, "mul_plain") for _, p in terms]))
        arr = (C.c_void_p * len(terms))(*[c.ptr for c, _ in terms])
        return OCt(self, lib().ock_mac_plain_lazy(self.ptr, arr, _dp(pts), len(terms)), lvl, None)

    def mul_plain_lazy(self, a, p):
        """a * p WITHOUT the rescale: the raw product at scale * q_top on the
        same limbs, charged as the reference's mul_plain; the rescale happens in
        a later rot_sum_rescale (the QK^T pack)."""
        self._check(a, "mul_plain")
        if a.level <= 0:
            raise LevelUnderflow("mul_plain: no multiplicative level left")
        self.ledger.count_ct_pt()
        pts = np.ascontiguousarray(self._slots(p, "mul_plain")[None, :])
        arr = (C.c_void_p * 1)(a.ptr)
        return OCt(self, lib().ock_mac_plain_lazy(self.ptr, arr, _dp(pts), 1), a.level, a.layout)

    def rot_sum_rescale(self, terms, hoisted: bool = False, scaled: bool = False):
        """rot_sum of unrescaled products (mul_plain_lazy) with the pending
        rescale merged into the sum's ModDown (one basis conversion from
        {q_top} u P); same charge as rot_sum, one level lower. scaled: the
        terms are still at scale >= 2^80, so their decomposition uses the wider
        digits of scaled_digit (the HE-VMM giants)."""
        for a, _ in terms:
            self._check(a, "rotate")
        for i, (a, r) in enumerate(terms):
            if r % self.N:
                self.ledger.count_rotation(hoisted)
        for _ in range(len(terms) - 1):
            self.ledger.count_add()
        arr = (C.c_void_p * len(terms))(*[a.ptr for a, _ in terms])
        rr = (C.c_int * len(terms))(*[int(r) for _, r in terms])
        lvl = min(a.level for a, _ in terms)
        if lvl <= 0:
            raise LevelUnderflow("mul_plain: no multiplicative level left")
        fn = lib().ock_rot_sum_rescale_scaled if scaled else lib().ock_rot_sum_rescale
        return OCt(self, fn(self.ptr, arr, rr, len(terms)), lvl - 1, None)

    def rotate(self, a, r: int, hoisted: bool = False):
        self._check(a, "rotate")
        if r % self.N == 0:
            return a
        self.ledger.count_rotation(hoisted)
        return OCt(self, lib().ock_rotate(self.ptr, a.ptr, int(r)), a.level, None)

    def rot_sum(self, terms, hoisted: bool = False, scaled: bool = False):
        """sum_i Rot(a_i, r_i) (one ModDown for the whole sum),
        charged as the reference's rotate/add chain: one rotation per r_i != 0
        (mod N) and len(terms) - 1 additions; layouts merge as that chain's."""
        for a, _ in terms:
            self._check(a, "rotate")
        ly = None
        for i, (a, r) in enumerate(terms):
            if r % self.N:
                self.ledger.count_rotation(hoisted)
            t_ly = a.layout if r % self.N == 0 else None
            ly = t_ly if i == 0 else (ly if (ly is not None and ly == t_ly) else None)
        for _ in range(len(terms) - 1):
            self.ledger.count_add()
        arr = (C.c_void_p * len(terms))(*[a.ptr for a, _ in terms])
        rr = (C.c_int * len(terms))(*[int(r) for _, r in terms])
        lvl = min(a.level for a, _ in terms)
        fn = lib().ock_rot_sum_scaled if scaled else lib().ock_rot_sum  # scaled: terms at scale >= 2^80
        return OCt(self, fn(self.ptr, arr, rr, len(terms)), lvl, ly)

    def fold_steps(self, c, rots, shift: int = 0):
        """The doubling chain c <- c + Rot(c, r_i), i = 0..m-1 (fold_within_head,
        replicate_lanes, fold_lanes, the VMM ladders: kv_attention.cpp:30-47,
        vmm.cpp:190-193, 226-230), i.e. sum_{k < 2^m} Rot(c, sum_i bit_i(k) r_i),
        evaluated as radix rotation sums (fold_radix) and charged
        as the reference's m rotate + add steps. shift: the value rotated by
        `shift` (every term of the last radix sum moves by it; uncharged)."""
        self._check(c, "rotate")
        m = len(rots)
        if m == 0:
            if shift % self.N == 0:
                return c
            led, self.ledger = self.ledger, CostLedger()
            try:
                return self.rot_sum([(c, shift)])
            finally:
                self.ledger = led
        for r in rots:
            if r % self.N:
                self.ledger.count_rotation(False)
        for _ in range(m):
            self.ledger.count_add()
        ly = c.layout if all(r % self.N == 0 for r in list(rots) + [shift]) else None
        led, self.ledger = self.ledger, CostLedger()
        try:
            lo = 0
            radix = fold_radix(1 << m)
            if self.fold_dh and len(radix) == 2:
                steps = []
                for si, bits in enumerate(radix):
                    rs = rots[lo:lo + bits]
                    s0 = shift if si == 1 else 0
                    steps.append([s0 + sum(rs[i] for i in range(bits) if (k >> i) & 1) for k in range(1 << bits)])
                    lo += bits
                a1 = (C.c_int * len(steps[0]))(*[int(r) for r in steps[0]])
                a2 = (C.c_int * len(steps[1]))(*[int(r) for r in steps[1]])
                out = OCt(self, lib().ock_fold2(self.ptr, c.ptr, a1, len(steps[0]), a2, len(steps[1])), c.level, None)
                return OCt._alias(out, ly)
            for si, bits in enumerate(radix):
                rs = rots[lo:lo + bits]
                s0 = shift if si + 1 == len(radix) else 0
                terms = []
                for k in range(1 << bits):
                    terms.append((c, s0 + sum(rs[i] for i in range(bits) if (k >> i) & 1)))
                c = self.rot_sum(terms)
                lo += bits
        finally:
            self.ledger = led
        return OCt._alias(c, ly)

    def fold(self, c, d_head: int, t: int):
        """fold_within_head (kv_attention.cpp:38-41)."""
        return self.fold_steps(c, [(1 << l) * t for l in range(d_head.bit_length() - 1)])

    def level_drop(self, a, target: int):
        self._check(a, "level_drop")
        if target < 0 or target > a.level:
            raise InvalidTarget(f"level_drop: target level {target} outside [0, level]")
        return OCt(self, lib().ock_level_drop(self.ptr, a.ptr, target + 1), target, a.layout)

    def bootstrap(self, a, target: int):
        """Oracle hook (client round trip): decrypt, re-encrypt at target."""
        self._check(a, "bootstrap")
        if target < 1 or target > self.L:
            raise InvalidTarget(f"bootstrap: target level {target} outside [1, L]")
        self.ledger.count_bootstrap()
        return self._reenc(self.decrypt(a), target, a.layout)

    def exact_transform(self, a, f):
        """Oracle hook: decrypt -> f -> re-encrypt at the same level (free)."""
        self._check(a, "exact_transform")
        out = np.asarray(f(self.decrypt(a)), dtype=np.float64)
        if len(out) != self.N:
            raise ShapeMismatch("exact_transform result: wrong slot count")
        return self._reenc(out, a.level, a.layout)

    def _reenc(self, slots, level, layout):
        ct = self.encrypt(slots, level, None)
        ct.layout = layout
        return ct

    def with_layout(self, c, layout):
        return OCt._alias(c, layout)


def _alias(c: OCt, layout):
    """Same C ciphertext, new layout tag (ciphertexts are immutable values)."""
    n = OCt.__new__(OCt)
    n.ctx, n.level, n.layout = c.ctx, c.level, layout
    n._owner = c  # keep the C handle alive
    n.ptr = c.ptr
    n.__dict__["_alias"] = True
    return n


OCt._alias = staticmethod(_alias)
_orig_del = OCt.__del__


def _del(self):
    if self.__dict__.get("_alias"):
        return
    _orig_del(self)


OCt.__del__ = _del
