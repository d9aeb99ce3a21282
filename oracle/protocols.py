"""Restatement of the reference's hot-path protocols, generic over a backend.

TEST INFRASTRUCTURE ONLY. Each function cites the reference lines it follows
(/root/reference/proj/src/...). The backend is any object with the slotforge
op set (encrypt, zeros, add, sub, mul, mul_plain, mac_plain, rotate,
level_drop, exact_transform, with_layout, ledger): the numpy SimBackend
(oracle/slot_sim.py) pins these restatements against the reference's golden
vectors, and the CKKS CPU oracle (oracle/ckks.py) runs the same op sequence on
real ciphertexts so the GPU product can be held to it bit for bit.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .errors import CacheEmpty, CacheFull, LayoutMismatch, ShapeMismatch
from .layout import (Layout, log2_exact, make_interleaved, make_mask, padded_dim, stride_mask,
                     validate_layout, block_mask)


# --------------------------------------------------------------------------- vmm.cpp

def ceil_sqrt(k: int) -> int:
    """vmm.cpp:10-15."""
    b = int(math.isqrt(k))
    while b * b < k:
        b += 1
    while b > 1 and (b - 1) * (b - 1) >= k:
        b -= 1
    return b


def bsgs_split(k: int):
    """vmm.cpp:23-28: baby = ceil(sqrt(k)), giant = ceil(k / baby)."""
    if k < 1:
        raise ShapeMismatch("bsgs_split: k must be >= 1")
    b = ceil_sqrt(k)
    return b, (k + b - 1) // b


@dataclass
class Shape:
    """vmm.cpp:124-153 (InterleavedShape)."""
    N: int
    d_in: int
    d_out: int
    t_in: int
    t_out: int
    k: int
    alpha_up: int
    ladder_T: int
    tau_in: int
    tau_out: int
    tau_u: int
    carry: int
    delta: int


def interleaved_shape(N: int, rows: int, cols: int, tau_in: int, tau_out: int) -> Shape:
    d_in, d_out = padded_dim(rows), padded_dim(cols)
    if d_in > N or d_out > N:
        raise ShapeMismatch("vmm_interleaved: padded dimension exceeds N")
    t_in, t_out = N // d_in, N // d_out
    if not (0 <= tau_in < t_in):
        raise ShapeMismatch("vmm_interleaved: input offset out of range")
    if not (0 <= tau_out < t_out):
        raise ShapeMismatch("vmm_interleaved: output offset out of range")
    tau_u = tau_in % t_out
    return Shape(N, d_in, d_out, t_in, t_out, max(d_in * d_out // N, 1), max(1, t_out // t_in),
                 max(t_in, t_out), tau_in, tau_out, tau_u, 1 if tau_out < tau_u else 0,
                 (tau_out - tau_u) % t_out)


def interleaved_diag(s: Shape, W: np.ndarray, g: int, j: np.ndarray) -> np.ndarray:
    """vmm.cpp:159-168 vectorised over slot indices j (pre-giant frame)."""
    N = s.N
    i0 = (j + g * s.t_in * s.t_out - s.tau_in) % N
    row = (i0 // s.t_in + (i0 % s.t_in) * s.alpha_up) % s.d_in
    rel = (j - s.tau_u) % N
    u = rel % s.t_out
    within = u // s.t_in + (u % s.t_in) * s.alpha_up
    col = (rel // s.t_out + s.carry) % s.d_out
    rows, cols = W.shape
    ok = (g * s.t_out + within < s.d_in) & (row < rows) & (col < cols)
    out = np.zeros(len(j))
    out[ok] = W[row[ok], col[ok]]
    return out


def interleaved_plain(s: Shape, W: np.ndarray, g: int, giant_shift: int) -> np.ndarray:
    """vmm.cpp:170-175: p[i] = diag(g, (i - giant_shift) mod N)."""
    i = np.arange(s.N, dtype=np.int64)
    return interleaved_diag(s, W, g, (i - giant_shift) % s.N)


GIANT_GROUPS = 8  # giant-step groups of the BSGS rotation sums


def ladder_rots(s):
    """Preprocess ladder rotation amounts (vmm.cpp:190-193)."""
    return [step * (s.ladder_T - 1) for step in (1 << i for i in range(s.t_in.bit_length() - 1))]


def reduce_rots(s):
    """Reduce ladder rotation amounts (vmm.cpp:226-230): -2^m if bit m of delta is set, else +2^m."""
    return [-(1 << m) if (s.delta >> m) & 1 else (1 << m) for m in range(s.t_out.bit_length() - 1)]


def vmm_interleaved(be, x, W: np.ndarray, bsgs: bool = False, out_offset: int = 0,
                    mask_output: bool = False):
    """vmm.cpp:179-236 (the scheme of record)."""
    N = be.N
    if x.layout is None or x.layout.kind != "interleaved":
        raise LayoutMismatch("vmm_interleaved: input must carry an interleaved layout")
    if x.layout.deferred_mask:
        raise LayoutMismatch("vmm_interleaved: mask (or fuse) deferred garbage before feeding a VMM")
    W = np.asarray(W, dtype=np.float64)
    s = interleaved_shape(N, W.shape[0], W.shape[1], x.layout.offset, out_offset)
    if x.layout.d != s.d_in:
        raise ShapeMismatch(f"vmm_interleaved: layout d={x.layout.d} but weights want {s.d_in}")
    # 1. ladder (vmm.cpp:190-193)
    stair = _fold_steps(be, x, ladder_rots(s))
    unit = s.t_in * s.t_out
    # 2. multiply-accumulate (vmm.cpp:196-224)
    if not bsgs:
        terms = [(be.rotate(stair, g * unit), interleaved_plain(s, W, g, 0)) for g in range(s.k)]
        acc = be.mac_plain(terms)
    else:
        b, giants = bsgs_split(s.k)
        baby = [stair] + [be.rotate(stair, g1 * unit, hoisted=True) for g1 in range(1, b)]
        acc = None
        for r in range(min(GIANT_GROUPS, giants)):
            grp = vmm_giant_group(be, s, W, baby, b, unit, range(r, giants, GIANT_GROUPS))
            acc = grp if acc is None else be.add(acc, grp)
    # 3. reduce (vmm.cpp:226-230)
    acc = _fold_steps(be, acc, reduce_rots(s))
    # 4. mask or defer (vmm.cpp:233-234)
    if mask_output:
        acc = be.mul_plain(acc, stride_mask(N, s.t_out, s.tau_out))
    return be.with_layout(acc, Layout("interleaved", s.d_out, s.t_out, s.tau_out, 1, not mask_output))


def vmm_giant_group(be, s, W, baby, b, unit, giants):
    """One giant group of vmm.cpp:206-222: every giant's partial MAC, aligned by its
    giant rotation, summed as ONE rotation sum (giants g2 = r mod
    GIANT_GROUPS share a ModDown, so shards owning whole groups reproduce the sum).
    CKKS backends keep the partials unrescaled (scale * q_top) and merge the
    rescale into the sum's ModDown, the rotations decomposed with the wider digits
    a >= 2^80 scale allows (csrc/protocols.cpp vmm_partial)."""
    scaled = getattr(be, "vmm_scaled_giants", False)
    mac = be.mac_plain_lazy if scaled else be.mac_plain
    partials = []
    for g2 in giants:
        shift = g2 * b * unit
        terms = [(baby[g1], interleaved_plain(s, W, g2 * b + g1, shift))
                 for g1 in range(b) if g2 * b + g1 < s.k]
        partials.append((mac(terms), shift))
    return be.rot_sum_rescale(partials, scaled=True) if scaled else be.rot_sum(partials)


def predict_interleaved_cost(N: int, rows: int, cols: int, bsgs: bool = False, mask_output: bool = False):
    """vmm.cpp:473-488 -> (rotations, ct_pt_mults, depth)."""
    d_in, d_out = padded_dim(rows), padded_dim(cols)
    t_in, t_out = N // d_in, N // d_out
    k = max(d_in * d_out // N, 1)
    rot = log2_exact(t_in) + log2_exact(t_out)
    if bsgs:
        b, g = bsgs_split(k)
        rot += (b - 1) + (g - 1)
    else:
        rot += k - 1
    return rot, k + (1 if mask_output else 0), 1 + (1 if mask_output else 0)


def valid_mask(ly: Layout, N: int) -> np.ndarray:
    """vmm.cpp:45-56."""
    return make_mask(ly, N, "valid")


def apply_deferred_mask(be, x):
    """vmm.cpp:58-64."""
    if x.layout is None or not x.layout.deferred_mask:
        return x
    out = be.mul_plain(x, valid_mask(x.layout, be.N))
    return be.with_layout(out, x.layout.with_(deferred_mask=False))


def rope_plaintexts(n: int, d_head: int, ly: Layout, N: int, base: float = 10000.0):
    """vmm.cpp:66-83: p0 = cos, p1 = sin on even elements, p2 = -sin on odd."""
    validate_layout(ly, N)
    if ly.kind != "interleaved":
        raise LayoutMismatch("rope_plaintexts: interleaved layout required")
    if d_head <= 0 or d_head % 2:
        raise ShapeMismatch("rope_plaintexts: d_head must be positive and even")
    p0, p1, p2 = np.zeros(N), np.zeros(N), np.zeros(N)
    for e in range(ly.d):
        pair = (e % d_head) // 2
        ang = float(n) * math.pow(base, -2.0 * pair / float(d_head))
        i = e * ly.t + ly.offset
        p0[i] = math.cos(ang)
        if e % 2 == 0:
            p1[i] = math.sin(ang)
        else:
            p2[i] = -math.sin(ang)
    return p0, p1, p2


def fused_extract(be, x, succ: str, rope: Optional[dict] = None, coeff=None):
    """vmm.cpp:85-109. succ in {rope, silu_mask, norm_mask, vcache_mask};
    rope = {n, d_head, s, base}."""
    N = be.N
    if x.layout is None:
        raise LayoutMismatch("fused_extract: input must carry a layout")
    ly = x.layout
    if succ == "rope":
        if rope is None:
            raise ShapeMismatch("fused_extract: rope successor needs RoPEParams")
        p0, p1, p2 = rope_plaintexts(rope["n"], rope["d_head"], ly, N, rope.get("base", 10000.0))
        s = rope["s"]
        if getattr(be, "rope_fused", False):
            # CKKS backends: ONE rotation sum of the unrescaled products with the
            # rescale merged into its ModDown (mirrors csrc/protocols.cpp rope_apply;
            # same charge: 3 ct-pt mults, 2 rotations, 2 additions)
            u = [be.with_layout(be.mul_plain_lazy(x, p), None) for p in (p0, p1, p2)]
            y = be.rot_sum_rescale([(u[0], 0), (u[1], -s), (u[2], s)], scaled=True)
            return be.with_layout(y, ly.with_(deferred_mask=False))
        y = be.mul_plain(x, p0)
        y = be.add(y, be.rotate(be.mul_plain(x, p1), -s))
        y = be.add(y, be.rotate(be.mul_plain(x, p2), s))
        return be.with_layout(y, ly.with_(deferred_mask=False))
    m = valid_mask(ly, N)
    if coeff is not None:
        m = m * np.asarray(coeff)
    y = be.mul_plain(x, m)
    return be.with_layout(y, ly.with_(deferred_mask=False))


# ----------------------------------------------------------------- kv_attention.cpp

@dataclass
class AttentionConfig:
    """kv_attention.hpp:32-42."""
    N: int
    d: int
    H: int = 1
    n0: int = 0
    n_max: int = 0

    @property
    def d_head(self):
        return self.d // self.H

    @property
    def t(self):
        return self.N // self.d

    @property
    def group_tokens(self):
        return self.N // self.H


def validate_attention_config(cfg: AttentionConfig, N_backend: int):
    """kv_attention.cpp:80-88."""
    from .layout import is_pow2
    if cfg.N != N_backend:
        raise ShapeMismatch("attention config N != backend slot count")
    if not (is_pow2(cfg.N) and is_pow2(cfg.d) and is_pow2(cfg.H)):
        raise ShapeMismatch("attention config: N, d and H must be powers of two")
    if cfg.H > cfg.d or cfg.d > cfg.N:
        raise ShapeMismatch("attention config: need H <= d <= N")
    if cfg.n0 < 0 or cfg.n_max < max(cfg.n0, 1):
        raise ShapeMismatch("attention config: need 0 <= n0 <= n_max, n_max >= 1")


@dataclass
class KVCache:
    """kv_attention.hpp:49-54 (copy-on-write value; appends return a new one)."""
    n_prime: int = 0
    k_cts: list = field(default_factory=list)
    v_cts: list = field(default_factory=list)  # [group][variant]
    # CKKS backends: giant-aligned variants Rot(v, G B t) kept by v_append (None:
    # not tracked)
    v_aligned: list = field(default_factory=list)

    def copy(self):
        return KVCache(self.n_prime, list(self.k_cts), [list(g) for g in self.v_cts],
                       [list(g) if g is not None else None for g in self.v_aligned])


def v_variant_count(cfg):
    return cfg.d_head if cfg.H == 1 else 2 * cfg.d_head - 1


def v_variant_index(cfg, w):
    dh = cfg.d_head
    if cfg.H == 1:
        if not (0 <= w < dh):
            raise ShapeMismatch("v_variant_index: merged variant out of range")
        return w
    if w <= -dh or w >= dh:
        raise ShapeMismatch("v_variant_index: variant out of range")
    return w + dh - 1


def v_variant_of(cfg, e, u_local):
    raw = e - u_local // cfg.t
    return raw % cfg.d_head if cfg.H == 1 else raw


def _require_clean_interleaved(x, cfg, offset, who):
    """kv_attention.cpp:15-27."""
    if x.layout is None or x.layout.kind != "interleaved":
        raise LayoutMismatch(f"{who}: input must carry an interleaved layout")
    if x.layout.d != cfg.d:
        raise ShapeMismatch(f"{who}: layout width {x.layout.d} != configured {cfg.d}")
    if x.layout.offset != offset:
        raise LayoutMismatch(f"{who}: expected slot offset {offset}, got {x.layout.offset}")
    if x.layout.deferred_mask:
        raise LayoutMismatch(f"{who}: input garbage must be cleared first")


def _fold_steps(be, c, rots):
    """c <- c + Rot(c, r) for r in rots; CKKS backends evaluate the chain as
    radix rotation sums with the same ledger charge."""
    if hasattr(be, "fold_steps"):
        return be.fold_steps(c, rots)
    for r in rots:
        c = be.add(c, be.rotate(c, r))
    return c


def replicate_lanes(be, q, t):
    """kv_attention.cpp:30-34."""
    if hasattr(be, "fold_steps"):
        return be.fold_steps(q, [-(1 << s) for s in range(t.bit_length() - 1)])
    r = q
    step = 1
    while step < t:
        r = be.add(r, be.rotate(r, -step))
        step <<= 1
    return r


def fold_within_head(be, c, d_head, t):
    """kv_attention.cpp:38-41 (CKKS backends evaluate it as radix rotation
    sums, with the reference's ledger charge)."""
    if hasattr(be, "fold"):
        return be.fold(c, d_head, t)
    l = 0
    while (1 << l) < d_head:
        c = be.add(c, be.rotate(c, (1 << l) * t))
        l += 1
    return c


def fold_lanes(be, c, t):
    """kv_attention.cpp:44-47."""
    if hasattr(be, "fold_steps"):
        return be.fold_steps(c, [1 << s for s in range(t.bit_length() - 1)])
    step = 1
    while step < t:
        c = be.add(c, be.rotate(c, step))
        step <<= 1
    return c


def touched_variants(cfg, tokens):
    """kv_attention.cpp:53-57."""
    u_max = (tokens - 1) // cfg.t
    if cfg.H == 1:
        return 0, cfg.d_head
    return -u_max, cfg.d_head


def rope_apply(be, x, cfg, position, base=10000.0):
    """kv_attention.cpp:111-117 (s = t)."""
    if x.layout is None or x.layout.kind != "interleaved" or x.layout.d != cfg.d:
        raise LayoutMismatch("rope_apply: input must be interleaved at the configured width")
    return fused_extract(be, x, "rope", dict(n=position, d_head=cfg.d_head, s=cfg.t, base=base))


def k_append(be, cache: KVCache, k_new, cfg):
    """kv_attention.cpp:131-143."""
    if cache.n_prime >= cfg.n_max:
        raise CacheFull("k_append: cache at capacity")
    t = cfg.t
    _require_clean_interleaved(k_new, cfg, cache.n_prime % t, "k_append")
    out = cache.copy()
    if cache.n_prime % t == 0:
        out.k_cts.append(k_new)
    else:
        out.k_cts[-1] = be.add(out.k_cts[-1], k_new)
    out.n_prime = cache.n_prime + 1
    return out


def v_piece_mask(cfg, e, position):
    """The mask of kv_attention.cpp:157-160: ones at (h*d_head+e)*t + pos%t."""
    m = np.zeros(cfg.N)
    j0 = position % cfg.t
    for h in range(cfg.H):
        m[(h * cfg.d_head + e) * cfg.t + j0] = 1.0
    return m


def make_v_pieces(be, v_open, cfg, position):
    """kv_attention.cpp:145-163."""
    if position < 0 or position >= cfg.n_max:
        raise ShapeMismatch("make_v_pieces: position outside cache capacity")
    if v_open.layout is None or v_open.layout.kind != "interleaved" or v_open.layout.d != cfg.d:
        raise LayoutMismatch("make_v_pieces: input must be interleaved at the configured width")
    if v_open.layout.offset != position % cfg.t:
        raise LayoutMismatch("make_v_pieces: value ct offset does not match the token position")
    parts = [fused_extract(be, v_open, "vcache_mask", coeff=v_piece_mask(cfg, e, position))
             for e in range(cfg.d_head)]
    if getattr(be, "sv_bsgs", False):
        _attach_aligned(be, v_open, parts, cfg, position)
    return parts


def _giant_shift(cfg, w):
    B = sv_baby(cfg)
    return (w // B) * B * cfg.t


def _attach_aligned(be, v_open, parts, cfg, position):
    """Aligned companions of the value pieces (mirrors csrc/protocols.cpp
    make_v_pieces): piece e lands in variant w of giant
    G = floor(w / B); its companion Rot(piece, G B t) is computed as
    RS(Rot(mask_e, G B t) (.) Rot(v_open, G B t)) with Rot(mask_e, G B t) =
    mask_{(e - G B) mod d_head} (valid slots invariant under a lane-block
    shift). Off-ledger."""
    N, t, dh = be.N, cfg.t, cfg.d_head
    valid = valid_mask(v_open.layout, N)
    if not np.array_equal(valid, np.roll(valid, -t)) or v_open.is_zero:
        return
    B = sv_baby(cfg)
    u_local = position % cfg.group_tokens
    led, be.ledger = be.ledger, type(be.ledger)()
    try:
        rot = {}
        for e in range(dh):
            w = v_variant_of(cfg, e, u_local)
            G = w // B
            r = G * B * t
            if r % N == 0:
                continue
            if r not in rot:
                rot[r] = be.rotate(v_open, r, hoisted=True)
            m = valid * v_piece_mask(cfg, (e - G * B) % dh, position)
            parts[e]._aligned = (be.mul_plain(rot[r], m), r)
    finally:
        be.ledger = led


def v_append(be, cache: KVCache, parts, cfg):
    """kv_attention.cpp:165-182."""
    if cache.n_prime >= cfg.n_max:
        raise CacheFull("v_append: cache at capacity")
    dh = cfg.d_head
    if len(parts) != dh:
        raise ShapeMismatch(f"v_append: expected d/H pieces, got {len(parts)}")
    gt = cfg.group_tokens
    g = cache.n_prime // gt
    u_local = cache.n_prime - g * gt
    out = cache.copy()
    if g == len(out.v_cts):
        z = be.zeros()
        out.v_cts.append([z] * v_variant_count(cfg))
    if getattr(be, "sv_bsgs", False):
        _append_aligned(be, cache, out, parts, cfg, g, u_local)
    for e in range(dh):
        idx = v_variant_index(cfg, v_variant_of(cfg, e, u_local))
        out.v_cts[g][idx] = be.add(out.v_cts[g][idx], parts[e])
    return out


def _append_aligned(be, cache, out, parts, cfg, g, u_local):
    """Giant-aligned variants (mirrors csrc/protocols.cpp v_append): aligned' =
    (aligned, or Rot(V_old) when untracked, or 0 for an empty variant) + the
    piece's aligned companion; untracked when a piece has none. Off-ledger."""
    N, nv = be.N, v_variant_count(cfg)
    while len(out.v_aligned) <= g:
        out.v_aligned.append(None)
    al = list(out.v_aligned[g]) if out.v_aligned[g] is not None else [None] * nv
    led, be.ledger = be.ledger, type(be.ledger)()
    try:
        for e in range(cfg.d_head):
            w = v_variant_of(cfg, e, u_local)
            idx = v_variant_index(cfg, w)
            r = _giant_shift(cfg, w)
            comp = getattr(parts[e], "_aligned", None)
            if r % N == 0 or comp is None or comp[1] != r or parts[e].is_zero:
                al[idx] = None
                continue
            if al[idx] is None:
                old = cache.v_cts[g][idx] if g < len(cache.v_cts) else None
                if old is None or old.is_zero:
                    al[idx] = comp[0]
                    continue
                al[idx] = be.rotate(old, r)
            al[idx] = be.add(al[idx], comp[0])
    finally:
        be.ledger = led
    out.v_aligned[g] = al


def _ceil_div(a, b):
    return (a + b - 1) // b


def qk_dot(be, q, cache: KVCache, cfg):
    """kv_attention.cpp:184-214."""
    if cache.n_prime == 0:
        raise CacheEmpty("qk_dot: no cached keys")
    _require_clean_interleaved(q, cfg, 0, "qk_dot")
    t, dh, gt = cfg.t, cfg.d_head, cfg.group_tokens
    if len(cache.k_cts) != _ceil_div(cache.n_prime, t):
        raise ShapeMismatch("qk_dot: key ct count does not match n_prime")
    q_rep = replicate_lanes(be, q, t)
    head_mask = make_mask(make_interleaved(cfg.d, cfg.N, 0, cfg.H), cfg.N, "replicate_extract")
    n_maps = _ceil_div(cache.n_prime, gt)
    terms = [[[] for _ in range(PACK_GROUPS)] for _ in range(n_maps)]
    for j, kc in enumerate(cache.k_cts):
        terms[(j * t) // gt][j % PACK_GROUPS].append(qk_term(be, q_rep, kc, cfg, head_mask, -((j * t) % gt)))
    # pack + accumulate (kv_attention.cpp:202-206), one sum per (map, key-ct
    # group j mod PACK_GROUPS)
    return [be.with_layout(pack_sum(be, grp), None) for grp in terms]


def qk_term(be, q_rep, kc, cfg, head_mask, r):
    """One key ciphertext's (masked product, pack rotation) of kv_attention.cpp:
    195-204. CKKS backends with a shiftable fold apply the pack rotation inside
    the fold (its last radix sum's terms move by r) and mask with Rot(mask, r):
    Rot(mask (.) F, r) = Rot(mask, r) (.) Rot(F, r) -- the returned product is
    already aligned (rotation 0) and still unrescaled."""
    prod = be.mul(q_rep, kc)
    if getattr(be, "qk_shift_fold", False):
        f = be.fold_steps(prod, [(1 << l) * cfg.t for l in range(cfg.d_head.bit_length() - 1)], shift=r)
        return be.mul_plain_lazy(f, np.roll(head_mask, -r)), r
    prod = fold_within_head(be, prod, cfg.d_head, cfg.t)
    return mask_lazy(be, prod, head_mask), r


def mask_lazy(be, x, mask):
    """The QK^T head mask (layouts.cpp:134-138) with its rescale deferred to the
    pack rotation sum (CKKS backends: mul_plain_lazy + rot_sum_rescale, one
    rescale per sum instead of one per key ciphertext)."""
    f = getattr(be, "mul_plain_lazy", None)
    return f(x, mask) if f else be.mul_plain(x, mask)


PACK_GROUPS = 8  # key-ct groups of the QK^T pack sums


def pack_sum(be, groups):
    """sum over non-empty groups of rot_sum(group), accumulated in group order
    (rot_sum_rescale where the backend deferred the mask's rescale; where the
    pack rotation already rode the fold, qk_term: the plain sum of the aligned
    products and one rescale, charged as the reference's rotate/add chain)."""
    rs = getattr(be, "rot_sum_rescale", None) if getattr(be, "mul_plain_lazy", None) else None
    shifted = getattr(be, "qk_shift_fold", False)
    acc = None
    for grp in groups:
        if not grp:
            continue
        if shifted:
            for _, r in grp:
                if r % be.N:
                    be.ledger.count_rotation(False)
            for _ in range(len(grp) - 1):
                be.ledger.count_add()
            led, be.ledger = be.ledger, type(be.ledger)()
            try:
                s = grp[0][0]
                for x, _ in grp[1:]:
                    s = be.add(s, x)
                s = be.rescale(s)
            finally:
                be.ledger = led
        else:
            s = rs(grp) if rs else be.rot_sum(grp)
        acc = s if acc is None else be.add(acc, s)
    return acc


def softmax_times_v(be, probs, cache: KVCache, cfg):
    """kv_attention.cpp:216-241."""
    if cache.n_prime == 0:
        raise CacheEmpty("softmax_times_v: no cached values")
    t, gt = cfg.t, cfg.group_tokens
    n_maps = _ceil_div(cache.n_prime, gt)
    if len(probs) != n_maps:
        raise ShapeMismatch(f"softmax_times_v: expected {n_maps} probability maps, got {len(probs)}")
    if len(cache.v_cts) < n_maps:
        raise ShapeMismatch("softmax_times_v: value cache is missing groups")
    if getattr(be, "sv_bsgs", False):
        # CKKS backends: the baby-step / giant-step form
        return sv_finish(be, [sv_partial(be, probs, cache, cfg, 0, 1)], cfg)
    pairs = []
    for g in range(n_maps):
        tokens = min(gt, cache.n_prime - g * gt)
        lo, hi = touched_variants(cfg, tokens)
        for w in range(lo, hi):
            scores = be.rotate(probs[g], -w * t) if w else probs[g]
            pairs.append((scores, cache.v_cts[g][v_variant_index(cfg, w)]))
    # sum of the products (kv_attention.cpp:230-235)
    acc = be.mul_sum(pairs)
    folded = fold_lanes(be, acc, t)
    out = be.mul_plain(folded, stride_mask(cfg.N, t, 0))
    return be.with_layout(out, make_interleaved(cfg.d, cfg.N, 0, cfg.H))


SV_GROUPS = 8  # giant groups of the Score*V giant rotation sums


def sv_baby(cfg):
    """Baby-step count B: the least power of two with B^2 >= #variants."""
    b, nv = 1, v_variant_count(cfg)
    while b * b < nv:
        b <<= 1
    return b


def sv_partial(be, probs, cache: KVCache, cfg, rank, world):
    """Score*V over the giant groups a rank owns, as a baby-step / giant-step
    sum (mirrors csrc/protocols.cpp softmax_times_v_partial):
    with w = G B + b,  sum_(g,w) Rot(P_g, -w t) (x) V[g][w]
      = sum_G Rot( sum_(g,b) Rot(P_g, -b t) (x) Rot(V[g][w], G B t), -G B t ),
    inner sums lazily relinearised (one relinearisation per giant), giants as
    one rotation sum per group G mod SV_GROUPS at the products' scale (the
    rescale happens once, in sv_finish). Charged as the reference's
    rotations / ct-ct mults / additions of the owned (g, w) pairs
    (kv_attention.cpp:227-235)."""
    t, gt, N = cfg.t, cfg.group_tokens, cfg.N
    B = sv_baby(cfg)
    own = []
    for g in range(len(probs)):
        tokens = min(gt, cache.n_prime - g * gt)
        lo, hi = touched_variants(cfg, tokens)
        for w in range(lo, hi):
            G = w // B
            if (G % SV_GROUPS) % world == rank:
                own.append((g, w, G, w - G * B))
    for g, w, _, _ in own:
        if (-w * t) % N:
            be.ledger.count_rotation(False)
    for _ in own:
        be.ledger.count_ct_ct()
    for _ in range(len(own) - 1):
        be.ledger.count_add()
    lvl = min(probs[0].level, cache.v_cts[0][0].level)
    if not own:
        return be.zeros(lvl)
    led, be.ledger = be.ledger, type(be.ledger)()
    try:
        babies = {}
        inner = {}
        for g, w, G, b in own:
            if (g, b) not in babies:
                babies[(g, b)] = be.rotate(probs[g], -b * t, hoisted=True) if b else probs[g]
            vi = v_variant_index(cfg, w)
            v = cache.v_cts[g][vi]
            tracked = (cache.v_aligned[g][vi] if G and g < len(cache.v_aligned) and cache.v_aligned[g] is not None
                       else None)
            if tracked is not None:
                v = tracked
            elif not v.is_zero and (G * B * t) % N:
                v = be.rotate(v, G * B * t)
            inner.setdefault(G, []).append((babies[(g, b)], v))
        rel = {}
        for G in sorted(inner):
            live = [(a, v) for a, v in inner[G] if not (a.is_zero or v.is_zero)]
            if live:
                rel[G] = be.relin(be.tensor_sum(live))
        if not rel:
            return be.zeros(lvl)
        acc = None
        for r in range(SV_GROUPS):
            terms = [(rel[G], -G * B * t) for G in sorted(rel) if G % SV_GROUPS == r]
            if terms:
                s = be.rot_sum(terms, scaled=True)  # the relinearised sums are at scale >= 2^80
                acc = s if acc is None else be.add(acc, s)
    finally:
        be.ledger = led
    return be.with_layout(acc, None)


def sv_finish(be, parts, cfg):
    """Sum of the ranks' Score*V partials (charged live - 1 additions), one
    rescale, then fold_lanes and the stride mask (kv_attention.cpp:236-240)."""
    live = [p for p in parts if not p.is_zero]
    for _ in range(len(live) - 1):
        be.ledger.count_add()
    led, be.ledger = be.ledger, type(be.ledger)()
    try:
        acc = parts[0] if not live else live[0]
        for p in live[1:]:
            acc = be.add(acc, p)
        acc = be.rescale(acc) if live else be.zeros(acc.level - 1)
    finally:
        be.ledger = led
    folded = fold_lanes(be, acc, cfg.t)
    out = be.mul_plain(folded, stride_mask(cfg.N, cfg.t, 0))
    return be.with_layout(out, make_interleaved(cfg.d, cfg.N, 0, cfg.H))


def plain_softmax(s):
    s = np.asarray(s, dtype=np.float64)
    if len(s) == 0:
        return s
    p = np.exp(s - s.max())
    return p / p.sum()


def exact_softmax_maps(be, maps, cfg, n_prime):
    """kv_attention.cpp:395-412: oracle softmax (zero cost, level preserving)."""
    gt = cfg.group_tokens
    if len(maps) != _ceil_div(n_prime, gt):
        raise ShapeMismatch("exact_softmax_maps: map count does not match n_prime")
    slots = [be.decrypt(m) for m in maps]
    out = [np.zeros(cfg.N) for _ in maps]
    v = np.arange(n_prime)
    for h in range(cfg.H):
        sc = np.array([slots[i // gt][h * gt + i % gt] for i in v])
        p = plain_softmax(sc)
        for i in v:
            out[i // gt][h * gt + i % gt] = p[i]
    return [be.exact_transform(m, (lambda _s, o=o: o)) for m, o in zip(maps, out)]


# --------------------------------------------------------------------- prefill
# kv_attention.cpp:119-129, 245-376, 414-454 and vmm.cpp:30-43, 417-467: the
# step before decode, which builds the KV cache a decode step consumes.

def inner_rotate(be, x, r, block, hoisted=False):
    """vmm.cpp:30-43: cyclic rotation by r inside every block of `block` slots."""
    N = be.N
    if block <= 0 or N % block:
        raise ShapeMismatch("inner_rotate: block must divide N")
    s = r % block
    if s == 0:
        return x
    i = np.arange(N)
    keep = (i % block < block - s).astype(np.float64)
    lo = be.mul_plain(be.rotate(x, s, hoisted), keep)
    hi = be.mul_plain(be.rotate(x, s - block, hoisted), 1.0 - keep)
    return be.add(lo, hi)


def batch_plain(W: np.ndarray, d: int, N: int, j: int, pre: int) -> np.ndarray:
    """vmm.cpp:426-433: slot i of the j-th token-batched diagonal, pre-shifted by pre."""
    t = N // d
    e = ((np.arange(N) - pre) % N) // t
    r = (e + j) % d
    rows, cols = W.shape
    out = np.zeros(N)
    ok = (r < rows) & (e < cols)
    out[ok] = W[r[ok], e[ok]]
    return out


def vmm_batch(be, x, W: np.ndarray, bsgs: bool = True):
    """vmm.cpp:417-467: square VMM over a token batch (lane tau = token tau)."""
    N = be.N
    if x.layout is None or x.layout.kind != "interleaved":
        raise LayoutMismatch("vmm_batch: input must carry an interleaved layout")
    if x.layout.deferred_mask:
        raise LayoutMismatch("vmm_batch: input garbage must be cleared first")
    W = np.asarray(W, dtype=np.float64)
    d = padded_dim(W.shape[0])
    if padded_dim(W.shape[1]) != d:
        raise ShapeMismatch("vmm_batch: square weights only")
    if x.layout.d != d:
        raise ShapeMismatch("vmm_batch: layout/weight dimension mismatch")
    t = N // d
    if not bsgs:
        acc = be.mac_plain([(be.rotate(x, j * t), batch_plain(W, d, N, j, 0)) for j in range(d)])
    else:
        b, giants = bsgs_split(d)
        baby = [x] + [be.rotate(x, g1 * t, hoisted=True) for g1 in range(1, b)]
        partials = []
        for g2 in range(giants):
            shift = g2 * b * t
            terms = [(baby[g1], batch_plain(W, d, N, g2 * b + g1, shift)) for g1 in range(b) if g2 * b + g1 < d]
            partials.append((be.mac_plain(terms), shift))
        acc = None  # giant alignment + sum, grouped as in vmm_interleaved
        for r in range(min(GIANT_GROUPS, giants)):
            grp = be.rot_sum(partials[r::GIANT_GROUPS])
            acc = grp if acc is None else be.add(acc, grp)
    return be.with_layout(acc, Layout("interleaved", d, t, 0, 1, False))


def rope_batch_plain(which: int, cfg, first_pos: int, base: float = 10000.0) -> np.ndarray:
    """kv_attention.cpp:59-76: lane tau carries position first_pos + tau."""
    N, t, dh = cfg.N, cfg.t, cfg.d_head
    p = np.zeros(N)
    for i in range(N):  # libm cos / sin / pow, as the C++ product computes them
        e = (i // t) % dh
        angle = float(first_pos + i % t) * math.pow(base, -2.0 * (e // 2) / float(dh))
        if which == 0:
            p[i] = math.cos(angle)
        elif which == 1 and e % 2 == 0:
            p[i] = math.sin(angle)
        elif which == 2 and e % 2 == 1:
            p[i] = -math.sin(angle)
    return p


def rope_apply_batch(be, x, cfg, first_pos, base=10000.0):
    """kv_attention.cpp:119-129."""
    _require_clean_interleaved(x, cfg, 0, "rope_apply_batch")
    if cfg.d_head % 2:
        raise ShapeMismatch("rope_apply_batch: d_head must be even")
    s = cfg.t
    y = be.mul_plain(x, rope_batch_plain(0, cfg, first_pos, base))
    y = be.add(y, be.rotate(be.mul_plain(x, rope_batch_plain(1, cfg, first_pos, base)), -s))
    y = be.add(y, be.rotate(be.mul_plain(x, rope_batch_plain(2, cfg, first_pos, base)), s))
    return be.with_layout(y, x.layout)


def prefill(be, x_prompt, Wq, Wk, Wv, cfg, softmax_fn, rope_base=10000.0):
    """kv_attention.cpp:245-376. Returns (attention cts, KVCache)."""
    t, dh, gt, N, n0 = cfg.t, cfg.d_head, cfg.group_tokens, cfg.N, cfg.n0
    if n0 < 1:
        raise ShapeMismatch("prefill: need a nonempty prompt")
    if n0 > cfg.n_max:
        raise CacheFull("prefill: prompt exceeds cache capacity")
    P = _ceil_div(n0, t)
    if len(x_prompt) != P:
        raise ShapeMismatch(f"prefill: expected {P} prompt cts, got {len(x_prompt)}")
    cache = KVCache()
    q_cts = []
    for p in range(P):
        q_cts.append(rope_apply_batch(be, vmm_batch(be, x_prompt[p], Wq), cfg, p * t, rope_base))
        cache.k_cts.append(rope_apply_batch(be, vmm_batch(be, x_prompt[p], Wk), cfg, p * t, rope_base))
    for p in range(P):
        v_raw = vmm_batch(be, x_prompt[p], Wv)
        g = (p * t) // gt
        u_cap = p - g * dh
        if g == len(cache.v_cts):
            z = be.zeros()
            cache.v_cts.append([z] * v_variant_count(cfg))
        for e in range(dh):
            m = np.zeros(N)
            for h in range(cfg.H):
                m[(h * dh + e) * t:(h * dh + e + 1) * t] = 1.0
            piece = be.mul_plain(v_raw, m)
            idx = v_variant_index(cfg, v_variant_of(cfg, e, u_cap * t))
            cache.v_cts[g][idx] = be.add(cache.v_cts[g][idx], piece)
    cache.n_prime = n0
    k_rot = [[cache.k_cts[j]] + [inner_rotate(be, cache.k_cts[j], rho, t) for rho in range(1, t)] for j in range(P)]
    acc = [[[None] * t for _ in range((p * t) // gt + 1)] for p in range(P)]
    for p in range(P):
        for j in range(p + 1):
            g_key, local = (j * t) // gt, (j * t) % gt
            for rho in range(t):
                m = np.zeros(N)
                any_ = False
                for tau in range(t):
                    key, query = j * t + (tau + rho) % t, p * t + tau
                    if key <= query and key < n0 and query < n0:
                        for h in range(cfg.H):
                            m[h * gt + tau] = 1.0
                        any_ = True
                if not any_:
                    continue
                prod = be.mul(q_cts[p], k_rot[j][rho])
                prod = fold_within_head(be, prod, dh, t)
                masked = be.mul_plain(prod, m)
                packed = be.rotate(masked, -local) if local else masked
                cell = acc[p][g_key][rho]
                acc[p][g_key][rho] = packed if cell is None else be.add(cell, packed)
    maps = []
    for p in range(P):
        rows = []
        for g in range(len(acc[p])):
            ref_level = acc[p][g][0].level
            rows.append([be.with_layout(c if c is not None else be.zeros(ref_level), None) for c in acc[p][g]])
        maps.append(rows)
    probs = softmax_fn(be, maps, cfg, n0)
    if len(probs) != len(maps):
        raise ShapeMismatch("prefill: softmax changed the map shape")
    groups = len(cache.v_cts)
    v_rot = []
    for g in range(groups):
        tokens = min(gt, n0 - g * gt)
        lo, hi = touched_variants(cfg, tokens)
        rows = []
        for w in range(lo, hi):
            base_ct = cache.v_cts[g][v_variant_index(cfg, w)]
            rows.append([base_ct] + [inner_rotate(be, base_ct, rho, t) for rho in range(1, t)])
        v_rot.append((lo, rows))
    att = []
    for p in range(P):
        pairs = []
        for g in range(len(probs[p])):
            tokens = min(gt, n0 - g * gt)
            lo, hi = touched_variants(cfg, tokens)
            for rho in range(t):
                pm = probs[p][g][rho]
                for w in range(lo, hi):
                    scores = be.rotate(pm, -w * t) if w else pm
                    pairs.append((scores, v_rot[g][1][w - lo][rho]))
        # sum of the products (kv_attention.cpp:358-368); CKKS backends relinearise
        # once, charged as the reference's mul/add chain
        a = be.mul_sum(pairs)
        att.append(be.with_layout(a, make_interleaved(cfg.d, N, 0, cfg.H)))
    return att, cache


def exact_softmax_prefill_maps(be, maps, cfg, n0):
    """kv_attention.cpp:414-454: oracle softmax over the packed prefill maps."""
    t, gt = cfg.t, cfg.group_tokens
    slots = [[[be.decrypt(c) for c in row] for row in mp] for mp in maps]
    out = [[[np.zeros(cfg.N) for _ in range(t)] for _ in mp] for mp in maps]
    for p in range(len(maps)):
        for tau in range(t):
            query = p * t + tau
            if query >= n0:
                continue
            for h in range(cfg.H):
                ks = np.arange(query + 1)
                g = ks // gt
                rho = (ks % t - tau) % t
                pos = h * gt + (ks - g * gt) // t * t + tau
                sc = np.array([slots[p][g[i]][rho[i]][pos[i]] for i in range(len(ks))])
                pr = plain_softmax(sc)
                for i in range(len(ks)):
                    out[p][g[i]][rho[i]][pos[i]] = pr[i]
    return [[[be.exact_transform(c, (lambda _s, o=out[p][g][r]: o)) for r, c in enumerate(row)]
             for g, row in enumerate(mp)] for p, mp in enumerate(maps)]
