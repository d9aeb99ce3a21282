"""Restatement of /root/reference/proj/src/layouts.cpp (TEST INFRASTRUCTURE)."""
from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .errors import ShapeMismatch


def is_pow2(v: int) -> bool:
    return v > 0 and (v & (v - 1)) == 0


def log2_exact(v: int) -> int:
    if not is_pow2(v):
        raise ShapeMismatch(f"log2_exact: {v} is not a power of two")
    return v.bit_length() - 1


def next_pow2(v: int) -> int:
    p = 1
    while p < v:
        p <<= 1
    return p


@dataclass(frozen=True)
class Layout:
    """layouts.hpp:22-33."""
    kind: str = "interleaved"  # contiguous | replicated | interleaved
    d: int = 0
    t: int = 0
    offset: int = 0
    heads: int = 1
    deferred_mask: bool = False

    def with_(self, **kw) -> "Layout":
        return replace(self, **kw)


def validate_layout(ly: Layout, N: int) -> None:
    """layouts.cpp:56-64."""
    def req(c, m):
        if not c:
            raise ShapeMismatch(m)
    req(is_pow2(N), "layout: N must be a power of two")
    req(ly.d > 0 and is_pow2(ly.d), f"layout: d must be a positive power of two, got {ly.d}")
    req(ly.t > 0 and is_pow2(ly.t), f"layout: t must be a positive power of two, got {ly.t}")
    req(ly.d * ly.t == N, "layout: d*t must equal N")
    req(0 <= ly.offset < ly.t, "layout: offset out of range")
    req(ly.heads >= 1 and is_pow2(ly.heads) and ly.heads <= ly.d, "layout: heads must be a power of two dividing d")


def make_interleaved(d: int, N: int, offset: int = 0, heads: int = 1) -> Layout:
    ly = Layout("interleaved", d, N // d if d else 0, offset, heads, False)
    validate_layout(ly, N)
    return ly


def make_contiguous(d: int, N: int) -> Layout:
    ly = Layout("contiguous", d, N // d, 0, 1, False)
    validate_layout(ly, N)
    return ly


def make_replicated(d: int, N: int) -> Layout:
    ly = Layout("replicated", d, N // d, 0, 1, False)
    validate_layout(ly, N)
    return ly


def encode(x, ly: Layout, N: int) -> np.ndarray:
    """layouts.cpp:66-84."""
    validate_layout(ly, N)
    x = np.asarray(x, dtype=np.float64)
    if len(x) > ly.d:
        raise ShapeMismatch("encode: input length exceeds d")
    s = np.zeros(N)
    n = len(x)
    if ly.kind == "contiguous":
        s[:n] = x
    elif ly.kind == "replicated":
        for c in range(ly.t):
            s[c * ly.d:c * ly.d + n] = x
    else:
        s[np.arange(n) * ly.t + ly.offset] = x
    return s


def decode(slots, ly: Layout) -> np.ndarray:
    """layouts.cpp:86-104."""
    slots = np.asarray(slots)
    validate_layout(ly, len(slots))
    if ly.kind in ("contiguous", "replicated"):
        return slots[:ly.d].copy()
    return slots[np.arange(ly.d) * ly.t + ly.offset].copy()


def stride_mask(N: int, t: int, offset: int) -> np.ndarray:
    """layouts.cpp:106-112."""
    if not (is_pow2(N) and is_pow2(t) and t <= N):
        raise ShapeMismatch("stride_mask: bad N/t")
    if not (0 <= offset < t):
        raise ShapeMismatch("stride_mask: offset out of range")
    m = np.zeros(N)
    m[offset::t] = 1.0
    return m


def block_mask(N: int, begin: int, length: int) -> np.ndarray:
    if begin < 0 or length < 0 or begin + length > N:
        raise ShapeMismatch("block_mask: range out of bounds")
    m = np.zeros(N)
    m[begin:begin + length] = 1.0
    return m


def make_mask(ly: Layout, N: int, kind: str, offset: int = 0) -> np.ndarray:
    """layouts.cpp:121-144: kind in {valid, replicate_extract, cache_slot}."""
    validate_layout(ly, N)
    if kind == "valid":
        if ly.kind == "interleaved":
            return stride_mask(N, ly.t, ly.offset)
        if ly.kind == "contiguous":
            return block_mask(N, 0, ly.d)
        return np.ones(N)
    if kind == "replicate_extract":
        hb = N // ly.heads
        m = np.zeros(N)
        for h in range(ly.heads):
            m[h * hb:h * hb + ly.t] = 1.0
        return m
    if kind == "cache_slot":
        return stride_mask(N, ly.t, offset)
    raise ShapeMismatch(f"make_mask: unknown kind {kind}")


def padded_dim(d: int) -> int:
    if d <= 0:
        raise ShapeMismatch("padded_dim: d must be positive")
    return next_pow2(d)


def pad_to(x, d: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    if len(x) > d:
        raise ShapeMismatch("pad_to: input longer than target")
    out = np.zeros(d)
    out[:len(x)] = x
    return out
