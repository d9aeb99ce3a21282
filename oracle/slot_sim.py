"""Slot-level oracle: numpy restatement of the reference's SimBackend.

TEST INFRASTRUCTURE ONLY (imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg; never by the product). Restates
/root/reference/proj/src/engine.cpp; pinned against golden vectors emitted by
the reference itself (oracle/ref_golden.cpp -> tests/golden/).

Level rules (engine.hpp:102-111): add/sub -> min level; add_plain keeps it;
mul/mul_plain -> min-1 and LevelUnderflow at 0; rotate keeps the level, r == 0
mod N is free; level_drop free; bootstrap -> target in [1, L].
"""
from __future__ import annotations

import copy
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from .errors import InvalidTarget, LevelUnderflow, ShapeMismatch
from .layout import Layout, is_pow2, validate_layout


@dataclass
class OpCounts:
    """engine.hpp:30-49."""
    rotations: int = 0
    hoisted_rotations: int = 0
    ct_pt_mults: int = 0
    ct_ct_mults: int = 0
    additions: int = 0
    bootstraps: int = 0

    def __add__(self, o: "OpCounts") -> "OpCounts":
        return OpCounts(*(a + b for a, b in zip(self.astuple(), o.astuple())))

    def __sub__(self, o: "OpCounts") -> "OpCounts":
        return OpCounts(*(a - b for a, b in zip(self.astuple(), o.astuple())))

    def astuple(self):
        return (self.rotations, self.hoisted_rotations, self.ct_pt_mults, self.ct_ct_mults,
                self.additions, self.bootstraps)

    def asdict(self):
        return dict(zip(("rotations", "hoisted_rotations", "ct_pt_mults", "ct_ct_mults",
                         "additions", "bootstraps"), self.astuple()))


class CostLedger:
    """engine.cpp:7-90: totals plus first-use-ordered phase breakdown."""
    DEFAULT = "(unphased)"

    def __init__(self):
        self.reset()

    def reset(self):
        self.total = OpCounts()
        self.by_phase: dict[str, OpCounts] = {}
        self.current = self.DEFAULT

    def _bump(self, attr: str, n: int = 1):
        setattr(self.total, attr, getattr(self.total, attr) + n)
        ph = self.by_phase.setdefault(self.current, OpCounts())
        setattr(ph, attr, getattr(ph, attr) + n)

    def count_rotation(self, hoisted: bool):
        self._bump("rotations")
        if hoisted:
            self._bump("hoisted_rotations")

    def count_ct_pt(self):
        self._bump("ct_pt_mults")

    def count_ct_ct(self):
        self._bump("ct_ct_mults")

    def count_add(self):
        self._bump("additions")

    def count_bootstrap(self):
        self._bump("bootstraps")

    def totals(self) -> OpCounts:
        return copy.copy(self.total)

    def phase_totals(self, name: str) -> OpCounts:
        return copy.copy(self.by_phase.get(name, OpCounts()))

    def conserved(self) -> bool:
        s = OpCounts()
        for v in self.by_phase.values():
            s = s + v
        return s == self.total

    class _Scope:
        def __init__(self, led, name):
            self.led, self.name = led, name

        def __enter__(self):
            self.prev, self.led.current = self.led.current, self.name
            return self

        def __exit__(self, *a):
            self.led.current = self.prev

    def phase(self, name: str):
        return CostLedger._Scope(self, name)


@dataclass
class SimCt:
    slots: np.ndarray
    level: int
    layout: Optional[Layout] = None


def _merge(a: SimCt, b: SimCt) -> Optional[Layout]:
    # engine.cpp:136-139: a binary result keeps a layout only if both agree
    return a.layout if (a.layout is not None and a.layout == b.layout) else None


class SimBackend:
    """engine.cpp:92-214 restated over float64 numpy arrays."""

    def __init__(self, N: int, L: int):
        if not is_pow2(N):
            raise ShapeMismatch("engine: N must be a power of two")
        if L < 1:
            raise InvalidTarget("engine: level budget L must be >= 1")
        self.N, self.L = N, L
        self.ledger = CostLedger()

    def phase(self, name):
        return self.ledger.phase(name)

    def _check_slots(self, s, what):
        if len(s) != self.N:
            raise ShapeMismatch(f"{what}: expected {self.N} slots, got {len(s)}")

    def _check(self, c: SimCt, what):
        self._check_slots(c.slots, what)
        if c.level < 0 or c.level > self.L:
            raise InvalidTarget(f"{what}: ciphertext level {c.level} out of [0, L]")

    # off-ledger client ops (engine.cpp:109-123)
    def encrypt(self, slots, level: int = -1, layout: Optional[Layout] = None) -> SimCt:
        if level < 0:
            level = self.L
        slots = np.asarray(slots, dtype=np.float64).copy()
        self._check_slots(slots, "encrypt")
        if level > self.L:
            raise InvalidTarget("encrypt: level exceeds budget L")
        if layout is not None:
            validate_layout(layout, self.N)
        return SimCt(slots, level, layout)

    def zeros(self, level: int = -1) -> SimCt:
        return self.encrypt(np.zeros(self.N), level)

    def decrypt(self, c: SimCt) -> np.ndarray:
        return c.slots.copy()

    def add(self, a, b):
        self._check(a, "add"), self._check(b, "add")
        self.ledger.count_add()
        return SimCt(a.slots + b.slots, min(a.level, b.level), _merge(a, b))

    def sub(self, a, b):
        self._check(a, "sub"), self._check(b, "sub")
        self.ledger.count_add()
        return SimCt(a.slots - b.slots, min(a.level, b.level), _merge(a, b))

    def add_plain(self, a, p):
        p = np.broadcast_to(np.asarray(p, dtype=np.float64), (self.N,))
        self._check(a, "add_plain")
        self.ledger.count_add()
        return SimCt(a.slots + p, a.level, a.layout)

    def mul(self, a, b):
        self._check(a, "mul"), self._check(b, "mul")
        lvl = min(a.level, b.level)
        if lvl <= 0:
            raise LevelUnderflow("mul: no multiplicative level left")
        self.ledger.count_ct_ct()
        return SimCt(a.slots * b.slots, lvl - 1, _merge(a, b))

    def mul_plain(self, a, p):
        p = np.broadcast_to(np.asarray(p, dtype=np.float64), (self.N,))
        self._check(a, "mul_plain")
        if a.level <= 0:
            raise LevelUnderflow("mul_plain: no multiplicative level left")
        self.ledger.count_ct_pt()
        return SimCt(a.slots * p, a.level - 1, a.layout)

    def mac_plain(self, terms):
        """sum_k ct_k * p_k, charged as the reference's mul_plain/add chain
        (vmm.cpp:214-219): len(terms) ct-pt mults and len(terms)-1 adds."""
        acc = None
        for c, p in terms:
            t = self.mul_plain(c, p)
            acc = t if acc is None else self.add(acc, t)
        return acc

    def mul_sum(self, pairs):
        """sum_i a_i * b_i charged as the reference's mul/add chain
        (kv_attention.cpp:230-235)."""
        acc = None
        for a, b in pairs:
            t = self.mul(a, b)
            acc = t if acc is None else self.add(acc, t)
        return acc

    def mul_plain_lazy(self, a, p):
        """CKKS backends defer this product's rescale to rot_sum_rescale; at
        slot level it is mul_plain (same charge, same level bookkeeping)."""
        return self.mul_plain(a, p)

    def rot_sum_rescale(self, terms, hoisted: bool = False):
        """rot_sum of mul_plain_lazy products (the deferred rescale is invisible
        at slot level)."""
        return self.rot_sum(terms, hoisted)

    def rot_sum(self, terms, hoisted: bool = False):
        """sum_i Rot(a_i, r_i) as the reference's rotate/add chain."""
        acc = None
        for a, r in terms:
            x = self.rotate(a, r, hoisted)
            acc = x if acc is None else self.add(acc, x)
        return acc

    def fold_steps(self, c, rots):
        """c <- c + Rot(c, r) for r in rots (the reference's doubling loops)."""
        for r in rots:
            c = self.add(c, self.rotate(c, r))
        return c

    def fold(self, c, d_head: int, t: int):
        """fold_within_head, kv_attention.cpp:38-41."""
        return self.fold_steps(c, [(1 << l) * t for l in range(d_head.bit_length() - 1)])

    def rotate(self, a, r: int, hoisted: bool = False):
        self._check(a, "rotate")
        s = r % self.N
        if s == 0:
            return a
        self.ledger.count_rotation(hoisted)
        return SimCt(np.roll(a.slots, -s), a.level, None)

    def bootstrap(self, a, target: int):
        self._check(a, "bootstrap")
        if target < 1 or target > self.L:
            raise InvalidTarget(f"bootstrap: target level {target} outside [1, L]")
        self.ledger.count_bootstrap()
        return SimCt(a.slots.copy(), target, a.layout)

    def level_drop(self, a, target: int):
        self._check(a, "level_drop")
        if target < 0 or target > a.level:
            raise InvalidTarget(f"level_drop: target level {target} outside [0, level]")
        return SimCt(a.slots.copy(), target, a.layout)

    def exact_transform(self, a, f: Callable[[np.ndarray], np.ndarray]):
        self._check(a, "exact_transform")
        out = np.asarray(f(a.slots.copy()), dtype=np.float64)
        self._check_slots(out, "exact_transform result")
        return SimCt(out, a.level, a.layout)

    def with_layout(self, c, layout):
        return SimCt(c.slots, c.level, layout)
