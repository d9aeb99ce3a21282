"""B200-native encrypted-decode hot path (arXiv 2602.11470, "Cachemir").

Python mirror of the reference's `slotforge` C++ API
(/root/reference/proj/include/slotforge/*.hpp) over the C ABI in
include/sf_b200.h. Names, argument meaning and error types follow the
reference so code written against slotforge reads the same:

    be = Backend(N=32768, L=13)                 # EngineParams{N, L}  (engine.hpp:19-22)
    x  = be.encrypt(slots, level, layout)       # Backend::encrypt    (engine.cpp:109-121)
    y  = vmm_interleaved(be, x, W, bsgs=True)   # vmm.hpp:74-75
    cache = k_append(be, cache, k_new)          # kv_attention.hpp:79-109 ...

Every operation runs on the GPU through libsf_b200.so (sm_100a kernels); the
package has no CPU fallback and fails loudly if the library is missing.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace
from typing import Optional, Sequence

import numpy as np

from . import _native
from ._native import SfLayout, SfOpCounts, SfParams

__all__ = [
    "Error", "LevelUnderflow", "InvalidTarget", "ShapeMismatch", "LayoutMismatch", "CacheFull", "CacheEmpty",
    "DomainViolation", "ScaleMismatch", "Layout", "make_interleaved", "OpCounts", "Backend", "Ciphertext",
    "VmmPlan", "vmm_interleaved", "predict_interleaved_cost", "AttentionConfig", "KVCache", "rope_apply", "rope_prepare",
    "fused_extract_mask", "k_append", "make_v_pieces", "v_append", "qk_dot", "softmax_times_v",
    "exact_softmax_maps", "kv_from_cts",
]


# --------------------------------------------------------------- errors (types.hpp:16-46)
class Error(RuntimeError):
    pass


class LevelUnderflow(Error):
    pass


class InvalidTarget(Error):
    pass


class ShapeMismatch(Error):
    pass


class LayoutMismatch(Error):
    pass


class CacheFull(Error):
    pass


class CacheEmpty(Error):
    pass


class DomainViolation(Error):
    pass


class ScaleMismatch(Error):
    pass


_CODES = {1: LevelUnderflow, 2: InvalidTarget, 3: ShapeMismatch, 4: LayoutMismatch, 5: CacheFull, 6: CacheEmpty,
          7: DomainViolation, 8: ScaleMismatch}


def _check(status: int):
    if status != 0:
        msg = _native.lib().sf_last_error().decode()
        raise _CODES.get(status, Error)(msg)


# ------------------------------------------------------------------- layouts.hpp:22-33
_KINDS = ["contiguous", "replicated", "interleaved"]


@dataclass(frozen=True)
class Layout:
    kind: str = "interleaved"
    d: int = 0
    t: int = 0
    offset: int = 0
    heads: int = 1
    deferred_mask: bool = False

    def with_(self, **kw) -> "Layout":
        return replace(self, **kw)


def make_interleaved(d: int, N: int, offset: int = 0, heads: int = 1) -> Layout:
    if d <= 0 or N % d:
        raise ShapeMismatch("layout: d*t must equal N")
    return Layout("interleaved", d, N // d, offset, heads, False)


def _to_sf(ly) -> Optional[SfLayout]:
    if ly is None:
        return None
    return SfLayout(1, _KINDS.index(ly.kind), ly.d, ly.t, ly.offset, ly.heads, int(bool(ly.deferred_mask)))


def _from_sf(s: SfLayout) -> Optional[Layout]:
    if not s.valid:
        return None
    return Layout(_KINDS[s.kind], s.d, s.t, s.offset, s.heads, bool(s.deferred_mask))


@dataclass
class OpCounts:
    """engine.hpp:30-49."""
    rotations: int = 0
    hoisted_rotations: int = 0
    ct_pt_mults: int = 0
    ct_ct_mults: int = 0
    additions: int = 0
    bootstraps: int = 0

    @staticmethod
    def _of(s: SfOpCounts) -> "OpCounts":
        return OpCounts(s.rotations, s.hoisted_rotations, s.ct_pt_mults, s.ct_ct_mults, s.additions, s.bootstraps)

    def __sub__(self, o):
        return OpCounts(*(getattr(self, f) - getattr(o, f) for f in self.__dataclass_fields__))

    def asdict(self):
        return {f: getattr(self, f) for f in self.__dataclass_fields__}


# ---------------------------------------------------------------------------- handles
class StepGraph:
    """A captured decode step (Backend.capture): launch() replays every kernel."""

    def __init__(self, be: "Backend", handle: int):
        self.be, self.h = be, handle

    def launch(self):
        _check(_native.lib().sf_graph_launch(self.be.ctx, self.h))

    @property
    def kernel_launches(self) -> int:
        return int(_native.lib().sf_graph_kernel_launches(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h and not _shutdown[0]:
            _native.lib().sf_graph_destroy(h)
            self.h = None


class Ciphertext:
    """Immutable device ciphertext (engine.hpp:24-28 + CKKS scale)."""

    __slots__ = ("be", "h")

    def __init__(self, be: "Backend", handle: int):
        self.be, self.h = be, handle

    def __del__(self):
        h = getattr(self, "h", None)
        if h and not _shutdown[0]:
            _native.lib().sf_ct_release(h)
            self.h = None

    def _info(self):
        lvl, sc, z, ly = C.c_int(), C.c_double(), C.c_int(), SfLayout()
        _check(_native.lib().sf_ct_info(self.h, C.byref(lvl), C.byref(sc), C.byref(z), C.byref(ly)))
        return lvl.value, sc.value, bool(z.value), _from_sf(ly)

    @property
    def level(self) -> int:
        return self._info()[0]

    @property
    def scale(self) -> float:
        return self._info()[1]

    @property
    def is_zero(self) -> bool:
        return self._info()[2]

    @property
    def layout(self) -> Optional[Layout]:
        return self._info()[3]

    def data(self) -> np.ndarray:
        """Raw RNS words [2][level+1][n] (NTT domain)."""
        out = np.empty((2, self.level + 1, self.be.n), dtype=np.uint64)
        _check(_native.lib().sf_ct_export(self.be.ctx, self.h, out.ctypes.data_as(_native.u64p)))
        return out


_shutdown = [False]


def _atexit():
    _shutdown[0] = True


import atexit  # noqa: E402

atexit.register(_atexit)


class _Ledger:
    """CostLedger view (engine.hpp:54-96)."""

    def __init__(self, be):
        self.be = be

    def totals(self) -> OpCounts:
        s = SfOpCounts()
        _check(_native.lib().sf_ledger_totals(self.be.ctx, C.byref(s)))
        return OpCounts._of(s)

    def phase_totals(self, name: str) -> OpCounts:
        s = SfOpCounts()
        _check(_native.lib().sf_ledger_phase_totals(self.be.ctx, name.encode(), C.byref(s)))
        return OpCounts._of(s)

    def reset(self):
        _check(_native.lib().sf_ledger_reset(self.be.ctx))


class _Phase:
    def __init__(self, be, name):
        self.be, self.name = be, name

    def __enter__(self):
        _check(_native.lib().sf_phase_push(self.be.ctx, self.name.encode()))
        return self

    def __exit__(self, *a):
        _check(_native.lib().sf_phase_pop(self.be.ctx))


def _slots(a, N) -> np.ndarray:
    return np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), (N,)))


class Backend:
    """slotforge::Backend over real RNS-CKKS on one B200 (engine.hpp:112-149).

    N is the reference's slot count; the ring degree defaults to 2N. Extra
    keyword arguments select the CKKS parameters (log_n, alpha, q0_bits,
    scale_bits, special_bits, seed, device); see DESIGN.md §3.1."""

    def __init__(self, N: int, L: int, log_n: int = 0, alpha: int = 0, q0_bits: int = 0, scale_bits: int = 0,
                 special_bits: int = 0, seed: int = 1, device: int = 0):
        p = SfParams(N, L, log_n, alpha, q0_bits, scale_bits, special_bits, device, seed)
        h = C.c_void_p()
        _check(_native.lib().sf_context_create(C.byref(p), C.byref(h)))
        self.ctx = h.value
        n, slots, LL, al, npr = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_native.lib().sf_context_info(self.ctx, C.byref(n), C.byref(slots), C.byref(LL), C.byref(al),
                                              C.byref(npr), None))
        self.N, self.L, self.n, self.alpha = slots.value, LL.value, n.value, al.value
        self.primes = np.empty(npr.value, dtype=np.uint64)
        _check(_native.lib().sf_context_info(self.ctx, None, None, None, None, None,
                                              self.primes.ctypes.data_as(_native.u64p)))
        self.ledger = _Ledger(self)
        self.seed = seed

    def __del__(self):
        if getattr(self, "ctx", None) and not _shutdown[0]:
            _native.lib().sf_context_destroy(self.ctx)
            self.ctx = None

    def params(self):
        return (self.N, self.L)

    def phase(self, name: str):
        return _Phase(self, name)

    def _ct(self, fn, *args) -> Ciphertext:
        out = C.c_void_p()
        _check(fn(self.ctx, *args, C.byref(out)))
        return Ciphertext(self, out.value)

    def synchronize(self):
        _check(_native.lib().sf_synchronize(self.ctx))

    # --- CUDA graphs of whole steps (include/sf_b200.h sf_graph_*)
    def capture(self, fn, *args, **kw):
        """Capture everything fn(*args, **kw) enqueues into one CUDA graph
        (nothing runs during the capture). Returns (graph, fn's result): the
        result's ciphertexts hold the latest replay's values; inputs created
        before the capture are fed with refill() between replays.

        Lazily built tables / keys / cached plaintexts need one host upload on
        first use, which a capture cannot contain: if fn hits one, the partial
        capture is discarded, fn runs once eagerly (warming every cache) and
        the capture is retried once."""
        lib = _native.lib()
        for attempt in range(2):
            _check(lib.sf_graph_capture_begin(self.ctx))
            err = None
            try:
                res = fn(*args, **kw)
            except Exception as e:  # noqa: BLE001 - the capture must be ended whatever fn raised
                err = e
            g = C.c_void_p()
            st = lib.sf_graph_capture_end(self.ctx, C.byref(g))
            if err is None:
                _check(st)
                return StepGraph(self, g.value), res
            if g.value:
                lib.sf_graph_destroy(g)
            if attempt == 0 and isinstance(err, InvalidTarget) and "eagerly" in str(err):
                fn(*args, **kw)  # warm-up run, then capture again
                self.synchronize()
                continue
            raise err

    def set_value_shard(self, rank: int, world: int) -> None:
        """Score*V giant groups this process owns (sf_set_value_shard): the appends build
        aligned companions for those only (automatic with the library-stream / peer
        exchanges)."""
        _check(_native.lib().sf_set_value_shard(self.ctx, rank, world))

    def mem_reserve(self, nbytes: int) -> None:
        """Grow the device pool once by nbytes (sf_mem_reserve): a setup step so
        that a later, larger working set never maps new memory mid-token."""
        _check(_native.lib().sf_mem_reserve(self.ctx, int(nbytes)))

    def key_stats(self):
        """(switching keys held, bytes, bytes if untruncated) (sf_key_stats)."""
        n, b, f = C.c_int(), C.c_size_t(), C.c_size_t()
        _check(_native.lib().sf_key_stats(self.ctx, C.byref(n), C.byref(b), C.byref(f)))
        return n.value, b.value, f.value

    def mem_stats(self):
        """(graph-node bytes, pool bytes) currently allocated (sf_mem_stats)."""
        g, p = C.c_size_t(), C.c_size_t()
        _check(_native.lib().sf_mem_stats(self.ctx, C.byref(g), C.byref(p)))
        return g.value, p.value

    def rotate_many(self, cts, r: int):
        """Rot(c, r) for every c, one batched key-switching pass (sf_rotate_many)."""
        k = len(cts)
        arr = (C.c_void_p * k)(*[c.h for c in cts])
        outs = (C.c_void_p * k)()
        _check(_native.lib().sf_rotate_many(self.ctx, arr, k, int(r), outs))
        return [Ciphertext(self, outs[i]) for i in range(k)]

    def bench_ntt(self, limbs: int, count: int, reps: int = 10) -> float:
        """Device ms per limb NTT of a batch of count x limbs limbs (sf_bench_ntt)."""
        ms = C.c_double()
        _check(_native.lib().sf_bench_ntt(self.ctx, limbs, count, reps, C.byref(ms)))
        return ms.value

    # --- wire format (include/sf_b200.h sf_ct_serialize / sf_ct_deserialize)
    def serialize(self, ct: "Ciphertext") -> bytes:
        n = C.c_size_t()
        _check(_native.lib().sf_ct_wire_size(self.ctx, ct.h, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        ln = C.c_size_t()
        _check(_native.lib().sf_ct_serialize(self.ctx, ct.h, buf, n.value, C.byref(ln)))
        return buf.raw[:ln.value]

    def deserialize(self, data: bytes) -> "Ciphertext":
        return self._ct(_native.lib().sf_ct_deserialize, data, len(data))

    def refill(self, ct: "Ciphertext", words: np.ndarray):
        """Overwrite ct's device words from (pinned) host memory, stream-ordered."""
        w = np.ascontiguousarray(words, dtype=np.uint64)
        _check(_native.lib().sf_ct_refill(self.ctx, ct.h, w.ctypes.data_as(_native.u64p)))

    def stage(self, ct: "Ciphertext", words: np.ndarray, slot: int):
        """refill() issued on a side stream that overlaps the work enqueued until
        stage_wait(slot) (sf_ct_stage). `words` is used in place (pinned, C-contiguous
        uint64; a captured graph re-reads it on every replay), so it must outlive the
        copy -- and the graph."""
        if not (isinstance(words, np.ndarray) and words.dtype == np.uint64 and words.flags.c_contiguous):
            raise TypeError("stage: words must be a C-contiguous uint64 array (used in place)")
        _check(_native.lib().sf_ct_stage(self.ctx, ct.h, words.ctypes.data_as(_native.u64p), int(slot)))

    def stage_out(self, ct: "Ciphertext", words: np.ndarray, slot: int):
        """Read ct's words [2][level+1][n] into `words` (pinned, C-contiguous uint64,
        used in place) on the side stream, overlapping the work enqueued until
        stage_wait(slot) (sf_ct_stage_out); valid after synchronize()."""
        if not (isinstance(words, np.ndarray) and words.dtype == np.uint64 and words.flags.c_contiguous):
            raise TypeError("stage_out: words must be a C-contiguous uint64 array (used in place)")
        if words.size != 2 * (ct.level + 1) * self.n:
            raise ValueError("stage_out: words must hold [2][level+1][n] words")
        _check(_native.lib().sf_ct_stage_out(self.ctx, ct.h, words.ctypes.data_as(_native.u64p), int(slot)))

    def stage_wait(self, slot: int):
        """Join the staged copy of `slot` back into the library stream (sf_ct_stage_wait)."""
        _check(_native.lib().sf_ct_stage_wait(self.ctx, int(slot)))

    # --- client side (off-ledger)
    def encrypt(self, slots, level: int = -1, layout=None, seed: Optional[int] = None) -> Ciphertext:
        s = np.asarray(slots, dtype=np.float64)
        if s.shape != (self.N,):
            raise ShapeMismatch(f"encrypt: expected {self.N} slots, got {s.size}")
        s = np.ascontiguousarray(s)
        ly = _to_sf(layout)
        return self._ct(_native.lib().sf_encrypt, s.ctypes.data_as(_native.dp), level,
                        C.byref(ly) if ly else None, C.c_uint64(seed or 0), int(seed is not None))

    def zeros(self, level: int = -1) -> Ciphertext:
        return self._ct(_native.lib().sf_zeros, level)

    def decrypt(self, ct: Ciphertext) -> np.ndarray:
        out = np.empty(self.N)
        _check(_native.lib().sf_decrypt(self.ctx, ct.h, out.ctypes.data_as(_native.dp)))
        return out

    def encode(self, slots, scale: float, limbs: int) -> np.ndarray:
        s = _slots(slots, self.N)
        out = np.empty((limbs, self.n), dtype=np.uint64)
        _check(_native.lib().sf_encode(self.ctx, s.ctypes.data_as(_native.dp), scale, limbs,
                                        out.ctypes.data_as(_native.u64p)))
        return out

    def import_ct(self, words, level, scale, layout=None, zero=False) -> Ciphertext:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        ly = _to_sf(layout)
        return self._ct(_native.lib().sf_ct_import, w.ctypes.data_as(_native.u64p), level, scale, int(zero),
                        C.byref(ly) if ly else None)

    def secret_key(self) -> np.ndarray:
        out = np.empty((len(self.primes), self.n), dtype=np.uint64)
        _check(_native.lib().sf_secret_key_export(self.ctx, out.ctypes.data_as(_native.u64p)))
        return out

    def switching_key(self, galois_elt: int) -> np.ndarray:
        beta = (self.L + 1 + self.alpha - 1) // self.alpha
        out = np.empty((beta, 2, len(self.primes), self.n), dtype=np.uint64)
        _check(_native.lib().sf_switching_key_export(self.ctx, C.c_uint64(galois_elt),
                                                      out.ctypes.data_as(_native.u64p)))
        return out

    def galois_elt(self, r: int) -> int:
        return _native.lib().sf_galois_elt(self.ctx, r)

    def gen_rotation_keys(self, rotations: Sequence[int]):
        arr = (C.c_int * len(rotations))(*rotations)
        _check(_native.lib().sf_gen_rotation_keys(self.ctx, arr, len(rotations)))

    # --- evaluator ops (ledger-charged, engine.cpp:143-214)
    def add(self, a, b):
        return self._ct(_native.lib().sf_add, a.h, b.h)

    def sub(self, a, b):
        return self._ct(_native.lib().sf_sub, a.h, b.h)

    def add_plain(self, a, p):
        s = _slots(p, self.N)
        return self._ct(_native.lib().sf_add_plain, a.h, s.ctypes.data_as(_native.dp))

    def mul(self, a, b):
        return self._ct(_native.lib().sf_mul, a.h, b.h)

    def mul_plain(self, a, p):
        s = _slots(p, self.N)
        return self._ct(_native.lib().sf_mul_plain, a.h, s.ctypes.data_as(_native.dp))

    def mac_plain(self, terms):
        cts = (C.c_void_p * len(terms))(*[c.h for c, _ in terms])
        pts = np.ascontiguousarray(np.stack([_slots(p, self.N) for _, p in terms]))
        return self._ct(_native.lib().sf_mac_plain, cts, pts.ctypes.data_as(_native.dp), len(terms))

    def rotate(self, a, r: int, hoisted: bool = False):
        return self._ct(_native.lib().sf_rotate, a.h, int(r), int(hoisted))

    def rotate_hoisted(self, a, rs: Sequence[int]):
        arr = (C.c_int * len(rs))(*rs)
        outs = (C.c_void_p * len(rs))()
        _check(_native.lib().sf_rotate_hoisted(self.ctx, a.h, arr, len(rs), outs))
        return [Ciphertext(self, o) for o in outs]

    def level_drop(self, a, target: int):
        return self._ct(_native.lib().sf_level_drop, a.h, target)

    def bootstrap(self, a, target: int):
        return self._ct(_native.lib().sf_bootstrap, a.h, target)

    def exact_transform(self, a, f):
        """Oracle hook (engine.cpp:208-214) as a client round trip: decrypt,
        apply f, re-encrypt at the same level (free, level-neutral)."""
        out = np.asarray(f(self.decrypt(a)), dtype=np.float64)
        if out.shape != (self.N,):
            raise ShapeMismatch("exact_transform result: wrong slot count")
        return self.encrypt(out, a.level, a.layout)

    def with_layout(self, ct, layout):
        ly = _to_sf(layout)
        return self._ct(_native.lib().sf_ct_with_layout, ct.h, C.byref(ly) if ly else None)

    # --- timing / accounting
    def event_record(self, slot: int):
        _check(_native.lib().sf_event_record(self.ctx, slot))

    def event_elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        _check(_native.lib().sf_event_elapsed_ms(self.ctx, a, b, C.byref(ms)))
        return ms.value

    def kernel_launches(self) -> int:
        return _native.lib().sf_kernel_launches(self.ctx)


# ------------------------------------------------------------------------------ VMM
class VmmPlan:
    """Pre-encoded interleaved diagonals (vmm.cpp:159-175) for one weight matrix
    at one input level; W=None selects the reference bench weight
    sin(0.001 (31 r + c) + 0.25) (slotforge_cli.cpp:88-92)."""

    def __init__(self, be: Backend, W, rows: int, cols: int, level: int, in_offset: int = 0, out_offset: int = 0,
                 bsgs: bool = True):
        self.be, self.rows, self.cols, self.level = be, rows, cols, level
        self.in_offset, self.out_offset, self.bsgs = in_offset, out_offset, bsgs
        h = C.c_void_p()
        if W is not None:
            W = np.ascontiguousarray(np.asarray(W, dtype=np.float64))
            if W.shape != (rows, cols):
                raise ShapeMismatch("vmm plan: W shape")
        _check(_native.lib().sf_vmm_plan_create(be.ctx, W.ctypes.data_as(_native.dp) if W is not None else None,
                                                 rows, cols, level, in_offset, out_offset, int(bsgs), C.byref(h)))
        self.h = h.value

    @classmethod
    def _wrap(cls, be, handle, level, in_offset, out_offset, bsgs):
        p = cls.__new__(cls)
        p.be, p.rows, p.cols, p.level = be, None, None, level
        p.in_offset, p.out_offset, p.bsgs, p.h = in_offset, out_offset, bsgs, handle
        return p

    def save(self, path: str) -> None:
        """Encoded-plan cache: diagonals (NTT words) + weights, reloadable with vmm_plan_load."""
        _check(_native.lib().sf_vmm_plan_save(self.be.ctx, self.h, path.encode()))

    def __del__(self):
        if getattr(self, "h", None) and not _shutdown[0]:
            _native.lib().sf_vmm_plan_destroy(self.h)
            self.h = None


def save_weight(dir: str, name: str, W) -> None:
    """The reference's weight files (layouts.cpp:158-170): <name>.bin row-major
    float64 + <name>.json {"name", "rows", "cols"}."""
    import json
    import os
    W = np.ascontiguousarray(np.asarray(W, dtype=np.float64))
    os.makedirs(dir, exist_ok=True)
    W.tofile(os.path.join(dir, name + ".bin"))
    with open(os.path.join(dir, name + ".json"), "w") as f:
        f.write(json.dumps({"name": name, "rows": int(W.shape[0]), "cols": int(W.shape[1])}, indent=2) + "\n")


def vmm_plan_from_file(be: Backend, dir: str, name: str, level: int, in_offset: int = 0, out_offset: int = 0,
                       bsgs: bool = True) -> "VmmPlan":
    """A VMM plan straight from the reference's weight files (load_weight, layouts.cpp:172-184)."""
    h = C.c_void_p()
    _check(_native.lib().sf_vmm_plan_create_from_file(be.ctx, dir.encode(), name.encode(), level, in_offset,
                                                       out_offset, int(bsgs), C.byref(h)))
    return VmmPlan._wrap(be, h.value, level, in_offset, out_offset, bsgs)


def vmm_plan_load(be: Backend, path: str) -> "VmmPlan":
    """Reload an encoded-plan cache written by VmmPlan.save (no re-encoding)."""
    h = C.c_void_p()
    _check(_native.lib().sf_vmm_plan_load(be.ctx, path.encode(), C.byref(h)))
    return VmmPlan._wrap(be, h.value, -1, 0, 0, True)


class VmmBatchPlan(VmmPlan):
    """Pre-encoded token-batched square diagonals (vmm.cpp:426-433) for vmm_batch."""

    def __init__(self, be: Backend, W, level: int, bsgs: bool = True):
        W = np.ascontiguousarray(np.asarray(W, dtype=np.float64))
        self.be, self.rows, self.cols, self.level, self.bsgs = be, W.shape[0], W.shape[1], level, bsgs
        self.in_offset = self.out_offset = 0
        h = C.c_void_p()
        _check(_native.lib().sf_vmm_batch_plan_create(be.ctx, W.ctypes.data_as(_native.dp), W.shape[0], W.shape[1],
                                                       level, int(bsgs), C.byref(h)))
        self.h = h.value


def predict_interleaved_cost(be: Backend, rows: int, cols: int, bsgs: bool = False, mask_output: bool = False):
    """vmm.cpp:473-488 -> (rotations, ct_pt_mults, depth)."""
    r, c, d = C.c_longlong(), C.c_longlong(), C.c_int()
    _check(_native.lib().sf_vmm_predict(be.ctx, rows, cols, int(bsgs), int(mask_output), C.byref(r), C.byref(c),
                                         C.byref(d)))
    return r.value, c.value, d.value


def vmm_interleaved_multi(be: Backend, x: Ciphertext, plans, mask_output: bool = False):
    """[vmm_interleaved(be, x, None, plan=p, mask_output=mask_output) for p in plans],
    word for word and in the ledger, with the input-only ladder and baby steps
    evaluated once (sf_vmm_interleaved_multi)."""
    k = len(plans)
    arr = (C.c_void_p * k)(*[p.h for p in plans])
    outs = (C.c_void_p * k)()
    _check(_native.lib().sf_vmm_interleaved_multi(be.ctx, x.h, arr, k, int(mask_output), outs))
    return [Ciphertext(be, outs[i]) for i in range(k)]


def vmm_interleaved_many(be: Backend, xs, plan: "VmmPlan", mask_output: bool = False):
    """[vmm_interleaved(be, x, None, plan=plan, mask_output=mask_output) for x in xs]
    word for word and in the ledger, every stage batched across the inputs
    (sf_vmm_interleaved_many)."""
    k = len(xs)
    arr = (C.c_void_p * k)(*[x.h for x in xs])
    outs = (C.c_void_p * k)()
    _check(_native.lib().sf_vmm_interleaved_many(be.ctx, arr, k, plan.h, int(mask_output), outs))
    return [Ciphertext(be, outs[i]) for i in range(k)]


def vmm_interleaved(be: Backend, x: Ciphertext, W, bsgs: bool = False, out_offset: int = 0,
                    mask_output: bool = False, plan: Optional[VmmPlan] = None) -> Ciphertext:
    """vmm_interleaved (vmm.hpp:74-75). Pass `plan` to reuse pre-encoded
    diagonals; otherwise a plan for W at x's level is built (offline cost)."""
    if plan is None:
        ly = x.layout
        if ly is None or ly.kind != "interleaved":
            raise LayoutMismatch("vmm_interleaved: input must carry an interleaved layout")
        W = np.asarray(W, dtype=np.float64)
        plan = VmmPlan(be, W, W.shape[0], W.shape[1], max(x.level, 1), ly.offset, out_offset, bsgs)
    return be._ct(_native.lib().sf_vmm_interleaved, x.h, plan.h, int(mask_output))


# ------------------------------------------------------------------------ attention
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


class KVCache:
    """Copy-on-write KV cache handle (kv_attention.hpp:49-54)."""

    def __init__(self, be: Backend, cfg: AttentionConfig, handle: Optional[int] = None):
        self.be, self.cfg = be, cfg
        if handle is None:
            h = C.c_void_p()
            _check(_native.lib().sf_kv_create(be.ctx, cfg.d, cfg.H, cfg.n0, cfg.n_max, C.byref(h)))
            handle = h.value
        self.h = handle

    def __del__(self):
        if getattr(self, "h", None) and not _shutdown[0]:
            _native.lib().sf_kv_release(self.h)
            self.h = None

    def _info(self):
        a, b, c, d = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_native.lib().sf_kv_info(self.h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return a.value, b.value, c.value, d.value

    @property
    def n_prime(self):
        return self._info()[0]

    @property
    def k_cts(self):
        n = self._info()[1]
        return [self._get(0, 0, i) for i in range(n)]

    @property
    def v_cts(self):
        _, _, g, nv = self._info()
        return [[self._get(1, gi, i) for i in range(nv)] for gi in range(g)]

    def _get(self, which, g, idx):
        out = C.c_void_p()
        _check(_native.lib().sf_kv_get(self.h, which, g, idx, C.byref(out)))
        return Ciphertext(self.be, out.value)


def kv_from_cts(be: Backend, cfg: AttentionConfig, n_prime: int, k_cts, v_cts) -> KVCache:
    ks = (C.c_void_p * max(1, len(k_cts)))(*[c.h for c in k_cts])
    flat = [c for g in v_cts for c in g]
    vs = (C.c_void_p * max(1, len(flat)))(*[c.h for c in flat])
    h = C.c_void_p()
    _check(_native.lib().sf_kv_from_cts(be.ctx, cfg.d, cfg.H, cfg.n0, cfg.n_max, n_prime, ks, len(k_cts), vs,
                                         len(v_cts), C.byref(h)))
    return KVCache(be, cfg, h.value)


def rope_apply(be: Backend, x: Ciphertext, cfg: AttentionConfig, position: int, base: float = 10000.0):
    """kv_attention.cpp:111-117."""
    return be._ct(_native.lib().sf_rope_apply, x.h, cfg.d, cfg.H, position, base)


def rope_prepare(be: Backend, cfg: AttentionConfig, position: int, level: int, offset: int = 0,
                 base: float = 10000.0) -> None:
    """Encode the RoPE plaintexts rope_apply will need for an input interleaved
    at `offset` with `level` at `position` ahead of time (stream-ordered upload,
    no host wait): a decode loop prepares token p+1 while token p runs."""
    _check(_native.lib().sf_rope_prepare(be.ctx, cfg.d, cfg.H, offset, level, int(position), base))


def fused_extract_mask(be: Backend, x: Ciphertext, coeff=None):
    """fused_extract with a mask successor (vmm.cpp:102-108)."""
    c = None if coeff is None else _slots(coeff, be.N)
    return be._ct(_native.lib().sf_fused_extract_mask, x.h, c.ctypes.data_as(_native.dp) if c is not None else None)


def k_append(be: Backend, cache: KVCache, k_new: Ciphertext) -> KVCache:
    out = C.c_void_p()
    _check(_native.lib().sf_k_append(be.ctx, cache.h, k_new.h, C.byref(out)))
    return KVCache(be, cache.cfg, out.value)


def make_v_pieces(be: Backend, cache: KVCache, v_open: Ciphertext, position: int):
    parts = (C.c_void_p * cache.cfg.d_head)()
    _check(_native.lib().sf_make_v_pieces(be.ctx, cache.h, v_open.h, position, parts))
    return [Ciphertext(be, p) for p in parts]


def v_append(be: Backend, cache: KVCache, parts) -> KVCache:
    arr = (C.c_void_p * max(1, len(parts)))(*[p.h for p in parts])
    out = C.c_void_p()
    _check(_native.lib().sf_v_append(be.ctx, cache.h, arr, len(parts), C.byref(out)))
    return KVCache(be, cache.cfg, out.value)


def qk_dot(be: Backend, q: Ciphertext, cache: KVCache):
    gt = cache.cfg.group_tokens
    cap = max(1, (max(cache.n_prime, 1) + gt - 1) // gt)
    maps = (C.c_void_p * cap)()
    n = C.c_int()
    _check(_native.lib().sf_qk_dot(be.ctx, q.h, cache.h, maps, C.byref(n)))
    return [Ciphertext(be, maps[i]) for i in range(n.value)]


def softmax_times_v(be: Backend, probs, cache: KVCache) -> Ciphertext:
    arr = (C.c_void_p * max(1, len(probs)))(*[p.h for p in probs])
    return be._ct(_native.lib().sf_softmax_times_v, arr, len(probs), cache.h)


def exact_softmax_maps(be: Backend, maps, cfg: AttentionConfig, n_prime: int):
    """Client-side oracle hook (kv_attention.cpp:395-412): decrypt the score
    maps, take the exact per-head softmax over the first n_prime scores,
    re-encrypt at the same level (no ledger cost)."""
    gt = cfg.group_tokens
    slots = [be.decrypt(m) for m in maps]
    out = [np.zeros(cfg.N) for _ in maps]
    for h in range(cfg.H):
        sc = np.array([slots[v // gt][h * gt + v % gt] for v in range(n_prime)])
        p = np.exp(sc - sc.max())
        p /= p.sum()
        for v in range(n_prime):
            out[v // gt][h * gt + v % gt] = p[v]
    return [be.exact_transform(m, (lambda _s, o=o: o)) for m, o in zip(maps, out)]


# --------------------------------------------------------------------- prefill
def inner_rotate(be: Backend, x: Ciphertext, r: int, block: int, hoisted: bool = False) -> Ciphertext:
    """vmm.cpp:30-43."""
    return be._ct(_native.lib().sf_inner_rotate, x.h, int(r), int(block), int(hoisted))


def vmm_batch(be: Backend, x: Ciphertext, W=None, bsgs: bool = True, plan: Optional[VmmBatchPlan] = None):
    """vmm.cpp:417-467 (pass `plan` to reuse the encoded diagonals)."""
    if plan is None:
        plan = VmmBatchPlan(be, W, x.level, bsgs)
    return be._ct(_native.lib().sf_vmm_batch, x.h, plan.h)


def rope_apply_batch(be: Backend, x: Ciphertext, cfg: AttentionConfig, first_pos: int, base: float = 10000.0):
    """kv_attention.cpp:119-129."""
    return be._ct(_native.lib().sf_rope_apply_batch, x.h, cfg.d, cfg.H, int(first_pos), base)


def prefill(be: Backend, x_prompt, Wq, Wk, Wv, cfg: AttentionConfig, softmax_fn, rope_base: float = 10000.0):
    """kv_attention.cpp:245-376 -> (attention cts, KVCache). The score maps are
    handed to softmax_fn(be, maps[p][g][rho], cfg, n0) between the two halves."""
    lib = _native.lib()
    t, gt, n0 = cfg.t, cfg.group_tokens, cfg.n0
    P = len(x_prompt)
    lvl = x_prompt[0].level if P else 0
    plans = [p if isinstance(p, VmmBatchPlan) else VmmBatchPlan(be, p, lvl) for p in (Wq, Wk, Wv)]
    xs = (C.c_void_p * max(1, P))(*[x.h for x in x_prompt])
    shape = [(p * t) // gt + 1 for p in range(P)]
    cap = max(1, sum(shape) * t)
    maps_out = (C.c_void_p * cap)()
    n = C.c_int()
    kv = C.c_void_p()
    _check(lib.sf_prefill_scores(be.ctx, xs, P, plans[0].h, plans[1].h, plans[2].h, cfg.d, cfg.H, n0, cfg.n_max,
                                 rope_base, C.byref(kv), maps_out, cap, C.byref(n)))
    cache = KVCache(be, cfg, kv.value)
    flat = [Ciphertext(be, maps_out[i]) for i in range(n.value)]
    maps, k = [], 0
    for p in range(P):
        rows = []
        for _ in range(shape[p]):
            rows.append(flat[k:k + t])
            k += t
        maps.append(rows)
    probs = softmax_fn(be, maps, cfg, n0)
    pf = [c for mp in probs for row in mp for c in row]
    arr = (C.c_void_p * max(1, len(pf)))(*[c.h for c in pf])
    att_out = (C.c_void_p * max(1, P))()
    na = C.c_int()
    _check(lib.sf_prefill_attend(be.ctx, arr, len(pf), cache.h, att_out, P, C.byref(na)))
    return [Ciphertext(be, att_out[i]) for i in range(na.value)], cache


def exact_softmax_prefill_maps(be: Backend, maps, cfg: AttentionConfig, n0: int):
    """Client-side oracle hook (kv_attention.cpp:414-454): decrypt the packed
    prefill maps, exact causal softmax per query and head, re-encrypt each map
    at its level (no ledger cost)."""
    t, gt = cfg.t, cfg.group_tokens
    slots = [[[be.decrypt(c) for c in row] for row in mp] for mp in maps]
    out = [[[np.zeros(cfg.N) for _ in range(t)] for _ in mp] for mp in maps]
    for p in range(len(maps)):
        for tau in range(t):
            query = p * t + tau
            if query >= n0:
                continue
            for h in range(cfg.H):
                idx = []
                for k in range(query + 1):
                    g, rho = k // gt, (k % t - tau) % t
                    idx.append((g, rho, h * gt + (k - g * gt) // t * t + tau))
                sc = np.array([slots[p][g][r][i] for g, r, i in idx])
                e = np.exp(sc - sc.max())
                pr = e / e.sum()
                for (g, r, i), v in zip(idx, pr):
                    out[p][g][r][i] = v
    return [[[be.exact_transform(c, (lambda _s, o=out[p][g][r]: o)) for r, c in enumerate(row)]
             for g, row in enumerate(mp)] for p, mp in enumerate(maps)]
