"""Decoder harness over the encrypted hot path.

A plan-driven decode loop for the reference's toy gated-FFN transformer
(harness.hpp:1-22), running every homomorphic stage on the GPU backend:
projections (vmm_interleaved), rotary + cache appends, QK^T, Score*V, the
residual adds and the gate product. Exact-mode nonlinearities (softmax, norm,
SiLU) and plan bootstraps are client round trips (decrypt -> f -> re-encrypt),
exactly the oracle hooks the reference runs them as (engine.cpp:193-214,
nonlinear.cpp:553-593, kv_attention.cpp:395-412).

Mirrors (file:line in /root/reference/proj):
  ModelConfig / validate_model_config     harness.hpp:38-60, harness.cpp:161-173
  make_weights (seeded draw order)        harness.cpp:197-223 (std::mt19937_64 +
                                          libstdc++ normal_distribution, ported below)
  seeded_prompt                           harness.cpp:280-287 (uniform_int_distribution)
  plaintext_reference                     harness.cpp:291-350
  run_decode_step                         harness.cpp:425-659
  prefill_prompt                          harness.cpp:719-857
  run_generation / Report                 harness.cpp:943-1053

The placement solver (placement.cpp) is out of scope: the plan
is an input -- PlacementPlan JSON as the reference writes it (plan.to_json) --
exactly as run_decode_step takes a `const PlacementPlan*`.

The stages are written against a small operator interface (`GpuOps` here);
tests drive the same loop with the slot-simulator oracle to pin the level
trace and per-phase ledger against the reference's own report.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field, asdict, replace
from typing import Dict, List, Optional

import numpy as np

STAGE_NAMES = ["Q, K, V", "RoPE & Cache", "QK^T", "Softmax", "Score*V", "Output projection", "Add & Norm",
               "Up & Gate projection", "SiLU", "Down projection", "Add & Norm"]  # harness.cpp:24-34
NORM_EPS = 1e-5  # harness.cpp:22
PHASE_ORDER = ["Amortized Prefilling"] + [n for i, n in enumerate(STAGE_NAMES) if i != 10] + ["Bootstrappings"]


class ShapeMismatch(ValueError):
    pass


class LevelUnderflow(RuntimeError):
    pass


# ----------------------------------------------------------------------- config
@dataclass
class ModelConfig:
    """harness.hpp:38-54 (defaults = the reference's desk configuration)."""
    d: int = 64
    H: int = 4
    n_layers: int = 2
    ffn_alpha: int = 4
    vocab: int = 32
    N: int = 256
    L: int = 13
    rope_base: float = 10000.0
    mode: str = "exact"
    seed: int = 1

    @staticmethod
    def from_json(obj) -> "ModelConfig":
        o = json.loads(obj) if isinstance(obj, str) else obj
        return ModelConfig(**{k: o[k] for k in ModelConfig.__dataclass_fields__ if k in o})


def _pow2(v):
    return v > 0 and (v & (v - 1)) == 0


def padded_dim(d: int) -> int:
    p = 1
    while p < d:
        p <<= 1
    return p


def validate_model_config(cfg: ModelConfig) -> None:
    """harness.cpp:161-173."""
    if not (_pow2(cfg.N) and _pow2(cfg.d) and _pow2(cfg.H)):
        raise ShapeMismatch("model config: N, d, H must be powers of two")
    if cfg.d > cfg.N:
        raise ShapeMismatch("model config: d must not exceed N")
    if cfg.H > cfg.d or (cfg.d // cfg.H) % 2:
        raise ShapeMismatch("model config: head width d/H must be a positive even number")
    if cfg.n_layers < 1:
        raise ShapeMismatch("model config: need at least one block")
    if cfg.ffn_alpha < 1 or padded_dim(cfg.ffn_alpha * cfg.d) > cfg.N:
        raise ShapeMismatch("model config: padded FFN width must fit the slot count")
    if cfg.vocab < 2:
        raise ShapeMismatch("model config: vocab must be at least 2")
    if cfg.L < 1:
        raise ShapeMismatch("model config: level budget must be at least 1")
    if not cfg.rope_base > 1.0:
        raise ShapeMismatch("model config: rope_base must exceed 1")
    if cfg.mode not in ("exact", "approx"):
        raise ShapeMismatch(f'model config: mode must be "exact" or "approx", got "{cfg.mode}"')


# ------------------------------------------------------------ seeded generators
class MT19937_64:
    """std::mt19937_64 (the standard's parameters), numpy-vectorised twist."""
    _N, _M = 312, 156
    _A = np.uint64(0xB5026F5AA96619E9)
    _UP, _LO = np.uint64(0xFFFFFFFF80000000), np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = [seed & 0xFFFFFFFFFFFFFFFF]
        for i in range(1, self._N):
            p = mt[-1]
            mt.append((6364136223846793005 * (p ^ (p >> 62)) + i) & 0xFFFFFFFFFFFFFFFF)
        self.mt = np.array(mt, dtype=np.uint64)
        self.buf: List[int] = []
        self.pos = 0

    def _twist(self):
        mt, N, M = self.mt, self._N, self._M
        one = np.uint64(1)

        def step(lo, hi, nxt, far):
            y = (mt[lo:hi] & self._UP) | (nxt & self._LO)
            return far ^ (y >> one) ^ np.where((y & one) != 0, self._A, np.uint64(0))
        mt[0:N - M] = step(0, N - M, mt[1:N - M + 1], mt[M:N])
        mt[N - M:N - 1] = step(N - M, N - 1, mt[N - M + 1:N], mt[0:M - 1])
        mt[N - 1:N] = step(N - 1, N, mt[0:1], mt[M - 1:M])
        y = mt.copy()
        y ^= (y >> np.uint64(29)) & np.uint64(0x5555555555555555)
        y ^= (y << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        y ^= (y << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        y ^= y >> np.uint64(43)
        self.buf = [int(v) for v in y]
        self.pos = 0

    def __call__(self) -> int:
        if self.pos >= len(self.buf):
            self._twist()
        v = self.buf[self.pos]
        self.pos += 1
        return v


class NormalDist:
    """libstdc++ std::normal_distribution<double> (Marsaglia polar method, one
    cached value) over generate_canonical<double, 53>: u = double(g()) / 2^64."""

    def __init__(self):
        self.saved = None

    @staticmethod
    def _canon(g) -> float:
        r = float(g()) / 18446744073709551616.0
        return r if r < 1.0 else math.nextafter(1.0, 0.0)

    def __call__(self, g) -> float:
        if self.saved is not None:
            v, self.saved = self.saved, None
            return v
        while True:
            x = 2.0 * self._canon(g) - 1.0
            y = 2.0 * self._canon(g) - 1.0
            r2 = x * x + y * y
            if not (r2 > 1.0 or r2 == 0.0):
                break
        mult = math.sqrt(-2 * math.log(r2) / r2)
        self.saved = x * mult
        return y * mult


def _randn(rows, cols, scale, g):  # harness.cpp:49-55: fresh distribution per matrix
    dist = NormalDist()
    return np.array([scale * dist(g) for _ in range(rows * cols)], dtype=np.float64).reshape(rows, cols)


def _randn_vec(n, base, spread, g):  # harness.cpp:57-62
    dist = NormalDist()
    return np.array([base + spread * dist(g) for _ in range(n)], dtype=np.float64)


@dataclass
class Block:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w_gate: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray
    gamma1: np.ndarray
    beta1: np.ndarray
    gamma2: np.ndarray
    beta2: np.ndarray


@dataclass
class ModelWeights:
    embedding: np.ndarray
    blocks: List[Block]


def make_weights(cfg: ModelConfig) -> ModelWeights:
    """harness.cpp:197-223: one generator, the reference's draw order."""
    validate_model_config(cfg)
    g = MT19937_64(cfg.seed)
    d, ad = cfg.d, cfg.ffn_alpha * cfg.d
    sd, sad = 1.0 / math.sqrt(d), 1.0 / math.sqrt(ad)
    score = 1.0 / math.sqrt(d // cfg.H)
    emb = _randn(cfg.vocab, d, 1.0, g)
    blocks = []
    for _ in range(cfg.n_layers):
        wq = _randn(d, d, sd * score, g)
        wk = _randn(d, d, sd, g)
        wv = _randn(d, d, sd, g)
        wo = _randn(d, d, sd, g)
        wg = _randn(d, ad, sd, g)
        wu = _randn(d, ad, sd, g)
        wd = _randn(ad, d, sad, g)
        g1 = _randn_vec(d, 1.0, 0.1, g)
        b1 = _randn_vec(d, 0.0, 0.01, g)
        g2 = _randn_vec(d, 1.0, 0.1, g)
        b2 = _randn_vec(d, 0.0, 0.01, g)
        blocks.append(Block(wq, wk, wv, wo, wg, wu, wd, g1, b1, g2, b2))
    return ModelWeights(emb, blocks)


def seeded_prompt(cfg: ModelConfig, n0: int) -> List[int]:
    """harness.cpp:280-287: uniform_int_distribution<int>(0, vocab-1) over
    mt19937_64(seed + golden ratio); libstdc++'s 128-bit Lemire reduction."""
    if n0 < 1:
        raise ShapeMismatch("prompt: need at least one token")
    g = MT19937_64((cfg.seed + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF)
    rng = cfg.vocab
    out = []
    for _ in range(n0):
        prod = g() * rng
        low = prod & 0xFFFFFFFFFFFFFFFF
        if low < rng:
            thr = ((1 << 64) - rng) % rng
            while low < thr:
                prod = g() * rng
                low = prod & 0xFFFFFFFFFFFFFFFF
        out.append(prod >> 64)
    return out


# ------------------------------------------------------------ plaintext model
def rope_rotate(x, d_head, n, base):  # harness.cpp:73-83
    y = x.copy()
    for e in range(0, x.size - 1, 2):
        pair = (e % d_head) // 2
        ang = float(n) * math.pow(base, -2.0 * pair / d_head)
        c, s = math.cos(ang), math.sin(ang)
        y[e] = x[e] * c - x[e + 1] * s
        y[e + 1] = x[e] * s + x[e + 1] * c
    return y


def layer_norm(v, gamma, beta):  # harness.cpp:85-90
    c = v - v.mean()
    var = float(c @ c) / v.size
    return gamma * c / math.sqrt(var + NORM_EPS) + beta


def silu(v):
    return v / (1.0 + np.exp(-v))


def argmax_low(v) -> int:  # harness.cpp:64-69: ties toward the lower id
    return int(np.argmax(v))


@dataclass
class ReferenceTrace:
    tokens: List[int]
    final_states: List[np.ndarray]
    logits: List[np.ndarray]


def plaintext_reference(cfg: ModelConfig, w: ModelWeights, prompt: List[int], gen_len: int) -> ReferenceTrace:
    """harness.cpp:291-350: exact double forward with greedy argmax."""
    validate_model_config(cfg)
    n0, dh = len(prompt), cfg.d // cfg.H
    positions = n0 if gen_len == 0 else n0 + gen_len - 1
    toks = list(prompt)
    K = [[] for _ in range(cfg.n_layers)]
    V = [[] for _ in range(cfg.n_layers)]
    states, logits = [], []
    for pos in range(positions):
        x = w.embedding[toks[pos]].copy()
        for b, blk in enumerate(w.blocks):
            q = rope_rotate(blk.wq.T @ x, dh, pos, cfg.rope_base)
            K[b].append(rope_rotate(blk.wk.T @ x, dh, pos, cfg.rope_base))
            V[b].append(blk.wv.T @ x)
            att = np.zeros(cfg.d)
            n = len(K[b])
            for h in range(cfg.H):
                sl = slice(h * dh, (h + 1) * dh)
                sc = np.array([q[sl] @ K[b][j][sl] for j in range(n)])
                p = np.exp(sc - sc.max())
                p /= p.sum()
                for j in range(n):
                    att[sl] += p[j] * V[b][j][sl]
            s = x + blk.wo.T @ att
            y = layer_norm(s, blk.gamma1, blk.beta1)
            act = silu(blk.w_gate.T @ y) * (blk.w_up.T @ y)
            x = layer_norm(y + blk.w_down.T @ act, blk.gamma2, blk.beta2)
        states.append(x)
        logits.append(w.embedding @ x)
        if pos + 1 >= n0 and len(toks) < n0 + gen_len:
            toks.append(argmax_low(logits[-1]))
    return ReferenceTrace(toks, states, logits)


# --------------------------------------------------------------------- plans
@dataclass
class PlanEntry:
    layer: str
    input_level: int
    bootstrap_to: Optional[int] = None
    drop_to: Optional[int] = None
    sublayer: Optional[str] = None


@dataclass
class PlacementPlan:
    """placement.hpp:125-144 (the solver's output; taken as input here)."""
    entries: List[PlanEntry]

    @staticmethod
    def from_json(obj) -> "PlacementPlan":
        arr = json.loads(obj) if isinstance(obj, str) else obj
        return PlacementPlan([PlanEntry(e["layer"], int(e["input_level"]), e.get("bootstrap_to"), e.get("drop_to"),
                                        e.get("sublayer")) for e in arr])

    def to_json(self) -> str:
        return json.dumps([{"layer": e.layer, "sublayer": e.sublayer, "input_level": e.input_level,
                            "bootstrap_to": e.bootstrap_to, "drop_to": e.drop_to} for e in self.entries])


# ------------------------------------------------------------ nonlinear schedule
@dataclass
class NonlinearSchedule:
    softmax: object
    norm: object
    silu: object


def nonlinear_schedule(cfg: ModelConfig) -> NonlinearSchedule:
    """harness.cpp:353-374: desk-shallow specs; exact mode marks them exact;
    approx mode trims the norm to 3 Goldschmidt iterations and clamps."""
    from . import nonlinear as NL
    s = NonlinearSchedule(NL.desk_spec("desk-shallow", "softmax"), NL.desk_spec("desk-shallow", "norm"),
                          NL.desk_spec("desk-shallow", "silu"))
    if cfg.mode == "exact":
        s.softmax.exact = s.norm.exact = s.silu.exact = True
        return s
    s.norm.iterations = 3
    s.norm.depth_budget = 0
    s.softmax.strict_domain = s.norm.strict_domain = s.silu.strict_domain = False
    return s


# ----------------------------------------------------------------- GPU operators
class GpuOps:
    """The harness's operator set on the GPU backend. VMM diagonals are encoded
    once per (matrix, level, offsets) and reused across tokens (offline cost,
    SPEC.md:174); everything homomorphic runs through the C ABI."""

    def __init__(self, be):
        from . import (AttentionConfig, KVCache, Layout, exact_softmax_maps, exact_softmax_prefill_maps, k_append,
                       kv_from_cts, make_interleaved, make_v_pieces, prefill, qk_dot, rope_apply, softmax_times_v,
                       v_append, vmm_batch, vmm_interleaved, VmmPlan, VmmBatchPlan)
        self.be, self.N, self.L = be, be.N, be.L
        self._m = dict(AttentionConfig=AttentionConfig, KVCache=KVCache, exact_softmax_maps=exact_softmax_maps,
                       exact_softmax_prefill_maps=exact_softmax_prefill_maps, k_append=k_append,
                       kv_from_cts=kv_from_cts, make_v_pieces=make_v_pieces, prefill=prefill, qk_dot=qk_dot,
                       rope_apply=rope_apply, softmax_times_v=softmax_times_v, v_append=v_append,
                       vmm_batch=vmm_batch, vmm_interleaved=vmm_interleaved, VmmPlan=VmmPlan,
                       VmmBatchPlan=VmmBatchPlan)
        self.make_interleaved = make_interleaved
        self._plans: Dict[tuple, object] = {}

    # layouts / containers
    def layout(self, d, offset=0, heads=1):
        return self.make_interleaved(d, self.N, offset, heads)

    def attention_config(self, cfg: ModelConfig, n_max: int, n0: int = 0):
        return self._m["AttentionConfig"](cfg.N, cfg.d, cfg.H, n0, n_max)

    def new_cache(self, acfg):
        return self._m["KVCache"](self.be, acfg)

    # projections
    def vmm(self, x, W, out_offset=0):
        key = (id(W), x.level, x.layout.offset, out_offset)
        plan = self._plans.get(key)
        if plan is None:
            plan = self._m["VmmPlan"](self.be, W, W.shape[0], W.shape[1], max(x.level, 1), x.layout.offset,
                                      out_offset, True)
            self._plans[key] = plan
        return self._m["vmm_interleaved"](self.be, x, None, plan=plan)

    def vmm_batch(self, x, W):
        key = ("batch", id(W), x.level)
        plan = self._plans.get(key)
        if plan is None:
            plan = self._m["VmmBatchPlan"](self.be, W, x.level, True)
            self._plans[key] = plan
        return self._m["vmm_batch"](self.be, x, plan=plan)

    # attention
    def rope(self, x, acfg, pos, base):
        return self._m["rope_apply"](self.be, x, acfg, pos, base)

    def make_v_pieces(self, cache, v, pos):
        return self._m["make_v_pieces"](self.be, cache, v, pos)

    def v_append(self, cache, pieces):
        return self._m["v_append"](self.be, cache, pieces)

    def k_append(self, cache, k):
        return self._m["k_append"](self.be, cache, k)

    def qk_dot(self, q, cache):
        return self._m["qk_dot"](self.be, q, cache)

    def exact_softmax(self, maps, acfg, n_prime):
        return self._m["exact_softmax_maps"](self.be, maps, acfg, n_prime)

    def softmax_times_v(self, probs, cache):
        return self._m["softmax_times_v"](self.be, probs, cache)

    def prefill(self, xs, wq, wk, wv, acfg, base):
        att, cache = self._m["prefill"](self.be, xs, wq, wk, wv, acfg, self._m["exact_softmax_prefill_maps"], base)
        dec = self._m["AttentionConfig"](acfg.N, acfg.d, acfg.H, 0, acfg.n_max)  # decode-side view of the cache
        return att, self._m["kv_from_cts"](self.be, dec, cache.n_prime, cache.k_cts, cache.v_cts)

    def fused_extract_norm(self, x):
        from . import fused_extract_mask
        return fused_extract_mask(self.be, x)

    def n_prime(self, cache):
        return cache.n_prime

    def k_cts(self, cache):
        return cache.k_cts

    def v_cts(self, cache):
        return cache.v_cts

    def cache_with(self, cache, k_cts, v_cts):
        return self._m["kv_from_cts"](self.be, cache.cfg, cache.n_prime, k_cts, v_cts)

    # ledger
    def totals(self):
        return self.be.ledger.totals().asdict()

    def phase_totals(self, name):
        return self.be.ledger.phase_totals(name).asdict()


# ------------------------------------------------------------ exact-mode hooks
def _valid_mask(ly, N):  # make_mask(ValidSlots) for interleaved layouts (layouts.cpp:121-131)
    m = np.zeros(N)
    m[ly.offset::ly.t] = 1.0
    return m


def exact_apply(be, x, f):
    """nonlinear.cpp:553-563: f on the valid slots, 0 elsewhere; clean layout."""
    mask = _valid_mask(x.layout, be.N) if x.layout is not None else np.ones(be.N)
    out = be.exact_transform(x, lambda s: np.where(mask != 0.0, f(s), 0.0))
    return be.with_layout(out, replace(x.layout, deferred_mask=False)) if x.layout is not None else out


def exact_norm(be, x, gamma, beta, eps=NORM_EPS):
    """nonlinear.cpp:569-593."""
    ly = x.layout
    if ly is None or ly.kind != "interleaved" or ly.heads != 1 or ly.deferred_mask:
        raise ShapeMismatch("exact_norm: clean head-merged interleaved input required")
    N, dl = be.N, gamma.size

    def f(s):
        idx = (np.arange(dl) * ly.t + ly.offset) % N
        v = s[idx]
        mean = 0.0
        for e in range(dl):
            mean += v[e]
        mean /= dl
        var = 0.0
        for e in range(dl):
            var += (v[e] - mean) * (v[e] - mean)
        var /= dl
        inv = 1.0 / math.sqrt(var + eps)
        out = np.zeros(N)
        out[idx] = (v - mean) * inv * gamma + beta
        return out
    return be.exact_transform(x, f)


def decode_hidden(slots, ly):
    return np.asarray(slots)[ly.offset::ly.t][:ly.d].copy()


# ------------------------------------------------------------------ decode step
@dataclass
class LevelEvent:
    step: int
    block: int
    phase: str
    level_in: int
    level_out: int
    bootstrap_to: Optional[int] = None


@dataclass
class EncryptedState:
    caches: list = field(default_factory=list)
    x: object = None
    position: int = 0
    n_max: int = 0


def run_decode_step(be, ops, cfg: ModelConfig, w: ModelWeights, plan: Optional[PlacementPlan],
                    state: EncryptedState, trace: Optional[List[LevelEvent]] = None, stage_counts=None):
    """harness.cpp:425-659: one token through every block, plan-driven."""
    validate_model_config(cfg)
    if len(state.caches) != cfg.n_layers:
        raise ShapeMismatch("decode step: expected one cache per block")
    if plan is not None and len(plan.entries) != 11 * cfg.n_layers:
        raise ShapeMismatch(f"decode step: plan has {len(plan.entries)} entries, decode chain has "
                            f"{11 * cfg.n_layers}")
    acfg = ops.attention_config(cfg, state.n_max)
    t = acfg.t
    pos = state.position
    from . import nonlinear as NL
    sched = nonlinear_schedule(cfg)
    exact = cfg.mode == "exact"

    def norm(v, gamma, beta):  # stages 6 / 10
        if exact:
            return exact_norm(be, exact_apply(be, v, lambda z: z), gamma, beta)
        return NL.approx_norm(be, ops.fused_extract_norm(v), gamma, beta, NORM_EPS, sched.norm)
    ffn_layout = ops.layout(padded_dim(cfg.ffn_alpha * cfg.d))
    x = state.x
    if plan is not None and x.level > plan.entries[0].input_level:
        x = be.level_drop(x, plan.entries[0].input_level)
    cur = {}

    def begin(chain, idx):
        if plan is not None and chain.level != plan.entries[idx].input_level:
            raise LevelUnderflow(f"decode step: stage {idx} entered at level {chain.level}, plan expects "
                                 f"{plan.entries[idx].input_level}")
        cur["before"], cur["lin"] = ops.totals(), chain.level

    def end(block, stage, chain):
        if stage_counts is not None:
            after = ops.totals()
            stage_counts.append({k: after[k] - cur["before"][k] for k in after})
        if trace is not None:
            trace.append(LevelEvent(0, block, STAGE_NAMES[stage], cur["lin"], chain.level))

    def post(idx, live, lift_k=False, lift_v=False, cache_slot=None):
        """harness.cpp:476-493: bootstrap every live ciphertext (and pending
        cache handles) or drop the chain."""
        if plan is None:
            return live
        e = plan.entries[idx]
        if e.bootstrap_to is not None:
            with be.phase("Bootstrappings"):
                live = [be.bootstrap(c, e.bootstrap_to) for c in live]
                if cache_slot is not None and (lift_k or lift_v):
                    cache = state.caches[cache_slot]
                    ks = ops.k_cts(cache)
                    vs = ops.v_cts(cache)
                    if lift_k:
                        ks = [be.bootstrap(c, e.bootstrap_to) for c in ks]
                    if lift_v:
                        vs = [[be.bootstrap(c, e.bootstrap_to) for c in g] for g in vs]
                    state.caches[cache_slot] = ops.cache_with(cache, ks, vs)
            if trace:
                trace[-1].bootstrap_to = e.bootstrap_to
        elif e.drop_to is not None:
            live = [be.level_drop(live[0], e.drop_to)] + live[1:]
        return live

    for b, blk in enumerate(w.blocks):
        base = 11 * b
        # [0] query / key / value projections
        begin(x, base + 0)
        with be.phase(STAGE_NAMES[0]):
            q_o = ops.vmm(x, blk.wq)
            k_o = ops.vmm(x, blk.wk, pos % t)
            v_o = ops.vmm(x, blk.wv, pos % t)
        end(b, 0, q_o)
        q_o, k_o, v_o, x = post(base + 0, [q_o, k_o, v_o, x])

        # [1] rotary + both appends
        begin(q_o, base + 1)
        with be.phase(STAGE_NAMES[1]):
            q = ops.rope(q_o, acfg, pos, cfg.rope_base)
            k = ops.rope(k_o, acfg, pos, cfg.rope_base)
            cache = state.caches[b]
            pieces = ops.make_v_pieces(cache, v_o, pos)
            cache = ops.v_append(cache, pieces)
            state.caches[b] = ops.k_append(cache, k)
        end(b, 1, q)
        q, x = post(base + 1, [q, x], True, True, b)

        # [2] scores against the whole cache
        begin(q, base + 2)
        with be.phase(STAGE_NAMES[2]):
            maps = ops.qk_dot(q, state.caches[b])
        end(b, 2, maps[0])
        live = post(base + 2, maps + [x], False, True, b)
        maps, x = live[:-1], live[-1]

        # [3] softmax (exact oracle hook; records no ops)
        begin(maps[0], base + 3)
        with be.phase(STAGE_NAMES[3]):
            probs = (ops.exact_softmax(maps, acfg, ops.n_prime(state.caches[b])) if exact else
                     NL.approx_softmax(be, maps, ops.n_prime(state.caches[b]), cfg.H, sched.softmax))
        end(b, 3, probs[0])
        live = post(base + 3, probs + [x], False, True, b)
        probs, x = live[:-1], live[-1]

        # [4] probability-weighted value sum
        begin(probs[0], base + 4)
        with be.phase(STAGE_NAMES[4]):
            att = ops.softmax_times_v(probs, state.caches[b])
        end(b, 4, att)
        att, x = post(base + 4, [att, x])

        # [5] output projection + level-free residual at the stage tail
        begin(att, base + 5)
        with be.phase(STAGE_NAMES[5]):
            s = ops.vmm(att, blk.wo)
        with be.phase(STAGE_NAMES[6]):
            deferred = s.layout
            s = be.with_layout(be.add(x, s), deferred)
        end(b, 5, s)
        (s,) = post(base + 5, [s])

        # [6] first norm
        begin(s, base + 6)
        with be.phase(STAGE_NAMES[6]):
            y = norm(s, blk.gamma1, blk.beta1)
        end(b, 6, y)
        (y,) = post(base + 6, [y])

        # [7] up and gate projections
        begin(y, base + 7)
        with be.phase(STAGE_NAMES[7]):
            gate_o = ops.vmm(y, blk.w_gate)
            up_o = ops.vmm(y, blk.w_up)
        end(b, 7, gate_o)
        gate_o, up_o, y = post(base + 7, [gate_o, up_o, y])

        # [8] gated activation (exact SiLU hook) times the up projection
        begin(gate_o, base + 8)
        with be.phase(STAGE_NAMES[8]):
            act = exact_apply(be, gate_o, silu) if exact else NL.approx_silu(be, gate_o, sched.silu)
            prod = be.with_layout(be.mul(act, up_o), ffn_layout)
        end(b, 8, prod)
        prod, y = post(base + 8, [prod, y])

        # [9] down projection + second residual
        begin(prod, base + 9)
        with be.phase(STAGE_NAMES[9]):
            s2 = ops.vmm(prod, blk.w_down)
        with be.phase(STAGE_NAMES[6]):
            deferred = s2.layout
            s2 = be.with_layout(be.add(y, s2), deferred)
        end(b, 9, s2)
        (s2,) = post(base + 9, [s2])

        # [10] second norm -> next block's input
        begin(s2, base + 10)
        with be.phase(STAGE_NAMES[6]):
            x = norm(s2, blk.gamma2, blk.beta2)
        end(b, 10, x)
        (x,) = post(base + 10, [x])

    state.position = pos + 1
    return x


# -------------------------------------------------------------------- prefill
def prefill_prompt(be, ops, cfg: ModelConfig, w: ModelWeights, tokens: List[int], state: EncryptedState,
                   n_max: int) -> List[np.ndarray]:
    """harness.cpp:719-857: batch prefill under the naive bootstrap rule."""
    validate_model_config(cfg)
    if not tokens:
        raise ShapeMismatch("prefill: need at least one token to cache")
    if len(tokens) > n_max:
        raise ShapeMismatch("prefill: more tokens than the cache capacity")
    m = len(tokens)
    acfg = ops.attention_config(cfg, n_max, n0=m)
    t = acfg.t
    P = (m + t - 1) // t
    batch_layout = ops.layout(cfg.d, 0, cfg.H)
    ffn_layout = ops.layout(padded_dim(cfg.ffn_alpha * cfg.d))
    state.caches, state.n_max = [], n_max
    L = be.L
    from . import nonlinear as NL
    sched = nonlinear_schedule(cfg)
    exact = cfg.mode == "exact"

    def ensure(c, need):
        return be.bootstrap(c, L) if c.level < need else c

    with be.phase("Amortized Prefilling"):
        xs = []
        for p in range(P):
            slots = np.zeros(cfg.N)
            for tau in range(t):
                if p * t + tau >= m:
                    break
                slots[np.arange(cfg.d) * t + tau] = w.embedding[tokens[p * t + tau]]
            xs.append(be.encrypt(slots, L, batch_layout))
        for blk in w.blocks:
            xs = [ensure(x, 7) for x in xs]
            att, cache = ops.prefill(xs, blk.wq, blk.wk, blk.wv, acfg, cfg.rope_base)
            nxt = []
            for p in range(P):
                a = ensure(att[p], 1)
                o = ops.vmm_batch(a, blk.wo)
                s = be.with_layout(be.add(xs[p], o), batch_layout)
                acc = None
                for tau in range(t):
                    if p * t + tau >= m:
                        break
                    s = ensure(s, 1)
                    mk = np.zeros(cfg.N)
                    mk[tau::t] = 1.0
                    lane = be.with_layout(be.mul_plain(s, mk), ops.layout(cfg.d, tau, 1))
                    if exact:
                        y = exact_norm(be, lane, blk.gamma1, blk.beta1)
                    else:
                        lane = ensure(lane, NL.norm_depth(sched.norm))
                        y = NL.approx_norm(be, lane, blk.gamma1, blk.beta1, NORM_EPS, sched.norm)
                    y = ensure(y, 1)
                    gate_o = ops.vmm(y, blk.w_gate)
                    up_o = ops.vmm(y, blk.w_up)
                    if exact:
                        act = ensure(exact_apply(be, gate_o, silu), 1)
                    else:
                        gate_o = ensure(gate_o, NL.silu_depth(sched.silu) + 1)
                        act = NL.approx_silu(be, gate_o, sched.silu)
                    up_o = ensure(up_o, 1)
                    prod = be.with_layout(be.mul(act, up_o), ffn_layout)
                    prod = ensure(prod, 1)
                    down = ops.vmm(prod, blk.w_down, tau)
                    s2 = be.with_layout(be.add(y, down), down.layout)
                    if exact:
                        z = exact_norm(be, exact_apply(be, s2, lambda v: v), blk.gamma2, blk.beta2)
                    else:
                        s2 = ensure(s2, 1 + NL.norm_depth(sched.norm))
                        z = NL.approx_norm(be, ops.fused_extract_norm(s2), blk.gamma2, blk.beta2, NORM_EPS,
                                           sched.norm)
                    acc = z if acc is None else be.add(acc, z)
                    acc = be.with_layout(acc, batch_layout)
                nxt.append(acc)
            # long-lived cache entries served at the level fresh decode appends reach
            serve = max(1, L - 2)
            ks = [be.bootstrap(c, serve) if c.level < serve else c for c in ops.k_cts(cache)]
            vs = [[be.bootstrap(c, serve) if c.level < serve else c for c in g] for g in ops.v_cts(cache)]
            state.caches.append(ops.cache_with(cache, ks, vs))
            xs = nxt
    states = []
    for p in range(P):
        sl = be.decrypt(xs[p])
        for tau in range(t):
            if p * t + tau >= m:
                break
            states.append(decode_hidden(sl, ops.layout(cfg.d, tau, 1)))
    return states


# ----------------------------------------------------------------- generation
@dataclass
class Report:
    config: ModelConfig
    prompt: List[int]
    generated: List[int] = field(default_factory=list)
    phases: List[dict] = field(default_factory=list)
    level_trace: List[LevelEvent] = field(default_factory=list)
    max_abs_error: float = 0.0
    bootstrap_count: int = 0
    hidden: List[np.ndarray] = field(default_factory=list)  # decoded last-block state per step

    def phase_rows(self) -> List[dict]:
        """Phase rows with the reference report's keys (harness.cpp:861-899)."""
        keys = {"rotations": "rotations", "hoisted_rotations": "hoisted", "ct_pt_mults": "ctpt_mult",
                "ct_ct_mults": "ctct_mult", "additions": "adds", "bootstraps": "bootstraps"}
        return [dict({keys[k]: v for k, v in p["ops"].items()}, name=p["name"], levels_in=p["levels_in"],
                     levels_out=p["levels_out"]) for p in self.phases]

    def to_csv(self) -> str:
        """harness.cpp:901-922 (pinned columns)."""
        def field_(v):
            if not any(ch in v for ch in ',"\n'):
                return v
            return '"' + v.replace('"', '""') + '"'
        out = "phase,rotations,hoisted,ctpt_mult,ctct_mult,adds,bootstraps,levels_in,levels_out\n"
        for r in self.phase_rows():
            cells = [field_(r["name"])] + [str(r[k]) for k in ("rotations", "hoisted", "ctpt_mult", "ctct_mult",
                                                                 "adds", "bootstraps")]
            cells += ["" if r[k] < 0 else str(r[k]) for k in ("levels_in", "levels_out")]
            out += ",".join(cells) + "\n"
        return out

    def to_json(self) -> str:
        return json.dumps({"config": asdict(self.config), "prompt": self.prompt, "generated": self.generated,
                           "phases": self.phase_rows(), "level_trace": [asdict(e) for e in self.level_trace],
                           "max_abs_error": self.max_abs_error, "bootstrap_count": self.bootstrap_count})


def run_generation(be, ops, cfg: ModelConfig, w: ModelWeights, prompt: List[int], gen_len: int,
                   plan: PlacementPlan) -> Report:
    """harness.cpp:943-1053 with the plan given (the solver is out of scope)."""
    validate_model_config(cfg)
    if not prompt:
        raise ShapeMismatch("generation: need a nonempty prompt")
    if gen_len < 1:
        raise ShapeMismatch("generation: gen_len must be >= 1")
    if plan is None:
        raise ShapeMismatch("generation: a placement plan is required (the solver is out of scope)")
    n0 = len(prompt)
    n_max = n0 + gen_len
    ref = plaintext_reference(cfg, w, prompt, gen_len)
    state = EncryptedState(n_max=n_max)
    err = 0.0
    if n0 > 1:
        pre = prefill_prompt(be, ops, cfg, w, prompt[:-1], state, n_max)
        for i, v in enumerate(pre):
            err = max(err, float(np.max(np.abs(v - ref.final_states[i]))))
    else:
        acfg = ops.attention_config(cfg, n_max)
        state.caches = [ops.new_cache(acfg) for _ in range(cfg.n_layers)]
    hl = ops.layout(cfg.d)

    def enc(tok):
        slots = np.zeros(cfg.N)
        slots[np.arange(cfg.d) * hl.t + hl.offset] = w.embedding[tok]
        return be.encrypt(slots, be.L, hl)

    state.x = enc(prompt[-1])
    state.position = n0 - 1
    rep = Report(cfg, list(prompt))
    for step in range(gen_len):
        first = len(rep.level_trace)
        h = run_decode_step(be, ops, cfg, w, plan, state, rep.level_trace)
        for ev in rep.level_trace[first:]:
            ev.step = step
        hv = decode_hidden(be.decrypt(h), hl)
        rep.hidden.append(hv)
        logits = w.embedding @ hv
        pos = n0 - 1 + step
        err = max(err, float(np.max(np.abs(hv - ref.final_states[pos]))))
        err = max(err, float(np.max(np.abs(logits - ref.logits[pos]))))
        tok = argmax_low(logits)
        rep.generated.append(tok)
        if step + 1 < gen_len:
            state.x = enc(tok)
    rep.max_abs_error = err
    tot = ops.totals()
    rep.bootstrap_count = tot["bootstraps"]
    for name in PHASE_ORDER:
        ops_ = ops.phase_totals(name)
        if any(ops_.values()):
            lv = next(((e.level_in, e.level_out) for e in rep.level_trace if e.phase == name), (-1, -1))
            rep.phases.append({"name": name, "ops": ops_, "levels_in": lv[0], "levels_out": lv[1]})
    return rep
