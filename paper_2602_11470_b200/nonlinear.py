"""Homomorphic nonlinearities over the encrypted hot path.

Chebyshev-basis polynomial evaluation at balanced depth, Goldschmidt
reciprocal / reciprocal square root, the overflow-free scaled exponential and
the softmax / layer-norm / SiLU (GeLU) compositions -- every one a program of
the backend's homomorphic operators (add, sub, mul, mul_plain, add_plain,
rotate), so on the GPU backend each step runs through the CUDA library.

Mirrors /root/reference/proj/src/nonlinear.cpp (file:line):
  guard_domain                  41-68     (domain check on the client: decrypt)
  cheb_divmod / eval_cheb_rec   72-119
  desk_spec / spec json         182-258
  fit_cheb_ls / cheb_fit_error  260-310
  eval_cheb / poly_depth        312-330
  goldschmidt(_depth)           334-384
  approx_exp / exp_depth        386-407
  approx_softmax / depth        409-462
  approx_norm / norm_depth      466-507
  approx_silu / silu_depth      509-549
  exact_apply / exact_norm      553-593
  sublayer_trace                600-633

Level and ledger behaviour is the reference's exactly (each function consumes
its declared depth; counts are the reference's). Two CKKS-specific notes:
  * `1 - x` in the inverse Goldschmidt is evaluated as (0 - x) + 1 (same two
    ledger additions, the same float64 result) because a trivial zero has no
    scale to encode a plaintext constant at;
  * the remainder / quotient adds of the balanced evaluation combine operands
    at different levels and scales -- the backend's add aligns them
    (DESIGN.md §3.5a).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np


class ShapeMismatch(ValueError):
    pass


class DomainViolation(RuntimeError):
    pass


class InfeasibleLayer(RuntimeError):
    pass


@dataclass
class ApproxSpec:
    """nonlinear.hpp:24-34."""
    function: str = ""
    domain_lo: float = 0.0
    domain_hi: float = 1.0
    depth_budget: int = 0
    iterations: int = 7
    degrees: List[int] = field(default_factory=list)
    scale_in: float = 1.0
    scale_out: float = 1.0
    strict_domain: bool = True
    exact: bool = False

    def to_json(self) -> str:
        return json.dumps({"function": self.function, "domain": [self.domain_lo, self.domain_hi],
                           "depth_budget": self.depth_budget, "iterations": self.iterations,
                           "degrees": list(self.degrees), "scale_in": self.scale_in, "scale_out": self.scale_out,
                           "strict_domain": self.strict_domain, "exact": self.exact})

    @staticmethod
    def from_json(text) -> "ApproxSpec":
        j = json.loads(text) if isinstance(text, str) else text
        s = ApproxSpec(function=j["function"])
        if "domain" in j:
            s.domain_lo, s.domain_hi = float(j["domain"][0]), float(j["domain"][1])
        s.depth_budget = j.get("depth_budget", 0)
        s.iterations = j.get("iterations", 7)
        s.degrees = list(j.get("degrees", []))
        s.scale_in = j.get("scale_in", 1.0)
        s.scale_out = j.get("scale_out", 1.0)
        s.strict_domain = j.get("strict_domain", True)
        s.exact = j.get("exact", False)
        return s


def ceil_log2(n: int) -> int:
    k = 0
    while (1 << k) < n:
        k += 1
    return k


def _validate_domain(spec, what):
    if not spec.domain_lo < spec.domain_hi:
        raise ShapeMismatch(f"{what}: empty domain [{spec.domain_lo}, {spec.domain_hi}]")


def _check_budget(spec, depth, what):
    if 0 < spec.depth_budget < depth:
        raise InfeasibleLayer(f"{what}: schedule needs depth {depth} but depth_budget is {spec.depth_budget}")


def _require_degrees(spec, count, what):
    if len(spec.degrees) != count:
        raise ShapeMismatch(f"{what}: expected {count} degree entries, got {len(spec.degrees)}")
    for i, d in enumerate(spec.degrees):
        if d < (1 if i == 0 else 0):
            raise ShapeMismatch(f"{what}: bad degree schedule entry {d}")


def _valid_mask(ly, N):  # make_mask(ValidSlots) (layouts.cpp:121-131)
    if ly.kind == "interleaved":
        m = np.zeros(N)
        m[ly.offset::ly.t] = 1.0
        return m
    if ly.kind == "contiguous":
        m = np.zeros(N)
        m[:ly.d] = 1.0
        return m
    return np.ones(N)


def _with_layout(be, c, ly):
    return be.with_layout(c, ly)


def guard_domain(be, c, spec: ApproxSpec, where: Optional[np.ndarray], what: str):
    """nonlinear.cpp:41-68: the client checks the valid slots against the
    spec's domain (decrypt); strict specs throw, others clamp (oracle hook)."""
    lo, hi = spec.domain_lo, spec.domain_hi
    s = np.asarray(be.decrypt(c))
    sel = np.ones(be.N, dtype=bool) if where is None else (np.asarray(where) != 0.0)
    bad_mask = sel & ((s < lo) | (s > hi))
    bad = int(bad_mask.sum())
    if bad == 0:
        return c
    worst = float(np.max(np.maximum(lo - s[bad_mask], s[bad_mask] - hi)))
    if spec.strict_domain:
        raise DomainViolation(f"{what}: {bad} slot(s) outside [{lo}, {hi}], worst excess {worst}")
    import sys
    print(f"[nonlinear] {what}: clamped {bad} slot(s) to [{lo:g}, {hi:g}]", file=sys.stderr)
    return be.exact_transform(c, lambda v: np.where(sel, np.clip(v, lo, hi), v))


# -------------------------------------------------------------- polynomial fits
def fit_cheb_ls(f: Callable[[float], float], lo: float, hi: float, degree: int) -> List[float]:
    """nonlinear.cpp:260-284: least squares on a uniform grid of max(8(d+1), 256)
    points in the Chebyshev basis of [lo, hi]."""
    if degree < 1:
        raise ShapeMismatch("fit_cheb_ls: degree must be >= 1")
    if not lo < hi:
        raise ShapeMismatch("fit_cheb_ls: empty interval")
    cols = degree + 1
    rows = max(8 * cols, 256)
    A = np.zeros((rows, cols))
    b = np.zeros(rows)
    for i in range(rows):
        x = lo + (hi - lo) * i / (rows - 1)
        z = (2.0 * x - lo - hi) / (hi - lo)
        tk2, tk1 = 1.0, z
        A[i, 0] = 1.0
        if cols > 1:
            A[i, 1] = z
        for k in range(2, cols):
            tk = 2.0 * z * tk1 - tk2
            A[i, k] = tk
            tk2, tk1 = tk1, tk
        b[i] = f(x)
    return list(np.linalg.lstsq(A, b, rcond=None)[0])


def cheb_value(coeffs, z: float) -> float:  # Clenshaw (nonlinear.cpp:288-297)
    b1 = b2 = 0.0
    for k in range(len(coeffs) - 1, 0, -1):
        b1, b2 = 2.0 * z * b1 - b2 + coeffs[k], b1
    return z * b1 - b2 + coeffs[0]


def cheb_fit_error(coeffs, f, lo, hi) -> float:
    worst = 0.0
    for i in range(4097):
        x = lo + (hi - lo) * i / 4096
        z = (2.0 * x - lo - hi) / (hi - lo)
        worst = max(worst, abs(cheb_value(coeffs, z) - f(x)))
    return worst


def poly_depth(degree: int) -> int:
    return 1 + ceil_log2(degree + 1)


def cheb_divmod(c, m):
    """p = q T_m + r with deg r < m (2 T_m T_k = T_{m+k} + T_{|m-k|})."""
    work = list(c)
    n = len(c)
    q = [0.0] * (n - m)
    for deg in range(n - 1, m - 1, -1):
        a = work[deg]
        work[deg] = 0.0
        if deg == m:
            q[0] += a
        else:
            q[deg - m] += 2.0 * a
            work[abs(deg - 2 * m)] -= a
    return q, work[:m]


def _coeff_plain(c, mask, N):
    return mask * c if mask is not None else np.full(N, c)


def _eval_rec(be, coeffs, tpow, mask):
    n = len(coeffs)
    if n == 1:
        return None, coeffs[0]
    if n == 2:
        ct = be.mul_plain(tpow[0], _coeff_plain(coeffs[1], mask, be.N))
        return be.add_plain(ct, _coeff_plain(coeffs[0], mask, be.N)), 0.0
    m = 1 << (ceil_log2(n) - 1)
    qc, rc = cheb_divmod(coeffs, m)
    tm = tpow[m.bit_length() - 1]
    qct, qplain = _eval_rec(be, qc, tpow, mask)
    prod = be.mul(tm, qct) if qct is not None else be.mul_plain(tm, _coeff_plain(qplain, mask, be.N))
    rct, _ = _eval_rec(be, rc, tpow, mask)
    return be.add(prod, rct), 0.0


def eval_cheb(be, x, lo, hi, coeffs, coeff_mask=None):
    """nonlinear.cpp:312-330: affine map to [-1, 1], T_{2^j} by doubling,
    balanced divide-and-conquer on the coefficients."""
    if len(coeffs) < 2:
        raise ShapeMismatch("eval_cheb: need at least degree 1")
    if not lo < hi:
        raise ShapeMismatch("eval_cheb: empty interval")
    t1 = be.add_plain(be.mul_plain(x, 2.0 / (hi - lo)), (-lo - hi) / (hi - lo))
    tpow = [t1]
    for _ in range(1, ceil_log2(len(coeffs))):
        sq = be.mul(tpow[-1], tpow[-1])
        tpow.append(be.add_plain(be.add(sq, sq), -1.0))
    out, _ = _eval_rec(be, list(coeffs), tpow, coeff_mask)
    return _with_layout(be, out, x.layout)


# ---------------------------------------------------------------- Goldschmidt
INVERSE, RSQRT = "inverse", "rsqrt"


def goldschmidt_depth(kind: str, spec: ApproxSpec) -> int:
    return (1 if spec.scale_in != 1.0 else 0) + (spec.iterations if kind == INVERSE else 2 * spec.iterations)


def goldschmidt(be, x, kind: str, spec: ApproxSpec):
    """nonlinear.cpp:339-384."""
    _validate_domain(spec, "goldschmidt")
    if spec.domain_lo <= 0.0 or spec.domain_hi > 1.0:
        raise ShapeMismatch("goldschmidt: domain must be a subinterval of (0, 1]")
    if spec.iterations < 2:
        raise ShapeMismatch("goldschmidt: need at least 2 iterations")
    _check_budget(spec, goldschmidt_depth(kind, spec), "goldschmidt")
    xs = be.mul_plain(x, spec.scale_in) if spec.scale_in != 1.0 else x
    sel = _valid_mask(xs.layout, be.N) if xs.layout is not None else None
    xs = guard_domain(be, xs, spec, sel, "goldschmidt")
    if kind == INVERSE:
        # 1/x = prod_i (1 + v^(2^i)), v = 1 - x
        v = be.add_plain(be.sub(be.zeros(xs.level), xs), 1.0)
        y = be.add_plain(v, 1.0)
        for _ in range(1, spec.iterations):
            v = be.mul(v, v)
            y = be.mul(y, be.add_plain(v, 1.0))
        return _with_layout(be, y, x.layout)
    # coupled Newton: g -> sqrt(x), h -> 1 / (2 sqrt(x))
    y1 = be.add_plain(be.mul_plain(xs, -0.5), 1.5)
    h = be.add_plain(be.mul_plain(xs, -0.25), 0.75)
    g = be.mul(xs, y1)
    for _ in range(1, spec.iterations):
        gh = be.mul(g, h)
        r = be.add_plain(be.sub(be.zeros(gh.level), gh), 0.5)
        g = be.mul(g, be.add_plain(r, 1.0))
        h = be.mul(h, be.add_plain(r, 1.0))
    return _with_layout(be, be.add(h, h), x.layout)


# ------------------------------------------------------------------ exponential
def exp_depth(spec: ApproxSpec) -> int:
    _require_degrees(spec, 2, "exp_depth")
    return poly_depth(spec.degrees[0]) + spec.degrees[1]


def approx_exp(be, x, spec: ApproxSpec, mask=None):
    """nonlinear.cpp:391-407: exp(x - M) as p((x - M) / 2^r)^(2^r)."""
    _validate_domain(spec, "approx_exp")
    _require_degrees(spec, 2, "approx_exp")
    _check_budget(spec, exp_depth(spec), "approx_exp")
    deg, r = spec.degrees
    M, scale = spec.domain_hi, float(1 << r)
    xg = guard_domain(be, x, spec, mask, "approx_exp")
    coeffs = fit_cheb_ls(lambda v: math.exp((v - M) / scale), spec.domain_lo, spec.domain_hi, deg)
    p = eval_cheb(be, xg, spec.domain_lo, spec.domain_hi, coeffs, mask)
    for _ in range(r):
        p = be.mul(p, p)
    return p


def fold_stride(be, acc, step, count):  # nonlinear.cpp:143-147
    s = step
    while s < step * count:
        acc = be.add(acc, be.rotate(acc, s))
        s <<= 1
    return acc


def replicate_block(be, acc, step, count):  # nonlinear.cpp:149-152
    s = step
    while s < step * count:
        acc = be.add(acc, be.rotate(acc, -s))
        s <<= 1
    return acc


def softmax_depth(spec: ApproxSpec) -> int:
    return exp_depth(spec) + 1 + spec.iterations + 1


def approx_softmax(be, maps, n_prime: int, heads: int, spec: ApproxSpec):
    """nonlinear.cpp:414-457: masked scaled exponentials, per-head normalizer
    (fold + extract + replicate), Goldschmidt inverse, renormalize."""
    N = be.N
    if heads < 1 or heads & (heads - 1) or heads > N:
        raise ShapeMismatch("approx_softmax: heads must be a power of two dividing N")
    if n_prime < 1:
        raise ShapeMismatch("approx_softmax: empty score range")
    gt = N // heads
    if len(maps) != (n_prime + gt - 1) // gt:
        raise ShapeMismatch(f"approx_softmax: expected {(n_prime + gt - 1) // gt} score maps, got {len(maps)}")
    if not 0.0 < spec.scale_in <= 1.0:
        raise ShapeMismatch("approx_softmax: scale_in must lie in (0, 1]")
    _check_budget(spec, softmax_depth(spec), "approx_softmax")
    _require_degrees(spec, 2, "approx_softmax")
    root = math.pow(spec.scale_in, 1.0 / (1 << spec.degrees[1]))
    es = []
    for m, mp in enumerate(maps):
        cnt = min(gt, n_prime - m * gt)
        mask = np.zeros(N)
        for h in range(heads):
            mask[h * gt:h * gt + cnt] = root
        es.append(approx_exp(be, mp, spec, mask))
    s = es[0]
    for e in es[1:]:
        s = be.add(s, e)
    s = fold_stride(be, s, 1, gt)
    sm = np.zeros(N)
    sm[0::gt] = 1.0
    total = replicate_block(be, be.mul_plain(s, sm), 1, gt)
    sub = ApproxSpec(function="inverse", domain_lo=1e-9, domain_hi=1.0, iterations=spec.iterations,
                     strict_domain=spec.strict_domain)
    inv = goldschmidt(be, total, INVERSE, sub)
    return [be.mul(e, inv) for e in es]


def approx_softmax_single(be, scores, n_prime: int, spec: ApproxSpec):
    return approx_softmax(be, [scores], n_prime, 1, spec)[0]


# ------------------------------------------------------------------- layer norm
def norm_depth(spec: ApproxSpec) -> int:
    return 5 + 2 * spec.iterations


def _require_norm_layout(x, what):
    ly = x.layout
    if ly is None or ly.kind != "interleaved":
        raise ShapeMismatch(f"{what}: interleaved input layout required")
    if ly.heads != 1:
        raise ShapeMismatch(f"{what}: head-merged input required (heads == 1)")
    if ly.deferred_mask:
        raise ShapeMismatch(f"{what}: clean input required (clear vmm garbage via fused_extract first)")
    return ly


def _logical_mask(ly, N, d_log, value):
    m = np.zeros(N)
    m[(np.arange(d_log) * ly.t + ly.offset) % N] = value
    return m


def _encode_logical(ly, N, v, scale):
    m = np.zeros(N)
    m[(np.arange(len(v)) * ly.t + ly.offset) % N] = np.asarray(v) * scale
    return m


def approx_norm(be, x, gamma, beta, eps: float, spec: ApproxSpec):
    """nonlinear.cpp:468-507."""
    ly = _require_norm_layout(x, "approx_norm")
    N = be.N
    gamma, beta = np.asarray(gamma, dtype=np.float64), np.asarray(beta, dtype=np.float64)
    d_log = gamma.size
    if beta.size != gamma.size:
        raise ShapeMismatch("approx_norm: gamma/beta size mismatch")
    if d_log < 1 or d_log > ly.d:
        raise ShapeMismatch("approx_norm: logical width must fit the layout")
    _check_budget(spec, norm_depth(spec), "approx_norm")
    s1 = fold_stride(be, x, ly.t, ly.d)
    mu = be.mul_plain(s1, _logical_mask(ly, N, d_log, 1.0 / d_log))
    xc = be.sub(x, mu)
    sq = be.mul(xc, xc)
    s2 = fold_stride(be, sq, ly.t, ly.d)
    vs = be.mul_plain(s2, _logical_mask(ly, N, d_log, spec.scale_in / d_log))
    vs = be.add_plain(vs, _logical_mask(ly, N, d_log, eps * spec.scale_in))
    valid = _logical_mask(ly, N, d_log, 1.0)
    vs = guard_domain(be, vs, spec, valid, "approx_norm")
    mid = 0.5 * (spec.domain_lo + spec.domain_hi)
    vs = be.add_plain(vs, (1.0 - valid) * mid)
    sub = ApproxSpec(function="rsqrt", domain_lo=spec.domain_lo, domain_hi=spec.domain_hi,
                     iterations=spec.iterations, strict_domain=spec.strict_domain)
    vs = _with_layout(be, vs, None)  # guarded already; the kernel runs slot-blind
    rs = goldschmidt(be, vs, RSQRT, sub)
    y = be.mul(xc, rs)
    out = be.mul_plain(y, _encode_logical(ly, N, gamma, math.sqrt(spec.scale_in)))
    out = be.add_plain(out, _encode_logical(ly, N, beta, 1.0))
    return _with_layout(be, out, ly)


# ------------------------------------------------------------------- SiLU / GeLU
def silu_ref(v):
    return v / (1.0 + math.exp(-v))


def gelu_ref(v):
    return 0.5 * v * (1.0 + math.erf(v / math.sqrt(2.0)))


def silu_depth(spec: ApproxSpec) -> int:
    _require_degrees(spec, 1, "silu_depth")
    return poly_depth(spec.degrees[0])


def approx_silu(be, x, spec: ApproxSpec, extra_coeff=None):
    """nonlinear.cpp:514-549: composite-polynomial SiLU (GeLU for
    spec.function == "gelu") with the valid mask fused into the coefficients."""
    _validate_domain(spec, "approx_silu")
    _require_degrees(spec, 1, "approx_silu")
    _check_budget(spec, silu_depth(spec), "approx_silu")
    gelu = spec.function == "gelu"
    mask = None
    if x.layout is not None:
        mask = _valid_mask(x.layout, be.N)
        if extra_coeff is not None:
            mask = mask * np.asarray(extra_coeff)
    elif extra_coeff is not None:
        mask = np.asarray(extra_coeff, dtype=np.float64)
    xg = guard_domain(be, x, spec, mask, "approx_gelu" if gelu else "approx_silu")
    coeffs = fit_cheb_ls(gelu_ref if gelu else silu_ref, spec.domain_lo, spec.domain_hi, spec.degrees[0])
    if spec.domain_lo < 0.0 < spec.domain_hi:  # pin the fixed point at zero
        z0 = (-spec.domain_lo - spec.domain_hi) / (spec.domain_hi - spec.domain_lo)
        coeffs[0] -= cheb_value(coeffs, z0)
    out = eval_cheb(be, xg, spec.domain_lo, spec.domain_hi, coeffs, mask)
    if out.layout is not None:
        from dataclasses import replace
        out = _with_layout(be, out, replace(out.layout, deferred_mask=False))
    return out


# --------------------------------------------------------------------- presets
def desk_spec(preset: str, function: str) -> ApproxSpec:
    """nonlinear.cpp:214-258."""
    shallow = preset == "desk-shallow"
    if not shallow and preset != "desk-default":
        raise ShapeMismatch(f"desk_spec: unknown preset '{preset}'")
    s = ApproxSpec(function=function)
    if function == "softmax":
        s.domain_lo, s.domain_hi = -8.0, 4.0
        s.degrees = [3, 1] if shallow else [7, 2]
        s.iterations = 6 if shallow else 14
        s.scale_in = 1.0 / 32.0
        s.depth_budget = softmax_depth(s)
    elif function == "norm":
        s.domain_lo, s.domain_hi = 0.02, 0.95
        s.iterations = 4 if shallow else 10
        s.scale_in = 1.0 / 8.0
        s.depth_budget = norm_depth(s)
    elif function in ("silu", "gelu"):
        s.domain_lo, s.domain_hi = -16.0, 12.0
        s.degrees = [15 if shallow else 63]
        s.depth_budget = silu_depth(s)
    elif function == "exp":
        s.domain_lo, s.domain_hi = -8.0, 4.0
        s.degrees = [3, 1] if shallow else [7, 2]
        s.depth_budget = exp_depth(s)
    elif function == "inverse":
        s.domain_lo, s.domain_hi = 1.0 / 64.0, 1.0
        s.iterations = 6 if shallow else 9
        s.depth_budget = goldschmidt_depth(INVERSE, s)
    elif function == "rsqrt":
        s.domain_lo, s.domain_hi = 1.0 / 16.0, 1.0
        s.iterations = 4 if shallow else 8
        s.depth_budget = goldschmidt_depth(RSQRT, s)
    else:
        raise ShapeMismatch(f"desk_spec: unknown function '{function}'")
    return s


# ----------------------------------------------------------- sub-layer traces
@dataclass
class SubLayerPhase:
    name: str
    depth: int
    ct_count: int = 1
    interruptible: bool = False


def sublayer_trace(function: str, spec: ApproxSpec) -> List[SubLayerPhase]:
    """nonlinear.cpp:606-633."""
    if spec.exact:
        return []
    if function == "softmax":
        return [SubLayerPhase("exponential", exp_depth(spec), 2, False), SubLayerPhase("normalizer", 1, 2, True),
                SubLayerPhase("reciprocal", spec.iterations, 2, False), SubLayerPhase("renormalize", 1, 2, True)]
    if function == "norm":
        return [SubLayerPhase("center", 1, 1, True), SubLayerPhase("variance", 2, 2, False),
                SubLayerPhase("inverse sqrt", 2 * spec.iterations, 3, False), SubLayerPhase("rescale", 2, 2, True)]
    if function in ("silu", "gelu"):
        return [SubLayerPhase("composite polynomial", silu_depth(spec), 2, False)]
    if function == "exp":
        return ([SubLayerPhase("shift", 1, 1, True), SubLayerPhase("polynomial", poly_depth(spec.degrees[0]) - 1, 2,
                                                                    False)]
                + [SubLayerPhase("squaring", 1, 1, True) for _ in range(spec.degrees[1])])
    if function == "inverse":
        return [SubLayerPhase("reciprocal", goldschmidt_depth(INVERSE, spec), 2, False)]
    if function == "rsqrt":
        return [SubLayerPhase("inverse sqrt", goldschmidt_depth(RSQRT, spec), 2, False)]
    raise ShapeMismatch(f"sublayer_trace: unknown function '{function}'")
