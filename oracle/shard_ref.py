"""Oracle restatement of the sharded hot path (TEST INFRASTRUCTURE ONLY).

Mirrors paper_2602_11470_b200/csrc/protocols.cpp (vmm_partial / vmm_finish,
qk_dot_partial, softmax_times_v_partial / _finish) over any slotforge-shaped
backend, so the multi-process tests can check on CPU (gloo, world_size 2) that
partial results exchanged between ranks and summed mod q reproduce the
single-device ciphertexts bit for bit. Ownership rules: VMM giant steps
g2 = rank mod world; K ciphertexts j = rank mod world; Score*V whole giant groups
(G mod 8) mod world == rank.
"""
from __future__ import annotations

import numpy as np

from . import protocols as P
from .layout import Layout, make_interleaved, make_mask, stride_mask


def vmm_partial(be, x, W, bsgs, out_offset, rank, world):
    N = be.N
    W = np.asarray(W, dtype=np.float64)
    s = P.interleaved_shape(N, W.shape[0], W.shape[1], x.layout.offset, out_offset)
    stair = P._fold_steps(be, x, P.ladder_rots(s))
    unit = s.t_in * s.t_out
    if not bsgs:
        own = list(range(rank, s.k, world))
        if not own:
            return be.zeros(x.level - 1)
        return be.mac_plain([(be.rotate(stair, g * unit), P.interleaved_plain(s, W, g, 0)) for g in own])
    b, giants = P.bsgs_split(s.k)
    G = P.GIANT_GROUPS
    groups = [r for r in range(min(G, giants)) if r % world == rank]
    if not groups:
        return be.zeros(x.level - 1)
    baby = [stair] + [be.rotate(stair, g1 * unit, hoisted=True) for g1 in range(1, b)]
    acc = None
    for r in groups:
        grp = P.vmm_giant_group(be, s, W, baby, b, unit, range(r, giants, G))
        acc = grp if acc is None else be.add(acc, grp)
    return acc


def vmm_finish(be, acc, W, in_offset, out_offset, mask_output=False):
    W = np.asarray(W)
    s = P.interleaved_shape(be.N, W.shape[0], W.shape[1], in_offset, out_offset)
    acc = P._fold_steps(be, acc, P.reduce_rots(s))
    if mask_output:
        acc = be.mul_plain(acc, stride_mask(be.N, s.t_out, s.tau_out))
    return be.with_layout(acc, Layout("interleaved", s.d_out, s.t_out, s.tau_out, 1, not mask_output))


def qk_dot_partial(be, q, cache, cfg, rank, world):
    t, dh, gt = cfg.t, cfg.d_head, cfg.group_tokens
    q_rep = P.replicate_lanes(be, q, t)
    head_mask = make_mask(make_interleaved(cfg.d, cfg.N, 0, cfg.H), cfg.N, "replicate_extract")
    n_maps = (cache.n_prime + gt - 1) // gt
    G = P.PACK_GROUPS
    terms = [[[] for _ in range(G)] for _ in range(n_maps)]
    for j in range(len(cache.k_cts)):
        if (j % G) % world != rank:  # whole pack groups per rank
            continue
        terms[(j * t) // gt][j % G].append(P.qk_term(be, q_rep, cache.k_cts[j], cfg, head_mask, -((j * t) % gt)))
    maps = [P.pack_sum(be, grp) for grp in terms]
    return [be.with_layout(m, None) if m is not None else be.zeros(q.level - 2) for m in maps]


def softmax_times_v_partial(be, probs, cache, cfg, rank, world):
    """The rank's share of the baby-step / giant-step Score*V sum (whole giant groups)."""
    return P.sv_partial(be, probs, cache, cfg, rank, world)


def softmax_times_v_finish(be, parts, cfg):
    """Sum the partials, fold the lanes, mask."""
    return P.sv_finish(be, parts, cfg)


def sum_partials(be, parts):
    live = [p for p in parts if not getattr(p, "is_zero", False)]
    if not live:
        return parts[0]
    acc = live[0]
    for p in live[1:]:
        acc = be.add(acc, p)
    return acc
