"""TEST INFRASTRUCTURE: the harness's operator interface over the CPU oracle
(oracle/slot_sim.SimBackend + oracle/protocols, the restatement pinned to the
reference), so paper_2602_11470_b200.harness can be checked against the
reference's own run_generation report on CPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import protocols as P  # noqa: E402
from oracle.layout import make_interleaved  # noqa: E402


class SimOps:
    def __init__(self, be):
        self.be, self.N, self.L = be, be.N, be.L

    def layout(self, d, offset=0, heads=1):
        return make_interleaved(d, self.N, offset, heads)

    def attention_config(self, cfg, n_max, n0=0):
        return P.AttentionConfig(cfg.N, cfg.d, cfg.H, n0, n_max)

    def new_cache(self, acfg):
        c = P.KVCache()
        c.cfg = acfg
        return c

    def _tag(self, cache, acfg):
        cache.cfg = acfg
        return cache

    def vmm(self, x, W, out_offset=0):
        return P.vmm_interleaved(self.be, x, W, bsgs=True, out_offset=out_offset)

    def vmm_batch(self, x, W):
        return P.vmm_batch(self.be, x, W, True)

    def rope(self, x, acfg, pos, base):
        return P.rope_apply(self.be, x, acfg, pos, base)

    def make_v_pieces(self, cache, v, pos):
        return P.make_v_pieces(self.be, v, cache.cfg, pos)

    def v_append(self, cache, pieces):
        return self._tag(P.v_append(self.be, cache, pieces, cache.cfg), cache.cfg)

    def k_append(self, cache, k):
        return self._tag(P.k_append(self.be, cache, k, cache.cfg), cache.cfg)

    def qk_dot(self, q, cache):
        return P.qk_dot(self.be, q, cache, cache.cfg)

    def exact_softmax(self, maps, acfg, n_prime):
        return P.exact_softmax_maps(self.be, maps, acfg, n_prime)

    def softmax_times_v(self, probs, cache):
        return P.softmax_times_v(self.be, probs, cache, cache.cfg)

    def prefill(self, xs, wq, wk, wv, acfg, base):
        att, cache = P.prefill(self.be, xs, wq, wk, wv, acfg, P.exact_softmax_prefill_maps, base)
        return att, self._tag(cache, P.AttentionConfig(acfg.N, acfg.d, acfg.H, 0, acfg.n_max))

    def fused_extract_norm(self, x):
        return P.fused_extract(self.be, x, "norm_mask")

    def n_prime(self, cache):
        return cache.n_prime

    def k_cts(self, cache):
        return list(cache.k_cts)

    def v_cts(self, cache):
        return [list(g) for g in cache.v_cts]

    def cache_with(self, cache, k_cts, v_cts):
        c = P.KVCache(cache.n_prime, list(k_cts), [list(g) for g in v_cts])
        c.cfg = cache.cfg
        return c

    def totals(self):
        return self.be.ledger.totals().asdict()

    def phase_totals(self, name):
        return self.be.ledger.phase_totals(name).asdict()
