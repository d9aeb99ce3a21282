// CPU reference arm: times the UNMODIFIED reference (oracle/_ref, compiled from
// /root/reference/proj/src by oracle/ref.mk) running the same hot-path op
// sequence that bench.py times on the GPU. TEST/BENCH INFRASTRUCTURE ONLY —
// bench.py --impl reference executes this binary; nothing in the product
// links it.
//
// Workloads (reference call sites):
//   llama   : one Llama-3-8B-shaped decoder-layer hot path at 2^15 slots
//             (ring 2^16): Q,K,V 4096^2 vmm_interleaved (vmm.cpp:179) ->
//             rope_apply x2 + make_v_pieces + v_append + k_append
//             (kv_attention.cpp:111-182) -> qk_dot (184) -> exact softmax (395)
//             -> softmax_times_v (216) -> W_O 4096^2 -> gate/up 4096->14336 ->
//             down 14336->4096, cache at n'=2047 -> 2048.
//   gpt2    : GPT-2 layer linear path at 2^15 slots (4x 768^2, 768->3072, 3072->768).
//   vmm768  : one 768x768 vmm at 2^14 slots (C1).
// Output: one JSON line {"workload", "ms_per_step", "steps", "warmup", "counts"}.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "slotforge/engine.hpp"
#include "slotforge/kv_attention.hpp"
#include "slotforge/layouts.hpp"
#include "slotforge/vmm.hpp"

using namespace slotforge;

namespace {

// slotforge_cli.cpp:88-92 convention: deterministic synthetic weights.
FunctorWeight bench_weight(int rows, int cols) {
  return FunctorWeight(rows, cols, [](int r, int c) {
    return std::sin(0.001 * (static_cast<double>(r) * 31.0 + c) + 0.25);
  });
}

SlotVector bench_vector(int N, unsigned seed) {
  std::mt19937_64 rng(seed);
  std::normal_distribution<double> dist(0.0, 1.0);
  SlotVector s(N);
  for (int i = 0; i < N; ++i) s[i] = dist(rng);
  return s;
}

Ciphertext fresh(SimBackend& be, int N, int d, int level, int offset, unsigned seed) {
  Layout ly = make_interleaved(d, N, offset);
  SlotVector s = SlotVector::Zero(N);
  SlotVector r = bench_vector(N, seed);
  for (int e = 0; e < d; ++e) s[e * ly.t + offset] = r[e];
  return be.encrypt(s, level, ly);
}

struct Llama {
  int N = 32768, d = 4096, H = 32, ff = 14336, np = 2048;
  AttentionConfig cfg{32768, 4096, 32, 0, 2048};
  KVCache base;
};

KVCache direct_cache(SimBackend& be, const AttentionConfig& cfg, int n, int level) {
  const int N = cfg.N, t = cfg.t(), dh = cfg.d_head(), gt = cfg.group_tokens();
  std::mt19937_64 rng(7);
  std::normal_distribution<double> dist(0.0, 1.0);
  KVCache c;
  c.n_prime = n;
  for (int j = 0; j * t < n; ++j) {
    SlotVector s = SlotVector::Zero(N);
    for (int tau = 0; tau < t && j * t + tau < n; ++tau)
      for (int E = 0; E < cfg.d; ++E) s[E * t + tau] = dist(rng);
    c.k_cts.push_back(be.encrypt(std::move(s), level));
  }
  for (int g = 0; g * gt < n; ++g) {
    std::vector<SlotVector> rows(v_variant_count(cfg), SlotVector::Zero(N));
    for (int u = g * gt; u < std::min(n, (g + 1) * gt); ++u) {
      const int ul = u - g * gt, j0 = ul % t;
      for (int h = 0; h < cfg.H; ++h)
        for (int e = 0; e < dh; ++e)
          rows[v_variant_index(cfg, v_variant_of(cfg, e, ul))][(h * dh + e) * t + j0] = dist(rng);
    }
    std::vector<Ciphertext> enc;
    for (auto& r : rows) enc.push_back(be.encrypt(std::move(r), level));
    c.v_cts.push_back(std::move(enc));
  }
  return c;
}

// Table-4 stage levels: QKV 4, RoPE&Cache 3, QK^T 2, S*V 2,
// out-proj 7, up/gate 3, down 1.
void llama_step(SimBackend& be, const Llama& m, int pos) {
  const int N = m.N, d = m.d, t = m.cfg.t();
  const auto wq = bench_weight(d, d), wk = bench_weight(d, d), wv = bench_weight(d, d), wo = bench_weight(d, d);
  const auto wg = bench_weight(d, m.ff), wu = bench_weight(d, m.ff), wd = bench_weight(m.ff, d);
  Ciphertext x = fresh(be, N, d, 4, 0, 42);
  Ciphertext q_raw, k_raw, v_raw;
  {
    auto ph = be.phase("Q, K, V");
    q_raw = vmm_interleaved(be, x, wq, {.bsgs = true});
    k_raw = vmm_interleaved(be, x, wk, {.bsgs = true, .out_offset = pos % t});
    v_raw = vmm_interleaved(be, x, wv, {.bsgs = true, .out_offset = pos % t});
  }
  KVCache cache;
  Ciphertext qc;
  {
    auto ph = be.phase("RoPE & Cache");
    qc = rope_apply(be, q_raw, m.cfg, pos);
    Ciphertext kc = rope_apply(be, k_raw, m.cfg, pos);
    cache = v_append(be, m.base, make_v_pieces(be, v_raw, m.cfg, pos), m.cfg);
    cache = k_append(be, cache, kc, m.cfg);
  }
  std::vector<Ciphertext> maps;
  {
    auto ph = be.phase("QK^T");
    maps = qk_dot(be, qc, cache, m.cfg);
  }
  auto probs = exact_softmax_maps(be, maps, m.cfg, cache.n_prime);
  for (auto& p : probs) p = be.encrypt(p.slots, 2);  // client re-encrypts at the S*V level (off-ledger)
  {
    auto ph = be.phase("Score*V");
    (void)softmax_times_v(be, probs, cache, m.cfg);
  }
  {
    auto ph = be.phase("Output projection");
    (void)vmm_interleaved(be, fresh(be, N, d, 7, 0, 43), wo, {.bsgs = true});
  }
  {
    auto ph = be.phase("Up & Gate projection");
    Ciphertext h = fresh(be, N, d, 3, 0, 44);
    (void)vmm_interleaved(be, h, wg, {.bsgs = true});
    (void)vmm_interleaved(be, h, wu, {.bsgs = true});
  }
  {
    auto ph = be.phase("Down projection");
    (void)vmm_interleaved(be, fresh(be, N, padded_dim(m.ff), 1, 0, 45), wd, {.bsgs = true});
  }
}

void gpt2_step(SimBackend& be) {
  const int N = 32768, d = 768, dp = 1024, ff = 3072;
  const auto w = bench_weight(d, d), wu = bench_weight(d, ff), wd = bench_weight(ff, d);
  Ciphertext x = fresh(be, N, dp, 4, 0, 42);
  for (int i = 0; i < 4; ++i) (void)vmm_interleaved(be, x, w, {.bsgs = true});
  (void)vmm_interleaved(be, fresh(be, N, dp, 3, 0, 44), wu, {.bsgs = true});
  (void)vmm_interleaved(be, fresh(be, N, ff > 2048 ? 4096 : ff, 1, 0, 45), wd, {.bsgs = true});
}

void vmm768_step(SimBackend& be) {
  const int N = 16384;
  (void)vmm_interleaved(be, fresh(be, N, 1024, 4, 0, 42), bench_weight(768, 768), {.bsgs = true});
}

}  // namespace

int main(int argc, char** argv) {
  std::string workload = "llama";
  int steps = 3, warmup = 1;
  for (int i = 1; i + 1 < argc; i += 2) {
    if (!std::strcmp(argv[i], "--workload")) workload = argv[i + 1];
    if (!std::strcmp(argv[i], "--steps")) steps = std::atoi(argv[i + 1]);
    if (!std::strcmp(argv[i], "--warmup")) warmup = std::atoi(argv[i + 1]);
  }
  const int N = workload == "vmm768" ? 16384 : 32768;
  SimBackend be({N, 13});
  Llama m;
  if (workload == "llama") m.base = direct_cache(be, m.cfg, m.np - 1, 2);
  auto run = [&](int pos) {
    if (workload == "llama")
      llama_step(be, m, pos);
    else if (workload == "gpt2")
      gpt2_step(be);
    else
      vmm768_step(be);
  };
  for (int i = 0; i < warmup; ++i) run(m.np - 1);
  be.ledger().reset();
  const auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < steps; ++i) run(m.np - 1);
  const auto t1 = std::chrono::steady_clock::now();
  const double ms = std::chrono::duration<double, std::milli>(t1 - t0).count() / std::max(steps, 1);
  const OpCounts c = be.ledger().totals();
  std::printf(
      "{\"workload\": \"%s\", \"ms_per_step\": %.3f, \"steps\": %d, \"warmup\": %d, \"cores\": 1, "
      "\"counts\": {\"rotations\": %lld, \"hoisted_rotations\": %lld, \"ct_pt_mults\": %lld, "
      "\"ct_ct_mults\": %lld, \"additions\": %lld}}\n",
      workload.c_str(), ms, steps, warmup, c.rotations / std::max(steps, 1),
      c.hoisted_rotations / std::max(steps, 1), c.ct_pt_mults / std::max(steps, 1),
      c.ct_ct_mults / std::max(steps, 1), c.additions / std::max(steps, 1));
  return 0;
}
