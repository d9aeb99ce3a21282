// Golden-vector generator: links the UNMODIFIED reference sources compiled
// into oracle/_ref (see oracle/ref.mk) and dumps, for a fixed set of seeded
// cases, the full slot content of every hot-path output together with the
// reference ledger counts and levels. TEST INFRASTRUCTURE ONLY; the emitted
// JSON is committed under tests/golden/ by tests/golden/make_golden.sh.
//
// Call sites exercised (reference file:line):
//   vmm_interleaved            proj/src/vmm.cpp:179-236
//   fused_extract (Rope/Mask)  proj/src/vmm.cpp:85-109
//   k_append / make_v_pieces / v_append   proj/src/kv_attention.cpp:131-182
//   qk_dot / softmax_times_v   proj/src/kv_attention.cpp:184-241
//   exact_softmax_maps         proj/src/kv_attention.cpp:395-412
//   prefill (vmm_batch, rope_apply_batch, inner_rotate, exact_softmax_prefill_maps)
//                              proj/src/kv_attention.cpp:119-129, 245-376, 414-454; vmm.cpp:30-43, 417-467
//   nonlinear ("nonlinear" set): eval_cheb, goldschmidt, approx_exp, approx_softmax,
//   approx_norm, approx_silu   proj/src/nonlinear.cpp:312-549
//   harness ("harness" set): make_weights / seeded_prompt / plaintext_reference /
//   plan_decode / run_generation (prefill_prompt + run_decode_step)
//                              proj/src/harness.cpp:197-352, 425-659, 712-857, 943-1053
#include <nlohmann/json.hpp>

#include <cstdio>
#include <functional>
#include <iostream>
#include <optional>
#include <random>
#include <string>
#include <vector>

#include "slotforge/engine.hpp"
#include "slotforge/harness.hpp"
#include "slotforge/nonlinear.hpp"
#include "slotforge/kv_attention.hpp"
#include "slotforge/layouts.hpp"
#include "slotforge/vmm.hpp"

using nlohmann::json;
using namespace slotforge;

namespace {

json vec_json(const double* p, long n) {
  json a = json::array();
  for (long i = 0; i < n; ++i) a.push_back(p[i]);
  return a;
}
json sv_json(const SlotVector& s) { return vec_json(s.data(), s.size()); }
json v_json(const Vector& s) { return vec_json(s.data(), s.size()); }
json m_json(const Matrix& m) { return vec_json(m.data(), m.size()); }

json counts_json(const OpCounts& c) {
  return json{{"rotations", c.rotations},   {"hoisted_rotations", c.hoisted_rotations},
              {"ct_pt_mults", c.ct_pt_mults}, {"ct_ct_mults", c.ct_ct_mults},
              {"additions", c.additions},   {"bootstraps", c.bootstraps}};
}
json layout_json(const std::optional<Layout>& ly) {
  if (!ly) return nullptr;
  return json{{"kind", to_string(ly->kind)}, {"d", ly->d},         {"t", ly->t},
              {"offset", ly->offset},       {"heads", ly->heads}, {"deferred_mask", ly->deferred_mask}};
}

Matrix random_matrix(std::mt19937_64& rng, int r, int c) {
  std::normal_distribution<double> dist(0.0, 1.0);
  Matrix m(r, c);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) m(i, j) = dist(rng);
  return m;
}
Vector random_vector(std::mt19937_64& rng, int n) {
  std::normal_distribution<double> dist(0.0, 1.0);
  Vector v(n);
  for (int i = 0; i < n; ++i) v[i] = dist(rng);
  return v;
}

json vmm_case(int N, int rows, int cols, int tau_in, int tau_out, bool bsgs, bool mask, unsigned seed) {
  const int L = 8;
  std::mt19937_64 rng(seed);
  Matrix w = random_matrix(rng, rows, cols);
  Vector x = random_vector(rng, rows);
  SimBackend be({N, L});
  const int d_in = padded_dim(rows);
  Layout lin = make_interleaved(d_in, N, tau_in);
  SlotVector xs = encode(pad_to(x, d_in), lin, N);
  Ciphertext cx = be.encrypt(xs, L, lin);
  Ciphertext cy = vmm_interleaved(be, cx, MatrixWeight(w), {.bsgs = bsgs, .out_offset = tau_out, .mask_output = mask});
  VmmCost pc = predict_interleaved_cost({N, L}, rows, cols, {.bsgs = bsgs, .out_offset = tau_out, .mask_output = mask});
  return json{{"kind", "vmm"},
              {"N", N},
              {"L", L},
              {"rows", rows},
              {"cols", cols},
              {"tau_in", tau_in},
              {"tau_out", tau_out},
              {"bsgs", bsgs},
              {"mask_output", mask},
              {"W", m_json(w)},
              {"x", v_json(x)},
              {"x_slots", sv_json(xs)},
              {"y_slots", sv_json(cy.slots)},
              {"y", v_json(decode(cy.slots, *cy.layout))},
              {"layout", layout_json(cy.layout)},
              {"level", cy.level},
              {"counts", counts_json(be.ledger().totals())},
              {"predicted", json{{"rotations", pc.rotations}, {"ct_pt_mults", pc.ct_pt_mults}, {"depth", pc.depth}}}};
}

json rope_case(int N, int d, int d_head, int offset, long long pos, unsigned seed) {
  const int L = 6;
  std::mt19937_64 rng(seed);
  Vector x = random_vector(rng, d);
  SimBackend be({N, L});
  Layout ly = make_interleaved(d, N, offset);
  ly.deferred_mask = true;
  SlotVector raw = encode(x, ly, N);
  for (int i = 0; i < N; ++i)
    if (i % ly.t != offset) raw[i] = 99.0 + i;  // garbage a vmm would leave
  Ciphertext cx = be.encrypt(raw, L, ly);
  RoPEParams p{10000.0, pos, d_head, ly.t};
  auto pts = rope_plaintexts(p, ly, N);
  Ciphertext cy = fused_extract(be, cx, Successor::Rope, &p);
  return json{{"kind", "rope"},   {"N", N},           {"L", L},
              {"d", d},           {"d_head", d_head}, {"offset", offset},
              {"pos", pos},       {"x_slots", sv_json(raw)},
              {"p0", sv_json(pts[0])}, {"p1", sv_json(pts[1])}, {"p2", sv_json(pts[2])},
              {"y_slots", sv_json(cy.slots)}, {"level", cy.level},
              {"layout", layout_json(cy.layout)}, {"counts", counts_json(be.ledger().totals())}};
}

// Decode-time attention over a cache built by the append protocol: every token
// goes through make_v_pieces / v_append / k_append (garbage-carrying V input,
// as in attn-bench, slotforge_cli.cpp:189-198), then one query runs qk_dot,
// exact softmax and softmax_times_v.
json attn_case(int N, int d, int H, int np, unsigned seed) {
  const int L = 12;
  AttentionConfig cfg{N, d, H, 0, np};
  SimBackend be({N, L});
  validate_attention_config(cfg, N);
  const int t = cfg.t();
  std::mt19937_64 rng(seed);
  Matrix K = random_matrix(rng, np, d), V = random_matrix(rng, np, d);
  Vector q = random_vector(rng, d);
  KVCache cache;
  json appends = json::array();
  for (int u = 0; u < np; ++u) {
    Layout vly = make_interleaved(d, N, u % t, H);
    vly.deferred_mask = true;
    SlotVector open = SlotVector::Constant(N, 7.5);
    for (int E = 0; E < d; ++E) open[E * t + u % t] = V(u, E);
    Ciphertext v_open = be.encrypt(open, L - 1, vly);
    OpCounts c0 = be.ledger().totals();
    auto parts = make_v_pieces(be, v_open, cfg, u);
    cache = v_append(be, cache, parts, cfg);
    Layout kly = make_interleaved(d, N, u % t, H);
    Vector krow(d);
    for (int E = 0; E < d; ++E) krow[E] = K(u, E);
    cache = k_append(be, cache, be.encrypt(encode(krow, kly, N), L - 2, kly), cfg);
    OpCounts c1 = be.ledger().totals();
    OpCounts delta;
    delta.rotations = c1.rotations - c0.rotations;
    delta.ct_pt_mults = c1.ct_pt_mults - c0.ct_pt_mults;
    delta.ct_ct_mults = c1.ct_ct_mults - c0.ct_ct_mults;
    delta.additions = c1.additions - c0.additions;
    appends.push_back(counts_json(delta));
  }
  json k_cts = json::array();
  for (const auto& c : cache.k_cts) k_cts.push_back(json{{"slots", sv_json(c.slots)}, {"level", c.level}});
  json v_cts = json::array();
  for (const auto& grp : cache.v_cts) {
    json g = json::array();
    for (const auto& c : grp) g.push_back(json{{"slots", sv_json(c.slots)}, {"level", c.level}});
    v_cts.push_back(g);
  }
  be.ledger().reset();
  Layout qly = make_interleaved(d, N, 0, H);
  Ciphertext qc = be.encrypt(encode(q, qly, N), L - 2, qly);
  std::vector<Ciphertext> maps;
  {
    auto ph = be.phase("QK^T");
    maps = qk_dot(be, qc, cache, cfg);
  }
  auto probs = exact_softmax_maps(be, maps, cfg, cache.n_prime);
  Ciphertext out;
  {
    auto ph = be.phase("Score*V");
    out = softmax_times_v(be, probs, cache, cfg);
  }
  json jm = json::array(), jp = json::array();
  for (auto& m : maps) jm.push_back(sv_json(m.slots));
  for (auto& p : probs) jp.push_back(sv_json(p.slots));
  return json{{"kind", "attn"},
              {"N", N},
              {"L", L},
              {"d", d},
              {"H", H},
              {"n_prime", np},
              {"K", m_json(K)},
              {"V", m_json(V)},
              {"q", v_json(q)},
              {"append_counts", appends},
              {"k_cts", k_cts},
              {"v_cts", v_cts},
              {"maps", jm},
              {"map_level", maps.front().level},
              {"probs", jp},
              {"out_slots", sv_json(out.slots)},
              {"out", v_json(decode(out.slots, *out.layout))},
              {"out_level", out.level},
              {"out_layout", layout_json(out.layout)},
              {"qk_counts", counts_json(be.ledger().phase_totals("QK^T"))},
              {"sv_counts", counts_json(be.ledger().phase_totals("Score*V"))}};
}

// Prefill of an n0-token prompt (kv_attention.cpp:245-376) with the exact
// softmax hook, as in test_kv.cpp:360-428.
json prefill_case(int N, int d, int H, int n0, unsigned seed) {
  const int L = 10;
  const int t = N / d;
  AttentionConfig cfg{N, d, H, n0, std::max(n0, 16)};
  SimBackend be({N, L});
  validate_attention_config(cfg, N);
  std::mt19937_64 rng(seed);
  Matrix Wq = random_matrix(rng, d, d), Wk = random_matrix(rng, d, d), Wv = random_matrix(rng, d, d);
  MatrixWeight wq(Wq), wk(Wk), wv(Wv);
  Matrix X = random_matrix(rng, n0, d);
  const int P = (n0 + t - 1) / t;
  std::vector<Ciphertext> xs;
  json xj = json::array();
  for (int p = 0; p < P; ++p) {
    SlotVector sl = SlotVector::Zero(N);
    for (int tau = 0; tau < t && p * t + tau < n0; ++tau)
      for (int E = 0; E < d; ++E) sl[E * t + tau] = X(p * t + tau, E);
    xj.push_back(sv_json(sl));
    xs.push_back(be.encrypt(std::move(sl), -1, make_interleaved(d, N, 0, H)));
  }
  PrefillResult pre = prefill(be, xs, {wq, wk, wv, 10000.0}, cfg,
                              [](Backend& b, const PrefillMaps& m, const AttentionConfig& c, int n) {
                                return exact_softmax_prefill_maps(b, m, c, n);
                              });
  json k_cts = json::array();
  for (const auto& c : pre.cache.k_cts) k_cts.push_back(json{{"slots", sv_json(c.slots)}, {"level", c.level}});
  json v_cts = json::array();
  for (const auto& grp : pre.cache.v_cts) {
    json g = json::array();
    for (const auto& c : grp) g.push_back(json{{"slots", sv_json(c.slots)}, {"level", c.level}});
    v_cts.push_back(g);
  }
  json att = json::array();
  for (const auto& a : pre.attention)
    att.push_back(json{{"slots", sv_json(a.slots)}, {"level", a.level}, {"layout", layout_json(a.layout)}});
  return json{{"kind", "prefill"}, {"N", N}, {"L", L}, {"d", d}, {"H", H}, {"n0", n0},
              {"Wq", m_json(Wq)}, {"Wk", m_json(Wk)}, {"Wv", m_json(Wv)}, {"X", m_json(X)},
              {"x_prompt", xj}, {"k_cts", k_cts}, {"v_cts", v_cts}, {"attention", att},
              {"n_prime", pre.cache.n_prime}, {"counts", counts_json(be.ledger().totals())}};
}

json engine_case() {
  SimBackend be({4, 3});
  SlotVector a(4);
  a << 1, 2, 3, 4;
  auto ct = be.encrypt(a, 3);
  json rots = json::array();
  for (int r : {1, -1, 0, 4, 5, 3}) rots.push_back(json{{"r", r}, {"slots", sv_json(be.rotate(ct, r).slots)}});
  return json{{"kind", "engine_rotate"}, {"N", 4}, {"input", sv_json(a)}, {"rotations", rots},
              {"counted", be.ledger().totals().rotations}};
}

json mat_stats(const Matrix& m) {
  double s = 0, s2 = 0;
  for (long i = 0; i < m.size(); ++i) s += m.data()[i], s2 += m.data()[i] * m.data()[i];
  return json{{"rows", m.rows()}, {"cols", m.cols()}, {"sum", s}, {"sumsq", s2},
              {"head", vec_json(m.data(), std::min<long>(4, m.size()))},
              {"last", m.data()[m.size() - 1]}};
}
json vec_stats(const Vector& v) {
  double s = 0;
  for (long i = 0; i < v.size(); ++i) s += v[i];
  return json{{"n", v.size()}, {"sum", s}, {"head", vec_json(v.data(), std::min<long>(4, v.size()))}};
}

// One seeded generation run of the reference harness: the config, weight
// fingerprints (Python port check), prompt, plaintext trace, the solver's plan
// (the harness port takes the plan as input), the full Report (tokens, level
// trace, per-phase ledger) and the prefill's final-block states.
json harness_case(const ModelConfig& cfg, int n0, int gen_len) {
  const ModelWeights w = make_weights(cfg);
  const std::vector<int> prompt = seeded_prompt(cfg, n0);
  const ReferenceTrace ref = plaintext_reference(cfg, w, prompt, gen_len);
  const PlacementPlan plan = plan_decode(cfg, w, n0 + gen_len);
  const Report rep = run_generation(cfg, w, prompt, gen_len, nullptr);
  json wj;
  wj["embedding"] = mat_stats(w.embedding);
  json blocks = json::array();
  for (const auto& b : w.blocks)
    blocks.push_back(json{{"wq", mat_stats(b.wq)},         {"wk", mat_stats(b.wk)},
                          {"wv", mat_stats(b.wv)},         {"wo", mat_stats(b.wo)},
                          {"w_gate", mat_stats(b.w_gate)}, {"w_up", mat_stats(b.w_up)},
                          {"w_down", mat_stats(b.w_down)}, {"gamma1", vec_stats(b.gamma1)},
                          {"beta1", vec_stats(b.beta1)},   {"gamma2", vec_stats(b.gamma2)},
                          {"beta2", vec_stats(b.beta2)}});
  wj["blocks"] = blocks;
  json states = json::array();
  for (const auto& v : ref.final_states) states.push_back(v_json(v));
  return json{{"kind", "harness"},
              {"config", json::parse(cfg.to_json())},
              {"n0", n0},
              {"gen_len", gen_len},
              {"weights", wj},
              {"prompt", prompt},
              {"ref_tokens", ref.tokens},
              {"ref_final_states", states},
              {"plan", json::parse(plan.to_json())},
              {"plan_terminal_level", plan.terminal_level},
              {"plan_bootstrap_count", plan.bootstrap_count},
              {"report", json::parse(rep.to_json())},
              {"report_csv", rep.to_csv()}};
}

SlotVector uniform_slots(std::mt19937_64& rng, int N, double lo, double hi) {
  std::uniform_real_distribution<double> u(lo, hi);
  SlotVector s(N);
  for (int i = 0; i < N; ++i) s[i] = u(rng);
  return s;
}

json spec_json(const ApproxSpec& s) { return json::parse(approx_spec_to_json(s)); }

// one nonlinear call on a fresh SimBackend: inputs, outputs, levels, ledger
json nl_case(const std::string& op, int N, int L, const std::vector<SlotVector>& ins, const ApproxSpec* spec,
             const std::function<std::vector<Ciphertext>(SimBackend&, const std::vector<Ciphertext>&)>& fn,
             json extra, const std::optional<Layout>& ly = std::nullopt) {
  SimBackend be({N, L});
  std::vector<Ciphertext> cts;
  json jin = json::array();
  for (const auto& s : ins) {
    cts.push_back(ly ? be.encrypt(s, L, *ly) : be.encrypt(s, L));
    jin.push_back(sv_json(s));
  }
  be.ledger().reset();
  auto outs = fn(be, cts);
  json jout = json::array(), lv = json::array();
  for (const auto& o : outs) {
    jout.push_back(sv_json(o.slots));
    lv.push_back(o.level);
  }
  json j{{"kind", "nonlinear"}, {"op", op},        {"N", N},
         {"L", L},              {"inputs", jin},   {"outputs", jout},
         {"out_levels", lv},    {"counts", counts_json(be.ledger().totals())},
         {"extra", extra},      {"layout", layout_json(ly)}};
  if (spec) j["spec"] = spec_json(*spec);
  return j;
}

json nonlinear_cases() {
  json cases = json::array();
  std::mt19937_64 rng(11);
  // eval_cheb at the degrees of test_nonlinear.cpp:49-70
  for (int deg : {1, 2, 3, 5, 8, 13, 20, 31}) {
    auto f = [](double x) { return std::sin(3.0 * x) + 0.25 * x; };
    auto coeffs = fit_cheb_ls(f, -2.0, 1.5, deg);
    cases.push_back(nl_case("eval_cheb", 64, 20, {uniform_slots(rng, 64, -2.0, 1.5)}, nullptr,
                            [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                              return std::vector<Ciphertext>{eval_cheb(be, x[0], -2.0, 1.5, coeffs)};
                            },
                            json{{"lo", -2.0}, {"hi", 1.5}, {"coeffs", coeffs}, {"deg", deg}}));
  }
  {  // coefficient mask (test_nonlinear.cpp:72-88)
    auto silu = [](double x) { return x / (1.0 + std::exp(-x)); };
    auto coeffs = fit_cheb_ls(silu, -4.0, 4.0, 15);
    SlotVector mask = SlotVector::Zero(32);
    for (int i = 0; i < 32; i += 2) mask[i] = 1.0;
    cases.push_back(nl_case("eval_cheb_masked", 32, 12, {uniform_slots(rng, 32, -4.0, 4.0)}, nullptr,
                            [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                              return std::vector<Ciphertext>{eval_cheb(be, x[0], -4.0, 4.0, coeffs, &mask)};
                            },
                            json{{"lo", -4.0}, {"hi", 4.0}, {"coeffs", coeffs}, {"mask", sv_json(mask)}}));
  }
  for (const char* preset : {"desk-default", "desk-shallow"}) {
    const ApproxSpec inv = desk_spec(preset, "inverse");
    cases.push_back(nl_case("inverse", 64, 24, {uniform_slots(rng, 64, 1.0 / 64.0, 1.0)}, &inv,
                            [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                              return std::vector<Ciphertext>{goldschmidt(be, x[0], GoldschmidtKind::Inverse, inv)};
                            },
                            json{{"preset", preset}}));
    const ApproxSpec rs = desk_spec(preset, "rsqrt");
    cases.push_back(nl_case("rsqrt", 64, 24, {uniform_slots(rng, 64, 1.0 / 16.0, 1.0)}, &rs,
                            [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                              return std::vector<Ciphertext>{goldschmidt(be, x[0], GoldschmidtKind::Rsqrt, rs)};
                            },
                            json{{"preset", preset}}));
    const ApproxSpec ex = desk_spec(preset, "exp");
    cases.push_back(nl_case("exp", 64, 24, {uniform_slots(rng, 64, -8.0, 4.0)}, &ex,
                            [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                              return std::vector<Ciphertext>{approx_exp(be, x[0], ex)};
                            },
                            json{{"preset", preset}}));
    const ApproxSpec sm = desk_spec(preset, "softmax");
    for (auto [heads, n] : std::vector<std::pair<int, int>>{{1, 20}, {2, 13}, {4, 19}}) {
      const int gt = 32 / heads;
      const int nm = (n + gt - 1) / gt;
      std::vector<SlotVector> maps;
      for (int m = 0; m < nm; ++m) {
        SlotVector s = SlotVector::Zero(32);
        const int cnt = std::min(gt, n - m * gt);
        for (int h = 0; h < heads; ++h) {
          SlotVector u = uniform_slots(rng, cnt, -6.0, 3.0);
          for (int k = 0; k < cnt; ++k) s[h * gt + k] = u[k];
        }
        maps.push_back(s);
      }
      cases.push_back(nl_case("softmax", 32, 26, maps, &sm,
                              [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                                return approx_softmax(be, x, n, heads, sm);
                              },
                              json{{"preset", preset}, {"heads", heads}, {"n_prime", n}}));
    }
    const ApproxSpec nm = desk_spec(preset, "norm");
    for (int d : {16, 8}) {
      const Layout ly = make_interleaved(d, 64, 1, 1);
      SlotVector s = SlotVector::Zero(64);
      SlotVector u = uniform_slots(rng, d, -1.5, 2.0);
      for (int e = 0; e < d; ++e) s[e * ly.t + ly.offset] = u[e];
      const SlotVector gs = uniform_slots(rng, d, 0.5, 1.5), bs = uniform_slots(rng, d, -0.2, 0.2);
      Vector gamma(d), beta(d);
      for (int e = 0; e < d; ++e) gamma[e] = gs[e], beta[e] = bs[e];
      cases.push_back(nl_case("norm", 64, 32, {s}, &nm,
                              [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                                return std::vector<Ciphertext>{approx_norm(be, x[0], gamma, beta, 1e-5, nm)};
                              },
                              json{{"preset", preset}, {"gamma", v_json(gamma)}, {"beta", v_json(beta)},
                                   {"eps", 1e-5}},
                              ly));
    }
    for (const char* fn : {"silu", "gelu"}) {
      const ApproxSpec si = desk_spec(preset, fn);
      Layout ly = make_interleaved(16, 64, 2, 1);
      ly.deferred_mask = true;  // vmm garbage on the invalid slots
      SlotVector s = uniform_slots(rng, 64, -10.0, 10.0);
      cases.push_back(nl_case("silu", 64, 16, {s}, &si,
                              [&](SimBackend& be, const std::vector<Ciphertext>& x) {
                                return std::vector<Ciphertext>{approx_silu(be, x[0], si)};
                              },
                              json{{"preset", preset}, {"function", fn}}, ly));
    }
  }
  return cases;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "small";
  json cases = json::array();
  unsigned seed = 1000;
  if (which == "small") {
    cases.push_back(engine_case());
    for (int N : {8, 64, 256}) {
      std::vector<std::pair<int, int>> shapes;
      for (int d : {2, 8, 32})
        if (d <= N) shapes.emplace_back(d, d);
      for (int d : {2, 8})
        for (int a : {2, 4})
          if (d * a <= N) {
            shapes.emplace_back(d, d * a);
            shapes.emplace_back(d * a, d);
          }
      if (N <= 64) shapes.emplace_back(N, N);
      shapes.emplace_back(3, 5);
      for (auto [r, c] : shapes) {
        const int t_in = N / padded_dim(r), t_out = N / padded_dim(c);
        for (bool bsgs : {false, true})
          for (int ti : {0, t_in - 1})
            for (int to : {0, t_out - 1}) {
              if (ti == t_in - 1 && to == t_out - 1 && t_in > 1 && !bsgs) continue;
              cases.push_back(vmm_case(N, r, c, ti, to, bsgs, (seed % 3) == 0, seed));
              ++seed;
            }
      }
    }
    for (int off : {0, 2}) cases.push_back(rope_case(32, 8, 4, off, 7, seed++));
    cases.push_back(rope_case(64, 16, 8, 3, 123, seed++));
    for (int d : {4, 16})
      for (int H : {1, 2, 4})
        for (int np : {1, 5, 13}) cases.push_back(attn_case(64, d, H, np, seed++));
    cases.push_back(attn_case(256, 64, 4, 21, seed++));
    cases.push_back(vmm_case(256, 256, 256, 0, 0, true, false, seed++));  // t = 1 edge
    // prefill shapes of test_kv.cpp:360-428 and a 1-token prompt (430-459)
    cases.push_back(prefill_case(16, 4, 2, 6, seed++));
    cases.push_back(prefill_case(16, 8, 2, 11, seed++));
    cases.push_back(prefill_case(16, 4, 1, 1, seed++));
    cases.push_back(prefill_case(64, 16, 4, 13, seed++));
  } else if (which == "nonlinear") {
    cases = nonlinear_cases();
  } else if (which == "harness") {
    // test_harness.cpp: desk_config (d 64, H 4, 2 blocks, vocab 32, N 256, L 13)
    // exact mode seeds 3 / 9 (prompt 8 + 8 generated; single-token prompt),
    // and tiny_config (d 8, H 2, 1 block, N 32)
    ModelConfig desk;
    desk.mode = NonlinearMode::Exact;
    desk.seed = 3;
    cases.push_back(harness_case(desk, 8, 8));
    desk.seed = 9;
    cases.push_back(harness_case(desk, 1, 1));
    ModelConfig tiny;
    tiny.d = 8, tiny.H = 2, tiny.n_layers = 1, tiny.ffn_alpha = 2, tiny.vocab = 8, tiny.N = 32, tiny.L = 13;
    tiny.seed = 11;
    cases.push_back(harness_case(tiny, 5, 3));
    // approx mode: homomorphic softmax / norm / SiLU under the solver's plan
    ModelConfig ap;
    ap.mode = NonlinearMode::Approx;
    ap.seed = 5;
    cases.push_back(harness_case(ap, 4, 2));
    tiny.mode = NonlinearMode::Approx;
    cases.push_back(harness_case(tiny, 3, 2));
  } else if (which == "medium") {
    // N = 2048 slots (ring degree 4096): the GPU parity size
    cases.push_back(vmm_case(2048, 64, 64, 0, 0, true, false, 7001));
    cases.push_back(vmm_case(2048, 64, 256, 5, 3, true, false, 7002));
    cases.push_back(vmm_case(2048, 256, 64, 0, 7, true, true, 7003));
    cases.push_back(vmm_case(2048, 100, 60, 3, 1, false, false, 7004));
    cases.push_back(rope_case(2048, 128, 32, 5, 77, 7005));
    cases.push_back(attn_case(2048, 128, 4, 40, 7006));
    cases.push_back(attn_case(2048, 64, 1, 70, 7007));
    cases.push_back(prefill_case(2048, 256, 4, 19, 7008));
  }
  std::cout << json{{"generator", "oracle/ref_golden.cpp over /root/reference/proj/src (unmodified)"},
                    {"set", which},
                    {"cases", cases}}
                   .dump()
            << "\n";
  return 0;
}
