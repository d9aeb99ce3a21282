// TEST INFRASTRUCTURE: the reference's own hot-path code, unmodified, run on
// the B200 binding (integration/b200_backend.hpp) next to the reference's
// SimBackend and the CPU CKKS twin (oracle/twin_backend.hpp).
//
// Each case runs ONE program of reference calls -- vmm_interleaved
// (vmm.cpp:179-236), rope_apply / make_v_pieces / v_append / k_append
// (kv_attention.cpp:111-182), qk_dot (:184-214), exact_softmax_maps on the
// simulator (:394-412), softmax_times_v (:216-241) -- three times:
//   Sim   the reference SimBackend (cleartext slots; the semantic truth),
//   B200  B200Backend (every virtual op through the C ABI on the GPU),
//   Twin  TwinBackend (the same ops on the CPU CKKS oracle).
// and prints one JSON line per case with: the max |decrypt(B200) - Sim| over
// ALL N slots of every output (deferred garbage included), whether the B200
// and Twin ciphertext words are identical, whether levels / layouts equal
// Sim's, and whether the ledgers (B200Backend::ledger(), the library's own
// sf_ledger_totals, TwinBackend::ledger()) equal SimBackend's.
//   ref_on_b200 [case ...]     cases: vmm_small vmm_bsgs_deferred decode_small vmm_ring16 decode_ring16 errors
#include <cmath>
#include <cstdio>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "../integration/b200_backend.hpp"
#include "slotforge/kv_attention.hpp"
#include "slotforge/layouts.hpp"
#include "slotforge/vmm.hpp"
#include "twin_backend.hpp"

using namespace slotforge;

namespace {

using Upload = std::function<Ciphertext(const Ciphertext&, uint64_t seed)>;
using ProbsFn = std::function<std::vector<Ciphertext>(Backend&, const std::vector<Ciphertext>&, int n_prime)>;

Matrix random_matrix(std::mt19937_64& rng, int r, int c, double scale) {
  std::normal_distribution<double> dist(0.0, 1.0);
  Matrix m(r, c);
  for (int i = 0; i < r; ++i)
    for (int j = 0; j < c; ++j) m(i, j) = dist(rng) * scale;
  return m;
}
Vector random_vector(std::mt19937_64& rng, int n) {
  std::normal_distribution<double> dist(0.0, 1.0);
  Vector v(n);
  for (int i = 0; i < n; ++i) v[i] = dist(rng);
  return v;
}

struct Case {
  std::string name;
  int N, L, log_n;
  // VMM-only cases
  int rows = 0, cols = 0, out_offset = 0;
  bool bsgs = false, mask = false;
  // decode cases
  int d = 0, H = 1, tokens = 0;
};

// The program: returns every ciphertext worth comparing.
std::vector<Ciphertext> program(Backend& be, const Case& c, const Upload& up, const ProbsFn& probs_fn) {
  std::mt19937_64 rng(1234);
  std::vector<Ciphertext> outs;
  const int N = c.N;
  if (c.tokens == 0) {  // one VMM (vmm.cpp:179-236)
    MatrixWeight W(random_matrix(rng, c.rows, c.cols, 1.0 / std::sqrt((double)c.rows)));
    const Layout ly = make_interleaved((int)next_pow2(c.rows), N, 0);
    Ciphertext x = up(be.encrypt(encode(random_vector(rng, c.rows), ly, N), c.L, ly), 11);
    outs.push_back(vmm_interleaved(be, x, W, {.bsgs = c.bsgs, .out_offset = c.out_offset, .mask_output = c.mask}));
    return outs;
  }
  // one decode step per token (test_kv.cpp:386-400's loop): Q/K/V projections,
  // RoPE, cache appends; then QK^T, exact softmax, Score*V at the last token
  AttentionConfig cfg{N, c.d, c.H, 0, 64};
  const int t = cfg.t();
  const double ws = 1.0 / std::sqrt((double)c.d);
  MatrixWeight wq(random_matrix(rng, c.d, c.d, ws)), wk(random_matrix(rng, c.d, c.d, ws)),
      wv(random_matrix(rng, c.d, c.d, ws));
  const Layout ly = make_interleaved(c.d, N, 0, c.H);
  KVCache cache;
  Ciphertext q;
  for (int u = 0; u < c.tokens; ++u) {
    Ciphertext xc = up(be.encrypt(encode(random_vector(rng, c.d), ly, N), c.L, ly), 100 + u);
    Ciphertext k_new = rope_apply(be, vmm_interleaved(be, xc, wk, {.out_offset = u % t}), cfg, u);
    Ciphertext v_raw = vmm_interleaved(be, xc, wv, {.out_offset = u % t});
    cache = v_append(be, cache, make_v_pieces(be, v_raw, cfg, u), cfg);
    cache = k_append(be, cache, k_new, cfg);
    q = rope_apply(be, vmm_interleaved(be, xc, wq, {}), cfg, u);
  }
  outs.push_back(q);
  for (const auto& k : cache.k_cts) outs.push_back(k);
  for (const auto& g : cache.v_cts)
    for (const auto& v : g) outs.push_back(v);
  std::vector<Ciphertext> maps = qk_dot(be, q, cache, cfg);
  for (const auto& m : maps) outs.push_back(m);
  std::vector<Ciphertext> probs = probs_fn(be, maps, cache.n_prime);
  outs.push_back(softmax_times_v(be, probs, cache, cfg));
  return outs;
}

bool same_layout(const std::optional<Layout>& a, const std::optional<Layout>& b) {
  if (a.has_value() != b.has_value()) return false;
  return !a || *a == *b;
}

void run_case(const Case& c) {
  const EngineParams ep{c.N, c.L};
  SimBackend sim(ep);
  B200Options opt;
  opt.log_n = c.log_n;
  opt.alpha = 2;
  opt.seed = 5;
  B200Backend gpu(ep, opt);
  TwinBackend twin(ep, c.log_n, 2, 5);

  // the simulator's exact softmax (the reference's client hook) -> cleartext
  // probability maps, handed to the encrypted runs as fresh encryptions
  std::vector<Ciphertext> sim_probs;
  ProbsFn sim_fn = [&](Backend& be, const std::vector<Ciphertext>& maps, int n_prime) {
    AttentionConfig cfg{c.N, c.d, c.H, 0, 64};
    sim_probs = exact_softmax_maps(be, maps, cfg, n_prime);
    return sim_probs;
  };
  auto enc_fn = [&sim_probs](auto& be) {
    auto* pb = &be;
    return ProbsFn([pb, &sim_probs](Backend&, const std::vector<Ciphertext>&, int) {
      std::vector<Ciphertext> r;
      for (size_t i = 0; i < sim_probs.size(); ++i)  // cleartext values, uploaded with fixed seeds
        r.push_back(pb->upload(sim_probs[i], 900 + i));
      return r;
    });
  };
  Upload sim_up = [](const Ciphertext& x, uint64_t) { return x; };
  Upload gpu_up = [&](const Ciphertext& x, uint64_t s) { return gpu.upload(x, s); };
  Upload twin_up = [&](const Ciphertext& x, uint64_t s) { return twin.upload(x, s); };

  std::vector<Ciphertext> so = program(sim, c, sim_up, sim_fn);
  std::vector<Ciphertext> go = program(gpu, c, gpu_up, enc_fn(gpu));
  std::vector<Ciphertext> to = program(twin, c, twin_up, enc_fn(twin));

  double max_err = 0.0, max_ref = 0.0;
  bool words_equal = go.size() == to.size(), levels_equal = go.size() == so.size(), layouts_equal = true;
  long long words_compared = 0;
  for (size_t i = 0; i < so.size() && i < go.size(); ++i) {
    const SlotVector got = gpu.decrypt(go[i]);
    max_err = std::max(max_err, (got - so[i].slots).abs().maxCoeff());
    max_ref = std::max(max_ref, so[i].slots.abs().maxCoeff());
    levels_equal = levels_equal && go[i].level == so[i].level && to[i].level == so[i].level;
    layouts_equal = layouts_equal && same_layout(go[i].layout, so[i].layout) && same_layout(to[i].layout, so[i].layout);
    const auto wg = gpu.words(go[i]), wt = twin.words(to[i]);
    words_equal = words_equal && wg == wt;
    words_compared += (long long)wg.size();
  }
  const OpCounts s = sim.ledger().totals(), g = gpu.ledger().totals(), tw = twin.ledger().totals();
  sf_op_counts lib{};
  sf_check(sf_ledger_totals(gpu.context(), &lib));
  const bool lib_equal = lib.rotations == s.rotations && lib.hoisted_rotations == s.hoisted_rotations &&
                         lib.ct_pt_mults == s.ct_pt_mults && lib.ct_ct_mults == s.ct_ct_mults &&
                         lib.additions == s.additions && lib.bootstraps == s.bootstraps;
  std::printf(
      "{\"case\": \"%s\", \"N\": %d, \"ring\": %d, \"outputs\": %zu, \"max_err\": %.3e, \"max_abs_ref\": %.3e, "
      "\"words_equal\": %s, \"words_compared\": %lld, \"levels_equal\": %s, \"layouts_equal\": %s, "
      "\"ledger_equal\": %s, \"lib_ledger_equal\": %s, \"twin_ledger_equal\": %s, "
      "\"ledger\": {\"rotations\": %lld, \"hoisted_rotations\": %lld, \"ct_pt_mults\": %lld, \"ct_ct_mults\": %lld, "
      "\"additions\": %lld}, \"live_handles\": %zu}\n",
      c.name.c_str(), c.N, 1 << c.log_n, so.size(), max_err, max_ref, words_equal ? "true" : "false",
      words_compared, levels_equal ? "true" : "false", layouts_equal ? "true" : "false",
      g == s ? "true" : "false", lib_equal ? "true" : "false", tw == s ? "true" : "false", s.rotations,
      s.hoisted_rotations, s.ct_pt_mults, s.ct_ct_mults, s.additions, gpu.live_handles());
  std::fflush(stdout);
}

// The reference's error contract through the binding: the same exception types
// the reference's tests expect (test_engine.cpp / test_kv.cpp).
void run_errors() {
  B200Options opt;
  opt.alpha = 2;
  B200Backend be({2048, 3}, opt);
  int ok = 0, total = 0;
  auto expect = [&](const char* what, auto&& f, auto tag) {
    ++total;
    try {
      f();
    } catch (const decltype(tag)&) {
      ++ok;
      return;
    } catch (const std::exception& e) {
      std::fprintf(stderr, "%s: wrong exception: %s\n", what, e.what());
      return;
    }
    std::fprintf(stderr, "%s: no exception\n", what);
  };
  Ciphertext z0 = be.upload(be.encrypt(SlotVector::Constant(2048, 0.5), 0), 1);
  expect("mul at level 0", [&] { be.mul(z0, z0); }, LevelUnderflow(""));
  expect("mul_plain at level 0", [&] { be.mul_plain(z0, 2.0); }, LevelUnderflow(""));
  expect("bootstrap target 0", [&] { be.bootstrap(z0, 0); }, InvalidTarget(""));
  expect("level_drop up", [&] { be.level_drop(z0, 2); }, InvalidTarget(""));
  Ciphertext x = be.upload(be.encrypt(SlotVector::Constant(2048, 0.5), 3), 2);
  expect("wrong slot count", [&] { be.mul_plain(x, SlotVector::Zero(1024)); }, ShapeMismatch(""));
  AttentionConfig cfg{2048, 128, 4, 0, 1};
  KVCache empty;
  expect("qk_dot on an empty cache", [&] { qk_dot(be, x, empty, cfg); }, CacheEmpty(""));
  expect("rope_apply without a layout", [&] { rope_apply(be, x, cfg, 0); }, LayoutMismatch(""));
  const Layout ly = make_interleaved(128, 2048, 0, 4);
  Ciphertext k = be.upload(be.encrypt(SlotVector::Zero(2048), 2, ly), 3);
  KVCache full = k_append(be, empty, k, cfg);
  expect("k_append past n_max", [&] { k_append(be, full, k, cfg); }, CacheFull(""));
  std::printf("{\"case\": \"errors\", \"expected\": %d, \"raised\": %d, \"ok\": %s}\n", total, ok,
              ok == total ? "true" : "false");
}

}  // namespace

int main(int argc, char** argv) {
  std::vector<Case> cases = {
      {"vmm_small", 2048, 4, 12, 64, 128, 0, false, true},
      {"vmm_bsgs_deferred", 2048, 4, 12, 256, 256, 3, true, false},
      {"decode_small", 2048, 7, 12, 0, 0, 0, false, false, 128, 4, 20},
      {"vmm_ring16", 32768, 4, 16, 1024, 1024, 0, true, true},
      {"decode_ring16", 32768, 7, 16, 0, 0, 0, false, false, 256, 4, 3},
  };
  std::vector<std::string> want(argv + 1, argv + argc);
  try {
    for (const auto& c : cases) {
      bool run = want.empty();
      for (const auto& w : want) run = run || w == c.name;
      if (run) run_case(c);
    }
    bool run_err = want.empty();
    for (const auto& w : want) run_err = run_err || w == "errors";
    if (run_err) run_errors();
  } catch (const std::exception& e) {
    std::printf("{\"error\": \"%s\"}\n", e.what());
    return 1;
  }
  return 0;
}
