// B200Backend: slotforge::Backend over the B200 C ABI. See b200_backend.hpp.
// Level rules, layout propagation, error types and ledger charges follow
// SimBackend (/root/reference/proj/src/engine.cpp:126-214) operator by
// operator; the arithmetic is the GPU's RNS-CKKS.
#include "b200_backend.hpp"

#include <atomic>
#include <cstring>
#include <string>

namespace slotforge {

namespace {

constexpr uint64_t kIdTag = 0x7FFAB20000000000ull;    // quiet NaN, payload = handle id
constexpr uint64_t kInstTag = 0x7FFAB20100000000ull;  // quiet NaN, payload = backend instance

std::atomic<uint64_t> g_instances{1};

uint64_t bits_of(double d) {
  uint64_t b;
  std::memcpy(&b, &d, 8);
  return b;
}
double double_of(uint64_t b) {
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

// engine.cpp:130-137: binary results keep a layout only when both operands agree
std::optional<Layout> merge_layouts(const Ciphertext& a, const Ciphertext& b) {
  if (a.layout && b.layout && *a.layout == *b.layout) return a.layout;
  return std::nullopt;
}

}  // namespace

void sf_check(sf_status s) {
  if (s == SF_OK) return;
  const std::string m = sf_last_error();
  switch (s) {
    case SF_ERR_LEVEL_UNDERFLOW: throw LevelUnderflow(m);
    case SF_ERR_INVALID_TARGET: throw InvalidTarget(m);
    case SF_ERR_SHAPE_MISMATCH: throw ShapeMismatch(m);
    case SF_ERR_LAYOUT_MISMATCH: throw LayoutMismatch(m);
    case SF_ERR_CACHE_FULL: throw CacheFull(m);
    case SF_ERR_CACHE_EMPTY: throw CacheEmpty(m);
    case SF_ERR_DOMAIN: throw DomainViolation(m);
    default: throw Error(m);
  }
}

B200Backend::B200Backend(EngineParams params, B200Options o) : Backend(params) {
  sf_params p{};
  p.slots = params.N;
  p.L = params.L;
  p.log_n = o.log_n;
  p.alpha = o.alpha;
  p.q0_bits = o.q0_bits;
  p.scale_bits = o.scale_bits;
  p.special_bits = o.special_bits;
  p.device = o.device;
  p.seed = o.seed;
  sf_check(sf_context_create(&p, &ctx_));
  instance_ = g_instances.fetch_add(1) & 0xFFFFFFFFull;
}

B200Backend::~B200Backend() {
  clear();
  sf_context_destroy(ctx_);
}

bool B200Backend::is_device(const Ciphertext& c) const {
  if (c.slots.size() < 2) return false;
  return (bits_of(c.slots(0)) >> 32) == (kIdTag >> 32);
}

sf_ct* B200Backend::resolve(const Ciphertext& c, bool* owned) {
  *owned = false;
  if (is_device(c)) {
    if (bits_of(c.slots(1)) != (kInstTag | instance_))
      throw Error("B200Backend: ciphertext belongs to another backend instance");
    const uint32_t id = (uint32_t)(bits_of(c.slots(0)) & 0xFFFFFFFFull);
    std::lock_guard<std::mutex> lk(mu_);
    auto it = handles_.find(id);
    if (it == handles_.end()) throw InvalidTarget("B200Backend: ciphertext was released");
    return it->second;
  }
  // a client value from the non-virtual Backend::encrypt / zeros
  check_ct(c, "encrypt");
  sf_ct* h = nullptr;
  bool all_zero = true;
  for (Eigen::Index i = 0; i < c.slots.size() && all_zero; ++i) all_zero = c.slots(i) == 0.0;
  if (all_zero) {
    sf_check(sf_zeros(ctx_, c.level, &h));  // zeros(): the trivial zero ciphertext
  } else {
    sf_check(sf_encrypt(ctx_, c.slots.data(), c.level, nullptr, 0, 0, &h));
  }
  *owned = true;
  return h;
}

Ciphertext B200Backend::wrap(sf_ct* h, std::optional<Layout> layout) {
  int level = 0, zero = 0;
  double scale = 0;
  sf_layout ly{};
  const sf_status s = sf_ct_info(h, &level, &scale, &zero, &ly);
  if (s != SF_OK) {
    sf_ct_release(h);
    sf_check(s);
  }
  uint32_t id;
  {
    std::lock_guard<std::mutex> lk(mu_);
    id = next_id_++;
    handles_.emplace(id, h);
  }
  Ciphertext c;
  c.slots = SlotVector::Zero(N());
  c.slots(0) = double_of(kIdTag | id);
  c.slots(1) = double_of(kInstTag | instance_);
  c.level = level;
  c.layout = std::move(layout);
  return c;
}

template <class F>
Ciphertext B200Backend::binary(F f, const Ciphertext& a, const Ciphertext& b, std::optional<Layout> ly) {
  bool oa, ob;
  sf_ct* ha = resolve(a, &oa);
  sf_ct* hb = nullptr;
  try {
    hb = resolve(b, &ob);
  } catch (...) {
    if (oa) sf_ct_release(ha);
    throw;
  }
  sf_ct* out = nullptr;
  const sf_status s = f(ctx_, ha, hb, &out);
  if (oa) sf_ct_release(ha);
  if (ob) sf_ct_release(hb);
  sf_check(s);
  return wrap(out, std::move(ly));
}

// --- virtual operators (SimBackend semantics, engine.cpp:143-214) -----------
Ciphertext B200Backend::add(const Ciphertext& a, const Ciphertext& b) {
  check_ct(a, "add");
  check_ct(b, "add");
  ledger_.count_addition();
  return binary(sf_add, a, b, merge_layouts(a, b));
}

Ciphertext B200Backend::sub(const Ciphertext& a, const Ciphertext& b) {
  check_ct(a, "sub");
  check_ct(b, "sub");
  ledger_.count_addition();
  return binary(sf_sub, a, b, merge_layouts(a, b));
}

Ciphertext B200Backend::add_plain(const Ciphertext& a, const SlotVector& p) {
  check_ct(a, "add_plain");
  check_slots(p, "add_plain");
  ledger_.count_addition();
  bool owned;
  sf_ct* h = resolve(a, &owned);
  sf_ct* out = nullptr;
  const sf_status s = sf_add_plain(ctx_, h, p.data(), &out);
  if (owned) sf_ct_release(h);
  sf_check(s);
  return wrap(out, a.layout);
}

Ciphertext B200Backend::mul(const Ciphertext& a, const Ciphertext& b) {
  check_ct(a, "mul");
  check_ct(b, "mul");
  if (std::min(a.level, b.level) <= 0) throw LevelUnderflow("mul: no multiplicative level left");
  ledger_.count_ct_ct_mult();
  return binary(sf_mul, a, b, merge_layouts(a, b));
}

Ciphertext B200Backend::mul_plain(const Ciphertext& a, const SlotVector& p) {
  check_ct(a, "mul_plain");
  check_slots(p, "mul_plain");
  if (a.level <= 0) throw LevelUnderflow("mul_plain: no multiplicative level left");
  ledger_.count_ct_pt_mult();
  bool owned;
  sf_ct* h = resolve(a, &owned);
  sf_ct* out = nullptr;
  const sf_status s = sf_mul_plain(ctx_, h, p.data(), &out);
  if (owned) sf_ct_release(h);
  sf_check(s);
  return wrap(out, a.layout);
}

Ciphertext B200Backend::rotate(const Ciphertext& a, int r, RotationHint hint) {
  check_ct(a, "rotate");
  if (pos_mod(r, N()) == 0) return a;  // a no-op and free (engine.cpp:184-185)
  ledger_.count_rotation(hint.hoisted);
  bool owned;
  sf_ct* h = resolve(a, &owned);
  sf_ct* out = nullptr;
  const sf_status s = sf_rotate(ctx_, h, r, hint.hoisted ? 1 : 0, &out);
  if (owned) sf_ct_release(h);
  sf_check(s);
  return wrap(out, std::nullopt);
}

Ciphertext B200Backend::bootstrap(const Ciphertext& a, int target_level) {
  check_ct(a, "bootstrap");
  if (target_level < 1 || target_level > L())
    throw InvalidTarget("bootstrap: target level " + std::to_string(target_level) + " outside [1, L]");
  ledger_.count_bootstrap();
  bool owned;
  sf_ct* h = resolve(a, &owned);
  sf_ct* out = nullptr;
  const sf_status s = sf_bootstrap(ctx_, h, target_level, &out);  // oracle hook: client round trip
  if (owned) sf_ct_release(h);
  sf_check(s);
  return wrap(out, a.layout);
}

Ciphertext B200Backend::level_drop(const Ciphertext& a, int target_level) {
  check_ct(a, "level_drop");
  if (target_level < 0 || target_level > a.level)
    throw InvalidTarget("level_drop: target level " + std::to_string(target_level) + " outside [0, level]");
  bool owned;
  sf_ct* h = resolve(a, &owned);
  sf_ct* out = nullptr;
  const sf_status s = sf_level_drop(ctx_, h, target_level, &out);
  if (owned) sf_ct_release(h);
  sf_check(s);
  return wrap(out, a.layout);
}

Ciphertext B200Backend::exact_transform(const Ciphertext& a,
                                        const std::function<SlotVector(const SlotVector&)>& f) {
  check_ct(a, "exact_transform");
  SlotVector out = f(decrypt(a));  // out-of-model oracle: client round trip, free
  check_slots(out, "exact_transform result");
  sf_ct* h = nullptr;
  sf_check(sf_encrypt(ctx_, out.data(), a.level, nullptr, 0, 0, &h));
  return wrap(h, a.layout);
}

// --- client side -------------------------------------------------------------
Ciphertext B200Backend::upload(const Ciphertext& c, std::optional<uint64_t> seed) {
  if (is_device(c)) return c;
  check_ct(c, "encrypt");
  sf_ct* h = nullptr;
  if (seed) {
    sf_check(sf_encrypt(ctx_, c.slots.data(), c.level, nullptr, *seed, 1, &h));
  } else {
    bool owned;
    h = resolve(c, &owned);
  }
  return wrap(h, c.layout);
}

SlotVector B200Backend::decrypt(const Ciphertext& c) {
  if (!is_device(c)) return c.slots;
  bool owned;
  sf_ct* h = resolve(c, &owned);
  SlotVector out(N());
  sf_check(sf_decrypt(ctx_, h, out.data()));
  return out;
}

std::vector<uint64_t> B200Backend::words(const Ciphertext& c) {
  bool owned;
  sf_ct* h = resolve(c, &owned);
  int level = 0, zero = 0, n = 0;
  double scale = 0;
  sf_layout ly{};
  sf_check(sf_ct_info(h, &level, &scale, &zero, &ly));
  sf_check(sf_context_info(ctx_, &n, nullptr, nullptr, nullptr, nullptr, nullptr));
  std::vector<uint64_t> w((size_t)2 * (level + 1) * n, 0);
  if (!zero) sf_check(sf_ct_export(ctx_, h, w.data()));
  if (owned) sf_ct_release(h);
  return w;
}

void B200Backend::release(const Ciphertext& c) {
  if (!is_device(c)) return;
  const uint32_t id = (uint32_t)(bits_of(c.slots(0)) & 0xFFFFFFFFull);
  std::lock_guard<std::mutex> lk(mu_);
  auto it = handles_.find(id);
  if (it == handles_.end()) return;
  sf_ct_release(it->second);
  handles_.erase(it);
}

void B200Backend::clear() {
  std::lock_guard<std::mutex> lk(mu_);
  for (auto& [id, h] : handles_) sf_ct_release(h);
  handles_.clear();
}

size_t B200Backend::live_handles() const {
  std::lock_guard<std::mutex> lk(mu_);
  return handles_.size();
}

}  // namespace slotforge
