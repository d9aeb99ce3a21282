// TwinBackend — TEST INFRASTRUCTURE ONLY: the CPU CKKS twin
// (oracle/ckks_oracle.cpp, `ock_*` C ABI) behind the reference's
// slotforge::Backend, with the same ciphertext-in-slots tagging as the
// product-side B200Backend (integration/b200_backend.hpp). Running the
// reference's own protocol code on both backends, op by op, gives the
// bit-exact expectation for the B200 binding. Level rules, error messages,
// layout merging and ledger charges follow SimBackend (engine.cpp:143-214),
// as oracle/ckks.py does; the seed of an encryption without an explicit one is
// DESIGN.md §3.4's fmix(key_seed ^ (0xE1C0000000000000 + k)).
#pragma once

#include <cstdint>
#include <cstring>
#include <optional>
#include <string>
#include <unordered_map>
#include <vector>

#include "slotforge/engine.hpp"

extern "C" {
const char* ock_last_error();
void* ock_context_new(int logn, int slots, int L, int q0_bits, int scale_bits, int alpha, int special_bits,
                      uint64_t seed);
void ock_context_free(void* c);
void* ock_encrypt(void* c, const double* slots, int limbs, double scale, uint64_t seed);
void* ock_zero(void* c, int limbs);
void ock_ct_free(void* ct);
void ock_ct_info(void* ct, int* limbs, double* scale, int* zero);
void ock_ct_data(void* ct, uint64_t* out);
void ock_decrypt(void* c, void* ct, double* slots);
void* ock_add(void* c, void* a, void* b);
void* ock_sub(void* c, void* a, void* b);
void* ock_add_plain(void* c, void* a, const double* slots);
void* ock_mac_plain(void* c, void** cts, const double* slots, int k);
void* ock_mul(void* c, void* a, void* b);
void* ock_rotate(void* c, void* a, int r);
void* ock_level_drop(void* c, void* a, int limbs);
}

namespace slotforge {

class TwinBackend final : public Backend {
 public:
  TwinBackend(EngineParams p, int log_n, int alpha, uint64_t seed, int q0_bits = 60, int scale_bits = 40,
              int special_bits = 60)
      : Backend(p), seed_(seed), delta_(std::ldexp(1.0, scale_bits)) {
    n_ = 1 << log_n;
    ctx_ = ock_context_new(log_n, p.N, p.L, q0_bits, scale_bits, alpha, special_bits, seed);
    if (!ctx_) throw Error(ock_last_error());
  }
  ~TwinBackend() override {
    for (auto& [id, h] : handles_) ock_ct_free(h);
    ock_context_free(ctx_);
  }

  Ciphertext add(const Ciphertext& a, const Ciphertext& b) override {
    check_ct(a, "add");
    check_ct(b, "add");
    ledger_.count_addition();
    return wrap(must(ock_add(ctx_, get(a), get(b))), std::min(a.level, b.level), merge(a, b));
  }
  Ciphertext sub(const Ciphertext& a, const Ciphertext& b) override {
    check_ct(a, "sub");
    check_ct(b, "sub");
    ledger_.count_addition();
    return wrap(must(ock_sub(ctx_, get(a), get(b))), std::min(a.level, b.level), merge(a, b));
  }
  Ciphertext add_plain(const Ciphertext& a, const SlotVector& p) override {
    check_ct(a, "add_plain");
    check_slots(p, "add_plain");
    ledger_.count_addition();
    return wrap(must(ock_add_plain(ctx_, get(a), p.data())), a.level, a.layout);
  }
  Ciphertext mul(const Ciphertext& a, const Ciphertext& b) override {
    check_ct(a, "mul");
    check_ct(b, "mul");
    const int lvl = std::min(a.level, b.level);
    if (lvl <= 0) throw LevelUnderflow("mul: no multiplicative level left");
    ledger_.count_ct_ct_mult();
    return wrap(must(ock_mul(ctx_, get(a), get(b))), lvl - 1, merge(a, b));
  }
  Ciphertext mul_plain(const Ciphertext& a, const SlotVector& p) override {
    check_ct(a, "mul_plain");
    check_slots(p, "mul_plain");
    if (a.level <= 0) throw LevelUnderflow("mul_plain: no multiplicative level left");
    ledger_.count_ct_pt_mult();
    void* h = get(a);
    return wrap(must(ock_mac_plain(ctx_, &h, p.data(), 1)), a.level - 1, a.layout);
  }
  Ciphertext rotate(const Ciphertext& a, int r, RotationHint hint = {}) override {
    check_ct(a, "rotate");
    if (pos_mod(r, N()) == 0) return a;
    ledger_.count_rotation(hint.hoisted);
    return wrap(must(ock_rotate(ctx_, get(a), r)), a.level, std::nullopt);
  }
  Ciphertext bootstrap(const Ciphertext& a, int target) override {
    check_ct(a, "bootstrap");
    if (target < 1 || target > L())
      throw InvalidTarget("bootstrap: target level " + std::to_string(target) + " outside [1, L]");
    ledger_.count_bootstrap();
    SlotVector s = decrypt(a);
    return wrap(must(ock_encrypt(ctx_, s.data(), target + 1, delta_, next_seed())), target, a.layout);
  }
  Ciphertext level_drop(const Ciphertext& a, int target) override {
    check_ct(a, "level_drop");
    if (target < 0 || target > a.level)
      throw InvalidTarget("level_drop: target level " + std::to_string(target) + " outside [0, level]");
    return wrap(must(ock_level_drop(ctx_, get(a), target + 1)), target, a.layout);
  }
  Ciphertext exact_transform(const Ciphertext& a, const std::function<SlotVector(const SlotVector&)>& f) override {
    check_ct(a, "exact_transform");
    SlotVector out = f(decrypt(a));
    check_slots(out, "exact_transform result");
    return wrap(must(ock_encrypt(ctx_, out.data(), a.level + 1, delta_, next_seed())), a.level, a.layout);
  }
  using Backend::add_plain;
  using Backend::mul_plain;

  Ciphertext upload(const Ciphertext& c, std::optional<uint64_t> seed = std::nullopt) {
    if (tagged(c)) return c;
    check_ct(c, "encrypt");
    bool all_zero = true;
    for (Eigen::Index i = 0; i < c.slots.size() && all_zero; ++i) all_zero = c.slots(i) == 0.0;
    void* h = all_zero && !seed ? ock_zero(ctx_, c.level + 1)
                                              : ock_encrypt(ctx_, c.slots.data(), c.level + 1, delta_,
                                                            seed ? *seed : next_seed());
    return wrap(must(h), c.level, c.layout);
  }
  SlotVector decrypt(const Ciphertext& c) {
    if (!tagged(c)) return c.slots;
    SlotVector out(N());
    ock_decrypt(ctx_, get(c), out.data());
    return out;
  }
  std::vector<uint64_t> words(const Ciphertext& c) {
    void* h = get(c);
    int limbs = 0, zero = 0;
    double scale = 0;
    ock_ct_info(h, &limbs, &scale, &zero);
    std::vector<uint64_t> w((size_t)2 * limbs * n_, 0);
    if (!zero) ock_ct_data(h, w.data());
    return w;
  }

 private:
  static constexpr uint64_t kTag = 0x7FFA7A0000000000ull;
  static uint64_t bits(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
  }
  static bool tagged(const Ciphertext& c) { return c.slots.size() >= 1 && (bits(c.slots(0)) >> 32) == (kTag >> 32); }
  static std::optional<Layout> merge(const Ciphertext& a, const Ciphertext& b) {
    if (a.layout && b.layout && *a.layout == *b.layout) return a.layout;
    return std::nullopt;
  }
  static void* must(void* h) {
    if (!h) throw Error(ock_last_error());
    return h;
  }
  uint64_t next_seed() {
    auto fmix = [](uint64_t z) {
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      return z ^ (z >> 31);
    };
    return fmix(seed_ ^ (0xE1C0000000000000ull + counter_++));
  }
  // a handle for c; untagged client values (Backend::encrypt / zeros) are
  // encrypted now, exactly when the B200 binding would
  void* get(const Ciphertext& c) {
    if (!tagged(c)) {
      Ciphertext u = upload(c);
      return handles_.at((uint32_t)(bits(u.slots(0)) & 0xFFFFFFFFull));
    }
    auto it = handles_.find((uint32_t)(bits(c.slots(0)) & 0xFFFFFFFFull));
    if (it == handles_.end()) throw InvalidTarget("TwinBackend: unknown ciphertext");
    return it->second;
  }
  Ciphertext wrap(void* h, int level, std::optional<Layout> layout) {
    const uint32_t id = next_id_++;
    handles_.emplace(id, h);
    Ciphertext c;
    c.slots = SlotVector::Zero(N());
    uint64_t b = kTag | id;
    std::memcpy(&c.slots(0), &b, 8);
    c.level = level;
    c.layout = std::move(layout);
    return c;
  }

  void* ctx_ = nullptr;
  int n_ = 0;
  uint64_t seed_ = 1, counter_ = 0;
  double delta_ = 0;
  std::unordered_map<uint32_t, void*> handles_;
  uint32_t next_id_ = 1;
};

}  // namespace slotforge
