// B200Backend — the reference-side binding of the B200 C ABI (include/sf_b200.h).
//
// A `slotforge::Backend` (/root/reference/proj/include/slotforge/engine.hpp:112-149)
// whose virtual operators run on the GPU through the C ABI, written against the
// UNMODIFIED reference headers: the reference's own protocol code
// (vmm_interleaved, rope_apply, k_append, make_v_pieces, v_append, qk_dot,
// softmax_times_v, ... in vmm.cpp / kv_attention.cpp) runs on it op by op.
//
// How a device ciphertext rides in the reference's value type. The reference's
// `Ciphertext` is {SlotVector slots, int level, optional<Layout> layout}
// (engine.hpp:24-28) with no room for a handle, and its `encrypt` / `zeros`
// (engine.cpp:109-123) and `ledger()` (engine.hpp:120) are non-virtual. So:
//   * a ciphertext produced by this backend keeps its N-slot vector, with slot 0
//     holding a quiet-NaN tag (0x7FFAB200'xxxxxxxx, x = handle id) and slot 1 the
//     backend's instance tag; the id indexes a side registry of sf_ct handles.
//     level and layout are the reference's fields and stay authoritative;
//   * a ciphertext WITHOUT a tag is a client value from the non-virtual
//     Backend::encrypt / zeros: on first use it is encrypted on the GPU at its
//     level (all-zero slots become the trivial zero ciphertext, exactly what
//     `zeros()` means to the reference's v_append, kv_attention.cpp:176);
//     upload() does that explicitly, with an optional fixed seed;
//   * every operator charges the inherited `ledger_` exactly as SimBackend does
//     (engine.cpp:143-206), so callers reading `be.ledger()` see the reference's
//     counts; the library's own ledger (sf_ledger_totals) counts the same ops.
// Handles live until release() / clear() / destruction (the reference copies
// Ciphertext values freely and has no destructor hook to refcount through).
//
// Client-side helpers of the reference that read `.slots` directly
// (exact_softmax_maps, kv_attention.cpp:403; harness checks) need decrypt()
// first: on this backend the slots of a device ciphertext are only a tag.
#pragma once

#include <cstdint>
#include <mutex>
#include <optional>
#include <unordered_map>
#include <vector>

#include "sf_b200.h"
#include "slotforge/engine.hpp"

namespace slotforge {

// CKKS parameters the reference leaves unhoused; see sf_params.
struct B200Options {
  int log_n = 0;  // 0: ring degree 2N
  int alpha = 2;  // special primes per key-switching digit
  int q0_bits = 0, scale_bits = 0, special_bits = 0;  // 0: 60 / 40 / 60
  int device = 0;
  uint64_t seed = 1;  // secret / evaluation key seed
};

// Rethrows an sf_status as the reference's exception type (types.hpp:16-46).
void sf_check(sf_status s);

class B200Backend final : public Backend {
 public:
  explicit B200Backend(EngineParams params, B200Options opts = {});
  ~B200Backend() override;
  B200Backend(const B200Backend&) = delete;
  B200Backend& operator=(const B200Backend&) = delete;

  Ciphertext add(const Ciphertext& a, const Ciphertext& b) override;
  Ciphertext sub(const Ciphertext& a, const Ciphertext& b) override;
  Ciphertext add_plain(const Ciphertext& a, const SlotVector& p) override;
  Ciphertext mul(const Ciphertext& a, const Ciphertext& b) override;
  Ciphertext mul_plain(const Ciphertext& a, const SlotVector& p) override;
  Ciphertext rotate(const Ciphertext& a, int r, RotationHint hint = {}) override;
  Ciphertext bootstrap(const Ciphertext& a, int target_level) override;
  Ciphertext level_drop(const Ciphertext& a, int target_level) override;
  Ciphertext exact_transform(const Ciphertext& a,
                             const std::function<SlotVector(const SlotVector&)>& f) override;
  using Backend::add_plain;
  using Backend::mul_plain;

  // --- client side (off-ledger)
  // Encrypts a client value (from Backend::encrypt / zeros) on the GPU now and
  // returns the device ciphertext; seed = nullopt uses the context's counter
  // (DESIGN.md §3.4). A device ciphertext is returned unchanged.
  Ciphertext upload(const Ciphertext& c, std::optional<uint64_t> seed = std::nullopt);
  SlotVector decrypt(const Ciphertext& c);           // device or client value
  std::vector<uint64_t> words(const Ciphertext& c);  // [2][level+1][n] RNS words (NTT domain)
  bool is_device(const Ciphertext& c) const;

  // --- handle management
  void release(const Ciphertext& c);  // drop one ciphertext's device words
  void clear();                       // drop every handle this backend made
  size_t live_handles() const;
  sf_context* context() { return ctx_; }
  const sf_context* context() const { return ctx_; }

 private:
  // resolves a ciphertext to a handle (uploading client values); the bool says
  // whether the caller owns the returned reference (a fresh upload)
  sf_ct* resolve(const Ciphertext& c, bool* owned);
  Ciphertext wrap(sf_ct* h, std::optional<Layout> layout);  // adopts h
  template <class F>
  Ciphertext binary(F f, const Ciphertext& a, const Ciphertext& b, std::optional<Layout> ly);

  sf_context* ctx_ = nullptr;
  uint64_t instance_ = 0;
  mutable std::mutex mu_;
  std::unordered_map<uint32_t, sf_ct*> handles_;
  uint32_t next_id_ = 1;
};

}  // namespace slotforge
