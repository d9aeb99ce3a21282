// Internal host-side declarations shared by the product's translation units.
// Product code: nothing here (or anywhere under csrc/) touches oracle/.
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace sf {

// Host-side cost accounting (SF_HOST_PROF=1; sf_host_profile): wall time per
// named scope, for finding what the host spends issuing a decode step.
bool host_prof_on();
void host_prof_add(const char* name, double us);
struct HostProfScope {
  const char* name;
  std::chrono::steady_clock::time_point t0;
  bool on;
  explicit HostProfScope(const char* n) : name(n), on(host_prof_on()) {
    if (on) t0 = std::chrono::steady_clock::now();
  }
  ~HostProfScope() {
    if (on) host_prof_add(name, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
  }
};
#define SF_HPROF_CAT2(a, b) a##b
#define SF_HPROF_CAT(a, b) SF_HPROF_CAT2(a, b)
#define SF_HPROF(name) ::sf::HostProfScope SF_HPROF_CAT(_hprof_, __LINE__)(name)

using u64 = uint64_t;
using i64 = int64_t;
using u128 = unsigned __int128;

// Status codes of include/sf_b200.h; thrown internally, mapped at the C ABI.
enum Code : int {
  kOk = 0,
  kLevelUnderflow = 1,
  kInvalidTarget = 2,
  kShapeMismatch = 3,
  kLayoutMismatch = 4,
  kCacheFull = 5,
  kCacheEmpty = 6,
  kDomain = 7,
  kScaleMismatch = 8,
  kCuda = 9,
  kInternal = 10,
};

struct Error : std::runtime_error {
  Code code;
  Error(Code c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(Code c, const std::string& m) { throw Error(c, m); }
inline void require(bool ok, Code c, const std::string& m) {
  if (!ok) fail(c, m);
}

constexpr bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }
inline int log2_exact(long long v) {
  require(is_pow2(v), kShapeMismatch, "log2_exact: " + std::to_string(v) + " is not a power of two");
  int k = 0;
  while (v > 1) v >>= 1, ++k;
  return k;
}
inline long long next_pow2(long long v) {
  long long p = 1;
  while (p < v) p <<= 1;
  return p;
}
constexpr long long pos_mod(long long a, long long m) { return ((a % m) + m) % m; }

// layouts.hpp:22-33
enum class LayoutKind : int { Contiguous = 0, Replicated = 1, Interleaved = 2 };
struct Layout {
  LayoutKind kind = LayoutKind::Interleaved;
  int d = 0, t = 0, offset = 0, heads = 1;
  bool deferred_mask = false;
  bool operator==(const Layout& o) const {
    return kind == o.kind && d == o.d && t == o.t && offset == o.offset && heads == o.heads &&
           deferred_mask == o.deferred_mask;
  }
};
using OptLayout = std::optional<Layout>;
void validate_layout(const Layout& ly, int N);
Layout make_interleaved(int d, int N, int offset = 0, int heads = 1);
int padded_dim(int d);

// host modular helpers (precomputation only)
inline u64 mulmod_h(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
inline u64 powmod_h(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod_h(r, b, m);
    b = mulmod_h(b, b, m);
    e >>= 1;
  }
  return r;
}
inline u64 invmod_h(u64 a, u64 m) { return powmod_h(a % m, m - 2, m); }
inline u64 shoup_h(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
inline u64 bitrev_h(u64 x, int bits) {
  u64 r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

// counter PRNG, shared by host and device code paths
#if defined(__CUDACC__)
#define SF_HD __host__ __device__ __forceinline__
#else
#define SF_HD inline
#endif
SF_HD u64 fmix64(u64 z) {
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}
// Key material and encryption randomness: a ChaCha20 counter stream
// (DESIGN.md §3.4). Word i of stream (seed, stream) is 64-bit word i mod 8 of
// the ChaCha20 block (20 rounds, 64-bit block counter, 64-bit nonce) with
//   key     = seed (2 words, little-endian) || "sf_b200 ckks rng" domain words || 1 || 0
//   counter = i / 8,  nonce = stream id.
struct RngKey {
  u64 seed, stream;
};
SF_HD RngKey stream_key(u64 seed, u64 stream) { return RngKey{seed, stream}; }
SF_HD uint32_t rotl32(uint32_t v, int c) { return (v << c) | (v >> (32 - c)); }
SF_HD void chacha_qr(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
  a += b, d ^= a, d = rotl32(d, 16);
  c += d, b ^= c, b = rotl32(b, 12);
  a += b, d ^= a, d = rotl32(d, 8);
  c += d, b ^= c, b = rotl32(b, 7);
}
// the 16 output words of the block (state after 20 rounds + input state)
SF_HD void chacha20_block(const uint32_t key[8], u64 counter, u64 nonce, uint32_t out[16]) {
  uint32_t in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key[0], key[1], key[2], key[3],
                     key[4], key[5], key[6], key[7], (uint32_t)counter, (uint32_t)(counter >> 32),
                     (uint32_t)nonce, (uint32_t)(nonce >> 32)};
  uint32_t x[16];
  for (int i = 0; i < 16; ++i) x[i] = in[i];
  for (int r = 0; r < 10; ++r) {
    chacha_qr(x[0], x[4], x[8], x[12]);
    chacha_qr(x[1], x[5], x[9], x[13]);
    chacha_qr(x[2], x[6], x[10], x[14]);
    chacha_qr(x[3], x[7], x[11], x[15]);
    chacha_qr(x[0], x[5], x[10], x[15]);
    chacha_qr(x[1], x[6], x[11], x[12]);
    chacha_qr(x[2], x[7], x[8], x[13]);
    chacha_qr(x[3], x[4], x[9], x[14]);
  }
  for (int i = 0; i < 16; ++i) out[i] = x[i] + in[i];
}
SF_HD u64 rand_at(RngKey k, u64 ctr) {
  const uint32_t key[8] = {(uint32_t)k.seed, (uint32_t)(k.seed >> 32), 0x625f6673u, 0x20303032u,
                           0x736b6b63u, 0x676e7220u, 1u, 0u};
  uint32_t o[16];
  chacha20_block(key, ctr >> 3, k.stream, o);
  const int w = (int)(ctr & 7);
  return (u64)o[2 * w] | ((u64)o[2 * w + 1] << 32);
}
constexpr u64 kStreamSk = 1ull << 56, kStreamKeyA = 2ull << 56, kStreamKeyE = 3ull << 56,
              kStreamEncA = 4ull << 56, kStreamEncE = 5ull << 56;

}  // namespace sf
