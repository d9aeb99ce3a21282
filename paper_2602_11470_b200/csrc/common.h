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
SF_HD u64 stream_key(u64 seed, u64 stream) { return fmix64(seed ^ fmix64(stream ^ 0x9E3779B97F4A7C15ull)); }
SF_HD u64 rand_at(u64 key, u64 ctr) { return fmix64(key + (ctr + 1) * 0x9E3779B97F4A7C15ull); }
constexpr u64 kStreamSk = 1ull << 56, kStreamKeyA = 2ull << 56, kStreamKeyE = 3ull << 56,
              kStreamEncA = 4ull << 56, kStreamEncE = 5ull << 56;

}  // namespace sf
