// Device modular arithmetic over 64-bit words, primes q < 2^61 (so 4q < 2^63
// and 64 lazily accumulated products of two residues fit in 128 bits).
//
//  * mul_shoup:   x * w mod q for a constant w with precomputed
//                 w' = floor(w 2^64 / q) (Shoup): 1 mul.hi + 2 mul.lo.
//  * reduce128:   (hi:lo) mod q for any 128-bit value via Barrett with
//                 mu = floor(2^128 / q) stored as (mu_hi, mu_lo); the quotient
//                 estimate is the exact floor(x mu / 2^128) so the remainder is
//                 < 3q and two conditional subtractions finish it.
//  * mac128:      lazy 128-bit multiply-accumulate (no reduction).
// All results leaving a kernel are canonical ([0, q)), which is what makes
// ciphertexts bit-identical to the CPU oracle regardless of evaluation order.
#pragma once
#include <cstdint>

namespace sf {

struct U128 {
  uint64_t lo, hi;
};

// The product is written as one 128-bit multiply: ptxas then emits the four
// 32x32 partial products (IMAD.WIDE.U32 with carry chaining) once, where the
// separate `a * b` and `__umul64hi(a, b)` recompute the low partials (5
// IMAD.WIDE + 2 IMAD per term instead of 4 IMAD.WIDE).
__device__ __forceinline__ void mac128(U128& acc, uint64_t a, uint64_t b) {
  const unsigned __int128 s = (((unsigned __int128)acc.hi << 64) | acc.lo) + (unsigned __int128)a * b;
  acc.lo = (uint64_t)s;
  acc.hi = (uint64_t)(s >> 64);
}

__device__ __forceinline__ uint64_t reduce128(uint64_t hi, uint64_t lo, uint64_t q, uint64_t mh, uint64_t ml) {
  const uint64_t t = __umul64hi(lo, ml);
  const uint64_t a_lo = lo * mh, a_hi = __umul64hi(lo, mh);
  const uint64_t b_lo = hi * ml, b_hi = __umul64hi(hi, ml);
  uint64_t s = t + a_lo;
  uint64_t c = s < a_lo;
  s += b_lo;
  c += s < b_lo;
  const uint64_t qhat = hi * mh + a_hi + b_hi + c;
  uint64_t r = lo - qhat * q;
  r = r >= q ? r - q : r;
  r = r >= q ? r - q : r;
  return r;
}

// 64-bit value mod q (hi = 0 specialisation of reduce128)
__device__ __forceinline__ uint64_t reduce64(uint64_t x, uint64_t q, uint64_t mh) {
  const uint64_t qhat = __umul64hi(x, mh);
  uint64_t r = x - qhat * q;
  r = r >= q ? r - q : r;
  r = r >= q ? r - q : r;
  return r;
}

// Montgomery reduction, R = 2^64: (hi:lo) R^-1 mod q for hi < q (any lo), with
// qn = -q^-1 mod 2^64. m = lo qn makes lo + m q = 0 mod 2^64 (a carry of 1
// unless lo = 0), so (T + m q) / 2^64 = hi + mulhi(m, q) + (lo != 0) < 2q.
// One 64-bit low product and one high product (reduce128: three high products).
__device__ __forceinline__ uint64_t redc128(uint64_t hi, uint64_t lo, uint64_t q, uint64_t qn) {
  const uint64_t m = lo * qn;
  const uint64_t r = hi + __umul64hi(m, q) + (lo != 0 ? 1u : 0u);
  return r >= q ? r - q : r;
}

// Montgomery-domain finish of a 128-bit sum T = sum x_i (k_i R) (R-scaled
// multipliers): T R^-1 mod q = sum x_i k_i mod q. The high word is first
// brought below q (T changes by a multiple of q 2^64), which bounds T < q 2^64.
__device__ __forceinline__ uint64_t mont_finish(const U128& t, uint64_t q, uint64_t mh, uint64_t qn) {
  return redc128(reduce64(t.hi, q, mh), t.lo, q, qn);
}

__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, uint64_t q, uint64_t mh, uint64_t ml) {
  return reduce128(__umul64hi(a, b), a * b, q, mh, ml);
}

__device__ __forceinline__ uint64_t mul_shoup(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  const uint64_t qh = __umul64hi(x, wp);
  const uint64_t r = x * w - qh * q;
  return r >= q ? r - q : r;
}

// Shoup product without the final correction: result in [0, 2q) for any x < 2^64
__device__ __forceinline__ uint64_t mul_shoup_lazy(uint64_t x, uint64_t w, uint64_t wp, uint64_t q) {
  return x * w - __umul64hi(x, wp) * q;
}

// L1 prefetch of one 128-byte line (no register result: the load latency of the
// next work item overlaps this one's arithmetic)
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ uint64_t add_mod(uint64_t a, uint64_t b, uint64_t q) {
  const uint64_t s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ uint64_t sub_mod(uint64_t a, uint64_t b, uint64_t q) {
  return a >= b ? a - b : a + q - b;
}

}  // namespace sf
