// Warp-level negacyclic sub-NTT building blocks (used by ntt.cu and fused.cu).
//
// A sub-transform of m = 32 * E points is owned by ONE warp: every lane holds E
// residues in registers, all butterflies of a group of log2(E) stages are
// register-local, and the warp re-distributes residues between groups through
// a private swizzled shared-memory region (__syncwarp only). Butterflies are
// Harvey-lazy: forward operands live in [0, 4q), inverse operands in [0, 2q);
// callers normalise at the end of a full transform.
#pragma once
#include "context.h"
#include "modarith.cuh"

namespace sf {
namespace wntt {

// 64-bit-bank swizzle inside a warp region (16 x 8-byte banks per half warp):
// i ^ T(bits 4..7 of i), T the GF(2) matrix with columns (2, 13, 4, 3). It is
// linear, so swz(lane part | register part) = swz(lane part) ^ swz(register
// part), and it makes every half warp hit 16 distinct banks in each relayout
// the warp NTTs issue (register bits at s0 = 0/2/5 for 8 registers per lane,
// 0/1/3/5 for 4, 0/1/5 for 16 -- checked exhaustively); the former
// i ^ (i >> 4) left the s0 = 2 relayouts of the 256-point transforms 2-way
// conflicted (profiles/r1_ncu_v16.md: 24 % of fused_col's shared wavefronts).
__device__ __forceinline__ int swz(int i) {
  const int h = i >> 4;
  return i ^ ((h & 1) ? 2 : 0) ^ ((h & 2) ? 13 : 0) ^ ((h & 4) ? 4 : 0) ^ ((h & 8) ? 3 : 0);
}
// the round-1 swizzle (2-way conflicted at s0 = 2, but cheaper to address);
// ks_row_kernel used it while it ran at 128 registers (the conflict-free form
// spilled there); at 80 registers it takes the conflict-free form (smem bank
// conflicts 26.6 % -> 5.6 % of shared wavefronts, same time: profiles/r2_ncu_v3_raw)
__device__ __forceinline__ int swz1(int i) { return i ^ ((i >> 4) & 15); }
template <bool XS>
__device__ __forceinline__ int swzx(int i) { return XS ? swz(i) : swz1(i); }

// index of register k of `lane` when register bits are [s0, s0 + LOGE)
template <int LOGE>
__device__ __forceinline__ int lay(int lane, int k, int s0) {
  return (lane & ((1 << s0) - 1)) | (k << s0) | ((lane >> s0) << (s0 + LOGE));
}

template <int LOGE, bool XS = true>
__device__ __forceinline__ void relayout(u64 (&x)[1 << LOGE], u64* sm, int lane, int from, int to) {
  if (from == to) return;
  const int wb = swzx<XS>(lay<LOGE>(lane, 0, from)), rb = swzx<XS>(lay<LOGE>(lane, 0, to));  // lane parts
#pragma unroll
  for (int k = 0; k < (1 << LOGE); ++k) sm[wb ^ swzx<XS>(k << from)] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < (1 << LOGE); ++k) x[k] = sm[rb ^ swzx<XS>(k << to)];
  __syncwarp();
}

// Register layouts: STRIDED (register bits = the top LOGE index bits, lane =
// the low 5 bits: element lane + 32k) or BLOCKED (register bits = the low LOGE
// bits: lane owns E consecutive elements, 16-byte vector loads/stores).
enum : int { kStrided = 0, kBlocked = 1 };

// Forward sub-NTT (Cooley-Tukey). Entry layout: strided. Exit layout: EXIT.
// tw(b, blk, w, ws) gives the twiddle (and Shoup companion) of the stage with
// butterfly distance 2^b for block blk.
template <int LOGM, int EXIT = kStrided, class TW, bool XS = true>
__device__ __forceinline__ void warp_fwd(u64 (&x)[1 << (LOGM - 5)], u64* sm, int lane, u64 q, const TW& tw) {
  constexpr int LOGE = LOGM - 5;
  constexpr int E = 1 << LOGE;
  const u64 q2 = 2 * q;
  int s0 = LOGM - LOGE;
#pragma unroll
  for (int hi = LOGM; hi > 0; hi -= LOGE) {
    const int lo = hi - LOGE > 0 ? hi - LOGE : 0;
    relayout<LOGE, XS>(x, sm, lane, s0, lo);
    s0 = lo;
#pragma unroll
    for (int b = hi - 1; b >= lo; --b) {
      const int rb = b - s0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << rb)) continue;
        const int idx = lay<LOGE>(lane, k, s0);
        u64 w, ws;
        tw(b, idx >> (b + 1), w, ws);
        u64 U = x[k];
        U = U >= q2 ? U - q2 : U;
        const u64 T = mul_shoup_lazy(x[k | (1 << rb)], w, ws, q);
        x[k] = U + T;
        x[k | (1 << rb)] = U - T + q2;
      }
    }
  }
  relayout<LOGE, XS>(x, sm, lane, s0, EXIT == kBlocked ? 0 : LOGM - LOGE);
}

// Inverse sub-NTT (Gentleman-Sande). Entry layout: ENTRY. Exit layout: strided.
template <int LOGM, int ENTRY = kStrided, class TW, bool XS = true>
__device__ __forceinline__ void warp_inv(u64 (&x)[1 << (LOGM - 5)], u64* sm, int lane, u64 q, const TW& tw) {
  constexpr int LOGE = LOGM - 5;
  constexpr int E = 1 << LOGE;
  const u64 q2 = 2 * q;
  int s0 = ENTRY == kBlocked ? 0 : LOGM - LOGE;
  // the forward transform's register groups in reverse ([0,2), [2,5), [5,8) at
  // 256 points): the relayouts use the register offsets s0 the swizzle is
  // conflict-free for (0/2/5, 0/1/5, 0/1/3/5); the former [0,3), [3,6), [6,8)
  // put s0 = 3 in between (2-way conflicts, profiles/r2_ncu_v2)
  constexpr int NG = (LOGM + LOGE - 1) / LOGE;
#pragma unroll
  for (int gi = NG - 1; gi >= 0; --gi) {
    const int hi = LOGM - gi * LOGE;
    const int lo = hi - LOGE > 0 ? hi - LOGE : 0;
    relayout<LOGE, XS>(x, sm, lane, s0, lo);
    s0 = lo;
#pragma unroll
    for (int b = lo; b < hi; ++b) {
      const int rb = b - s0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << rb)) continue;
        const int idx = lay<LOGE>(lane, k, s0);
        u64 w, ws;
        tw(b, idx >> (b + 1), w, ws);
        const u64 U = x[k], V = x[k | (1 << rb)];
        const u64 S = U + V;
        x[k] = S >= q2 ? S - q2 : S;
        x[k | (1 << rb)] = mul_shoup_lazy(U - V + q2, w, ws, q);
      }
    }
  }
  relayout<LOGE, XS>(x, sm, lane, s0, LOGM - LOGE);
}

// NC independent sub-transforms of the same prime in one warp (e.g. NC adjacent
// columns of a column pass): every butterfly of a stage is issued for all NC
// columns with one twiddle fetch, doubling the warp's independent work (ILP).
template <int LOGE, int NC>
__device__ __forceinline__ void relayout_n(u64 (&x)[NC][1 << LOGE], u64* const (&sm)[NC], int lane, int from, int to) {
  if (from == to) return;
  const int wb = swz(lay<LOGE>(lane, 0, from)), rb = swz(lay<LOGE>(lane, 0, to));  // lane parts
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int k = 0; k < (1 << LOGE); ++k) sm[c][wb ^ swz(k << from)] = x[c][k];
  __syncwarp();
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int k = 0; k < (1 << LOGE); ++k) x[c][k] = sm[c][rb ^ swz(k << to)];
  __syncwarp();
}

template <int LOGM, int NC, class TW>
__device__ __forceinline__ void warp_fwd_n(u64 (&x)[NC][1 << (LOGM - 5)], u64* const (&sm)[NC], int lane, u64 q,
                                           const TW& tw) {
  constexpr int LOGE = LOGM - 5;
  constexpr int E = 1 << LOGE;
  const u64 q2 = 2 * q;
  int s0 = LOGM - LOGE;
#pragma unroll
  for (int hi = LOGM; hi > 0; hi -= LOGE) {
    const int lo = hi - LOGE > 0 ? hi - LOGE : 0;
    relayout_n<LOGE, NC>(x, sm, lane, s0, lo);
    s0 = lo;
#pragma unroll
    for (int b = hi - 1; b >= lo; --b) {
      const int rb = b - s0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << rb)) continue;
        const int idx = lay<LOGE>(lane, k, s0);
        u64 w, ws;
        tw(b, idx >> (b + 1), w, ws);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          u64 U = x[c][k];
          U = U >= q2 ? U - q2 : U;
          const u64 T = mul_shoup_lazy(x[c][k | (1 << rb)], w, ws, q);
          x[c][k] = U + T;
          x[c][k | (1 << rb)] = U - T + q2;
        }
      }
    }
  }
  relayout_n<LOGE, NC>(x, sm, lane, s0, LOGM - LOGE);
}

// FS: the last stage also applies a constant factor f to every output (the
// caller's post-transform scale, e.g. n^-1 times a conversion factor): the
// sum gets f, the difference f * w (fw precomputed); outputs canonical
template <int LOGM, int NC, class TW, bool FS = false>
__device__ __forceinline__ void warp_inv_n(u64 (&x)[NC][1 << (LOGM - 5)], u64* const (&sm)[NC], int lane, u64 q,
                                           const TW& tw, u64 f = 0, u64 fs = 0, u64 fw = 0, u64 fws = 0) {
  constexpr int LOGE = LOGM - 5;
  constexpr int E = 1 << LOGE;
  const u64 q2 = 2 * q;
  int s0 = LOGM - LOGE;
  constexpr int NG = (LOGM + LOGE - 1) / LOGE;  // forward groups reversed (see warp_inv)
#pragma unroll
  for (int gi = NG - 1; gi >= 0; --gi) {
    const int hi = LOGM - gi * LOGE;
    const int lo = hi - LOGE > 0 ? hi - LOGE : 0;
    relayout_n<LOGE, NC>(x, sm, lane, s0, lo);
    s0 = lo;
#pragma unroll
    for (int b = lo; b < hi; ++b) {
      const int rb = b - s0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << rb)) continue;
        const int idx = lay<LOGE>(lane, k, s0);
        u64 w, ws;
        tw(b, idx >> (b + 1), w, ws);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const u64 U = x[c][k], V = x[c][k | (1 << rb)];
          const u64 S = U + V;
          if (FS && b == LOGM - 1) {
            x[c][k] = mul_shoup(S, f, fs, q);
            x[c][k | (1 << rb)] = mul_shoup(U - V + q2, fw, fws, q);
          } else {
            x[c][k] = S >= q2 ? S - q2 : S;
            x[c][k | (1 << rb)] = mul_shoup_lazy(U - V + q2, w, ws, q);
          }
        }
      }
    }
  }
  relayout_n<LOGE, NC>(x, sm, lane, s0, LOGM - LOGE);
}

__device__ __forceinline__ u64 canon4(u64 v, u64 q) {  // [0, 4q) -> [0, q)
  v = v >= 2 * q ? v - 2 * q : v;
  return v >= q ? v - q : v;
}

__device__ __forceinline__ uint32_t brev(uint32_t x, int logn) { return __brev(x) >> (32 - logn); }
__device__ __forceinline__ uint32_t auto_perm(uint32_t i, u64 g, int logn) {
  const u64 e = 2ull * brev(i, logn) + 1;
  const u64 e2 = (e * g) & ((2ull << logn) - 1);
  return brev((uint32_t)((e2 - 1) >> 1), logn);
}

// Row-granular automorphism X -> X^g in the bit-reversed evaluation order with
// n = R x C: position i = rd*C + c maps to perm_g(i), whose row
// and bit-reversed column are
//   row(perm_g(i))        = br_R(B mod R)
//   br_C(col(perm_g(i)))  = (floor(B / R) + g * br_C(c)) mod C
// with B = ((2 br_R(rd) + 1) g - 1) / 2: the source row depends on rd only and
// the in-row position is affine in br_C(c) (odd slope g).
template <int LOGR, int LOGC>
struct RowPerm {
  uint32_t src_row, base, slope;  // position(bc) = (base + slope * bc) mod C
  __device__ __forceinline__ RowPerm(int rd, u64 g) {
    constexpr uint32_t R = 1u << LOGR, C = 1u << LOGC;
    const u64 B = ((2ull * (__brev((uint32_t)rd) >> (32 - LOGR)) + 1) * g - 1) >> 1;
    src_row = __brev((uint32_t)(B & (R - 1))) >> (32 - LOGR);
    base = (uint32_t)(B >> LOGR) & (C - 1);
    slope = (uint32_t)g & (C - 1);
  }
  // bit-reversed source column of the element whose own column has br_C = bc
  __device__ __forceinline__ uint32_t pos(uint32_t bc) const { return (base + slope * bc) & ((1u << LOGC) - 1); }
};

}  // namespace wntt
}  // namespace sf
