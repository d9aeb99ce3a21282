// Batched negacyclic NTT / inverse NTT over 64-bit RNS limbs, sm_100a.
//
// n = R x C (R = 2^r rows, C = 2^c columns, element (row, col) at row*C+col).
// Forward (Cooley-Tukey, natural -> bit-reversed): the first r stages have
// butterfly distance >= C and act within columns (column pass), the last c
// stages act within rows (row pass). Inverse (Gentleman-Sande) runs the row
// pass first, then the column pass, folding n^-1 into the last stage.
//
// Each sub-NTT of m = 32 * E points is owned by ONE warp: every lane holds E
// residues in registers, all butterflies of a group of log2(E) stages are
// register-local, and the warp re-distributes residues between groups through a
// private swizzled shared-memory region (no __syncthreads inside a transform).
// Global loads/stores are 256-byte coalesced rows (row pass) or 64-byte row
// segments staged through shared memory (column pass). A launch covers any
// number of limbs (the LimbBatch), so one launch of a ModUp / ModDown / rescale
// touches every limb of every ciphertext in the batch.
#include "context.h"
#include "kernels.cuh"
#include "modarith.cuh"

namespace sf {
namespace {

constexpr int kWarps = 8;  // sub-NTTs per CTA

// 64-bit-bank swizzle inside a warp region (16 x 8-byte banks per half warp)
__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 4) & 15); }

// index of register k of `lane` when register bits are [s0, s0 + LOGE)
template <int LOGE>
__device__ __forceinline__ int lay(int lane, int k, int s0) {
  return (lane & ((1 << s0) - 1)) | (k << s0) | ((lane >> s0) << (s0 + LOGE));
}

template <int LOGE>
__device__ __forceinline__ void relayout(u64 (&x)[1 << LOGE], u64* sm, int lane, int from, int to) {
  if (from == to) return;
#pragma unroll
  for (int k = 0; k < (1 << LOGE); ++k) sm[swz(lay<LOGE>(lane, k, from))] = x[k];
  __syncwarp();
#pragma unroll
  for (int k = 0; k < (1 << LOGE); ++k) x[k] = sm[swz(lay<LOGE>(lane, k, to))];
  __syncwarp();
}

// Forward sub-NTT (CT). Entry/exit layout: s0 = LOGM - LOGE (lane = low 5 bits).
// tw(b, blk) -> (w, w_shoup) for the stage of butterfly distance 2^b.
template <int LOGM, class TW>
__device__ __forceinline__ void warp_fwd(u64 (&x)[1 << (LOGM - 5)], u64* sm, int lane, u64 q, const TW& tw) {
  constexpr int LOGE = LOGM - 5;
  constexpr int E = 1 << LOGE;
  const u64 q2 = 2 * q;
  int s0 = LOGM - LOGE;
#pragma unroll
  for (int hi = LOGM; hi > 0; hi -= LOGE) {
    const int lo = hi - LOGE > 0 ? hi - LOGE : 0;
    relayout<LOGE>(x, sm, lane, s0, lo);
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
        // Harvey lazy CT butterfly: operands in [0, 4q), T in [0, 2q)
        u64 U = x[k];
        U = U >= q2 ? U - q2 : U;
        const u64 T = mul_shoup_lazy(x[k | (1 << rb)], w, ws, q);
        x[k] = U + T;
        x[k | (1 << rb)] = U - T + q2;
      }
    }
  }
  relayout<LOGE>(x, sm, lane, s0, LOGM - LOGE);
}

// Inverse sub-NTT (GS), same entry/exit layout.
template <int LOGM, class TW>
__device__ __forceinline__ void warp_inv(u64 (&x)[1 << (LOGM - 5)], u64* sm, int lane, u64 q, const TW& tw) {
  constexpr int LOGE = LOGM - 5;
  constexpr int E = 1 << LOGE;
  const u64 q2 = 2 * q;
  int s0 = LOGM - LOGE;
#pragma unroll
  for (int lo = 0; lo < LOGM; lo += LOGE) {
    const int hi = lo + LOGE < LOGM ? lo + LOGE : LOGM;
    const int ns0 = hi - LOGE > 0 ? hi - LOGE : 0;
    relayout<LOGE>(x, sm, lane, s0, ns0);
    s0 = ns0;
#pragma unroll
    for (int b = lo; b < hi; ++b) {
      const int rb = b - s0;
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if (k & (1 << rb)) continue;
        const int idx = lay<LOGE>(lane, k, s0);
        u64 w, ws;
        tw(b, idx >> (b + 1), w, ws);
        // Harvey lazy GS butterfly: operands in [0, 2q)
        const u64 U = x[k], V = x[k | (1 << rb)];
        const u64 S = U + V;
        x[k] = S >= q2 ? S - q2 : S;
        x[k | (1 << rb)] = mul_shoup_lazy(U - V + q2, w, ws, q);
      }
    }
  }
  relayout<LOGE>(x, sm, lane, s0, LOGM - LOGE);
}

// ---------------------------------------------------------------- row pass
// Warp w of a CTA transforms row (tile*kWarps + w) of its limb (C = 2^LOGC).
template <int LOGR, int LOGC, bool INV>
__global__ void __launch_bounds__(kWarps * 32) ntt_row_pass(LimbBatch B, Tabs T) {
  constexpr int C = 1 << LOGC, E = C / 32, LOGN = LOGR + LOGC;
  constexpr int tiles = (1 << LOGR) / kWarps;
  __shared__ u64 sm_all[kWarps * C];
  const int entry = blockIdx.x / tiles, tile = blockIdx.x - entry * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = tile * kWarps + warp;
  const int p = B.prime[entry];
  const u64 q = T.q[p];
  u64* a = B.ptr[entry] + (size_t)row * C;
  u64* sm = sm_all + warp * C;
  u64 x[E];
#pragma unroll
  for (int k = 0; k < E; ++k) x[k] = a[lane + 32 * k];
  if (!INV) {
    const u64* W = T.psi + ((size_t)p << LOGN);
    const u64* Ws = T.psi_s + ((size_t)p << LOGN);
    // row stage with in-row distance 2^b is global stage s = r + (c-1-b):
    // twiddle index 2^s + row * 2^(c-1-b) + blk
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int sp = LOGC - 1 - b;
      const int i = (1 << (LOGR + sp)) + (row << sp) + blk;
      w = W[i];
      ws = Ws[i];
    };
    warp_fwd<LOGC>(x, sm, lane, q, tw);
#pragma unroll
    for (int k = 0; k < E; ++k) {  // [0, 4q) -> canonical
      u64 v = x[k];
      v = v >= 2 * q ? v - 2 * q : v;
      x[k] = v >= q ? v - q : v;
    }
  } else {
    const u64* W = T.ipsi + ((size_t)p << LOGN);
    const u64* Ws = T.ipsi_s + ((size_t)p << LOGN);
    // GS stage with distance t = 2^b: h = n/(2t); blocks per row C/(2t)
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int i = (1 << (LOGN - 1 - b)) + (row << (LOGC - 1 - b)) + blk;
      w = W[i];
      ws = Ws[i];
    };
    warp_inv<LOGC>(x, sm, lane, q, tw);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) a[lane + 32 * k] = x[k];
}

// ------------------------------------------------------------- column pass
// A CTA owns kWarps adjacent columns x R rows: the tile is staged through
// shared memory with 64-byte coalesced row segments, each warp transforms one
// column (R = 2^LOGR points, stride C in global memory).
template <int LOGR, int LOGC, bool INV>
__global__ void __launch_bounds__(kWarps * 32) ntt_col_pass(LimbBatch B, Tabs T) {
  constexpr int R = 1 << LOGR, C = 1 << LOGC, E = R / 32, LOGN = LOGR + LOGC;
  constexpr int tiles = C / kWarps;
  constexpr int PAD = R + 1;  // column regions offset by one bank
  __shared__ u64 sm_all[kWarps * PAD];
  __shared__ u64 tw_s[2 * R];
  const int entry = blockIdx.x / tiles, tile = blockIdx.x - entry * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = B.prime[entry];
  const u64 q = T.q[p];
  u64* a = B.ptr[entry] + tile * kWarps;
  {
    const u64* W = (INV ? T.ipsi : T.psi) + ((size_t)p << LOGN);
    const u64* Ws = (INV ? T.ipsi_s : T.psi_s) + ((size_t)p << LOGN);
    for (int i = threadIdx.x; i < R; i += blockDim.x) {
      tw_s[i] = W[i];
      tw_s[R + i] = Ws[i];
    }
  }
  // stage the R x kWarps tile: element (row, col) -> column region col
  for (int e = threadIdx.x; e < R * kWarps; e += blockDim.x) {
    const int row = e / kWarps, col = e % kWarps;
    sm_all[col * PAD + swz(row)] = a[(size_t)row * C + col];
  }
  __syncthreads();
  u64* sm = sm_all + warp * PAD;
  u64 x[E];
#pragma unroll
  for (int k = 0; k < E; ++k) x[k] = sm[swz(lane + 32 * k)];
  __syncwarp();
  if (!INV) {
    // column stage with distance 2^b (rows) is global stage r-1-b: psi[2^(r-1-b) + blk]
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int i = (1 << (LOGR - 1 - b)) + blk;
      w = tw_s[i];
      ws = tw_s[R + i];
    };
    warp_fwd<LOGR>(x, sm, lane, q, tw);
  } else {
    // GS distance 2^b rows = 2^b * C words: h = n / (2 t) = 2^(r-1-b)
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int i = (1 << (LOGR - 1 - b)) + blk;
      w = tw_s[i];
      ws = tw_s[R + i];
    };
    warp_inv<LOGR>(x, sm, lane, q, tw);
    const u64 ni = T.ninv[p], nis = T.ninv_s[p];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = mul_shoup(x[k], ni, nis, q);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) sm[swz(lane + 32 * k)] = x[k];
  __syncthreads();
  for (int e = threadIdx.x; e < R * kWarps; e += blockDim.x) {
    const int row = e / kWarps, col = e % kWarps;
    a[(size_t)row * C + col] = sm_all[col * PAD + swz(row)];
  }
}

template <int LOGR, int LOGC>
void run_two_pass(Context& c, const LimbBatch& b, bool inverse) {
  const unsigned rows_grid = (unsigned)b.count * ((1u << LOGR) / kWarps);
  const unsigned cols_grid = (unsigned)b.count * ((1u << LOGC) / kWarps);
  if (!inverse) {
    ntt_col_pass<LOGR, LOGC, false><<<cols_grid, kWarps * 32, 0, c.stream>>>(b, c.tabs);
    ntt_row_pass<LOGR, LOGC, false><<<rows_grid, kWarps * 32, 0, c.stream>>>(b, c.tabs);
  } else {
    ntt_row_pass<LOGR, LOGC, true><<<rows_grid, kWarps * 32, 0, c.stream>>>(b, c.tabs);
    ntt_col_pass<LOGR, LOGC, true><<<cols_grid, kWarps * 32, 0, c.stream>>>(b, c.tabs);
  }
}

}  // namespace

bool ntt_two_pass(Context& c, const LimbBatch& b, bool inverse) {
  switch (c.logn) {
    case 12: run_two_pass<6, 6>(c, b, inverse); return true;
    case 13: run_two_pass<6, 7>(c, b, inverse); return true;
    case 14: run_two_pass<7, 7>(c, b, inverse); return true;
    case 15: run_two_pass<7, 8>(c, b, inverse); return true;
    case 16: run_two_pass<8, 8>(c, b, inverse); return true;
    case 17: run_two_pass<8, 9>(c, b, inverse); return true;
    default: return false;
  }
}

}  // namespace sf
