// Batched negacyclic NTT / inverse NTT over 64-bit RNS limbs, sm_100a, and the
// fused column kernel of ModUp / ModDown / rescale.
//
// n = R x C (R = 2^r rows, C = 2^c columns, element (row, col) at row*C+col).
// Forward (Cooley-Tukey, natural -> bit-reversed): the first r stages have
// butterfly distance >= C and act within columns (column pass), the last c
// stages act within rows (row pass). Inverse (Gentleman-Sande) runs the row
// pass first, then the column pass, folding n^-1 into the last stage. Every
// sub-transform is owned by one warp (warp_ntt.cuh). A launch covers any number
// of limbs (LimbBatch), so one launch touches every limb of a whole batch of
// ciphertexts.
//
// Fusion: basis conversion / rescale lifting is elementwise over
// coefficients, so it runs in shared memory between the inverse column pass of
// its source limbs and the forward column pass of its destination limbs, and
// the ModDown / rescale combine runs as the epilogue of the forward row pass:
// ModUp, ModDown and rescale each cost three passes over HBM instead of six.
#include "batch.cuh"
#include "warp_ntt.cuh"

namespace sf {
namespace {

using namespace wntt;
constexpr int kWarps = 8;  // sub-NTTs per CTA

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
  const u64* a = B.ptr[entry] + (size_t)row * C;
  u64* o = (B.optr[entry] ? B.optr[entry] : B.ptr[entry]) + (size_t)row * C;
  u64* sm = sm_all + warp * C;
  u64 x[E];
  if (!INV) {
    // strided 256-byte coalesced loads in, blocked 16-byte vector stores out
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = a[lane + 32 * k];
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
    warp_fwd<LOGC, kBlocked>(x, sm, lane, q, tw);
#pragma unroll
    for (int k = 0; k < E; k += 2)
      reinterpret_cast<ulonglong2*>(o + lane * E)[k / 2] = make_ulonglong2(canon4(x[k], q), canon4(x[k + 1], q));
  } else {
    // blocked 16-byte vector loads in, strided coalesced stores out
#pragma unroll
    for (int k = 0; k < E; k += 2) {
      const ulonglong2 v = reinterpret_cast<const ulonglong2*>(a + lane * E)[k / 2];
      x[k] = v.x;
      x[k + 1] = v.y;
    }
    const u64* W = T.ipsi + ((size_t)p << LOGN);
    const u64* Ws = T.ipsi_s + ((size_t)p << LOGN);
    // GS stage with distance t = 2^b: h = n/(2t); blocks per row C/(2t)
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int i = (1 << (LOGN - 1 - b)) + (row << (LOGC - 1 - b)) + blk;
      w = W[i];
      ws = Ws[i];
    };
    warp_inv<LOGC, kBlocked>(x, sm, lane, q, tw);
#pragma unroll
    for (int k = 0; k < E; ++k) o[lane + 32 * k] = x[k];
  }
}

// Forward row pass + combine epilogue (EpiBatch): out = (acc - v) * inv (+ addend);
// NOMUL: out = acc - v (+ addend) (ModDown with P^-1 folded into the keys and the conversion).
template <int LOGR, int LOGC, bool NOMUL>
__global__ void __launch_bounds__(kWarps * 32) ntt_row_epi(EpiBatch B, Tabs T) {
  constexpr int C = 1 << LOGC, E = C / 32, LOGN = LOGR + LOGC;
  constexpr int tiles = (1 << LOGR) / kWarps;
  __shared__ u64 sm_all[kWarps * C];
  const int entry = blockIdx.x / tiles, tile = blockIdx.x - entry * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = tile * kWarps + warp;
  const int p = B.prime[entry];
  const u64 q = T.q[p];
  const u64* a = B.buf[entry] + (size_t)row * C;
  u64* sm = sm_all + warp * C;
  u64 x[E];
#pragma unroll
  for (int k = 0; k < E; ++k) x[k] = a[lane + 32 * k];
  const u64* W = T.psi + ((size_t)p << LOGN);
  const u64* Ws = T.psi_s + ((size_t)p << LOGN);
  auto tw = [&](int b, int blk, u64& w, u64& ws) {
    const int sp = LOGC - 1 - b;
    const int i = (1 << (LOGR + sp)) + (row << sp) + blk;
    w = W[i];
    ws = Ws[i];
  };
  warp_fwd<LOGC, kBlocked>(x, sm, lane, q, tw);
  const u64* acc = B.acc[entry];
  const u64* addend = B.addend[entry];
  const u64* post = B.post[entry];
  const u64 g = B.g[entry], inv = B.inv[entry], inv_s = B.inv_s[entry];
  u64* out = B.out[entry];
  const int base = row * C + lane * E;  // blocked: this lane owns E consecutive outputs
#pragma unroll
  for (int k = 0; k < E; k += 2) {
    const ulonglong2 av = *reinterpret_cast<const ulonglong2*>(acc + base + k);
    u64 v0 = sub_mod(av.x, canon4(x[k], q), q);
    u64 v1 = sub_mod(av.y, canon4(x[k + 1], q), q);
    if constexpr (!NOMUL) {
      v0 = mul_shoup(v0, inv, inv_s, q);
      v1 = mul_shoup(v1, inv, inv_s, q);
    }
    if (addend) {
      if (g > 1) {
        v0 = add_mod(v0, addend[auto_perm((uint32_t)(base + k), g, LOGN)], q);
        v1 = add_mod(v1, addend[auto_perm((uint32_t)(base + k + 1), g, LOGN)], q);
      } else {
        const ulonglong2 dv = *reinterpret_cast<const ulonglong2*>(addend + base + k);
        v0 = add_mod(v0, dv.x, q);
        v1 = add_mod(v1, dv.y, q);
      }
    }
    if (post) {  // fused ct x pt (the plaintext product mul_plain_batch would apply next)
      const ulonglong2 pv = *reinterpret_cast<const ulonglong2*>(post + base + k);
      v0 = mulmod(v0, pv.x, q, T.mh[p], T.ml[p]);
      v1 = mulmod(v1, pv.y, q, T.mh[p], T.ml[p]);
    }
    *reinterpret_cast<ulonglong2*>(out + base + k) = make_ulonglong2(v0, v1);
  }
}

// ------------------------------------------------------------- column pass
// A CTA owns kWarps adjacent columns x R rows: the tile is staged through
// shared memory with 64-byte coalesced row segments, each warp transforms one
// column (R = 2^LOGR points, stride C in global memory).
template <int LOGR, int LOGC, bool INV>
__global__ void __launch_bounds__(kWarps * 32) ntt_col_pass(LimbBatch B, Tabs T) {
  constexpr int R = 1 << LOGR, C = 1 << LOGC, E = R / 32, LOGN = LOGR + LOGC;
  constexpr int tiles = C / kWarps;
  constexpr int PAD = R + 2;  // column regions offset by one 8-byte bank pair (conflict-free row-major staging)
  __shared__ u64 sm_all[kWarps * PAD];
  __shared__ u64 tw_s[2 * R];
  const int entry = blockIdx.x / tiles, tile = blockIdx.x - entry * tiles;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int swl = swz(lane);  // lane part of the (linear) swizzle
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
  for (int e = threadIdx.x; e < R * kWarps; e += blockDim.x) {
    const int row = e / kWarps, col = e % kWarps;
    sm_all[col * PAD + swz(row)] = a[(size_t)row * C + col];
  }
  __syncthreads();
  u64* sm = sm_all + warp * PAD;
  u64 x[E];
#pragma unroll
  for (int k = 0; k < E; ++k) x[k] = sm[(swl ^ swz(32 * k))];
  __syncwarp();
  // column stage with distance 2^b rows: forward global stage r-1-b uses
  // psi[2^(r-1-b) + blk]; GS: h = n / (2 * 2^b * C) = 2^(r-1-b)
  auto tw = [&](int b, int blk, u64& w, u64& ws) {
    const int i = (1 << (LOGR - 1 - b)) + blk;
    w = tw_s[i];
    ws = tw_s[R + i];
  };
  if (!INV) {
    warp_fwd<LOGR>(x, sm, lane, q, tw);  // lazy output in [0, 4q): the row pass accepts it
  } else {
    warp_inv<LOGR>(x, sm, lane, q, tw);
    const u64 ni = T.ninv[p], nis = T.ninv_s[p];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = mul_shoup(x[k], ni, nis, q);
  }
#pragma unroll
  for (int k = 0; k < E; ++k) sm[(swl ^ swz(32 * k))] = x[k];
  __syncthreads();
  for (int e = threadIdx.x; e < R * kWarps; e += blockDim.x) {
    const int row = e / kWarps, col = e % kWarps;
    a[(size_t)row * C + col] = sm_all[col * PAD + swz(row)];
  }
}

// ------------------------------------------------------------ fused column
// One CTA = one job x TCF adjacent columns, one warp per column (TCF warps).
// Shared memory holds the ns source tiles and two destination tiles; the
// destinations are produced one prime at a time (conversion -> forward column
// NTT -> store), so shared memory does not grow with nd and every phase keeps
// all warps busy. TCF = 8 gives 64-byte row segments for big batches; TCF = 2
// gives 4x more CTAs for single-ciphertext launches.
template <int LOGR, int LOGC, int TCF, int CPW, bool FC>
__global__ void __launch_bounds__(TCF / CPW * 32, TCF / CPW == 8 ? (CPW == 1 && LOGR + LOGC < 17 ? 3 : 2)
                                                                  : (TCF / CPW == 4 ? (LOGR + LOGC < 17 ? 6 : 4) : 8))
    fused_col_kernel(FusedColArgs A, Tabs T) {
  // CPW columns per warp (TCF / CPW warps): the column transforms of one warp
  // run interleaved (shared twiddles, CPW x the independent butterflies)
  constexpr int R = 1 << LOGR, C = 1 << LOGC, E = R / 32, LOGN = LOGR + LOGC;
  // column regions offset by 2 banks pairs: a half warp staging TCF = 8 columns
  // of two adjacent rows (swz(row) and swz(row ^ 1) differ in bit 0) hits 16
  // distinct 8-byte banks; PAD = R + 1 made those 2-way conflicts
  constexpr int PAD = R + 2;
  constexpr int tiles = C / TCF;
  constexpr int NT = TCF / CPW * 32;
  extern __shared__ u64 sm_all[];  // [ns][TCF][PAD] sources, [TCF][PAD] destination
  // blockIdx.x = (job * dgroups + dgroup) * tiles + tile; a CTA converts the
  // destinations [dgroup * dpc, +dpc) (dpc = nd: all of them)
  const int dpc = A.d_per_cta > 0 ? A.d_per_cta : A.nd;
  const int dgroups = (A.nd + dpc - 1) / dpc;
  const int tile = blockIdx.x % tiles, jd = blockIdx.x / tiles;
  const int job = jd / dgroups, dgroup = jd - job * dgroups;
  const int d_lo = dgroup * dpc, d_hi = min(A.nd, d_lo + dpc);
  const int col0 = tile * TCF;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int swl = swz(lane);  // lane part of the (linear) swizzle
  constexpr int n = 1 << LOGN;
  const u64* src = A.src[job];
  u64* dst = A.dst[job];
  auto region = [&](int limb, int col) { return sm_all + (size_t)(limb * TCF + col) * PAD; };
  // 1. stage the source tiles (TCF*8-byte row segments): per source limb, all
  //    of a thread's loads are issued before its shared-memory stores (R*TCF/NT
  //    loads in flight per thread instead of one)
  constexpr int kStage = R * TCF / NT;
  for (int s = 0; s < A.ns; ++s) {
    u64 v[kStage];
#pragma unroll
    for (int i = 0; i < kStage; ++i) {
      const int e = threadIdx.x + i * NT, row = e / TCF, col = e - row * TCF;
      v[i] = src[(size_t)s * n + (size_t)row * C + col0 + col];
    }
#pragma unroll
    for (int i = 0; i < kStage; ++i) {
      const int e = threadIdx.x + i * NT, row = e / TCF, col = e - row * TCF;
      region(s, col)[swz(row)] = v[i];
    }
  }
  __syncthreads();
  // 2. inverse column NTT of every (source limb, column); the epilogue applies
  //    n^-1 (mode 1) or n^-1 qhat_s^-1 (mode 0: the conversion's first factor)
  for (int s = 0; s < A.ns; ++s) {
    const int p = A.src_prime[s];
    const u64 q = T.q[p];
    const u64* W = T.ipsi + ((size_t)p << LOGN);
    const u64* Ws = T.ipsi_s + ((size_t)p << LOGN);
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int i = (1 << (LOGR - 1 - b)) + blk;
      w = W[i];
      ws = Ws[i];
    };
    u64* sm[CPW];
    u64 x[CPW][E];
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      sm[c] = region(s, warp * CPW + c);
#pragma unroll
      for (int k = 0; k < E; ++k) x[c][k] = sm[c][(swl ^ swz(32 * k))];
    }
    __syncwarp();
    // canonical y_s: the basis conversion's [x q^_s^-1]_{q_s} (and the centred lift) need it;
    // the factor rides the last inverse stage (its twiddle is ipsi[1] for every butterfly)
    const u64 ym = A.mode == 0 ? A.ymul[s] : T.ninv[p], yms = A.mode == 0 ? A.ymul_s[s] : T.ninv_s[p];
    const u64 ymw = A.mode == 0 ? A.ymulw[s] : T.ninvw[p], ymws = A.mode == 0 ? A.ymulw_s[s] : T.ninvw_s[p];
    warp_inv_n<LOGR, CPW, decltype(tw), true>(x, sm, lane, q, tw, ym, yms, ymw, ymws);
#pragma unroll
    for (int c = 0; c < CPW; ++c)
#pragma unroll
      for (int k = 0; k < E; ++k) sm[c][(swl ^ swz(32 * k))] = x[c][k];
    __syncwarp();
  }
  __syncthreads();
  for (int d = d_lo; d < d_hi; ++d) {
    const int pd = A.dst_prime[d];
    const u64 q = T.q[pd];
    u64* out = region(A.ns, 0);
    if constexpr (FC) {
      // 3+4. each warp converts its own column(s) straight into registers and
      // transforms them (no destination-tile round trip, one barrier less)
      u64 x[CPW][E];
      u64* sm[CPW];
      if (A.mode == 0) {
        u64 h[8], hs[8];
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < A.ns) h[s] = A.qhat[(size_t)s * A.nd + d], hs[s] = A.qhat_s[(size_t)s * A.nd + d];
        const u64 q4 = 4 * q, q8 = 8 * q;
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
          const int col = warp * CPW + c;
          sm[c] = out + (size_t)col * PAD;
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const int r = (swl ^ swz(32 * k));
            u64 acc = 0;
#pragma unroll
            for (int s = 0; s < 8; ++s)
              if (s < A.ns) acc += mul_shoup_lazy(region(s, col)[r], h[s], hs[s], q);
            if (A.ns > 4) acc = acc >= q8 ? acc - q8 : acc;
            if (A.ns > 2) acc = acc >= q4 ? acc - q4 : acc;
            x[c][k] = acc;
          }
        }
      } else {
        const u64 mh = T.mh[pd];
        const u64 ql = reduce64(A.q_last, q, mh), half = A.q_last >> 1;
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
          const int col = warp * CPW + c;
          sm[c] = out + (size_t)col * PAD;
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const u64 v = region(0, col)[(swl ^ swz(32 * k))];
            const u64 rr = reduce64(v, q, mh);
            x[c][k] = v > half ? sub_mod(rr, ql, q) : rr;
          }
        }
      }
      const u64* W = T.psi + ((size_t)pd << LOGN);
      const u64* Ws = T.psi_s + ((size_t)pd << LOGN);
      auto tw = [&](int b, int blk, u64& w, u64& ws) {
        const int i = (1 << (LOGR - 1 - b)) + blk;
        w = W[i];
        ws = Ws[i];
      };
      warp_fwd_n<LOGR, CPW>(x, sm, lane, q, tw);
#pragma unroll
      for (int c = 0; c < CPW; ++c)
#pragma unroll
        for (int k = 0; k < E; ++k) sm[c][(swl ^ swz(32 * k))] = x[c][k];
      __syncthreads();
      u64* o = dst + (size_t)A.out_slot[d] * n + col0;
      for (int e = threadIdx.x; e < R * TCF; e += NT) {
        const int row = e / TCF, col = e - row * TCF;
        o[(size_t)row * C + col] = out[(size_t)col * PAD + swz(row)];
      }
      if (d + 1 < d_hi) __syncthreads();
      continue;
    }
    // 3. conversion (coefficient domain) into destination tile d & 1
    if (A.mode == 0) {
      u64 h[8], hs[8];
#pragma unroll
      for (int s = 0; s < 8; ++s)
        if (s < A.ns) h[s] = A.qhat[(size_t)s * A.nd + d], hs[s] = A.qhat_s[(size_t)s * A.nd + d];
      // the forward column NTT accepts [0, 4q): the ns lazy Shoup products (each
      // in [0, 2q), q < 2^60) are summed and brought below 4q only as needed
      const u64 q4 = 4 * q, q8 = 8 * q;
      for (int e = threadIdx.x; e < R * TCF; e += NT) {
        const int row = e / TCF, col = e - row * TCF;
        const int r = swz(row);
        u64 acc = 0;
#pragma unroll
        for (int s = 0; s < 8; ++s)
          if (s < A.ns) acc += mul_shoup_lazy(region(s, col)[r], h[s], hs[s], q);
        if (A.ns > 4) acc = acc >= q8 ? acc - q8 : acc;
        if (A.ns > 2) acc = acc >= q4 ? acc - q4 : acc;
        out[(size_t)col * PAD + r] = acc;
      }
    } else {  // rescale lift: centred x mod q_last reduced mod each destination prime
      const u64 mh = T.mh[pd];
      const u64 ql = reduce64(A.q_last, q, mh), half = A.q_last >> 1;
      for (int e = threadIdx.x; e < R * TCF; e += NT) {
        const int row = e / TCF, col = e - row * TCF;
        const int r = swz(row);
        const u64 v = region(0, col)[r];
        const u64 rr = reduce64(v, q, mh);
        out[(size_t)col * PAD + r] = v > half ? sub_mod(rr, ql, q) : rr;
      }
    }
    __syncthreads();
    // 4. forward column NTT, one column per warp
    {
      const u64* W = T.psi + ((size_t)pd << LOGN);
      const u64* Ws = T.psi_s + ((size_t)pd << LOGN);
      auto tw = [&](int b, int blk, u64& w, u64& ws) {
        const int i = (1 << (LOGR - 1 - b)) + blk;
        w = W[i];
        ws = Ws[i];
      };
      u64* sm[CPW];
      u64 x[CPW][E];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        sm[c] = out + (size_t)(warp * CPW + c) * PAD;
#pragma unroll
        for (int k = 0; k < E; ++k) x[c][k] = sm[c][(swl ^ swz(32 * k))];
      }
      __syncwarp();
      warp_fwd_n<LOGR, CPW>(x, sm, lane, q, tw);
#pragma unroll
      for (int c = 0; c < CPW; ++c)
#pragma unroll
        for (int k = 0; k < E; ++k) sm[c][(swl ^ swz(32 * k))] = x[c][k];
    }
    __syncthreads();
    // 5. store (lazy [0, 4q) values; the row pass accepts them); one
    //    destination tile, so the next conversion waits for the stores
    u64* o = dst + (size_t)A.out_slot[d] * n + col0;
    for (int e = threadIdx.x; e < R * TCF; e += NT) {
      const int row = e / TCF, col = e - row * TCF;
      o[(size_t)row * C + col] = out[(size_t)col * PAD + swz(row)];
    }
    if (d + 1 < d_hi) __syncthreads();
  }
}

// ------------------------------------------------------ fused key-switch row
// One CTA = (source s, target slot t, kWarps source rows); warp w owns source
// row rs. Automorphisms map whole rows to whole rows in the bit-reversed
// evaluation order (the row index is the top LOGR bits of the position, which
// fix e = 2 br(i) + 1 mod 2C and hence e*g mod 2C), so every output row of a
// job reads exactly one source row: rd = perm_{g^-1}(rs), and within it the
// column perm_g(rd*C + c) mod C.
template <int LOGR, int LOGC>
// ring 2^17 rows hold 16 residues per lane: one CTA per SM lifts the register cap (no spills)
__global__ void __launch_bounds__(kWarps * 32, LOGC >= 9 ? 1 : 3) ks_row_kernel(KsRowArgs A, Tabs T) {
  constexpr int C = 1 << LOGC, E = C / 32, LOGN = LOGR + LOGC;
  auto rbr = [](uint32_t col) { return __brev(col) >> (32 - LOGC); };
  // row buffers hold bit-reversed columns; lane L's blocked segment lands at
  // brev5(L) + 32 k, whose bit 4 (= bit 0 of L) is folded into bit 0 so the 16
  // lanes of a half warp (and the affine gathers below) hit 16 distinct banks
  auto xp = [](uint32_t i) { return i ^ ((i >> 4) & 1u); };
  constexpr int tiles = (1 << LOGR) / kWarps;
  constexpr int n = 1 << LOGN;
  extern __shared__ u64 ks_sm[];  // [kWarps][ndig + 1][C]
  const int tile = blockIdx.x % tiles, rest = blockIdx.x / tiles;
  const int t = rest % A.nt, s = rest / A.nt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rs = tile * kWarps + warp;
  const int m = A.tprime[t];
  const u64 q = T.q[m];
  u64* wsm = ks_sm + (size_t)warp * (A.ndig + 1) * C;
  if (lane < C / 16 && A.job_begin[s] < A.job_begin[s + 1]) {  // the first job's key rows: in flight during the row NTTs
    const int j0 = A.job_begin[s];
    const u64 g0 = A.g[j0];
    const int rd0 = g0 > 1 ? (int)RowPerm<LOGR, LOGC>(rs, A.ginv[j0]).src_row : rs;
    for (int j = 0; j < A.ndig; ++j)
      for (int part = 0; part < 2; ++part)
        prefetch_l1(A.key[j0] + ((size_t)(j * 2 + part) * A.np + m) * n + (size_t)rd0 * C + (size_t)lane * 16);
  }
  // 1. row rs of every digit's extended polynomial, NTT domain, natural order
  for (int j = 0; j < A.ndig; ++j) {
    u64* X = wsm + j * C;
    const int lo = j * A.alpha, hi = min(lo + A.alpha, A.limbs);
    if (t >= lo && t < hi) {  // own prime: the exact NTT-domain source residues
      const u64* a = A.c1[s] + (size_t)t * n + (size_t)rs * C + lane * E;
#pragma unroll
      for (int k = 0; k < E; k += 2) {
        const ulonglong2 v = reinterpret_cast<const ulonglong2*>(a)[k / 2];
        X[xp(rbr(lane * E + k))] = v.x;
        X[xp(rbr(lane * E + k + 1))] = v.y;
      }
    } else {
      const u64* a = A.ext[s] + ((size_t)j * A.nt + t) * n + (size_t)rs * C;
      u64 x[E];
#pragma unroll
      for (int k = 0; k < E; ++k) x[k] = a[lane + 32 * k];
      const u64* W = T.psi + ((size_t)m << LOGN);
      const u64* Ws = T.psi_s + ((size_t)m << LOGN);
      auto tw = [&](int b, int blk, u64& w, u64& ws) {
        const int sp = LOGC - 1 - b;
        const int i = (1 << (LOGR + sp)) + (rs << sp) + blk;
        w = W[i];
        ws = Ws[i];
      };
      warp_fwd<LOGC, kBlocked, decltype(tw), true>(x, X, lane, q, tw);
#pragma unroll
      for (int k = 0; k < E; ++k) X[xp(rbr(lane * E + k))] = canon4(x[k], q);
    }
  }
  __syncwarp();
  const u64 mh = T.mh[m], qn = T.qn[m];  // keys (and pm) are Montgomery-scaled: get_key_mont
  u64* scratch = wsm + A.ndig * C;
  // 2. every job of this source: permuted inner product with its key
  for (int jb = A.job_begin[s]; jb < A.job_begin[s + 1]; ++jb) {
    const u64 g = A.g[jb];
    const int rd = g > 1 ? (int)RowPerm<LOGR, LOGC>(rs, A.ginv[jb]).src_row : rs;
    const size_t rowoff = (size_t)rd * C + lane * E;
    uint32_t sc[E];  // positions in the bit-reversed row buffers (bank-conflict free gathers)
#pragma unroll
    for (int k = 0; k < E; ++k)
      sc[k] = xp(g > 1 ? RowPerm<LOGR, LOGC>(rd, g).pos(rbr(lane * E + k)) : rbr(lane * E + k));
    // the b and a parts one after the other: half the accumulator registers
    // (3 CTAs per SM instead of 2); the gathered words are re-read from shared memory
#pragma unroll 1
    for (int part = 0; part < 2; ++part) {
      U128 acc[E];
#pragma unroll
      for (int k = 0; k < E; ++k) acc[k] = U128{0, 0};
      for (int j = 0; j < A.ndig; ++j) {
        const u64* X = wsm + j * C;
        const u64* kp = A.key[jb] + ((size_t)(j * 2 + part) * A.np + m) * n + rowoff;
#pragma unroll
        for (int k = 0; k < E; k += 2) {
          const ulonglong2 kv = reinterpret_cast<const ulonglong2*>(kp)[k / 2];
          mac128(acc[k], X[sc[k]], kv.x);
          mac128(acc[k + 1], X[sc[k + 1]], kv.y);
        }
      }
      if (A.merged && t < A.limbs) {  // + P * (d0, d1): the relinearised pair in the extended basis
        const u64 pmt = A.pm[t];
        const u64* ad = (part ? A.add1[jb] : A.add0[jb]) + (size_t)t * n + rowoff;
#pragma unroll
        for (int k = 0; k < E; k += 2) {
          const ulonglong2 v = reinterpret_cast<const ulonglong2*>(ad)[k / 2];
          mac128(acc[k], v.x, pmt);
          mac128(acc[k + 1], v.y, pmt);
        }
      }
      u64 v[E];
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = mont_finish(acc[k], q, mh, qn);
      u64* out = A.acc[jb] + (size_t)(part * A.nt + t) * n;
      if (t < A.limbs && !(A.merged && t == A.limbs - 1)) {
#pragma unroll
        for (int k = 0; k < E; k += 2)
          reinterpret_cast<ulonglong2*>(out + rowoff)[k / 2] = make_ulonglong2(v[k], v[k + 1]);
      } else {  // special prime: ModDown's inverse row pass, strided stores
        const u64* W = T.ipsi + ((size_t)m << LOGN);
        const u64* Ws = T.ipsi_s + ((size_t)m << LOGN);
        auto tw = [&](int b, int blk, u64& w, u64& ws) {
          const int i = (1 << (LOGN - 1 - b)) + (rd << (LOGC - 1 - b)) + blk;
          w = W[i];
          ws = Ws[i];
        };
        warp_inv<LOGC, kBlocked, decltype(tw), true>(v, scratch, lane, q, tw);
#pragma unroll
        for (int k = 0; k < E; ++k) out[(size_t)rd * C + lane + 32 * k] = v[k];
      }
    }
  }
}

// ------------------------------------------------------- rotation-sum row
// One CTA = (output o, target slot t, kWarps destination rows); warp w owns
// destination row rd and walks the jobs of o: each non-identity job reads its
// source rows rs = perm_g(rd) (digit ext rows / own c1 row and the c0 row),
// staged through the warp's shared row buffer for the in-row permutation.
// Automorphism gather of one row held blocked in registers (lane L owns the 8
// natural columns 8L..8L+7), by warp shuffles instead of a shared-memory round
// trip (ks_sum is L1TEX-bound; profiles/r1_ncu_v8.md). Destination register k
// of lane L needs the source at bit-reversed position
//   pos = (base + slope * ((brev3(k) << 5) | brev5(L))) mod 256,
// i.e. source lane brev5(pos & 31) -- a function of L alone -- and source
// register brev3(((A_L >> 5) + slope * brev3(k)) & 7) with A_L = base +
// slope * brev5(L). Each source lane therefore pre-rotates its registers by
// the c = (A_L >> 5) & 7 of the lane that will read it (3 select stages),
// applies the warp-uniform multiplier permutation (4 static cases, slope odd)
// and every register moves with one 64-bit shuffle.
struct ShflPerm {
  int src_lane;   // lane this lane reads from
  int c;          // rotation this lane applies for its reader
  int smod;       // slope mod 8 (odd)
  __device__ __forceinline__ ShflPerm(uint32_t base, uint32_t slope, int lane) {
    const uint32_t u = __brev((uint32_t)lane) >> 27;  // brev5(lane)
    src_lane = (int)(__brev((base + slope * u) & 31) >> 27);
    uint32_t inv = slope;  // slope^-1 mod 32 (Newton, slope odd)
    inv *= 2 - slope * inv;
    inv *= 2 - slope * inv;
    inv *= 2 - slope * inv;
    const uint32_t ur = (inv * ((__brev((uint32_t)lane) >> 27) - base)) & 31;  // reader's brev5(L)
    c = (int)(((base + slope * ur) >> 5) & 7);
    smod = (int)(slope & 7);
#pragma unroll
    for (int b = 0; b < 3; ++b) rm[b] = 0ull - (u64)((c >> b) & 1);
  }
  u64 rm[3];  // all-ones where rotation stage b applies (bit b of c)
  // v: natural-order registers of this lane's row segment -> permuted row
  __device__ __forceinline__ void apply(u64 (&v)[8]) const {
    u64 z[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) z[m] = v[__brev((uint32_t)m) >> 29];  // z[m] = v[brev3(m)]
    // z[i] <- z[(i + c) & 7]: a barrel rotation by 1, 2, 4 as bitwise blends
    // x ^ ((x ^ y) & m) (one LOP3 per 32-bit half on the ALU pipe; the branchy
    // in-place form compiled to predicated IMAD.MOVs on the FMA-heavy pipe that
    // the key-switch products saturate)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const u64 m = rm[b];
      u64 t[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) t[i] = z[i] ^ ((z[i] ^ z[(i + (1 << b)) & 7]) & m);
#pragma unroll
      for (int i = 0; i < 8; ++i) z[i] = t[i];
    }
    switch (smod) {  // y[k] = z[(slope * brev3(k)) & 7], then one shuffle per register
#define SF_SHFL_CASE(M)                                                                 \
  case M:                                                                               \
    _Pragma("unroll") for (int k = 0; k < 8; ++k) v[k] =                                \
        __shfl_sync(0xffffffffu, z[(M * (__brev((uint32_t)k) >> 29)) & 7], src_lane);  \
    break;
      SF_SHFL_CASE(1)
      SF_SHFL_CASE(3)
      SF_SHFL_CASE(5)
      SF_SHFL_CASE(7)
#undef SF_SHFL_CASE
    }
  }
};

// Automorphism gather for the pair-strided row layout of ks_sum (C = 256):
// register k = 2a + b of lane L holds column 64a + 2L + b, so every row load
// and store is one fully coalesced 16-byte access per lane per quarter a (the
// blocked layout's 64-byte lane stride cost 4x the L1 wavefronts: ks_sum was
// L1TEX-bound). In bit-reversed positions, brev8(64a + 2L + b) = brev2(a) +
// 4 brev5(L) + 128 b, so destination (L, a, b) reads position
//   p = (S_a + 4 slope brev5(L) + 128 b) mod 256,  S_a = base + slope brev2(a),
// i.e. source lane brev5((p >> 2) & 31) -- the same for b = 0, 1 -- source
// quarter brev2(S_a & 3) -- warp-uniform: 8 static cases of (base & 3, slope & 3)
// -- and source pair element b ^ (bit 7 of p at b = 0). Each source lane swaps
// its pair for the lane that reads it (one blend per quarter) and every
// register moves with one 64-bit shuffle.
struct ShflPermQ {
  int sl[4];        // per destination quarter: the lane this lane reads from
  uint32_t fm[4];   // per quarter: all-ones when this lane's reader needs the pair swapped
  int cs;           // quarter map case: (base & 3) | (slope & 2) << 1
  __device__ __forceinline__ ShflPermQ(uint32_t base, uint32_t slope, int lane) {
    const uint32_t u = __brev((uint32_t)lane) >> 27;  // brev5(lane)
    uint32_t inv = slope;  // slope^-1 mod 32 (Newton, slope odd)
    inv *= 2 - slope * inv;
    inv *= 2 - slope * inv;
    inv *= 2 - slope * inv;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const uint32_t S = (base + slope * (uint32_t)(((a & 1) << 1) | (a >> 1))) & 255;
      sl[a] = (int)(__brev(((S >> 2) + slope * u) & 31) >> 27);
      const uint32_t ur = (inv * (u - (S >> 2))) & 31;  // brev5 of the lane reading this one
      fm[a] = 0u - ((((S >> 2) + slope * ur) >> 5) & 1u);
    }
    cs = (int)((base & 3) | ((slope & 2) << 1));
  }
  __device__ __forceinline__ static u64 blend(u64 x, u64 y, uint32_t m) {  // m ? y : x, per 32-bit half
    const uint32_t lo = (uint32_t)x ^ (((uint32_t)x ^ (uint32_t)y) & m);
    const uint32_t hi = (uint32_t)(x >> 32) ^ (((uint32_t)(x >> 32) ^ (uint32_t)(y >> 32)) & m);
    return ((u64)hi << 32) | lo;
  }
  __device__ __forceinline__ void apply(u64 (&v)[8]) const {
    u64 y[8];
    switch (cs) {
#define SF_Q_CASE(K)                                                                          \
  case K:                                                                                     \
    _Pragma("unroll") for (int a = 0; a < 4; ++a) {                                           \
      constexpr int b3 = K & 3, s3 = (K & 4) ? 3 : 1;                                         \
      const int al = ((a & 1) << 1) | (a >> 1);                                               \
      const int pa = (b3 + s3 * al) & 3;                                                      \
      const int ap = ((pa & 1) << 1) | (pa >> 1);                                            \
      y[2 * a] = blend(v[2 * ap], v[2 * ap + 1], fm[a]);                                      \
      y[2 * a + 1] = blend(v[2 * ap + 1], v[2 * ap], fm[a]);                                  \
    }                                                                                         \
    break;
      SF_Q_CASE(0)
      SF_Q_CASE(1)
      SF_Q_CASE(2)
      SF_Q_CASE(3)
      SF_Q_CASE(4)
      SF_Q_CASE(5)
      SF_Q_CASE(6)
      SF_Q_CASE(7)
#undef SF_Q_CASE
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      v[2 * a] = __shfl_sync(0xffffffffu, y[2 * a], sl[a]);
      v[2 * a + 1] = __shfl_sync(0xffffffffu, y[2 * a + 1], sl[a]);
    }
  }
};

__device__ __forceinline__ void add128(U128& acc, uint64_t a) {
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, 0;" : "+l"(acc.lo), "+l"(acc.hi) : "l"(a));
}

// PM1: the keys' Q limbs carry P^-1 (get_key_pinv), so the P * sigma(c0) and
// P * (c0, c1) terms are plain additions
template <int LOGR, int LOGC, bool PF, bool SH, bool PM1>
__global__ void __launch_bounds__(kWarps * 32, LOGC >= 9 ? 1 : 2) ks_sum_kernel(KsSumArgs A, Tabs T) {
  constexpr int C = 1 << LOGC, E = C / 32, LOGN = LOGR + LOGC;
  auto rbr = [](uint32_t col) { return __brev(col) >> (32 - LOGC); };
  auto xp = [](uint32_t i) { return i ^ ((i >> 4) & 1u); };  // bank fold, as in ks_row_kernel
  constexpr int tiles = (1 << LOGR) / kWarps;
  constexpr int n = 1 << LOGN;
  __shared__ u64 rowbuf[kWarps][C];
  const int tile = blockIdx.x % tiles, rest = blockIdx.x / tiles;
  const int t = rest % A.nt, o = rest / A.nt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rd = tile * kWarps + warp;
  const int m = A.tprime[t];
  const u64 q = T.q[m], mh = T.mh[m], qn = T.qn[m];
  const bool qt = t < A.limbs;
  const bool c0t = qt || A.ext_c0;  // targets receiving the c0 (b part) terms
  const u64 pm = qt ? A.pm[t] : 0;
  u64* buf = rowbuf[warp];
  // register layout of a row: pair-strided on the shuffle path at C = 256
  // (register pair k of lane L = columns 64 (k/2) + 2L, +1: coalesced), blocked
  // otherwise (lane L owns columns E L .. E L + E - 1)
  constexpr bool PS = SH && LOGC == 8;
  auto eoff = [&](int k) { return PS ? 64 * (k >> 1) + 2 * lane : lane * E + k; };
  const size_t rowoff = (size_t)rd * C;
  U128 sb[E], sa[E];
#pragma unroll
  for (int k = 0; k < E; ++k) sb[k] = U128{0, 0}, sa[k] = U128{0, 0};
  // Montgomery-domain sums (keys and pm carry R = 2^64: get_key_mont): a product
  // adds < 2^56 to the high word, a plain term c (P * sigma(c0) with P^-1 folded
  // into the keys) enters as c R = c * 2^64, i.e. c added to the high word. A job
  // raises the high word by at most 2^60 + ndig 2^56 (q < 2^60: one product's high
  // word <= 2^56 per digit, one plain c < 2^60), so from a reduced high word (< q)
  // J jobs stay below 2^60 (1 + J (1 + ndig / 16)) < 2^64 for J <= 239 / (16 + ndig)
  // (14 single-digit jobs, 13 at two digits, 11 at four): the high word is brought
  // back below q every fold_at jobs (T changes by multiples of q 2^64) and the sum
  // finishes with one REDC.
  const int fold_at = 239 / (16 + A.ndig);
  int terms = 0;  // jobs since the last high-word reduction
  auto fold = [&]() {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      sb[k].hi = reduce64(sb[k].hi, q, mh);
      sa[k].hi = reduce64(sa[k].hi, q, mh);
    }
    terms = 0;
  };
  for (int jb = A.out_begin[o]; jb < A.out_begin[o + 1]; ++jb) {
    const int s = A.jsrc[jb];
    const u64 g = A.g[jb];
    if (terms >= fold_at) fold();
    if (g <= 1) {  // identity term: P * (c0, c1) on the Q primes (ext_c0: c0 on every target)
      if (!c0t) continue;
      const u64* a0 = A.c0[s] + (size_t)t * n + rowoff;
      const u64* a1 = A.c1[s] + (size_t)t * n + rowoff;
#pragma unroll
      for (int k = 0; k < E; k += 2) {
        const ulonglong2 v0 = *reinterpret_cast<const ulonglong2*>(a0 + eoff(k));
        const ulonglong2 v1 = qt ? *reinterpret_cast<const ulonglong2*>(a1 + eoff(k)) : make_ulonglong2(0, 0);
        if constexpr (PM1) {
          sb[k].hi += v0.x;
          sb[k + 1].hi += v0.y;
          sa[k].hi += v1.x;
          sa[k + 1].hi += v1.y;
        } else {
          mac128(sb[k], v0.x, pm);
          mac128(sb[k + 1], v0.y, pm);
          mac128(sa[k], v1.x, pm);
          mac128(sa[k + 1], v1.y, pm);
        }
      }
      ++terms;
      continue;
    }
    const RowPerm<LOGR, LOGC> rp(rd, g);
    const int rs = (int)rp.src_row;
    if constexpr (PS) {  // shuffle gather (no shared-memory round trip)
      const ShflPermQ sp(rp.base, rp.slope, lane);
      for (int j = 0; j < A.ndig; ++j) {
        const int lo = j * A.alpha, hi = min(lo + A.alpha, A.limbs);
        const u64* src = (t >= lo && t < hi) ? A.c1[s] + (size_t)t * n + (size_t)rs * C
                                             : A.ext[s] + ((size_t)j * A.nt + t) * n + (size_t)rs * C;
        const u64* kb = A.key[jb] + ((size_t)(j * 2 + 0) * A.np + m) * n + rowoff;
        const u64* ka = A.key[jb] + ((size_t)(j * 2 + 1) * A.np + m) * n + rowoff;
        u64 x[8];
#pragma unroll
        for (int k = 0; k < E; k += 2) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + eoff(k));
          x[k] = v.x, x[k + 1] = v.y;
        }
        sp.apply(x);
        ulonglong2 kv[E];
#pragma unroll
        for (int k = 0; k < E; k += 2)
          kv[k] = *reinterpret_cast<const ulonglong2*>(kb + eoff(k)),
          kv[k + 1] = *reinterpret_cast<const ulonglong2*>(ka + eoff(k));
#pragma unroll
        for (int k = 0; k < E; k += 2) {
          mac128(sb[k], x[k], kv[k].x);
          mac128(sa[k], x[k], kv[k + 1].x);
          mac128(sb[k + 1], x[k + 1], kv[k].y);
          mac128(sa[k + 1], x[k + 1], kv[k + 1].y);
        }
      }
      if (c0t) {  // P * sigma_g(c0)
        const u64* src = A.c0[s] + (size_t)t * n + (size_t)rs * C;
        u64 x[8];
#pragma unroll
        for (int k = 0; k < E; k += 2) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(src + eoff(k));
          x[k] = v.x, x[k + 1] = v.y;
        }
        sp.apply(x);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if constexpr (PM1)
            sb[k].hi += x[k];
          else
            mac128(sb[k], x[k], pm);
        }
      }
      ++terms;
      continue;
    }
    // source positions in the bit-reversed row buffer: an affine map of
    // br(column) with odd slope g, so every 16 lanes hit 16 distinct banks
    uint32_t sc[E];
#pragma unroll
    for (int k = 0; k < E; ++k) sc[k] = xp(rp.pos(rbr(lane * E + k)));
    for (int j = 0; j < A.ndig; ++j) {
      const int lo = j * A.alpha, hi = min(lo + A.alpha, A.limbs);
      const u64* src = (t >= lo && t < hi) ? A.c1[s] + (size_t)t * n + (size_t)rs * C
                                           : A.ext[s] + ((size_t)j * A.nt + t) * n + (size_t)rs * C;
      const u64* kb = A.key[jb] + ((size_t)(j * 2 + 0) * A.np + m) * n + rowoff + lane * E;
      const u64* ka = A.key[jb] + ((size_t)(j * 2 + 1) * A.np + m) * n + rowoff + lane * E;
      ulonglong2 kv[PF ? E : 1];  // PF: the key words are in flight while the row is staged
      if constexpr (PF) {
#pragma unroll
        for (int k = 0; k < E; k += 2) {
          kv[k] = reinterpret_cast<const ulonglong2*>(kb)[k / 2];
          kv[k + 1] = reinterpret_cast<const ulonglong2*>(ka)[k / 2];
        }
      }
#pragma unroll
      for (int k = 0; k < E; k += 2) {
        const ulonglong2 v = reinterpret_cast<const ulonglong2*>(src + lane * E)[k / 2];
        buf[xp(rbr(lane * E + k))] = v.x;
        buf[xp(rbr(lane * E + k + 1))] = v.y;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < E; k += 2) {
        ulonglong2 vb, va;
        if constexpr (PF) {
          vb = kv[k], va = kv[k + 1];
        } else {
          vb = reinterpret_cast<const ulonglong2*>(kb)[k / 2];
          va = reinterpret_cast<const ulonglong2*>(ka)[k / 2];
        }
        const u64 x0 = buf[sc[k]], x1 = buf[sc[k + 1]];
        mac128(sb[k], x0, vb.x);
        mac128(sa[k], x0, va.x);
        mac128(sb[k + 1], x1, vb.y);
        mac128(sa[k + 1], x1, va.y);
      }
      __syncwarp();
    }
    if (c0t) {  // P * sigma_g(c0)
      const u64* src = A.c0[s] + (size_t)t * n + (size_t)rs * C;
#pragma unroll
      for (int k = 0; k < E; k += 2) {
        const ulonglong2 v = reinterpret_cast<const ulonglong2*>(src + lane * E)[k / 2];
        buf[xp(rbr(lane * E + k))] = v.x;
        buf[xp(rbr(lane * E + k + 1))] = v.y;
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (PM1)
          sb[k].hi += buf[sc[k]];
        else
          mac128(sb[k], buf[sc[k]], pm);
      }
      __syncwarp();
    }
    ++terms;
  }
  u64 vb[E], va[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    vb[k] = mont_finish(sb[k], q, mh, qn);
    va[k] = mont_finish(sa[k], q, mh, qn);
  }
  u64* accb = A.acc[o] + (size_t)t * n;
  u64* acca = A.acc[o] + (size_t)(A.nt + t) * n;
  // NTT-domain stores on the Q targets; the special primes (and a merged q_top)
  // get ModDown's inverse row pass and strided stores -- except a kept b part
  const bool ntt_a = qt && t < A.inv_from, ntt_b = ntt_a || A.keep_b;
  if (ntt_b) {
#pragma unroll
    for (int k = 0; k < E; k += 2)
      *reinterpret_cast<ulonglong2*>(accb + rowoff + eoff(k)) = make_ulonglong2(vb[k], vb[k + 1]);
  }
  if (ntt_a) {
#pragma unroll
    for (int k = 0; k < E; k += 2)
      *reinterpret_cast<ulonglong2*>(acca + rowoff + eoff(k)) = make_ulonglong2(va[k], va[k + 1]);
  } else {
    const u64* W = T.ipsi + ((size_t)m << LOGN);
    const u64* Ws = T.ipsi_s + ((size_t)m << LOGN);
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int i = (1 << (LOGN - 1 - b)) + (rd << (LOGC - 1 - b)) + blk;
      w = W[i];
      ws = Ws[i];
    };
    if constexpr (PS) {  // pair-strided -> strided (lane + 32 k) through the row buffer, then the transform
      auto restride = [&](u64 (&v)[E]) {
#pragma unroll
        for (int k = 0; k < E; ++k) buf[xp(eoff(k & ~1) + (k & 1))] = v[k];
        __syncwarp();
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = buf[xp(lane + 32 * k)];
        __syncwarp();
      };
      if (!ntt_b) {
        restride(vb);
        warp_inv<LOGC, kStrided>(vb, buf, lane, q, tw);
      }
      restride(va);
      warp_inv<LOGC, kStrided>(va, buf, lane, q, tw);
    } else {
      if (!ntt_b) warp_inv<LOGC, kBlocked>(vb, buf, lane, q, tw);
      warp_inv<LOGC, kBlocked>(va, buf, lane, q, tw);
    }
    if (!ntt_b) {
#pragma unroll
      for (int k = 0; k < E; ++k) accb[(size_t)rd * C + lane + 32 * k] = vb[k];
    }
#pragma unroll
    for (int k = 0; k < E; ++k) acca[(size_t)rd * C + lane + 32 * k] = va[k];
  }
}

// ------------------------------------------ rotation-sum row, TMA pipelined
// Single-digit rotation sums at C = 256 (the QK^T folds and pack at level 1,
// two thirds of the rotation-sum time): ks_sum_kernel's pair-strided register
// math, but every row a job reads (its digit row, the two key rows, the c0 row;
// 2 KB each, contiguous) arrives in shared memory by 1D bulk copies
// (cp.async.bulk, the TMA engine) on a per-warp double-buffered mbarrier ring:
// lane 0 issues job i+1's copies before the warp computes job i, so the L2
// latency that left ks_sum long-scoreboard bound (profiles/r2_ncu: 3.4 stall
// cycles per issue) overlaps the previous job's arithmetic, with no registers
// held for the prefetch. Four warps (rows) per CTA, 72 KB of shared memory.
namespace tma1d {
__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(saddr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
}  // namespace tma1d

constexpr int kTmaWarps = 4;
constexpr int kTmaRows = 4;  // per stage: digit row, key b row, key a row, c0 row
// GATHER: the automorphism read straight out of the staged rows -- register k
// of lane L (natural column c = 64 (k/2) + 2L + (k & 1)) loads column
// br8((base + slope br8(c)) mod 256) with one 8-byte shared load -- instead of
// natural-order loads plus the ShflPermQ blend/shuffle network (the rows are in
// shared memory anyway; ~2-way bank conflicts, far fewer instructions per job)
// ONE: single-digit sums (the QKᵀ folds), the digit loop compiled away
template <int LOGR, bool PM1, bool GATHER, bool ONE>
__global__ void __launch_bounds__(kTmaWarps * 32, 3) ks_sum_tma_kernel(KsSumArgs A, Tabs T) {
  constexpr int LOGC = 8, C = 1 << LOGC, E = 8, LOGN = LOGR + LOGC;
  constexpr int tiles = (1 << LOGR) / kTmaWarps;
  constexpr int n = 1 << LOGN;
  extern __shared__ __align__(128) u64 tma_sm[];  // [warp][2 stages][kTmaRows][C], [warp][C], mbarriers
  const int tile = blockIdx.x % tiles, rest = blockIdx.x / tiles;
  const int t = rest % A.nt, o = rest / A.nt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rd = tile * kTmaWarps + warp;
  const int m = A.tprime[t];
  const u64 q = T.q[m], mh = T.mh[m], qn = T.qn[m];
  const bool qt = t < A.limbs;
  const bool c0t = qt || A.ext_c0;  // targets receiving the c0 (b part) terms
  const u64 pm = qt ? A.pm[t] : 0;
  u64* stage_base = tma_sm + (size_t)warp * 2 * kTmaRows * C;
  u64* buf = tma_sm + (size_t)kTmaWarps * 2 * kTmaRows * C + (size_t)warp * C;
  uint64_t* bars = reinterpret_cast<uint64_t*>(tma_sm + (size_t)kTmaWarps * (2 * kTmaRows + 1) * C) + warp * 2;
  auto eoff = [&](int k) { return 64 * (k >> 1) + 2 * lane; };
  auto xp = [](uint32_t i) { return i ^ ((i >> 4) & 1u); };
  const size_t rowoff = (size_t)rd * C;
  const int b0 = A.out_begin[o], b1 = A.out_begin[o + 1];
  if (lane == 0) {
    tma1d::mbar_init(&bars[0], 1);
    tma1d::mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint32_t row_bytes = C * sizeof(u64);
  // lane 0: arm stage st's barrier and copy the rows of job jb's digit j into it
  // (the digit row, its two key rows; with digit 0, the c0 row)
  auto issue = [&](int jb, int j, int st) {
    if (lane != 0) return;
    const int s = A.jsrc[jb];
    const int rs = (int)RowPerm<LOGR, LOGC>(rd, A.g[jb]).src_row;
    u64* dst = stage_base + (size_t)st * kTmaRows * C;
    const bool wc0 = c0t && j == 0;
    tma1d::fence_proxy_async();  // the warp's earlier shared-memory reads of this stage come first
    tma1d::mbar_expect_tx(&bars[st], (wc0 ? 4 : 3) * row_bytes);
    const int lo = j * A.alpha, hi = min(lo + A.alpha, A.limbs);
    const u64* src = (t >= lo && t < hi) ? A.c1[s] + (size_t)t * n : A.ext[s] + ((size_t)j * A.nt + t) * n;
    tma1d::bulk_g2s(dst, src + (size_t)rs * C, row_bytes, &bars[st]);
    tma1d::bulk_g2s(dst + C, A.key[jb] + ((size_t)(2 * j) * A.np + m) * n + rowoff, row_bytes, &bars[st]);
    tma1d::bulk_g2s(dst + 2 * C, A.key[jb] + ((size_t)(2 * j + 1) * A.np + m) * n + rowoff, row_bytes, &bars[st]);
    if (wc0) tma1d::bulk_g2s(dst + 3 * C, A.c0[s] + (size_t)t * n + (size_t)rs * C, row_bytes, &bars[st]);
  };
  auto next_rot = [&](int jb) {  // first non-identity job at or after jb
    while (jb < b1 && A.g[jb] <= 1) ++jb;
    return jb;
  };
  U128 sb[E], sa[E];
#pragma unroll
  for (int k = 0; k < E; ++k) sb[k] = U128{0, 0}, sa[k] = U128{0, 0};
  const int ndig = ONE ? 1 : A.ndig;
  const int fold_at = ONE ? 14 : 239 / (16 + ndig);  // see ks_sum_kernel
  int terms = 0;  // jobs since the last high-word reduction (see ks_sum_kernel)
  auto fold = [&]() {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      sb[k].hi = reduce64(sb[k].hi, q, mh);
      sa[k].hi = reduce64(sa[k].hi, q, mh);
    }
    terms = 0;
  };
  int cur = next_rot(b0), st = 0;
  uint32_t phase = 0;  // bit st: parity of stage st's next completion
  if (cur < b1) issue(cur, 0, 0);
  for (int jb = b0; jb < b1; ++jb) {
    const int s = A.jsrc[jb];
    const u64 g = A.g[jb];
    if (terms >= fold_at) fold();
    if (g <= 1) {  // identity term: P * (c0, c1) on the Q primes (ext_c0: c0 on every target), from global memory
      if (!c0t) continue;
#pragma unroll
      for (int k = 0; k < E; k += 2) {
        ulonglong2 v0, v1;
        if constexpr (GATHER) {  // strided: register k holds column 32 k + lane
          const u64* a0 = A.c0[s] + (size_t)t * n + rowoff + lane;
          const u64* a1 = A.c1[s] + (size_t)t * n + rowoff + lane;
          v0 = make_ulonglong2(a0[32 * k], a0[32 * (k + 1)]);
          v1 = qt ? make_ulonglong2(a1[32 * k], a1[32 * (k + 1)]) : make_ulonglong2(0, 0);
        } else {
          v0 = *reinterpret_cast<const ulonglong2*>(A.c0[s] + (size_t)t * n + rowoff + eoff(k));
          v1 = qt ? *reinterpret_cast<const ulonglong2*>(A.c1[s] + (size_t)t * n + rowoff + eoff(k))
                  : make_ulonglong2(0, 0);
        }
        if constexpr (PM1) {
          sb[k].hi += v0.x;
          sb[k + 1].hi += v0.y;
          sa[k].hi += v1.x;
          sa[k + 1].hi += v1.y;
        } else {
          mac128(sb[k], v0.x, pm);
          mac128(sb[k + 1], v0.y, pm);
          mac128(sa[k], v1.x, pm);
          mac128(sa[k + 1], v1.y, pm);
        }
      }
      ++terms;
      continue;
    }
    const RowPerm<LOGR, LOGC> rp(rd, g);
    for (int j = 0; j < ndig; ++j) {
    // (jb, j): its rows are in (or on their way to) stage st; start the next step's copies
    if (j + 1 < ndig) {
      issue(jb, j + 1, st ^ 1);
    } else {
      const int nxt = next_rot(jb + 1);
      if (nxt < b1) issue(nxt, 0, st ^ 1);
    }
    tma1d::mbar_wait(&bars[st], (phase >> st) & 1);
    phase ^= 1u << st;
    const u64* X = stage_base + (size_t)st * kTmaRows * C;
    u64 x[E];
    // GATHER: strided registers (register k of lane L = column c = 32 k + L);
    // source column br8(base + slope br8(c)), br8(c) = br8(L) | br8(32 k): one
    // product per job, a constant per register. The 16 lanes of a half warp then
    // read 16 distinct banks (br8(c) varies in its top four bits)
    const uint32_t gb = rp.base + rp.slope * (__brev((uint32_t)lane) >> 24);
    auto src_col = [&](int k) {
      const uint32_t kb = (__brev((uint32_t)(32 * k)) >> 24);
      return __brev((gb + rp.slope * kb) & 255u) >> 24;
    };
    if constexpr (GATHER) {
#pragma unroll
      for (int k = 0; k < E; ++k) x[k] = X[src_col(k)];
    } else {
      const ShflPermQ sp(rp.base, rp.slope, lane);
#pragma unroll
      for (int k = 0; k < E; k += 2) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(X + eoff(k));
        x[k] = v.x, x[k + 1] = v.y;
      }
      sp.apply(x);
    }
#pragma unroll
    for (int k = 0; k < E; k += 2) {
      ulonglong2 kb, ka;
      if constexpr (GATHER) {
        kb = make_ulonglong2(X[C + 32 * k + lane], X[C + 32 * (k + 1) + lane]);
        ka = make_ulonglong2(X[2 * C + 32 * k + lane], X[2 * C + 32 * (k + 1) + lane]);
      } else {
        kb = *reinterpret_cast<const ulonglong2*>(X + C + eoff(k));
        ka = *reinterpret_cast<const ulonglong2*>(X + 2 * C + eoff(k));
      }
      mac128(sb[k], x[k], kb.x);
      mac128(sa[k], x[k], ka.x);
      mac128(sb[k + 1], x[k + 1], kb.y);
      mac128(sa[k + 1], x[k + 1], ka.y);
    }
    if (c0t && j == 0) {  // P * sigma_g(c0)
      if constexpr (GATHER) {
#pragma unroll
        for (int k = 0; k < E; ++k) x[k] = X[3 * C + src_col(k)];
      } else {
        const ShflPermQ sp(rp.base, rp.slope, lane);
#pragma unroll
        for (int k = 0; k < E; k += 2) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(X + 3 * C + eoff(k));
          x[k] = v.x, x[k + 1] = v.y;
        }
        sp.apply(x);
      }
#pragma unroll
      for (int k = 0; k < E; ++k) {
        if constexpr (PM1)
          sb[k].hi += x[k];
        else
          mac128(sb[k], x[k], pm);
      }
    }
    __syncwarp();  // every lane is done with stage st before lane 0 refills it
    st ^= 1;
    }
    ++terms;
  }
  u64 vb[E], va[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    vb[k] = mont_finish(sb[k], q, mh, qn);
    va[k] = mont_finish(sa[k], q, mh, qn);
  }
  u64* accb = A.acc[o] + (size_t)t * n;
  u64* acca = A.acc[o] + (size_t)(A.nt + t) * n;
  // NTT-domain stores on the Q targets; the special primes (and a merged q_top)
  // get ModDown's inverse row pass and strided stores -- except a kept b part
  const bool ntt_a = qt && t < A.inv_from, ntt_b = ntt_a || A.keep_b;
  if (ntt_b) {
#pragma unroll
    for (int k = 0; k < E; k += 2) {
      if constexpr (GATHER) {
        accb[rowoff + 32 * k + lane] = vb[k];
        accb[rowoff + 32 * (k + 1) + lane] = vb[k + 1];
      } else {
        *reinterpret_cast<ulonglong2*>(accb + rowoff + eoff(k)) = make_ulonglong2(vb[k], vb[k + 1]);
      }
    }
  }
  if (ntt_a) {
#pragma unroll
    for (int k = 0; k < E; k += 2) {
      if constexpr (GATHER) {
        acca[rowoff + 32 * k + lane] = va[k];
        acca[rowoff + 32 * (k + 1) + lane] = va[k + 1];
      } else {
        *reinterpret_cast<ulonglong2*>(acca + rowoff + eoff(k)) = make_ulonglong2(va[k], va[k + 1]);
      }
    }
  } else {
    const u64* W = T.ipsi + ((size_t)m << LOGN);
    const u64* Ws = T.ipsi_s + ((size_t)m << LOGN);
    auto tw = [&](int b, int blk, u64& w, u64& ws) {
      const int i = (1 << (LOGN - 1 - b)) + (rd << (LOGC - 1 - b)) + blk;
      w = W[i];
      ws = Ws[i];
    };
    auto restride = [&](u64 (&v)[E]) {
      if constexpr (GATHER) return;  // the registers are strided already
#pragma unroll
      for (int k = 0; k < E; ++k) buf[xp(eoff(k & ~1) + (k & 1))] = v[k];
      __syncwarp();
#pragma unroll
      for (int k = 0; k < E; ++k) v[k] = buf[xp(lane + 32 * k)];
      __syncwarp();
    };
    if (!ntt_b) {
      restride(vb);
      warp_inv<LOGC, kStrided>(vb, buf, lane, q, tw);
#pragma unroll
      for (int k = 0; k < E; ++k) accb[(size_t)rd * C + lane + 32 * k] = vb[k];
    }
    restride(va);
    warp_inv<LOGC, kStrided>(va, buf, lane, q, tw);
#pragma unroll
    for (int k = 0; k < E; ++k) acca[(size_t)rd * C + lane + 32 * k] = va[k];
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

template <int LOGR, int LOGC>
void run_row(Context& c, const LimbBatch& b, bool inverse) {
  const unsigned grid = (unsigned)b.count * ((1u << LOGR) / kWarps);
  if (inverse)
    ntt_row_pass<LOGR, LOGC, true><<<grid, kWarps * 32, 0, c.stream>>>(b, c.tabs);
  else
    ntt_row_pass<LOGR, LOGC, false><<<grid, kWarps * 32, 0, c.stream>>>(b, c.tabs);
}

template <int LOGR, int LOGC>
void run_epi(Context& c, const EpiBatch& e) {
  const unsigned grid = (unsigned)e.count * ((1u << LOGR) / kWarps);
  if (e.nomul)
    ntt_row_epi<LOGR, LOGC, true><<<grid, kWarps * 32, 0, c.stream>>>(e, c.tabs);
  else
    ntt_row_epi<LOGR, LOGC, false><<<grid, kWarps * 32, 0, c.stream>>>(e, c.tabs);
}

template <int LOGR, int LOGC, int TCF, int CPW>
void run_fused_t(Context& c, const FusedColArgs& a) {
  constexpr int R = 1 << LOGR;
  const size_t sm = (size_t)(a.ns + 1) * TCF * (R + 2) * sizeof(u64);
  static int configured = 0;
  if (!configured) {
    SF_CUDA(cudaFuncSetAttribute(fused_col_kernel<LOGR, LOGC, TCF, CPW, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    SF_CUDA(cudaFuncSetAttribute(fused_col_kernel<LOGR, LOGC, TCF, CPW, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = 1;
  }
  require(sm <= 200 * 1024, kInternal, "fused column stage: too many source limbs for shared memory");
  const int dpc = a.d_per_cta > 0 ? a.d_per_cta : a.nd;
  const unsigned grid = (unsigned)a.count * ((a.nd + dpc - 1) / dpc) * ((1u << LOGC) / TCF);
  // per-warp conversion into registers for the batched 8-column CTAs (-4% family
  // time); the 2-column single-ciphertext CTAs keep the block-wide conversion
  // (measured faster there: 1.49 vs 1.69 ms/step); SF_VARIANT bit 4 forces it everywhere
  if ((c.variant & 16) || TCF < 8)
    fused_col_kernel<LOGR, LOGC, TCF, CPW, false><<<grid, TCF / CPW * 32, sm, c.stream>>>(a, c.tabs);
  else
    fused_col_kernel<LOGR, LOGC, TCF, CPW, true><<<grid, TCF / CPW * 32, sm, c.stream>>>(a, c.tabs);
}

template <int LOGR, int LOGC>
void run_fused(Context& c, const FusedColArgs& a) {
  if ((size_t)a.count * ((1u << LOGC) / 8) >= 444) {
    if (c.fused_cpw == 2 && (1 << LOGC) >= 16)
      run_fused_t<LOGR, LOGC, 16, 2>(c, a);
    else if (c.fused_cpw == 4)  // A/B: 4-column, 4-warp CTAs
      run_fused_t<LOGR, LOGC, 4, 1>(c, a);
    else
      run_fused_t<LOGR, LOGC, 8, 1>(c, a);
    return;
  }
  // small launch (single ciphertexts): 2-column CTAs, and the destinations
  // spread over CTAs (each recomputes the few source inverse transforms) so the
  // chain of per-destination transforms does not serialise inside one warp
  FusedColArgs b = a;
  b.d_per_cta = 1;
  run_fused_t<LOGR, LOGC, 2, 1>(c, b);
}

template <int LOGR, int LOGC>
void run_ks_row(Context& c, const KsRowArgs& a) {
  constexpr int C = 1 << LOGC;
  const size_t sm = (size_t)kWarps * (a.ndig + 1) * C * sizeof(u64);
  static int configured = 0;
  if (!configured) {
    SF_CUDA(cudaFuncSetAttribute(ks_row_kernel<LOGR, LOGC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 200 * 1024));
    configured = 1;
  }
  require(sm <= 200 * 1024, kInternal, "key-switch row stage: too many digits for shared memory");
  const unsigned grid = (unsigned)(a.nsrc * a.nt * ((1 << LOGR) / kWarps));
  ks_row_kernel<LOGR, LOGC><<<grid, kWarps * 32, sm, c.stream>>>(a, c.tabs);
}

template <int LOGR, int LOGC>
void run_ks_sum(Context& c, const KsSumArgs& a) {
  if constexpr (LOGC == 8) {
    // the TMA-pipelined row stage, one (job, digit) step per stage (SF_VARIANT bit 6:
    // ks_sum_kernel, for A/B; bit 11: TMA for single-digit sums only)
    if ((a.ndig == 1 || !(c.variant & 2048)) && !(c.variant & 64)) {
      constexpr size_t sm = (size_t)kTmaWarps * (2 * kTmaRows + 1) * 256 * sizeof(u64) + kTmaWarps * 2 * sizeof(u64);
      static bool attr = false;
      if (!attr) {
        SF_CUDA(cudaFuncSetAttribute(ks_sum_tma_kernel<LOGR, true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        SF_CUDA(cudaFuncSetAttribute(ks_sum_tma_kernel<LOGR, false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        SF_CUDA(cudaFuncSetAttribute(ks_sum_tma_kernel<LOGR, true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        SF_CUDA(cudaFuncSetAttribute(ks_sum_tma_kernel<LOGR, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        SF_CUDA(cudaFuncSetAttribute(ks_sum_tma_kernel<LOGR, true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        SF_CUDA(cudaFuncSetAttribute(ks_sum_tma_kernel<LOGR, false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        attr = true;
      }
      const unsigned grid = (unsigned)(a.nout * a.nt * ((1 << LOGR) / kTmaWarps));
      // SF_VARIANT bit 10: the shuffle-network automorphism instead of the shared-memory gather (A/B)
      const bool gather = !(c.variant & 1024);
      const dim3 blk(kTmaWarps * 32);
      if (a.ndig == 1) {
        if (a.pm_one && gather)
          ks_sum_tma_kernel<LOGR, true, true, true><<<grid, blk, sm, c.stream>>>(a, c.tabs);
        else if (a.pm_one)
          ks_sum_tma_kernel<LOGR, true, false, true><<<grid, blk, sm, c.stream>>>(a, c.tabs);
        else if (gather)
          ks_sum_tma_kernel<LOGR, false, true, true><<<grid, blk, sm, c.stream>>>(a, c.tabs);
        else
          ks_sum_tma_kernel<LOGR, false, false, true><<<grid, blk, sm, c.stream>>>(a, c.tabs);
      } else if (a.pm_one) {
        ks_sum_tma_kernel<LOGR, true, true, false><<<grid, blk, sm, c.stream>>>(a, c.tabs);
      } else {
        ks_sum_tma_kernel<LOGR, false, true, false><<<grid, blk, sm, c.stream>>>(a, c.tabs);
      }
      return;
    }
  }
  const unsigned grid = (unsigned)(a.nout * a.nt * ((1 << LOGR) / kWarps));
  // default: automorphism gather by warp shuffles (-2% family time vs shared-memory staging);
  // SF_VARIANT bit 3: shared-memory staging with the key loads issued first (-4% vs bit 0:
  // key words loaded after the row is staged)
  if (a.pm_one)
    ks_sum_kernel<LOGR, LOGC, true, true, true><<<grid, kWarps * 32, 0, c.stream>>>(a, c.tabs);
  else if (c.variant & 1)
    ks_sum_kernel<LOGR, LOGC, false, false, false><<<grid, kWarps * 32, 0, c.stream>>>(a, c.tabs);
  else if (c.variant & 8)
    ks_sum_kernel<LOGR, LOGC, true, false, false><<<grid, kWarps * 32, 0, c.stream>>>(a, c.tabs);
  else
    ks_sum_kernel<LOGR, LOGC, true, true, false><<<grid, kWarps * 32, 0, c.stream>>>(a, c.tabs);
}

#define SF_NTT_DISPATCH(FN, ...)                        \
  switch (c.logn) {                                     \
    case 12: FN<6, 6>(c, __VA_ARGS__); return true;     \
    case 13: FN<6, 7>(c, __VA_ARGS__); return true;     \
    case 14: FN<7, 7>(c, __VA_ARGS__); return true;     \
    case 15: FN<7, 8>(c, __VA_ARGS__); return true;     \
    case 16: FN<8, 8>(c, __VA_ARGS__); return true;     \
    case 17: FN<8, 9>(c, __VA_ARGS__); return true;     \
    default: return false;                              \
  }

}  // namespace

bool ntt_two_pass(Context& c, const LimbBatch& b, bool inverse) { SF_NTT_DISPATCH(run_two_pass, b, inverse) }
bool ntt_row_only(Context& c, const LimbBatch& b, bool inverse) { SF_NTT_DISPATCH(run_row, b, inverse) }
bool ntt_row_epi(Context& c, const EpiBatch& e) { SF_NTT_DISPATCH(run_epi, e) }
bool ntt_fused_col(Context& c, const FusedColArgs& a) { SF_NTT_DISPATCH(run_fused, a) }
bool ntt_ks_row(Context& c, const KsRowArgs& a) { SF_NTT_DISPATCH(run_ks_row, a) }
bool ntt_ks_sum(Context& c, const KsSumArgs& a) { SF_NTT_DISPATCH(run_ks_sum, a) }

}  // namespace sf
