// Batched elementwise / basis-conversion / key-switch kernels.
//
// Each launch processes up to kJobs independent jobs (ciphertexts, key
// switches) whose device pointers travel in the kernel parameter block
// (CUDA 12.1+ allows 32 KB of parameters). grid.y indexes the job, grid.x
// strides over limbs x coefficients with 16-byte vector accesses where the
// layout allows. This turns the thousands of per-ciphertext operations of an
// attention decode step (256 K ciphertexts, 510 V handles, 2.5k rotations)
// into a few hundred full-GPU launches.
#include <algorithm>

#include "batch.cuh"
#include "modarith.cuh"

namespace sf {
namespace {

constexpr int kT = 256;

inline void post(Context& c) {
  c.launches.fetch_add(1, std::memory_order_relaxed);
  SF_CUDA(cudaGetLastError());
}

// butterflies of one half (row or column pass) of a limb NTT: n/2 per stage
inline double half_bfly(const Context& c, bool column) {
  const int logr = c.logn / 2, logc = c.logn - logr;
  return 0.5 * c.n * (column ? logr : logc);
}

inline dim3 grid2(size_t per_job_threads, int jobs) {
  size_t bx = (per_job_threads + kT - 1) / kT;
  if (bx > 2048) bx = 2048;
  return dim3((unsigned)(bx ? bx : 1), (unsigned)jobs);
}

__device__ __forceinline__ uint32_t brev_(uint32_t x, int logn) { return __brev(x) >> (32 - logn); }
__device__ __forceinline__ uint32_t perm_(uint32_t i, u64 g, int logn) {
  const u64 e = 2ull * brev_(i, logn) + 1;
  const u64 e2 = (e * g) & ((2ull << logn) - 1);
  return brev_((uint32_t)((e2 - 1) >> 1), logn);
}

// ------------------------------------------------------------------ kernels
__global__ void copy_batch_kernel(CopyBatch B, size_t words) {
  const int j = blockIdx.y;
  const ulonglong2* s = reinterpret_cast<const ulonglong2*>(B.src[j]);
  ulonglong2* d = reinterpret_cast<ulonglong2*>(B.dst[j]);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words / 2; i += (size_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}

__global__ void add_batch_kernel(AddBatch B, int limbs, int n, const u64* Q) {
  const int j = blockIdx.y;
  const size_t half = (size_t)limbs * n / 2;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < 2 * half; v += (size_t)gridDim.x * blockDim.x) {
    const int poly = v >= half;
    const size_t w = v - poly * half;
    const int l = (int)((w * 2) / n);
    const u64 q = Q[l];
    const ulonglong2 x = reinterpret_cast<const ulonglong2*>(poly ? B.a1[j] : B.a0[j])[w];
    const ulonglong2 y = reinterpret_cast<const ulonglong2*>(poly ? B.b1[j] : B.b0[j])[w];
    ulonglong2 z;
    z.x = B.sub ? sub_mod(x.x, y.x, q) : add_mod(x.x, y.x, q);
    z.y = B.sub ? sub_mod(x.y, y.y, q) : add_mod(x.y, y.y, q);
    reinterpret_cast<ulonglong2*>(poly ? B.o1[j] : B.o0[j])[w] = z;
  }
}

__global__ void sum_kernel(SumArgs A, int limbs, int n, const u64* Q) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * total; i += (size_t)gridDim.x * blockDim.x) {
    const int poly = i >= total;
    const size_t w = i - poly * total;
    const int l = (int)(w / n);
    const u64 q = Q[l];
    u64 acc = 0;
    for (int k = 0; k < A.k; ++k) acc = add_mod(acc, (poly ? A.in1[k] : A.in0[k])[w], q);
    (poly ? A.out1 : A.out0)[w] = acc;
  }
}

__global__ void sum_multi_kernel(SumMultiArgs A, int limbs, int n, const u64* Q) {
  const int o = blockIdx.y;
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * total; i += (size_t)gridDim.x * blockDim.x) {
    const int poly = i >= total;
    const size_t w = i - poly * total;
    const u64 q = Q[w / n];
    u64 acc = 0;
    for (int k = A.begin[o]; k < A.begin[o + 1]; ++k) acc = add_mod(acc, (poly ? A.in1[k] : A.in0[k])[w], q);
    (poly ? A.out1[o] : A.out0[o])[w] = acc;
  }
}

__global__ void mulpt_batch_kernel(MulPtBatch B, int limbs, int n, const u64* Q, const u64* MH, const u64* ML) {
  const int j = blockIdx.y;
  const size_t total = (size_t)limbs * n;
  if (const u64* cs = B.cs[j]) {  // shared ciphertext: Shoup products, two coefficients per thread
    for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 2; i < total;
         i += (size_t)gridDim.x * blockDim.x * 2) {
      const u64 q = Q[i / n];
      const ulonglong2 p = *reinterpret_cast<const ulonglong2*>(B.pt[j] + i);
      const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(B.c0[j] + i);
      const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(B.c1[j] + i);
      const ulonglong2 w0 = *reinterpret_cast<const ulonglong2*>(cs + i);
      const ulonglong2 w1 = *reinterpret_cast<const ulonglong2*>(cs + total + i);
      *reinterpret_cast<ulonglong2*>(B.o0[j] + i) =
          make_ulonglong2(mul_shoup(p.x, x0.x, w0.x, q), mul_shoup(p.y, x0.y, w0.y, q));
      *reinterpret_cast<ulonglong2*>(B.o1[j] + i) =
          make_ulonglong2(mul_shoup(p.x, x1.x, w1.x, q), mul_shoup(p.y, x1.y, w1.y, q));
    }
    return;
  }
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const u64 p = B.pt[j][i];
    B.o0[j][i] = mulmod(B.c0[j][i], p, Q[l], MH[l], ML[l]);
    B.o1[j][i] = mulmod(B.c1[j][i], p, Q[l], MH[l], ML[l]);
  }
}

// Shoup companions floor(a 2^64 / q) of `polys` polynomials of `limbs` limbs (contiguous)
__global__ void shoup_companion_kernel(const u64* a, u64* out, int limbs, int n, int polys, const u64* Q) {
  const size_t total = (size_t)polys * limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const u64 q = Q[(i / n) % limbs];
    out[i] = (u64)(((unsigned __int128)a[i] << 64) / q);
  }
}

// the shared-a form: d0 = b0 a0, d1 = b0 a1 + b1 a0, d2 = b1 a1 as Shoup products
// (a's companions precomputed once for the batch); two coefficients per thread
__global__ void tensor_shared_kernel(TensorBatch B, int limbs, int n, const u64* Q) {
  const int j = blockIdx.y;
  const size_t total = (size_t)limbs * n;
  const u64* a0s = B.as;
  const u64* a1s = B.as + total;
  for (size_t i = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) * 2; i < total;
       i += (size_t)gridDim.x * blockDim.x * 2) {
    const u64 q = Q[i / n];
    const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(B.a0[j] + i);
    const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(B.a1[j] + i);
    const ulonglong2 w0 = *reinterpret_cast<const ulonglong2*>(a0s + i);
    const ulonglong2 w1 = *reinterpret_cast<const ulonglong2*>(a1s + i);
    const ulonglong2 y0 = *reinterpret_cast<const ulonglong2*>(B.b0[j] + i);
    const ulonglong2 y1 = *reinterpret_cast<const ulonglong2*>(B.b1[j] + i);
    *reinterpret_cast<ulonglong2*>(B.d0[j] + i) =
        make_ulonglong2(mul_shoup(y0.x, x0.x, w0.x, q), mul_shoup(y0.y, x0.y, w0.y, q));
    *reinterpret_cast<ulonglong2*>(B.d1[j] + i) =
        make_ulonglong2(add_mod(mul_shoup(y1.x, x0.x, w0.x, q), mul_shoup(y0.x, x1.x, w1.x, q), q),
                        add_mod(mul_shoup(y1.y, x0.y, w0.y, q), mul_shoup(y0.y, x1.y, w1.y, q), q));
    *reinterpret_cast<ulonglong2*>(B.d2[j] + i) =
        make_ulonglong2(mul_shoup(y1.x, x1.x, w1.x, q), mul_shoup(y1.y, x1.y, w1.y, q));
  }
}

__global__ void tensor_batch_kernel(TensorBatch B, int limbs, int n, const u64* Q, const u64* MH, const u64* ML) {
  const int j = blockIdx.y;
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const u64 q = Q[l], mh = MH[l], ml = ML[l];
    const u64 x0 = B.a0[j][i], x1 = B.a1[j][i], y0 = B.b0[j][i], y1 = B.b1[j][i];
    B.d0[j][i] = mulmod(x0, y0, q, mh, ml);
    U128 m{0, 0};
    mac128(m, x0, y1);
    mac128(m, x1, y0);
    B.d1[j][i] = reduce128(m.hi, m.lo, q, mh, ml);
    B.d2[j][i] = mulmod(x1, y1, q, mh, ml);
  }
}

// Lazily relinearised sum of ct x ct products (Score*V): 128-bit accumulation,
// folded back to a residue every 16 terms (16 * 2 * q^2 < 2^127 for q < 2^61).
__global__ void tensor_sum_kernel(TensorSumArgs A, int limbs, int n, const u64* Q, const u64* MH, const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const u64 q = Q[l], mh = MH[l], ml = ML[l];
    U128 s0{A.accumulate ? A.d0[i] : 0, 0}, s1{A.accumulate ? A.d1[i] : 0, 0}, s2{A.accumulate ? A.d2[i] : 0, 0};
    for (int k = 0; k < A.k; ++k) {
      const u64 x0 = A.a0[k][i], x1 = A.a1[k][i], y0 = A.b0[k][i], y1 = A.b1[k][i];
      mac128(s0, x0, y0);
      mac128(s1, x0, y1);
      mac128(s1, x1, y0);
      mac128(s2, x1, y1);
      if ((k & 15) == 15) {
        s0 = {reduce128(s0.hi, s0.lo, q, mh, ml), 0};
        s1 = {reduce128(s1.hi, s1.lo, q, mh, ml), 0};
        s2 = {reduce128(s2.hi, s2.lo, q, mh, ml), 0};
      }
    }
    A.d0[i] = reduce128(s0.hi, s0.lo, q, mh, ml);
    A.d1[i] = reduce128(s1.hi, s1.lo, q, mh, ml);
    A.d2[i] = reduce128(s2.hi, s2.lo, q, mh, ml);
  }
}

// One block = 128 threads x 2 adjacent coefficients of one limb (16-byte loads);
// the block walks all outputs, so the operands shared between outputs stay in L1.
__global__ void __launch_bounds__(128) tensor_sum_multi_kernel(TensorSumMultiArgs A, int limbs, int n, const u64* Q,
                                                              const u64* MH, const u64* ML) {
  const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i >= (size_t)limbs * n) return;
  const int l = (int)(i / n);
  const u64 q = Q[l], mh = MH[l], ml = ML[l];
  for (int o = 0; o < A.nout; ++o) {
    U128 s0[2] = {{0, 0}, {0, 0}}, s1[2] = {{0, 0}, {0, 0}}, s2[2] = {{0, 0}, {0, 0}};
    for (int k = A.begin[o], c = 0; k < A.begin[o + 1]; ++k, ++c) {
      const ulonglong2 x0 = *reinterpret_cast<const ulonglong2*>(A.a0[k] + i);
      const ulonglong2 x1 = *reinterpret_cast<const ulonglong2*>(A.a1[k] + i);
      const ulonglong2 y0 = *reinterpret_cast<const ulonglong2*>(A.b0[k] + i);
      const ulonglong2 y1 = *reinterpret_cast<const ulonglong2*>(A.b1[k] + i);
      mac128(s0[0], x0.x, y0.x);
      mac128(s1[0], x0.x, y1.x);
      mac128(s1[0], x1.x, y0.x);
      mac128(s2[0], x1.x, y1.x);
      mac128(s0[1], x0.y, y0.y);
      mac128(s1[1], x0.y, y1.y);
      mac128(s1[1], x1.y, y0.y);
      mac128(s2[1], x1.y, y1.y);
      if ((c & 15) == 15) {  // 16 * 2 * q^2 < 2^127 for q < 2^61
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          s0[h] = {reduce128(s0[h].hi, s0[h].lo, q, mh, ml), 0};
          s1[h] = {reduce128(s1[h].hi, s1[h].lo, q, mh, ml), 0};
          s2[h] = {reduce128(s2[h].hi, s2[h].lo, q, mh, ml), 0};
        }
      }
    }
    *reinterpret_cast<ulonglong2*>(A.d0[o] + i) =
        make_ulonglong2(reduce128(s0[0].hi, s0[0].lo, q, mh, ml), reduce128(s0[1].hi, s0[1].lo, q, mh, ml));
    *reinterpret_cast<ulonglong2*>(A.d1[o] + i) =
        make_ulonglong2(reduce128(s1[0].hi, s1[0].lo, q, mh, ml), reduce128(s1[1].hi, s1[1].lo, q, mh, ml));
    *reinterpret_cast<ulonglong2*>(A.d2[o] + i) =
        make_ulonglong2(reduce128(s2[0].hi, s2[0].lo, q, mh, ml), reduce128(s2[1].hi, s2[1].lo, q, mh, ml));
  }
}

__global__ void lift_batch_kernel(LiftBatch B, int limbs, int n, u64 ql, const u64* Q, const u64* MH) {
  const int j = blockIdx.y;
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const size_t k = i - (size_t)l * n;
    const u64 q = Q[l];
    const u64 v = B.x[j][k];
    const u64 r = reduce64(v, q, MH[l]);
    B.out[j][i] = v > (ql >> 1) ? sub_mod(r, reduce64(ql, q, MH[l]), q) : r;
  }
}

__global__ void conv_batch_kernel(ConvBatch A, const u64* Q, const u64* MH, const u64* ML) {
  const int j = blockIdx.y;
  const int n = A.n;
  const u64* in = A.in[j];
  u64* out = A.out[j];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    u64 y[kMaxPrimes];
#pragma unroll 4
    for (int i = 0; i < A.nsrc; ++i)
      y[i] = mul_shoup(in[(size_t)i * n + k], A.qinv[i], A.qinv_s[i], Q[A.src_prime[i]]);
    for (int d = 0; d < A.ndst; ++d) {
      U128 acc{0, 0};
      const u64* h = A.qhat + d;
      for (int i = 0; i < A.nsrc; ++i) mac128(acc, y[i], h[(size_t)i * A.ndst]);
      const int pd = A.dst_prime[d];
      out[(size_t)A.out_slot[d] * n + k] = reduce128(acc.hi, acc.lo, Q[pd], MH[pd], ML[pd]);
    }
  }
}

__global__ void ks_batch_kernel(KsBatch A, const u64* Q, const u64* MH, const u64* ML) {
  const int j = blockIdx.y;
  const int n = 1 << A.logn;
  const size_t total = (size_t)A.nt * n;
  const u64 g = A.g[j];
  const u64* ext = A.ext[j];
  const u64* key = A.key[j];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i >> A.logn);
    const uint32_t k = (uint32_t)(i & (n - 1));
    const uint32_t src = g > 1 ? perm_(k, g, A.logn) : k;
    const int m = A.tprime[t];
    U128 sb{0, 0}, sa{0, 0};
    for (int d = 0; d < A.ndig; ++d) {
      const u64 x = ext[((size_t)d * A.nt + t) * n + src];
      const u64* kb = key + (((size_t)d * 2 + 0) * A.np + m) * n;
      const u64* ka = key + (((size_t)d * 2 + 1) * A.np + m) * n;
      mac128(sb, x, kb[k]);
      mac128(sa, x, ka[k]);
    }
    A.accb[j][i] = reduce128(sb.hi, sb.lo, Q[m], MH[m], ML[m]);
    A.acca[j][i] = reduce128(sa.hi, sa.lo, Q[m], MH[m], ML[m]);
  }
}

__global__ void subscale_batch_kernel(SubScaleBatch B, int limbs, int logn, const u64* inv, const u64* inv_s,
                                      const u64* Q) {
  const int j = blockIdx.y;
  const int n = 1 << logn;
  const size_t total = (size_t)limbs * n;
  const u64 g = B.g[j];
  const u64* addend = B.addend[j];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i >> logn);
    const u64 q = Q[l];
    u64 v = mul_shoup(sub_mod(B.acc[j][i], B.conv[j][i], q), inv[l], inv_s[l], q);
    if (addend) {
      const uint32_t k = (uint32_t)(i & (n - 1));
      const uint32_t src = g > 1 ? perm_(k, g, logn) : k;
      v = add_mod(v, addend[((size_t)l << logn) + src], q);
    }
    B.out[j][i] = v;
  }
}

// Fused VMM multiply-accumulate over ALL giant steps (vmm.cpp:210-219):
// partial[g2] = sum_g1 baby[g1] (.) pt[g2*b + g1], lazily reduced once.
// A CTA owns 64 coefficients of one limb: it stages the b babies' (c0, c1)
// words for those coefficients in shared memory once, then each warp streams
// the plaintext diagonals of its giants (16-byte loads, 512 B per warp row).
// D > 0: each lane streams its 16-byte share of the diagonal tiles through a
// private D+1-slot shared-memory ring with cp.async (no registers held by the
// in-flight loads; every lane reads back only what it copied, so no barrier).
template <int D>
__global__ void vmm_mac_kernel(VmmMacArgs A, const u64* Q, const u64* MH, const u64* ML) {
  extern __shared__ u64 sb[];  // [b][2][64] babies, then (D > 0) [warps][D + 1][64] diagonal ring
  const int n = A.n;
  const int tiles_per_limb = n / 64;
  const int l = blockIdx.x / tiles_per_limb;
  const int k0 = (blockIdx.x - l * tiles_per_limb) * 64;
  const size_t base = (size_t)l * n + k0;
  for (int e = threadIdx.x; e < A.b * 2 * 64; e += blockDim.x) {
    const int g1 = e / 128, rem = e - g1 * 128, poly = rem >> 6, kk = rem & 63;
    sb[e] = (poly ? A.baby1[g1] : A.baby0[g1])[base + kk];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const u64 q = Q[l], mh = MH[l], ml = ML[l];
  for (int g2 = warp; g2 < A.giants; g2 += nw) {
    U128 a0{0, 0}, a1{0, 0}, b0{0, 0}, b1{0, 0};
    const int gbase = A.gidx[g2] * A.b;
    const int cnt = min(A.b, A.k - gbase);
    u64* ring = sb + (size_t)A.b * 128 + (size_t)warp * (D + 1) * 64;
    auto issue = [&](int g1) {
      if (g1 < cnt) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(ring + (g1 % (D + 1)) * 64 + 2 * lane);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(A.pt[gbase + g1] + base + 2 * lane)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if constexpr (D > 0)
      for (int u = 0; u < D; ++u) issue(u);
    for (int g1 = 0; g1 < cnt; ++g1) {
      ulonglong2 p;
      if constexpr (D > 0) {
        issue(g1 + D);
        asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory");
        p = reinterpret_cast<const ulonglong2*>(ring + (g1 % (D + 1)) * 64)[lane];
      } else {
        p = reinterpret_cast<const ulonglong2*>(A.pt[gbase + g1] + base)[lane];
      }
      const u64* s = sb + g1 * 128;
      mac128(a0, s[2 * lane], p.x);
      mac128(b0, s[2 * lane + 1], p.y);
      mac128(a1, s[64 + 2 * lane], p.x);
      mac128(b1, s[64 + 2 * lane + 1], p.y);
    }
    ulonglong2 r0, r1;
    r0.x = reduce128(a0.hi, a0.lo, q, mh, ml);
    r0.y = reduce128(b0.hi, b0.lo, q, mh, ml);
    r1.x = reduce128(a1.hi, a1.lo, q, mh, ml);
    r1.y = reduce128(b1.hi, b1.lo, q, mh, ml);
    reinterpret_cast<ulonglong2*>(A.out0[g2] + base)[lane] = r0;
    reinterpret_cast<ulonglong2*>(A.out1[g2] + base)[lane] = r1;
  }
}

__global__ void axpy_pm_kernel(AxpyBatch B, int limbs, int logn, const u64* pm, const u64* Q, const u64* MH,
                               const u64* ML) {
  const int j = blockIdx.y;
  const size_t total = (size_t)limbs << logn;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i >> logn);
    const u64 q = Q[l];
    B.acc[j][i] = add_mod(B.acc[j][i], mulmod(B.d[j][i], pm[l], q, MH[l], ML[l]), q);
  }
}

// Rotation-sum inner products for ring degrees without the two-pass kernels:
// one thread per (output, extended limb, coefficient), every limb written in
// the NTT domain (the generic ModDown follows).
__global__ void ks_sum_generic_kernel(KsSumArgs A, const u64* Q, const u64* MH, const u64* ML, int logn) {
  const int o = blockIdx.y;
  const int n = 1 << logn;
  const size_t total = (size_t)A.nt * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i >> logn);
    const uint32_t k = (uint32_t)(i & (n - 1));
    const int m = A.tprime[t];
    const u64 q = Q[m], mh = MH[m], ml = ML[m];
    const bool qt = t < A.limbs;
    U128 sb{0, 0}, sa{0, 0};
    int terms = 0;
    for (int jb = A.out_begin[o]; jb < A.out_begin[o + 1]; ++jb) {
      if (terms > 200) {
        sb = U128{reduce128(sb.hi, sb.lo, q, mh, ml), 0};
        sa = U128{reduce128(sa.hi, sa.lo, q, mh, ml), 0};
        terms = 0;
      }
      const int s = A.jsrc[jb];
      const u64 g = A.g[jb];
      if (g <= 1) {
        if (qt) {
          mac128(sb, A.c0[s][(size_t)t * n + k], A.pm[t]);
          mac128(sa, A.c1[s][(size_t)t * n + k], A.pm[t]);
          ++terms;
        }
        continue;
      }
      const uint32_t src = perm_(k, g, logn);
      for (int j = 0; j < A.ndig; ++j) {
        const int lo = j * A.alpha, hi = min(lo + A.alpha, A.limbs);
        const u64 x = (t >= lo && t < hi) ? A.c1[s][(size_t)t * n + src] : A.ext[s][((size_t)j * A.nt + t) * n + src];
        mac128(sb, x, A.key[jb][((size_t)(j * 2 + 0) * A.np + m) * n + k]);
        mac128(sa, x, A.key[jb][((size_t)(j * 2 + 1) * A.np + m) * n + k]);
      }
      if (qt) mac128(sb, A.c0[s][(size_t)t * n + src], A.pm[t]);
      terms += A.ndig + 1;
    }
    A.acc[o][i] = reduce128(sb.hi, sb.lo, q, mh, ml);
    A.acc[o][total + i] = reduce128(sa.hi, sa.lo, q, mh, ml);
  }
}

}  // namespace

// --------------------------------------------------------------------- wrappers
void b_copy(Context& c, const CopyBatch& B, size_t words) {
  SF_HPROF("b_copy");
  if (!B.count) return;
  ProfScope prof(c, kFamElem, 16.0 * words * B.count);
  copy_batch_kernel<<<grid2(words / 2, B.count), kT, 0, c.stream>>>(B, words);
  post(c);
}

void b_add(Context& c, const AddBatch& B, int limbs) {
  SF_HPROF("b_add");
  if (!B.count) return;
  ProfScope prof(c, kFamElem, 48.0 * limbs * c.n * B.count);
  add_batch_kernel<<<grid2((size_t)limbs * c.n, B.count), kT, 0, c.stream>>>(B, limbs, c.n, c.tabs.q);
  post(c);
}

void b_sum(Context& c, const SumArgs& A, int limbs) {
  SF_HPROF("b_sum");
  ProfScope prof(c, kFamElem, 16.0 * limbs * c.n * (A.k + 1));
  sum_kernel<<<grid2((size_t)limbs * c.n * 2, 1), kT, 0, c.stream>>>(A, limbs, c.n, c.tabs.q);
  post(c);
}

void b_sum_multi(Context& c, const SumMultiArgs& A, int limbs) {
  SF_HPROF("b_sum_multi");
  if (!A.nout) return;
  ProfScope prof(c, kFamElem, 16.0 * limbs * c.n * (A.begin[A.nout] + A.nout));
  sum_multi_kernel<<<grid2((size_t)limbs * c.n * 2, A.nout), kT, 0, c.stream>>>(A, limbs, c.n, c.tabs.q);
  post(c);
}

void b_mulpt(Context& c, const MulPtBatch& B, int limbs) {
  SF_HPROF("b_mulpt");
  if (!B.count) return;
  ProfScope prof(c, kFamMac, 40.0 * limbs * c.n * B.count);
  mulpt_batch_kernel<<<grid2((size_t)limbs * c.n, B.count), kT, 0, c.stream>>>(B, limbs, c.n, c.tabs.q, c.tabs.mh,
                                                                                c.tabs.ml);
  post(c);
}

void b_tensor(Context& c, const TensorBatch& B, int limbs) {
  SF_HPROF("b_tensor");
  if (!B.count) return;
  ProfScope prof(c, kFamElem, 56.0 * limbs * c.n * B.count);
  if (B.as)
    tensor_shared_kernel<<<grid2((size_t)limbs * c.n / 2, B.count), kT, 0, c.stream>>>(B, limbs, c.n, c.tabs.q);
  else
    tensor_batch_kernel<<<grid2((size_t)limbs * c.n, B.count), kT, 0, c.stream>>>(B, limbs, c.n, c.tabs.q,
                                                                                    c.tabs.mh, c.tabs.ml);
  post(c);
}

void b_shoup_companion(Context& c, const u64* a, u64* out, int limbs, int polys) {
  SF_HPROF("b_shoup_companion");
  shoup_companion_kernel<<<grid2((size_t)polys * limbs * c.n, 1), kT, 0, c.stream>>>(a, out, limbs, c.n, polys,
                                                                                      c.tabs.q);
  post(c);
}

// One NTT row pass moves 8n bytes in and 8n out per limb; the fused column
// stage reads ns and writes nd limbs (its transforms stay in shared memory).
void b_row(Context& c, const LimbBatch& b, bool inverse) {
  SF_HPROF("b_row");
  if (!b.count) return;
  ProfScope prof(c, kFamNtt, 16.0 * c.n * b.count, half_bfly(c, false) * b.count);
  ntt_row_only(c, b, inverse);
  post(c);
}

void b_fused_col(Context& c, const FusedColArgs& A) {
  SF_HPROF("b_fused_col");
  if (!A.count) return;
  ProfScope prof(c, kFamConv, 8.0 * c.n * (A.ns + A.nd) * A.count, half_bfly(c, true) * (A.ns + A.nd) * A.count);
  ntt_fused_col(c, A);
  post(c);
}

void b_row_epi(Context& c, const EpiBatch& E) {
  SF_HPROF("b_row_epi");
  if (!E.count) return;
  // row pass in + acc + addend + out
  double bytes = 0;
  for (int i = 0; i < E.count; ++i) bytes += 8.0 * c.n * (E.addend[i] ? 4 : 3);
  ProfScope prof(c, kFamNtt, bytes, half_bfly(c, false) * E.count);
  ntt_row_epi(c, E);
  post(c);
}

void b_tensor_sum(Context& c, const TensorSumArgs& A, int limbs) {
  SF_HPROF("b_tensor_sum");
  ProfScope prof(c, kFamMac, 8.0 * limbs * c.n * (4.0 * A.k + 3));
  tensor_sum_kernel<<<grid2((size_t)limbs * c.n, 1), kT, 0, c.stream>>>(A, limbs, c.n, c.tabs.q, c.tabs.mh,
                                                                        c.tabs.ml);
  post(c);
}

void b_tensor_sum_multi(Context& c, const TensorSumMultiArgs& A, int limbs) {
  SF_HPROF("b_tensor_sum_multi");
  if (!A.nout) return;
  ProfScope prof(c, kFamMac, 8.0 * limbs * c.n * (4.0 * A.begin[A.nout] + 3.0 * A.nout));
  const size_t threads = (size_t)limbs * c.n / 2;
  tensor_sum_multi_kernel<<<(unsigned)((threads + 127) / 128), 128, 0, c.stream>>>(A, limbs, c.n, c.tabs.q,
                                                                                    c.tabs.mh, c.tabs.ml);
  post(c);
}

void b_lift(Context& c, const LiftBatch& B, int limbs, int last_prime) {
  SF_HPROF("b_lift");
  if (!B.count) return;
  ProfScope prof(c, kFamElem, 8.0 * c.n * (limbs + 1) * B.count);
  lift_batch_kernel<<<grid2((size_t)limbs * c.n, B.count), kT, 0, c.stream>>>(B, limbs, c.n, c.primes[last_prime],
                                                                                c.tabs.q, c.tabs.mh);
  post(c);
}

void b_conv(Context& c, const ConvBatch& A) {
  SF_HPROF("b_conv");
  if (!A.count) return;
  ProfScope prof(c, kFamConv, 8.0 * c.n * (A.nsrc + A.ndst) * A.count);
  conv_batch_kernel<<<grid2(c.n, A.count), kT, 0, c.stream>>>(A, c.tabs.q, c.tabs.mh, c.tabs.ml);
  post(c);
}

void b_ks(Context& c, const KsBatch& A) {
  SF_HPROF("b_ks");
  if (!A.count) return;
  // ext (one read per job) + key (2 polys per digit) + 2 outputs
  ProfScope prof(c, kFamKs, 8.0 * c.n * ((double)A.ndig * A.nt * 3 + 2.0 * A.nt) * A.count);
  ks_batch_kernel<<<grid2((size_t)A.nt * c.n, A.count), kT, 0, c.stream>>>(A, c.tabs.q, c.tabs.mh, c.tabs.ml);
  post(c);
}

void b_ks_row(Context& c, const KsRowArgs& A) {
  SF_HPROF("b_ks_row");
  if (!A.nsrc) return;
  // sources: ndig rows per target; jobs: 2 key rows per digit + 2 outputs per target
  const double jobs = A.job_begin[A.nsrc];
  // row NTTs: every non-own digit row of every unit and target; two inverse rows per job and special prime
  double rows = 0;
  for (int t = 0; t < A.nt; ++t)
    for (int j = 0; j < A.ndig; ++j) {
      const int lo = j * A.alpha, hi = std::min(lo + A.alpha, A.limbs);
      if (!(t >= lo && t < hi)) rows += A.nsrc;
    }
  rows += jobs * 2.0 * (A.nt - A.limbs);
  ProfScope prof(c, kFamKs, 8.0 * c.n * A.nt * ((double)A.nsrc * A.ndig + jobs * (2.0 * A.ndig + 2.0)),
                 half_bfly(c, false) * rows);
  ntt_ks_row(c, A);
  post(c);
}

void b_ks_sum(Context& c, const KsSumArgs& A) {
  SF_HPROF("b_ks_sum");
  if (!A.nout) return;
  const double jobs = A.out_begin[A.nout];
  ProfScope prof(c, kFamKs, 8.0 * c.n * A.nt * (jobs * (3.0 * A.ndig + 2.0) + 2.0 * A.nout),
                 half_bfly(c, false) * 2.0 * A.nout * (A.nt - A.limbs));
  if (!ntt_ks_sum(c, A))
    ks_sum_generic_kernel<<<grid2((size_t)A.nt * c.n, A.nout), kT, 0, c.stream>>>(A, c.tabs.q, c.tabs.mh, c.tabs.ml,
                                                                                   c.logn);
  post(c);
}

void b_axpy_pm(Context& c, const AxpyBatch& B, int limbs, const u64* pm_dev) {
  if (!B.count) return;
  ProfScope prof(c, kFamElem, 24.0 * limbs * c.n * B.count);
  axpy_pm_kernel<<<grid2((size_t)limbs * c.n, B.count), kT, 0, c.stream>>>(B, limbs, c.logn, pm_dev, c.tabs.q,
                                                                            c.tabs.mh, c.tabs.ml);
  post(c);
}

void b_subscale(Context& c, const SubScaleBatch& B, int limbs, const u64* inv, const u64* inv_s) {
  SF_HPROF("b_subscale");
  if (!B.count) return;
  ProfScope prof(c, kFamElem, 32.0 * limbs * c.n * B.count);
  subscale_batch_kernel<<<grid2((size_t)limbs * c.n, B.count), kT, 0, c.stream>>>(B, limbs, c.logn, inv, inv_s,
                                                                                    c.tabs.q);
  post(c);
}

void b_vmm_mac(Context& c, const VmmMacArgs& A, int limbs) {
  SF_HPROF("b_vmm_mac");
  // diagonal ring depth: 4 (measured best: 6.1 -> 5.8 ms/step vs direct loads; 8 and 12 lose
  // occupancy); SF_VARIANT bits 5-6 select 0 / 8 / 12 for A/B
  static const int kDepth[4] = {4, 0, 8, 12};
  const int D = kDepth[(c.variant >> 5) & 3];
  const size_t sm = (size_t)A.b * 2 * 64 * sizeof(u64) + (D ? (size_t)8 * (D + 1) * 64 * sizeof(u64) : 0);
  // algorithmic bytes: every diagonal once, babies once, partials once
  ProfScope prof(c, kFamMac, 8.0 * c.n * limbs * ((double)A.k + 2.0 * A.b + 2.0 * A.giants));
  static bool attr = false;
  if (!attr) {
    SF_CUDA(cudaFuncSetAttribute(vmm_mac_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    SF_CUDA(cudaFuncSetAttribute(vmm_mac_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    SF_CUDA(cudaFuncSetAttribute(vmm_mac_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    SF_CUDA(cudaFuncSetAttribute(vmm_mac_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  const unsigned grid = (unsigned)(limbs * (c.n / 64));
  switch (D) {
    case 4: vmm_mac_kernel<4><<<grid, 256, sm, c.stream>>>(A, c.tabs.q, c.tabs.mh, c.tabs.ml); break;
    case 8: vmm_mac_kernel<8><<<grid, 256, sm, c.stream>>>(A, c.tabs.q, c.tabs.mh, c.tabs.ml); break;
    case 12: vmm_mac_kernel<12><<<grid, 256, sm, c.stream>>>(A, c.tabs.q, c.tabs.mh, c.tabs.ml); break;
    default: vmm_mac_kernel<0><<<grid, 256, sm, c.stream>>>(A, c.tabs.q, c.tabs.mh, c.tabs.ml);
  }
  post(c);
}

}  // namespace sf
