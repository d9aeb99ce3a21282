// sm_100a kernels for the RNS-CKKS hot path. Every kernel leaves canonical
// residues in [0, q), so results are bit-identical to the CPU oracle
// (oracle/ckks_oracle.cpp) for the same inputs, whatever the evaluation order.
//
// Memory layout: a polynomial is `limbs` consecutive rows of
// n u64 residues (limb-major); limb l of a ciphertext is reduced mod primes[l].
// Elementwise kernels stream 16-byte (ulonglong2) vectors; the NTT stages a
// column or row tile in shared memory (two passes for n > 4096).
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.cuh"
#include "modarith.cuh"

namespace sf {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
}

static cudaEvent_t prof_event(Context& c) {
  if (c.prof_pool_next == c.prof_pool.size()) {
    cudaEvent_t e;
    SF_CUDA(cudaEventCreate(&e));
    c.prof_pool.push_back(e);
  }
  return c.prof_pool[c.prof_pool_next++];
}

ProfScope::ProfScope(Context& ctx, int family, double algorithmic_bytes, double butterflies)
    : c(ctx), fam(family), bytes(algorithmic_bytes), on(((ctx.prof_mask >> family) & 1) != 0) {
  if (!on) return;
  cudaEvent_t a = prof_event(c);
  b = prof_event(c);
  SF_CUDA(cudaEventRecord(a, c.stream));
  c.prof_recs.push_back({fam, a, b, bytes, butterflies});
}
ProfScope::~ProfScope() {
  if (on) cudaEventRecord(b, c.stream);
}

namespace {

constexpr int kThreads = 256;
constexpr int kMaxL = 64;

struct IntArr {
  int v[kMaxL];
};
struct RngArr {
  RngKey v[kMaxL];
};
struct U64Arr {
  u64 v[kMaxL];
};

inline void post_launch(Context& c) {
  c.launches.fetch_add(1, std::memory_order_relaxed);
#ifdef SF_DEBUG_SYNC
  host_sync(c);
#endif
  SF_CUDA(cudaGetLastError());
}

inline unsigned blocks_for(size_t work, int per_thread = 1) {
  size_t b = (work + (size_t)kThreads * per_thread - 1) / ((size_t)kThreads * per_thread);
  return (unsigned)(b ? b : 1);
}

__device__ __forceinline__ uint32_t brev(uint32_t x, int logn) { return __brev(x) >> (32 - logn); }

// NTT-domain automorphism index: out[i] = in[perm(i)].
__device__ __forceinline__ uint32_t auto_perm(uint32_t i, u64 g, int logn) {
  const u64 e = 2ull * brev(i, logn) + 1;
  const u64 e2 = (e * g) & ((2ull << logn) - 1);
  return brev((uint32_t)((e2 - 1) >> 1), logn);
}

// ----------------------------------------------------------------------------- NTT
// Forward: Cooley-Tukey, natural order in, bit-reversed evaluation order out:
// out[i] = a(psi^(2 br(i) + 1)). Inverse: Gentleman-Sande + n^-1.

template <bool INV>
__global__ void __launch_bounds__(512) ntt_single(LimbBatch B, Tabs T) {
  extern __shared__ u64 s[];
  const int n = T.n;
  u64* a = B.ptr[blockIdx.x];
  const int p = B.prime[blockIdx.x];
  const u64 q = T.q[p];
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = a[i];
  __syncthreads();
  const int half = n >> 1;
  if (!INV) {
    const u64* W = T.psi + (size_t)p * n;
    const u64* Ws = T.psi_s + (size_t)p * n;
    for (int m = 1, t = half; m < n; m <<= 1, t >>= 1) {
      for (int bf = threadIdx.x; bf < half; bf += blockDim.x) {
        const int i = bf / t, j = bf - i * t;
        const int idx = 2 * i * t + j;
        const u64 U = s[idx];
        const u64 V = mul_shoup(s[idx + t], W[m + i], Ws[m + i], q);
        s[idx] = add_mod(U, V, q);
        s[idx + t] = sub_mod(U, V, q);
      }
      __syncthreads();
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = s[i];
  } else {
    const u64* W = T.ipsi + (size_t)p * n;
    const u64* Ws = T.ipsi_s + (size_t)p * n;
    for (int m = n, t = 1; m > 1; m >>= 1, t <<= 1) {
      const int h = m >> 1;
      for (int bf = threadIdx.x; bf < half; bf += blockDim.x) {
        const int i = bf / t, j = bf - i * t;
        const int idx = 2 * i * t + j;
        const u64 U = s[idx], V = s[idx + t];
        s[idx] = add_mod(U, V, q);
        s[idx + t] = mul_shoup(sub_mod(U, V, q), W[h + i], Ws[h + i], q);
      }
      __syncthreads();
    }
    const u64 ni = T.ninv[p], nis = T.ninv_s[p];
    for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = mul_shoup(s[i], ni, nis, q);
  }
}

// ----------------------------------------------------------------------- elementwise
__global__ void addsub_kernel(u64* out, const u64* a, const u64* b, int limbs, int n, const u64* Q, bool sub) {
  const size_t total = (size_t)limbs * n / 2;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < total; v += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)((v * 2) / n);
    const u64 q = Q[l];
    const ulonglong2 x = reinterpret_cast<const ulonglong2*>(a)[v];
    const ulonglong2 y = reinterpret_cast<const ulonglong2*>(b)[v];
    ulonglong2 z;
    z.x = sub ? sub_mod(x.x, y.x, q) : add_mod(x.x, y.x, q);
    z.y = sub ? sub_mod(x.y, y.y, q) : add_mod(x.y, y.y, q);
    reinterpret_cast<ulonglong2*>(out)[v] = z;
  }
}

__global__ void copy_kernel(u64* out, const u64* in, size_t words) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < words / 2; i += (size_t)gridDim.x * blockDim.x)
    reinterpret_cast<ulonglong2*>(out)[i] = reinterpret_cast<const ulonglong2*>(in)[i];
}

__global__ void mac_kernel(u64* out0, u64* out1, MacTerms t, int limbs, int n, const u64* Q, const u64* MH,
                           const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    U128 a0{0, 0}, a1{0, 0};
    for (int k = 0; k < t.k; ++k) {
      const u64 p = t.pt[k][i];
      mac128(a0, t.c0[k][i], p);
      mac128(a1, t.c1[k][i], p);
    }
    out0[i] = reduce128(a0.hi, a0.lo, Q[l], MH[l], ML[l]);
    out1[i] = reduce128(a1.hi, a1.lo, Q[l], MH[l], ML[l]);
  }
}

__global__ void tensor_kernel(u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0, const u64* b1,
                              int limbs, int n, const u64* Q, const u64* MH, const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const u64 q = Q[l], mh = MH[l], ml = ML[l];
    const u64 x0 = a0[i], x1 = a1[i], y0 = b0[i], y1 = b1[i];
    d0[i] = mulmod(x0, y0, q, mh, ml);
    U128 m{0, 0};
    mac128(m, x0, y1);
    mac128(m, x1, y0);
    d1[i] = reduce128(m.hi, m.lo, q, mh, ml);
    d2[i] = mulmod(x1, y1, q, mh, ml);
  }
}

__global__ void hadamard_kernel(u64* out, const u64* a, const u64* b, int limbs, int n, const u64* Q, const u64* MH,
                                const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    out[i] = mulmod(a[i], b[i], Q[l], MH[l], ML[l]);
  }
}

__global__ void automorph_kernel(u64* out, const u64* in, const u64* add, u64 g, int limbs, int logn,
                                 const u64* Q) {
  const int n = 1 << logn;
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i >> logn);
    const uint32_t k = (uint32_t)(i & (n - 1));
    u64 v = in[((size_t)l << logn) + auto_perm(k, g, logn)];
    if (add) v = add_mod(v, add[i], Q[l]);
    out[i] = v;
  }
}

struct ConvArgs {
  int nsrc, ndst, n;
  const u64* qinv;    // [nsrc]
  const u64* qinv_s;  // [nsrc]
  const u64* qhat;    // [nsrc][ndst]
  int src_prime[kMaxL];
  int dst_prime[kMaxL];
  int out_slot[kMaxL];
};

__global__ void conv_kernel(ConvArgs A, const u64* in, u64* out, const u64* Q, const u64* MH, const u64* ML) {
  const int n = A.n;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    u64 y[kMaxL];
#pragma unroll 4
    for (int i = 0; i < A.nsrc; ++i) {
      const u64 q = Q[A.src_prime[i]];
      y[i] = mul_shoup(in[(size_t)i * n + k], A.qinv[i], A.qinv_s[i], q);
    }
    for (int d = 0; d < A.ndst; ++d) {
      U128 acc{0, 0};
      const u64* h = A.qhat + d;
      for (int i = 0; i < A.nsrc; ++i) mac128(acc, y[i], h[(size_t)i * A.ndst]);
      const int pd = A.dst_prime[d];
      out[(size_t)A.out_slot[d] * n + k] = reduce128(acc.hi, acc.lo, Q[pd], MH[pd], ML[pd]);
    }
  }
}

struct KsArgs {
  int ndig, nt, np, logn;
  u64 g;
  int tprime[kMaxL];
};

__global__ void ks_inner_kernel(u64* accb, u64* acca, const u64* ext, const u64* key, KsArgs A, const u64* Q,
                                const u64* MH, const u64* ML) {
  const int n = 1 << A.logn;
  const size_t total = (size_t)A.nt * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(i >> A.logn);
    const uint32_t k = (uint32_t)(i & (n - 1));
    const uint32_t src = A.g > 1 ? auto_perm(k, A.g, A.logn) : k;
    const int m = A.tprime[t];
    U128 sb{0, 0}, sa{0, 0};
    for (int j = 0; j < A.ndig; ++j) {
      const u64 x = ext[((size_t)j * A.nt + t) * n + src];
      const u64* kb = key + (((size_t)j * 2 + 0) * A.np + m) * n;
      const u64* ka = key + (((size_t)j * 2 + 1) * A.np + m) * n;
      mac128(sb, x, kb[k]);
      mac128(sa, x, ka[k]);
    }
    accb[i] = reduce128(sb.hi, sb.lo, Q[m], MH[m], ML[m]);
    acca[i] = reduce128(sa.hi, sa.lo, Q[m], MH[m], ML[m]);
  }
}

__global__ void sub_scale_kernel(u64* out, const u64* acc, const u64* conv, const u64* inv, const u64* inv_s,
                                 const u64* addend, u64 g, int limbs, int logn, const u64* Q) {
  const int n = 1 << logn;
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i >> logn);
    const u64 q = Q[l];
    u64 v = mul_shoup(sub_mod(acc[i], conv[i], q), inv[l], inv_s[l], q);
    if (addend) {
      const uint32_t k = (uint32_t)(i & (n - 1));
      const uint32_t src = g > 1 ? auto_perm(k, g, logn) : k;
      v = add_mod(v, addend[((size_t)l << logn) + src], q);
    }
    out[i] = v;
  }
}

__global__ void rescale_lift_kernel(u64* out, const u64* x, u64 ql, int limbs, int n, const u64* Q, const u64* MH) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const size_t k = i - (size_t)l * n;
    const u64 q = Q[l];
    const u64 v = x[k];
    const u64 r = reduce64(v, q, MH[l]);
    if (v > (ql >> 1))
      out[i] = sub_mod(r, reduce64(ql, q, MH[l]), q);
    else
      out[i] = r;
  }
}

// --- sampling ----------------------------------------------------------------------
// uniform residue k of a limb: two stream words as a 128-bit integer, reduced
// mod q (bias < 2^-67; a single 64-bit word mod a 60-bit prime would be biased)
__global__ void uniform_kernel(u64* out, RngArr keys, IntArr prime, int limbs, int n, const u64* Q, const u64* MH,
                               const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const size_t k = i - (size_t)l * n;
    const int p = prime.v[l];
    const u64 lo = rand_at(keys.v[l], 2 * k), hi = rand_at(keys.v[l], 2 * k + 1);
    out[i] = reduce128(hi, lo, Q[p], MH[p], ML[p]);
  }
}

__device__ __forceinline__ u64 signed_to_mod(i64 v, u64 q) {
  if (v >= 0) return (u64)v % q;
  u64 r = ((u64)(-(v + 1)) % q + 1) % q;
  return r == 0 ? 0 : q - r;
}

__global__ void ternary_kernel(u64* out, RngKey key, int limbs, int n, int first_prime, const u64* Q) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const size_t k = i - (size_t)l * n;
    const i64 v = (i64)(rand_at(key, k) % 3) - 1;
    out[i] = signed_to_mod(v, Q[first_prime + l]);
  }
}

__global__ void small_rns_kernel(u64* out, RngKey ekey, bool noise, const i64* m, IntArr prime, int limbs, int n,
                                 const u64* Q) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const size_t k = i - (size_t)l * n;
    const u64 q = Q[prime.v[l]];
    u64 res = 0;
    if (noise) {
      const u64 r = rand_at(ekey, k);
      const i64 v = (i64)__popcll(r & 0x1FFFFFull) - (i64)__popcll((r >> 21) & 0x1FFFFFull);
      res = signed_to_mod(v, q);
    }
    if (m) res = add_mod(res, signed_to_mod(m[k], q), q);
    out[i] = res;
  }
}

__global__ void key_combine_kernel(u64* b, const u64* a, const u64* s, const u64* e, const u64* sp, U64Arr pm,
                                   IntArr prime, int limbs, int n, const u64* Q, const u64* MH, const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const size_t k = i - (size_t)l * n;
    const int p = prime.v[l];
    const u64 q = Q[p], mh = MH[p], ml = ML[p];
    const size_t sidx = (size_t)p * n + k;  // s and s' are stored over all primes
    u64 v = sub_mod(e[i], mulmod(a[i], s[sidx], q, mh, ml), q);
    if (pm.v[l]) v = add_mod(v, mulmod(pm.v[l], sp[sidx], q, mh, ml), q);
    b[i] = v;
  }
}

__global__ void enc_combine_kernel(u64* c0, const u64* a, const u64* s, const u64* em, int limbs, int n,
                                   const u64* Q, const u64* MH, const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    const u64 q = Q[l];
    c0[i] = add_mod(sub_mod(0, mulmod(a[i], s[i], q, MH[l], ML[l]), q), em[i], q);
  }
}

__global__ void dec_combine_kernel(u64* out, const u64* c0, const u64* c1, const u64* s, int n, const u64* Q,
                                   const u64* MH, const u64* ML) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = add_mod(c0[i], mulmod(c1[i], s[i], Q[0], MH[0], ML[0]), Q[0]);
}

// data[blk][m][n] *= F[m] (mod prime m) for the primes with F[m] != 1 (blk = nblk blocks of np primes)
__global__ void scale_limbs_kernel(u64* data, size_t total, int np, int n, const u64* F, const u64* Q, const u64* MH,
                                   const u64* ML) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)((i / n) % np);
    const u64 f = F[m];
    if (f != 1) data[i] = mulmod(data[i], f, Q[m], MH[m], ML[m]);
  }
}

__global__ void square_kernel(u64* out, const u64* s, int limbs, int n, const u64* Q, const u64* MH,
                              const u64* ML) {
  const size_t total = (size_t)limbs * n;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total; i += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(i / n);
    out[i] = mulmod(s[i], s[i], Q[l], MH[l], ML[l]);
  }
}

unsigned grid_cap(size_t work) {
  const size_t b = blocks_for(work);
  return (unsigned)(b < 148 * 16 ? b : 148 * 16);
}

const u64* QP(Context& c) { return c.tabs.q; }

}  // namespace

// ------------------------------------------------------------------------ wrappers
void launch_ntt(Context& c, const LimbBatch& b, bool inverse) {
  if (b.count == 0) return;
  const int n = c.n;
  ProfScope prof(c, kFamNtt, 16.0 * n * b.count, 0.5 * n * c.logn * b.count);
  if (c.logn >= 12) {
    ntt_two_pass(c, b, inverse);
    post_launch(c);
    c.launches.fetch_add(1, std::memory_order_relaxed);  // two kernels per transform
    return;
  }
  const int th = std::min(512, std::max(32, n / 2));
  const size_t sm = (size_t)n * sizeof(u64);
  if (inverse)
    ntt_single<true><<<b.count, th, sm, c.stream>>>(b, c.tabs);
  else
    ntt_single<false><<<b.count, th, sm, c.stream>>>(b, c.tabs);
  post_launch(c);
}

void ntt_limbs(Context& c, u64* base, int count, int first_prime, bool inverse) {
  LimbBatch b;
  for (int i = 0; i < count; ++i) {
    b.add(base + (size_t)i * c.n, first_prime + i);
    if (b.count == kMaxBatch) launch_ntt(c, b, inverse), b.count = 0;
  }
  launch_ntt(c, b, inverse);
}

void ntt_list(Context& c, const std::vector<std::pair<u64*, int>>& limbs, bool inverse) {
  LimbBatch b;
  for (const auto& l : limbs) {
    b.add(l.first, l.second);
    if (b.count == kMaxBatch) launch_ntt(c, b, inverse), b.count = 0;
  }
  launch_ntt(c, b, inverse);
}

void k_addsub(Context& c, u64* out, const u64* a, const u64* b, int limbs, bool sub) {
  const size_t w = (size_t)limbs * c.n / 2;
  ProfScope prof(c, kFamElem, 24.0 * limbs * c.n);
  addsub_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, a, b, limbs, c.n, QP(c), sub);
  post_launch(c);
}

void k_copy(Context& c, u64* out, const u64* in, size_t words) {
  ProfScope prof(c, kFamElem, 16.0 * words);
  copy_kernel<<<grid_cap(words / 2), kThreads, 0, c.stream>>>(out, in, words);
  post_launch(c);
}

void k_mac(Context& c, u64* out0, u64* out1, const MacTerms& t, int limbs) {
  const size_t w = (size_t)limbs * c.n;
  ProfScope prof(c, kFamMac, 8.0 * c.n * limbs * (3.0 * t.k + 2));
  mac_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out0, out1, t, limbs, c.n, QP(c), c.tabs.mh, c.tabs.ml);
  post_launch(c);
}

void k_tensor(Context& c, u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0, const u64* b1,
              int limbs) {
  const size_t w = (size_t)limbs * c.n;
  ProfScope prof(c, kFamElem, 56.0 * limbs * c.n);
  tensor_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(d0, d1, d2, a0, a1, b0, b1, limbs, c.n, QP(c), c.tabs.mh,
                                                        c.tabs.ml);
  post_launch(c);
}

void k_hadamard(Context& c, u64* out, const u64* a, const u64* b, int limbs, int first_prime) {
  const size_t w = (size_t)limbs * c.n;
  ProfScope prof(c, kFamElem, 24.0 * limbs * c.n);
  hadamard_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, a, b, limbs, c.n, QP(c) + first_prime,
                                                          c.tabs.mh + first_prime, c.tabs.ml + first_prime);
  post_launch(c);
}

void k_automorph(Context& c, u64* out, const u64* in, const u64* add, u64 g, int limbs) {
  const size_t w = (size_t)limbs * c.n;
  ProfScope prof(c, kFamElem, (add ? 24.0 : 16.0) * limbs * c.n);
  automorph_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, in, add, g, limbs, c.logn, QP(c));
  post_launch(c);
}

void k_conv(Context& c, const ConvPlan& p, const u64* in, u64* out, const std::vector<int>& out_slot) {
  require(p.nsrc <= kMaxL && p.ndst <= kMaxL, kInternal, "conv: too many primes");
  ConvArgs A;
  A.nsrc = p.nsrc;
  A.ndst = p.ndst;
  A.n = c.n;
  A.qinv = p.tab->p;
  A.qinv_s = p.tab->p + p.nsrc;
  A.qhat = p.tab->p + 2 * p.nsrc;
  for (int i = 0; i < p.nsrc; ++i) A.src_prime[i] = p.src[i];
  for (int d = 0; d < p.ndst; ++d) {
    A.dst_prime[d] = p.dst[d];
    A.out_slot[d] = out_slot[d];
  }
  ProfScope prof(c, kFamConv, 8.0 * c.n * (p.nsrc + p.ndst));
  conv_kernel<<<grid_cap(c.n), kThreads, 0, c.stream>>>(A, in, out, QP(c), c.tabs.mh, c.tabs.ml);
  post_launch(c);
}

void k_ks_inner(Context& c, u64* accb, u64* acca, const u64* ext, int ndig, int nt, const int* tprime, const u64* key,
                u64 g) {
  require(nt <= kMaxL, kInternal, "ks: too many limbs");
  KsArgs A;
  A.ndig = ndig;
  A.nt = nt;
  A.np = c.np;
  A.logn = c.logn;
  A.g = g;
  for (int t = 0; t < nt; ++t) A.tprime[t] = tprime[t];
  const size_t w = (size_t)nt * c.n;
  ProfScope prof(c, kFamKs, 8.0 * c.n * ((double)ndig * nt * 3 + 2.0 * nt));
  ks_inner_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(accb, acca, ext, key, A, QP(c), c.tabs.mh, c.tabs.ml);
  post_launch(c);
}

void k_sub_scale(Context& c, u64* out, const u64* acc, const u64* conv, const u64* inv, const u64* inv_s,
                 const u64* addend, u64 g, int limbs) {
  const size_t w = (size_t)limbs * c.n;
  ProfScope prof(c, kFamElem, 8.0 * c.n * limbs * (addend ? 4 : 3));
  sub_scale_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, acc, conv, inv, inv_s, addend, g, limbs, c.logn,
                                                           QP(c));
  post_launch(c);
}

void k_rescale_lift(Context& c, u64* out, const u64* x, int last_prime, int limbs) {
  const size_t w = (size_t)limbs * c.n;
  ProfScope prof(c, kFamElem, 8.0 * c.n * (limbs + 1));
  rescale_lift_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, x, c.primes[last_prime], limbs, c.n, QP(c),
                                                              c.tabs.mh);
  post_launch(c);
}

void k_sample_uniform(Context& c, u64* out, const RngKey* stream_keys, const int* prime_of_limb, int limbs) {
  require(limbs <= kMaxL, kInternal, "sample: too many limbs");
  RngArr k;
  IntArr p;
  for (int l = 0; l < limbs; ++l) k.v[l] = stream_keys[l], p.v[l] = prime_of_limb[l];
  const size_t w = (size_t)limbs * c.n;
  uniform_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, k, p, limbs, c.n, QP(c), c.tabs.mh, c.tabs.ml);
  post_launch(c);
}

void k_ternary(Context& c, u64* out, RngKey key, int limbs, int first_prime) {
  const size_t w = (size_t)limbs * c.n;
  ternary_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, key, limbs, c.n, first_prime, QP(c));
  post_launch(c);
}

void k_small_rns(Context& c, u64* out, RngKey ekey, bool noise, const i64* m, const int* prime_of_limb, int limbs) {
  require(limbs <= kMaxL, kInternal, "small_rns: too many limbs");
  IntArr p;
  for (int l = 0; l < limbs; ++l) p.v[l] = prime_of_limb[l];
  const size_t w = (size_t)limbs * c.n;
  small_rns_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, ekey, noise, m, p, limbs, c.n, QP(c));
  post_launch(c);
}

void k_key_combine(Context& c, u64* b, const u64* a, const u64* s, const u64* e, const u64* sp, const u64* pm,
                   const int* prime_of_limb, int limbs) {
  U64Arr P;
  IntArr p;
  for (int l = 0; l < limbs; ++l) P.v[l] = pm[l], p.v[l] = prime_of_limb[l];
  const size_t w = (size_t)limbs * c.n;
  key_combine_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(b, a, s, e, sp, P, p, limbs, c.n, QP(c), c.tabs.mh,
                                                             c.tabs.ml);
  post_launch(c);
}

void k_enc_combine(Context& c, u64* c0, const u64* a, const u64* s, const u64* em, int limbs) {
  const size_t w = (size_t)limbs * c.n;
  enc_combine_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(c0, a, s, em, limbs, c.n, QP(c), c.tabs.mh,
                                                             c.tabs.ml);
  post_launch(c);
}

void k_dec_combine(Context& c, u64* out, const u64* c0, const u64* c1, const u64* s) {
  dec_combine_kernel<<<grid_cap(c.n), kThreads, 0, c.stream>>>(out, c0, c1, s, c.n, QP(c), c.tabs.mh, c.tabs.ml);
  post_launch(c);
}

void k_scale_limbs(Context& c, u64* data, int nblk, const u64* F_dev) {
  const size_t total = (size_t)nblk * c.np * c.n;
  scale_limbs_kernel<<<grid_cap(total), kThreads, 0, c.stream>>>(data, total, c.np, c.n, F_dev, c.tabs.q, c.tabs.mh,
                                                                 c.tabs.ml);
  post_launch(c);
}

void k_square(Context& c, u64* out, const u64* s, int limbs) {
  const size_t w = (size_t)limbs * c.n;
  square_kernel<<<grid_cap(w), kThreads, 0, c.stream>>>(out, s, limbs, c.n, QP(c), c.tabs.mh, c.tabs.ml);
  post_launch(c);
}

}  // namespace sf
