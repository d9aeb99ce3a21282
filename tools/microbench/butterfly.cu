// Butterfly throughput microbenchmark (B200): exact vs approximate-hi Shoup.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o butterfly butterfly.cu
#include <cstdint>
#include <cstdio>
typedef uint64_t u64;
typedef uint32_t u32;

__device__ __forceinline__ u64 shoup_exact(u64 x, u64 w, u64 wp, u64 q) { return x * w - __umul64hi(x, wp) * q; }
__device__ __forceinline__ u64 hi_approx(u64 x, u64 wp) {
  const u32 xl = (u32)x, xh = (u32)(x >> 32), wl = (u32)wp, wh = (u32)(wp >> 32);
  return (u64)xh * wh + __umulhi(xh, wl) + __umulhi(xl, wh);
}
__device__ __forceinline__ u64 shoup_approx(u64 x, u64 w, u64 wp, u64 q) { return x * w - hi_approx(x, wp) * q; }

template <int V>
__global__ void bench(u64* out, const u64* in, u64 q, u64 w0, u64 wp0, int iters, double wq0) {
  u64 x[8];
  for (int k = 0; k < 8; ++k) x[k] = in[(threadIdx.x + blockIdx.x * blockDim.x) * 8 + k] % q;
  const u64 q2 = 2 * q;
  u64 w = w0, wp = wp0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int b = 0; b < 3; ++b) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k & (1 << b)) continue;
        u64 U = x[k];
        U = U >= q2 ? U - q2 : U;
        u64 T;
        if (V == 0) {
          T = shoup_exact(x[k | (1 << b)], w, wp, q);
        } else if (V == 1) {
          T = shoup_approx(x[k | (1 << b)], w, wp, q);
          T = T >= q2 ? T - q2 : T;
        } else if (V == 3) {  // FP64 quotient (q < 2^42 primes): qt = floor(x * (w / q)) +- 1
          const u64 V_ = x[k | (1 << b)];
          const u64 qt = (u64)(__ull2double_rn(V_) * wq0);
          u64 r = V_ * w - qt * q;
          T = (long long)r < 0 ? r + q : r;
        } else {  // V2: [0, 8q) invariant, approximate high product, one correction
          U = x[k];
          U = U >= 2 * q2 ? U - 2 * q2 : U;
          T = shoup_approx(x[k | (1 << b)], w, wp, q);
          x[k] = U + T;
          x[k | (1 << b)] = U - T + 2 * q2;
          continue;
        }
        x[k] = U + T;
        x[k | (1 << b)] = U - T + q2;
      }
    }
    w ^= (u64)it & 1;  // keep twiddles loop-variant
  }
  u64 s = 0;
  for (int k = 0; k < 8; ++k) s ^= x[k];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}

int main() {
  const int blocks = 148 * 8, threads = 256, iters = 2000;
  const size_t nth = (size_t)blocks * threads;
  u64 *in, *out;
  cudaMalloc(&in, nth * 8 * 8);
  cudaMalloc(&out, nth * 8);
  cudaMemset(in, 0x5a, nth * 64);
  const u64 q = 1152921504606584833ull;  // < 2^60
  const u64 w = 123456789123456789ull % q;
  const u64 wp = (u64)(((unsigned __int128)w << 64) / q);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const u64 q40 = 1099511480321ull;  // a 40-bit NTT prime (any q < 2^42 works for V3)
  const u64 w40 = 123456789123ull % q40;
  const u64 wp40 = (u64)(((unsigned __int128)w40 << 64) / q40);
  const double wq40 = (double)w40 / (double)q40;
  for (int v = 0; v < 4; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v == 0) bench<0><<<blocks, threads>>>(out, in, q40, w40, wp40, iters, wq40);
      else if (v == 1) bench<1><<<blocks, threads>>>(out, in, q40, w40, wp40, iters, wq40);
      else if (v == 2) bench<2><<<blocks, threads>>>(out, in, q40, w40, wp40, iters, wq40);
      else bench<3><<<blocks, threads>>>(out, in, q40, w40, wp40, iters, wq40);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bf = (double)nth * iters * 12;
      if (rep) printf("variant %d: %.3f ms, %.1f G butterflies/s\n", v, ms, bf / ms / 1e6);
    }
  }
  return 0;
}
