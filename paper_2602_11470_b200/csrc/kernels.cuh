// Kernel launch wrappers (kernels.cu). All launches go on ctx.stream and bump
// ctx.launches (reported as bench.py's gpu_launches).
#pragma once
#include "context.h"

namespace sf {

constexpr int kMaxTerms = 64;  // lazy 128-bit MAC bound for q < 2^61

// Pointer bundle for a MAC over `k` terms: sum_t ct[t] (.) pt[t].
struct MacTerms {
  const u64* c0[kMaxTerms];
  const u64* c1[kMaxTerms];
  const u64* pt[kMaxTerms];
  int k;
};

void k_addsub(Context& c, u64* out, const u64* a, const u64* b, int limbs, bool sub);
void k_copy(Context& c, u64* out, const u64* in, size_t words);
void k_mac(Context& c, u64* out0, u64* out1, const MacTerms& t, int limbs);
void k_tensor(Context& c, u64* d0, u64* d1, u64* d2, const u64* a0, const u64* a1, const u64* b0,
              const u64* b1, int limbs);
void k_hadamard(Context& c, u64* out, const u64* a, const u64* b, int limbs, int first_prime = 0);
// out[l][i] = in[l][perm_g(i)] (+ add[l][i]); prime of limb l = l
void k_automorph(Context& c, u64* out, const u64* in, const u64* add, u64 g, int limbs);

// fast basis conversion (coefficient domain): in limbs (src primes, at in +
// s*n), out limbs (dst primes, at out_slots[d]*n from out)
void k_conv(Context& c, const ConvPlan& p, const u64* in, u64* out, const std::vector<int>& out_slot);

// key-switch inner product over extended basis T (nt limbs with prime idx
// primes[t]); ext = [ndig][nt][n]; key = [beta][2][np][n]; automorphism g
// applied to ext on the fly (g <= 1: identity).
void k_ks_inner(Context& c, u64* accb, u64* acca, const u64* ext, int ndig, int nt, const int* tprime,
                const u64* key, u64 g);

// out[l] = (acc[l] - conv[l]) * inv_l (+ addend permuted by g)
void k_sub_scale(Context& c, u64* out, const u64* acc, const u64* conv, const u64* inv, const u64* inv_s,
                 const u64* addend, u64 g, int limbs);
// rescale lift: x = coefficient limb mod q_last -> r_i = centred(x) mod q_i, i < limbs
void k_rescale_lift(Context& c, u64* out, const u64* x, int last_prime, int limbs);

// sampling
void k_sample_uniform(Context& c, u64* out, const RngKey* stream_keys, const int* prime_of_limb, int limbs);
void k_ternary(Context& c, u64* out, RngKey key, int limbs, int first_prime);  // sk coefficients
// small signed coefficients v = cbd(rand(key, k)) + (m ? m[k] : 0) reduced mod each prime
void k_small_rns(Context& c, u64* out, RngKey ekey, bool noise, const i64* m, const int* prime_of_limb, int limbs);
// b = -a*s + e (+ pm * s') ; operands per limb via prime index
void k_key_combine(Context& c, u64* b, const u64* a, const u64* s, const u64* e, const u64* sp, const u64* pm,
                   const int* prime_of_limb, int limbs);
// c0 = -a*s + em ; over limbs 0..limbs-1
void k_enc_combine(Context& c, u64* c0, const u64* a, const u64* s, const u64* em, int limbs);
// mu = c0 + c1*s on limb 0
void k_dec_combine(Context& c, u64* out, const u64* c0, const u64* c1, const u64* s);
// sk' = sigma_g(s) or s*s over all primes
void k_square(Context& c, u64* out, const u64* s, int limbs);
void k_scale_limbs(Context& c, u64* data, int nblk, const u64* F_dev);  // data[blk][m][n] *= F[m] mod prime m

}  // namespace sf
