// Job descriptors for the batched kernels (batch.cu). Each struct is passed by
// value as the kernel parameter block (<= 32 KB, CUDA 12.1+).
#pragma once
#include <map>

#include "context.h"

namespace sf {

constexpr int kMaxPrimes = 64;
constexpr int kJobs = 128;      // jobs per key-switch / tensor launch
constexpr int kJobsWide = 256;  // jobs per light elementwise launch

struct CopyBatch {
  int count = 0;
  const u64* src[kJobsWide];
  u64* dst[kJobsWide];
};

struct AddBatch {
  int count = 0;
  bool sub = false;
  const u64 *a0[kJobsWide], *a1[kJobsWide], *b0[kJobsWide], *b1[kJobsWide];
  u64 *o0[kJobsWide], *o1[kJobsWide];
};

struct SumArgs {  // out = sum of k ciphertexts
  int k = 0;
  const u64* in0[512];
  const u64* in1[512];
  u64 *out0, *out1;
};

struct SumMultiArgs {  // out_o = sum of the inputs [begin[o], begin[o+1]) (several sums, one launch)
  int nout = 0;
  int begin[65];
  const u64 *in0[512], *in1[512];
  u64 *out0[64], *out1[64];
};

struct MulPtBatch {  // (c0, c1) (.) pt, reduced, no rescale
  int count = 0;
  const u64 *c0[kJobsWide], *c1[kJobsWide], *pt[kJobsWide];
  u64 *o0[kJobsWide], *o1[kJobsWide];
  // per job: Shoup companions of (c0, c1) ([2][limbs][n]) when the ciphertext feeds
  // several products of the batch (computed once; the products become Shoup products)
  const u64* cs[kJobsWide] = {};
};

struct TensorBatch {
  int count = 0;
  const u64 *a0[kJobs], *a1[kJobs], *b0[kJobs], *b1[kJobs];
  u64 *d0[kJobs], *d1[kJobs], *d2[kJobs];
  // every job's a is the same ciphertext (QK^T: the replicated query): its Shoup
  // companions floor(a 2^64 / q) ([2][limbs][n]) turn the four products into Shoup products
  const u64* as = nullptr;
};

struct LiftBatch {  // rescale lift of one coefficient-domain limb into `limbs` limbs
  int count = 0;
  const u64* x[512];
  u64* out[512];
};

struct ConvBatch {  // fast basis conversion, same plan for every job
  int count = 0;
  int nsrc = 0, ndst = 0, n = 0;
  const u64 *qinv = nullptr, *qinv_s = nullptr, *qhat = nullptr;
  int src_prime[kMaxPrimes];
  int dst_prime[kMaxPrimes];
  int out_slot[kMaxPrimes];
  const u64* in[kJobsWide];
  u64* out[kJobsWide];
};

struct KsBatch {  // key-switch inner products over the extended basis
  int count = 0;
  int ndig = 0, nt = 0, np = 0, logn = 0;
  int tprime[kMaxPrimes];
  const u64* ext[kJobs];
  const u64* key[kJobs];
  u64 g[kJobs];
  u64* accb[kJobs];
  u64* acca[kJobs];
};

struct AxpyBatch {  // acc[l] += pm[l] * d[l] (mod q_l), l < limbs
  int count = 0;
  u64* acc[kJobsWide];
  const u64* d[kJobsWide];
};

struct SubScaleBatch {  // out = (acc - conv) * inv (+ addend permuted by g)
  int count = 0;
  const u64 *acc[kJobsWide], *conv[kJobsWide], *addend[kJobsWide];
  u64 g[kJobsWide];
  u64* out[kJobsWide];
};

struct VmmMacArgs {
  int n = 0, b = 0, giants = 0, k = 0;  // giants = number of outputs
  int gidx[64];                          // global giant-step index of output i
  const u64* baby0[64];
  const u64* baby1[64];
  const u64* pt[2048];
  u64* out0[64];
  u64* out1[64];
};

struct TensorSumArgs {  // (D0, D1, D2) = sum_i tensor(a_i, b_i), no relinearisation
  int k = 0;
  const u64 *a0[512], *a1[512], *b0[512], *b1[512];
  u64 *d0, *d1, *d2;
  bool accumulate = false;  // add into existing (D0, D1, D2)
};

// Several lazily relinearised sums at once (the Score*V giants):
// output o = sum over terms [begin[o], begin[o+1]) of tensor(a_i, b_i). A block
// walks every output for one coefficient tile, so operands shared by several
// outputs (the babies) are re-read from L1 / L2 and each distinct operand
// streams from HBM about once.
constexpr int kTsmTerms = 600, kTsmOuts = 32;
struct TensorSumMultiArgs {
  int nout = 0;
  int begin[kTsmOuts + 1];
  u64 *d0[kTsmOuts], *d1[kTsmOuts], *d2[kTsmOuts];
  const u64 *a0[kTsmTerms], *a1[kTsmTerms], *b0[kTsmTerms], *b1[kTsmTerms];
};

// Fused column stage of ModUp / ModDown / rescale (fused.cu): per job, the
// inverse column NTT of ns source limbs (already inverse-row-passed), the
// basis conversion (mode 0) or rescale lift (mode 1) into nd destination limbs
// in shared memory, and their forward column NTT; the destination limbs then
// need only the forward row pass. Source limbs of job j: src[j] + s*n;
// destination limb d: dst[j] + out_slot[d]*n.
struct FusedColArgs {
  int d_per_cta = 0;  // destinations per CTA (0: all); the launcher sets it for small launches
  void set_plan(const u64* tab, int nsrc, int ndst) {
    const size_t base2 = 2 * (size_t)nsrc + (size_t)nsrc * ndst;
    qhat = tab + 2 * nsrc;
    ymul = tab + base2;
    ymul_s = tab + base2 + nsrc;
    qhat_s = tab + base2 + 2 * nsrc;
    ymulw = tab + 2 * base2;
    ymulw_s = tab + 2 * base2 + nsrc;
  }
  int count = 0, ns = 0, nd = 0, mode = 0;
  int src_prime[kMaxPrimes], dst_prime[kMaxPrimes], out_slot[kMaxPrimes];
  // mode 0 (ConvPlan tables): y_s = x_s * (n^-1 qhat_s^-1) (Shoup), out_d = sum_s y_s * qhat[s][d] (Shoup)
  const u64 *ymul = nullptr, *ymul_s = nullptr, *qhat = nullptr, *qhat_s = nullptr;
  const u64 *ymulw = nullptr, *ymulw_s = nullptr;  // ymul * ipsi[1]: folded into the last inverse stage
  u64 q_last = 0;  // mode 1
  const u64* src[kJobsWide];
  u64* dst[kJobsWide];
};

// Forward row pass with the ModDown / rescale combine as epilogue:
// out = (acc - NTT(buf)) * inv (+ addend[perm_g]) on limb `prime`.
struct EpiBatch {
  int count = 0;
  u64* buf[kJobsWide];
  const u64* acc[kJobsWide];
  const u64* addend[kJobsWide];
  u64* out[kJobsWide];
  u64 g[kJobsWide];
  u64 inv[kJobsWide], inv_s[kJobsWide];
  const u64* post[kJobsWide] = {};  // optional NTT-domain plaintext limb multiplied into the output
  uint8_t prime[kJobsWide];
  bool nomul = false;  // out = acc - v (+ addend): P^-1 already folded in (rotation sums)
};

// Fused key-switch row stage (ntt.cu ks_row_kernel): per (source, target prime
// t, row), the forward row pass of the ModUp output of every digit (own limbs
// read straight from the NTT-domain source), then per job of that source the
// automorphism + inner product with the switching key, reduced, written in
// the NTT domain for t < limbs and inverse-row-passed (ModDown's first pass)
// for the special primes. Jobs are grouped by source (CSR in job_begin).
struct KsRowArgs {
  int nsrc = 0, limbs = 0, nt = 0, ndig = 0, alpha = 0, np = 0;
  int run_len = 0;  // host-side scratch (jobs of the current source while splitting)
  // merged relinearise + rescale: Q targets accumulate
  // P * (add0, add1) and the top Q prime is inverse-row-passed like the P primes
  int merged = 0;
  u64 pm[kMaxPrimes];
  const u64* add0[kJobs];
  const u64* add1[kJobs];
  int tprime[kMaxPrimes];
  // per work unit (a source, or a chunk of one source's jobs):
  const u64* c1[kJobs];   // NTT-domain source polynomial (limbs x n)
  const u64* ext[kJobs];  // column-pass ModUp output [ndig][nt][n] (own slots unused)
  int job_begin[kJobs + 1];
  u64 g[kJobs], ginv[kJobs];
  const u64* key[kJobs];  // [beta][2][np][n]
  u64* acc[kJobs];        // [2][nt][n]
};

// Rotation-sum row stage (ntt.cu ks_sum_kernel): per output o,
// target slot t and destination row, the extended-basis accumulation
//   acc_o = sum_{jobs of o} [ <sigma_g(ModUp(c1_s)), key_g> + P * sigma_g(c0_s) ]
// (identity jobs, g <= 1: P * (c0_s, c1_s)), reduced once, written NTT-domain
// for t < limbs and inverse-row-passed for the special primes (ModDown input).
// ext holds the FULLY NTT'd ModUp output of every non-own target.
constexpr int kSumOuts = 128, kSumJobs = 1024, kSumSrcs = 128;
struct KsSumArgs {
  int nout = 0, limbs = 0, nt = 0, ndig = 0, alpha = 0, np = 0;
  int tprime[kMaxPrimes];
  u64 pm[kMaxPrimes];  // P mod q_t, t < limbs
  bool pm_one = false;  // keys carry P^-1 on the Q limbs (get_key_pinv): pm == 1, ModDown without P^-1
  // targets t >= inv_from (and all special primes) are written inverse-row-passed:
  // inv_from = limbs - 1 feeds the merged ModDown + rescale (M = {q_top} u P)
  int inv_from = 1 << 30;
  // double hoisting (fold_steps_batch; PM1 only):
  // keep_b: the b part stays extended and NTT-domain on every target (the next
  //   radix sum's c0 input), only the a part is inverse-row-passed for its ModDown
  // ext_c0: c0[s] is such an extended b part ([nt][n]); sigma_g(c0) (identity: c0)
  //   enters on every target, c1 on the Q targets only
  bool keep_b = false, ext_c0 = false;
  int out_begin[kSumOuts + 1];
  u64* acc[kSumOuts];  // [2][nt][n]
  int jsrc[kSumJobs];
  u64 g[kSumJobs];
  const u64* key[kSumJobs];
  const u64* c0[kSumSrcs];
  const u64* c1[kSumSrcs];
  const u64* ext[kSumSrcs];  // [ndig][nt][n]
};

// ntt.cu dispatchers (false when the ring degree has no two-pass kernels)
bool ntt_row_only(Context& c, const LimbBatch& b, bool inverse);
bool ntt_row_epi(Context& c, const EpiBatch& e);
bool ntt_fused_col(Context& c, const FusedColArgs& a);
bool ntt_ks_row(Context& c, const KsRowArgs& a);
bool ntt_ks_sum(Context& c, const KsSumArgs& a);
inline bool fused_path(const Context& c) { return c.logn >= 12 && c.logn <= 17 && c.alpha <= 7; }
// profiled launch wrappers (batch.cu)
void b_row(Context& c, const LimbBatch& b, bool inverse);
void b_fused_col(Context& c, const FusedColArgs& A);
void b_row_epi(Context& c, const EpiBatch& E);
void b_ks_row(Context& c, const KsRowArgs& A);
void b_ks_sum(Context& c, const KsSumArgs& A);

void b_copy(Context& c, const CopyBatch& B, size_t words);
void b_tensor_sum(Context& c, const TensorSumArgs& A, int limbs);
void b_tensor_sum_multi(Context& c, const TensorSumMultiArgs& A, int limbs);
void b_add(Context& c, const AddBatch& B, int limbs);
void b_sum(Context& c, const SumArgs& A, int limbs);
void b_sum_multi(Context& c, const SumMultiArgs& A, int limbs);
void b_mulpt(Context& c, const MulPtBatch& B, int limbs);
void b_tensor(Context& c, const TensorBatch& B, int limbs);
void b_shoup_companion(Context& c, const u64* a, u64* out, int limbs, int polys);  // out = floor(a 2^64 / q_l)
void b_lift(Context& c, const LiftBatch& B, int limbs, int last_prime);
void b_conv(Context& c, const ConvBatch& A);
void b_ks(Context& c, const KsBatch& A);
void b_subscale(Context& c, const SubScaleBatch& B, int limbs, const u64* inv, const u64* inv_s);
void b_axpy_pm(Context& c, const AxpyBatch& B, int limbs, const u64* pm_dev);
void b_vmm_mac(Context& c, const VmmMacArgs& A, int limbs);

// ---- batched evaluator (keyswitch.cu) ------------------------------------------
// One rotation job: rotate srcs[src] by r (galois element derived from r).
struct RotJob {
  int src;
  int r;
};
// Rotations of a set of same-level ciphertexts; each distinct source is
// ModUp'd once (hoisting), key switches and ModDowns run batched.
std::vector<Ct> rotate_batch(Context& c, const std::vector<const Ct*>& srcs, const std::vector<RotJob>& jobs,
                             bool hoisted, bool count = true);
std::vector<Ct> mul_batch(Context& c, const std::vector<const Ct*>& a, const std::vector<const Ct*>& b,
                          bool count = true);
std::vector<Ct> rescale_batch(Context& c, const std::vector<const Ct*>& xs);
// x_i (.) p_i, rescaled (scale preserved: p_i encoded at q_top)
// rescale = false: the raw products at scale * q_top, same limbs (the caller rescales)
std::vector<Ct> mul_plain_batch(Context& c, const std::vector<const Ct*>& xs, const std::vector<const Pt*>& ps,
                                bool count = true, bool rescale = true);
std::vector<Ct> add_batch(Context& c, const std::vector<const Ct*>& a, const std::vector<const Ct*>& b,
                          bool count = true);
// sum_i Rot(a_i, r_i) per group with one ModDown per part
struct SumTerm {
  const Ct* ct;
  int r;
};
// rescale: the sum is rescaled by its top prime in the same basis conversion as
// its ModDown (merged): one conversion from {q_top} u P
// dig: digit size of the terms' decomposition (0: alpha; scaled_digit(limbs) for
// sums of products still at scale >= 2^80, with the rescale merged)
// Double hoisting (fused path, PM1 sums, no rescale): keep_b (one entry per
// group) receives each sum's b part extended and NTT-domain ([nt][n], the
// buffer kept alive) and the returned Ct holds only the a part (c0 undefined);
// ext_b feeds such kept b parts back as the c0 of their source ciphertexts.
struct ExtPoly {
  BufPtr buf;
  const u64* p = nullptr;
};
std::vector<Ct> rot_sum_batch(Context& c, const std::vector<std::vector<SumTerm>>& groups, bool hoisted,
                              bool count = true, const std::vector<const Pt*>* post = nullptr, bool rescale = false,
                              int dig = 0, std::vector<ExtPoly>* keep_b = nullptr,
                              const std::map<const Ct*, const u64*>* ext_b = nullptr);
// doubling chains x <- x + Rot(x, r) over rots[i] (radix rotation sums); charged
// as the reference's rotate + add steps when count && lead
// post (fused path only): per chain an NTT-domain plaintext multiplied into the
// result in the last ModDown's epilogue (a fused ct x pt; the caller rescales)
// shift (per chain): Rot(chain value, shift[i]) -- every term of the last radix
// sum moves by shift[i] (one rotation sum, no extra key switch)
std::vector<Ct> fold_steps_batch(Context& c, const std::vector<const Ct*>& xs, const std::vector<std::vector<int>>& rots,
                                 bool count = true, bool lead = true, const std::vector<const Pt*>* post = nullptr,
                                 const std::vector<int>* shift = nullptr);
// fold_within_head of every x (radix rotation sums), reference ledger charge
std::vector<Ct> fold_batch(Context& c, const std::vector<const Ct*>& xs, int d_head, int t, bool count = true,
                           const std::vector<const Pt*>* post = nullptr, const std::vector<int>* shift = nullptr);
// sum of k same-level ciphertexts, charged k-1 additions
Ct sum_cts(Context& c, const std::vector<const Ct*>& xs, bool count = true);
// several such sums in one launch (uncharged; the caller charges)
std::vector<Ct> sum_cts_multi(Context& c, const std::vector<std::vector<const Ct*>>& groups);

// Degree-2 ciphertext (d0, d1, d2) decrypting under (1, s, s^2): the lazily
// relinearised sum of ct x ct products. d01 holds (d0, d1); d2 lives in the
// c0 polynomial of its own Ct (c1 unused, zero).
struct Ct3 {
  Ct d01, d2;
  bool zero = true;
};
// sum_i a_i (x) b_i without relinearisation; charged k ct-ct mults and k-1 additions
Ct3 tensor_sum(Context& c, const std::vector<const Ct*>& a, const std::vector<const Ct*>& b, bool count = true);
// several such sums in one pass (operands shared between sums read once); charged like
// separate tensor_sum calls when count
std::vector<Ct3> tensor_sum_multi(Context& c, const std::vector<std::vector<const Ct*>>& a,
                                  const std::vector<std::vector<const Ct*>>& b, bool count = true);
// component-wise sum of degree-2 partials (no ledger charge)
Ct3 add_ct3(Context& c, const std::vector<const Ct3*>& xs);
// relinearise (key switch d2 under s^2) and rescale
Ct relin_rescale(Context& c, const Ct3& x);
// relinearise many degree-2 ciphertexts (one batched ModUp and key switch),
// rescaled in the ModDown's conversion (merged) or not (same level and scale)
std::vector<Ct> relin_batch(Context& c, const std::vector<const Ct3*>& xs, bool rescale);

}  // namespace sf
