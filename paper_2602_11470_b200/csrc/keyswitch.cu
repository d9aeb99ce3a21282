// Batched hybrid key switching, rescaling and ciphertext arithmetic
// (DESIGN.md §3.5-3.6, §5). Every per-ciphertext result is bit-identical to
// the scalar definition (and to the CPU oracle): batching changes only how
// many ciphertexts one launch covers.
//
// rotate(ct, r)  = ( sigma_g(c0) + ModDown(<sigma_g(ModUp(c1)), evk_g.b>),
//                                  ModDown(<sigma_g(ModUp(c1)), evk_g.a>) )
// mul(a, b)      = Rescale( (d0, d1) + ModDown(<ModUp(d2), rlk>) )
// Hoisting falls out of the definition: jobs that share a source share one
// ModUp (RotationHint{hoisted}, engine.hpp:98-100).
#include <algorithm>
#include <cmath>
#include <map>

#include "batch.cuh"

namespace sf {

int scaled_digit(const Context& c, int limbs) {
  double lp = 0.0;
  for (int k = 0; k < c.alpha; ++k) lp += std::log2((double)c.primes[c.P_index(k)]);
  int best = c.alpha;
  for (int d = c.alpha + 1; d <= std::min(8, limbs); ++d) {
    bool ok = true;
    for (int lo = 0; lo < limbs && ok; lo += d) {
      double lq = 0.0;
      for (int l = lo; l < std::min(limbs, lo + d); ++l) lq += std::log2((double)c.primes[l]);
      ok = lq - lp <= 30.0;
    }
    if (ok) best = d;
  }
  return best;
}

int relin_digit(const Context& c, int limbs) {
  double lq = 0.0, lp = 0.0;
  for (int l = 0; l < limbs; ++l) lq += std::log2((double)c.primes[l]);
  for (int k = 0; k < c.alpha; ++k) lp += std::log2((double)c.primes[c.P_index(k)]);
  return (limbs > c.alpha && limbs <= 8 && lq - lp <= 30.0) ? limbs : c.alpha;
}


BufPtr make_buf(Context& c, size_t words);
const u64* level_consts(Context& c, int limbs);
const ConvPlan& conv_plan(Context& c, const std::vector<int>& src, const std::vector<int>& dst, bool pinv = false);
OptLayout merge_layouts(const Ct& a, const Ct& b);

namespace {

struct ExtB {
  BufPtr buf;
  int S = 0, ndig = 0, nt = 0, limbs = 0, dig = 0;  // dig: limbs per digit
  bool col_only = false;        // ext holds column-pass output; ks_row_kernel finishes it
  std::vector<const u64*> src;  // the NTT-domain sources (own-prime rows)
  std::vector<int> tprime;
  size_t per = 0;  // words per source
  const u64* ext(int s) const { return buf->p + (size_t)s * per; }
};

// one polynomial for ModDown (mod_down_polys / mod_down_rescale_polys)
struct MdPoly {
  const u64* acc;
  const u64* addend;
  u64 g;
  u64* out;
  const u64* post = nullptr;  // optional NTT-domain plaintext multiplied into the result (fused ct x pt)
};

void fill_conv(ConvBatch& B, Context& c, const ConvPlan& p) {
  SF_HPROF("fill_conv");
  B.nsrc = p.nsrc;
  B.ndst = p.ndst;
  B.n = c.n;
  B.qinv = p.tab->p;
  B.qinv_s = p.tab->p + p.nsrc;
  B.qhat = p.tab->p + 2 * p.nsrc;
  for (int i = 0; i < p.nsrc; ++i) B.src_prime[i] = p.src[i];
  for (int d = 0; d < p.ndst; ++d) B.dst_prime[d] = p.dst[d];
}

void ntt_batch(Context& c, LimbBatch& b, bool inverse) {
  SF_HPROF("ntt_batch");
  if (b.count) launch_ntt(c, b, inverse);
  b.count = 0;
}
void ntt_push(Context& c, LimbBatch& b, u64* p, int prime, bool inverse) {
  SF_HPROF("ntt_push");
  b.add(p, prime);
  if (b.count == kMaxBatch) ntt_batch(c, b, inverse);
}

// ModUp of S distinct NTT-domain polynomials d[s] (limbs limbs each).
// full_ext: the ext limbs are fully NTT'd (forward row pass run here) and the
// digit's own limbs are not copied (the consumer reads the source) -- the
// layout ks_sum_kernel expects; otherwise ks_row_kernel's column-only layout.
// dig: digit size of the decomposition (0: alpha; a wide relinearisation: all limbs)
ExtB mod_up_batch(Context& c, const std::vector<const u64*>& d, int limbs, bool full_ext = false, int dig = 0) {
  SF_HPROF("mod_up_batch");
  ExtB x;
  const size_t n = c.n;
  x.S = (int)d.size();
  x.limbs = limbs;
  x.dig = dig > 0 ? dig : c.alpha;
  x.ndig = (limbs + x.dig - 1) / x.dig;
  x.nt = limbs + c.alpha;
  for (int t = 0; t < x.nt; ++t) x.tprime.push_back(t < limbs ? t : c.P_index(t - limbs));
  x.per = (size_t)x.ndig * x.nt * n;
  x.src = d;
  BufPtr dcoef = make_buf(c, (size_t)x.S * limbs * n);
  if (fused_path(c)) {
    x.col_only = c.ks_row && !full_ext;
    // inverse row pass (out of place) -> per digit: fused [inverse column pass,
    // conversion, forward column pass] straight into ext -> forward row pass
    LimbBatch lb;
    for (int s = 0; s < x.S; ++s)
      for (int l = 0; l < limbs; ++l) {
        lb.add(const_cast<u64*>(d[s]) + (size_t)l * n, l, dcoef->p + ((size_t)s * limbs + l) * n);
        if (lb.count == kMaxBatch) b_row(c, lb, true), lb.count = 0;
      }
    if (lb.count) b_row(c, lb, true), lb.count = 0;
    x.buf = make_buf(c, (size_t)x.S * x.per);
    for (int j = 0; j < x.ndig; ++j) {
      const int lo = j * x.dig, hi = std::min((j + 1) * x.dig, limbs);
      std::vector<int> src, dst, slot;
      for (int i = lo; i < hi; ++i) src.push_back(i);
      for (int t = 0; t < x.nt; ++t)
        if (t < lo || t >= hi) dst.push_back(x.tprime[t]), slot.push_back(t);
      const ConvPlan& plan = conv_plan(c, src, dst);
      FusedColArgs A;
      A.ns = hi - lo;
      A.nd = (int)dst.size();
      A.mode = 0;
      A.set_plan(plan.tab->p, plan.nsrc, plan.ndst);
      for (int i = 0; i < A.ns; ++i) A.src_prime[i] = src[i];
      for (int k = 0; k < A.nd; ++k) A.dst_prime[k] = dst[k], A.out_slot[k] = slot[k];
      CopyBatch cb;
      auto ext_of = [&](int s) { return x.buf->p + (size_t)s * x.per + (size_t)j * x.nt * n; };
      for (int s = 0; s < x.S; ++s) {
        A.src[A.count] = dcoef->p + ((size_t)s * limbs + lo) * n;
        A.dst[A.count++] = ext_of(s);
        if (A.count == kJobsWide) b_fused_col(c, A), A.count = 0;
        if (x.col_only || full_ext) continue;
        cb.src[cb.count] = d[s] + (size_t)lo * n;  // own primes: the exact NTT-domain residues
        cb.dst[cb.count++] = ext_of(s) + (size_t)lo * n;
        if (cb.count == kJobsWide) b_copy(c, cb, (size_t)(hi - lo) * n), cb.count = 0;
      }
      if (A.count) b_fused_col(c, A);
      if (x.col_only) continue;
      if (!full_ext) b_copy(c, cb, (size_t)(hi - lo) * n);
      for (int s = 0; s < x.S; ++s)
        for (size_t k = 0; k < slot.size(); ++k) {
          lb.add(ext_of(s) + (size_t)slot[k] * n, dst[k]);
          if (lb.count == kMaxBatch) b_row(c, lb, false), lb.count = 0;
        }
      if (lb.count) b_row(c, lb, false), lb.count = 0;
    }
    return x;
  }
  {
    CopyBatch cb;
    for (int s = 0; s < x.S; ++s) {
      cb.src[cb.count] = d[s];
      cb.dst[cb.count++] = dcoef->p + (size_t)s * limbs * n;
      if (cb.count == kJobsWide) b_copy(c, cb, (size_t)limbs * n), cb.count = 0;
    }
    b_copy(c, cb, (size_t)limbs * n);
    LimbBatch lb;
    for (int s = 0; s < x.S; ++s)
      for (int l = 0; l < limbs; ++l) ntt_push(c, lb, dcoef->p + ((size_t)s * limbs + l) * n, l, true);
    ntt_batch(c, lb, true);
  }
  x.buf = make_buf(c, (size_t)x.S * x.per);
  LimbBatch lb;
  for (int j = 0; j < x.ndig; ++j) {
    const int lo = j * x.dig, hi = std::min((j + 1) * x.dig, limbs);
    std::vector<int> src, dst, slot;
    for (int i = lo; i < hi; ++i) src.push_back(i);
    for (int t = 0; t < x.nt; ++t)
      if (t < lo || t >= hi) dst.push_back(x.tprime[t]), slot.push_back(t);
    const ConvPlan& plan = conv_plan(c, src, dst);
    ConvBatch cv;
    fill_conv(cv, c, plan);
    for (size_t k = 0; k < slot.size(); ++k) cv.out_slot[k] = slot[k];
    CopyBatch cb;
    auto ext_of = [&](int s) { return x.buf->p + (size_t)s * x.per + (size_t)j * x.nt * n; };
    for (int s = 0; s < x.S; ++s) {
      u64* e = ext_of(s);
      cv.in[cv.count] = dcoef->p + ((size_t)s * limbs + lo) * n;
      cv.out[cv.count++] = e;
      if (cv.count == kJobsWide) b_conv(c, cv), cv.count = 0;
      cb.src[cb.count] = d[s] + (size_t)lo * n;  // own primes: the exact NTT-domain residues
      cb.dst[cb.count++] = e + (size_t)lo * n;
      if (cb.count == kJobsWide) b_copy(c, cb, (size_t)(hi - lo) * n), cb.count = 0;
    }
    b_conv(c, cv);
    b_copy(c, cb, (size_t)(hi - lo) * n);
    // forward NTT of the converted limbs, enqueued after every conversion
    for (int s = 0; s < x.S; ++s)
      for (size_t k = 0; k < slot.size(); ++k) ntt_push(c, lb, ext_of(s) + (size_t)slot[k] * n, dst[k], false);
    ntt_batch(c, lb, false);
  }
  return x;
}

struct KsJob {
  int src;
  u64 g;             // automorphism applied to ext and to the addends (<= 1: none)
  const u64* add0;   // added to the b-part after ModDown (c0 / d0) or null
  const u64* add1;   // added to the a-part (d1) or null
  u64* out0;
  u64* out1;
};

// Inner products + ModDown for every job (chunks of kJobs).
// (q_top * P)^-1 mod q_l (+ Shoup), l < limbs - 1: the merged relinearise + rescale constants
const std::vector<u64>& merged_consts(Context& c, int limbs, const u64** dev) {
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.merged_consts_h.find(limbs);
  if (it == c.merged_consts_h.end()) {
    std::vector<u64> h(2 * (size_t)(limbs - 1));
    const u64 qt = c.primes[limbs - 1];
    for (int l = 0; l < limbs - 1; ++l) {
      const u64 q = c.primes[l];
      u64 m = qt % q;
      for (int k = 0; k < c.alpha; ++k) m = mulmod_h(m, c.primes[c.P_index(k)] % q, q);
      h[l] = invmod_h(m, q);
      h[limbs - 1 + l] = shoup_h(h[l], q);
    }
    BufPtr b = make_buf(c, h.size());
    SF_CUDA(cudaMemcpyAsync(b->p, h.data(), h.size() * sizeof(u64), cudaMemcpyHostToDevice, c.stream));
    host_sync(c);
    c.merged_consts[limbs] = b;
    it = c.merged_consts_h.emplace(limbs, std::move(h)).first;
  }
  *dev = c.merged_consts[limbs]->p;
  return it->second;
}

// ModDown and rescale by the top prime as one conversion:
// out = (X_Q' - conv_{M -> Q'}(X_M)) * M^-1, M = {q_top} u P, Q' = q_0..q_{limbs-2};
// X = [limbs + alpha][n] with the q_top and P limbs inverse-row-passed (fused
// path) or NTT domain (generic path).
void mod_down_rescale_polys(Context& c, int limbs, const std::vector<MdPoly>& P, bool rowpassed) {
  SF_HPROF("mod_down_rescale_polys");
  const size_t n = c.n;
  const int L1 = limbs - 1;
  std::vector<int> mp{L1}, qidx;
  for (int k = 0; k < c.alpha; ++k) mp.push_back(c.P_index(k));
  for (int l = 0; l < L1; ++l) qidx.push_back(l);
  const ConvPlan& plan = conv_plan(c, mp, qidx);
  const u64* kd = nullptr;
  const std::vector<u64>& kh = merged_consts(c, limbs, &kd);
  for (size_t s0 = 0; s0 < P.size(); s0 += kJobsWide) {
    const int J = (int)std::min<size_t>(kJobsWide, P.size() - s0);
    BufPtr conv = make_buf(c, (size_t)J * L1 * n);
    if (fused_path(c)) {
      require(rowpassed, kInternal, "mod_down_rescale: fused path expects row-passed inputs");
      FusedColArgs A;
      A.ns = (int)mp.size();
      A.nd = L1;
      A.set_plan(plan.tab->p, plan.nsrc, plan.ndst);
      for (int k = 0; k < A.ns; ++k) A.src_prime[k] = mp[k];
      for (int l = 0; l < L1; ++l) A.dst_prime[l] = l, A.out_slot[l] = l;
      for (int j = 0; j < J; ++j) {
        A.src[A.count] = P[s0 + j].acc + (size_t)L1 * n;
        A.dst[A.count++] = conv->p + (size_t)j * L1 * n;
      }
      b_fused_col(c, A);
      EpiBatch E;
      for (int j = 0; j < J; ++j)
        for (int l = 0; l < L1; ++l) {
          E.buf[E.count] = conv->p + ((size_t)j * L1 + l) * n;
          E.acc[E.count] = P[s0 + j].acc + (size_t)l * n;
          E.addend[E.count] = nullptr;
          E.out[E.count] = P[s0 + j].out + (size_t)l * n;
          E.g[E.count] = 0;
          E.inv[E.count] = kh[l];
          E.inv_s[E.count] = kh[L1 + l];
          E.prime[E.count++] = (uint8_t)l;
          if (E.count == kJobsWide) b_row_epi(c, E), E.count = 0;
        }
      b_row_epi(c, E);
      continue;
    }
    LimbBatch lb;
    for (int j = 0; j < J; ++j)
      for (size_t k = 0; k < mp.size(); ++k)
        ntt_push(c, lb, const_cast<u64*>(P[s0 + j].acc) + (size_t)(L1 + k) * n, mp[k], true);
    ntt_batch(c, lb, true);
    ConvBatch cv;
    fill_conv(cv, c, plan);
    for (int l = 0; l < L1; ++l) cv.out_slot[l] = l;
    for (int j = 0; j < J; ++j) {
      cv.in[cv.count] = P[s0 + j].acc + (size_t)L1 * n;
      cv.out[cv.count++] = conv->p + (size_t)j * L1 * n;
    }
    b_conv(c, cv);
    for (int j = 0; j < J; ++j)
      for (int l = 0; l < L1; ++l) ntt_push(c, lb, conv->p + ((size_t)j * L1 + l) * n, l, false);
    ntt_batch(c, lb, false);
    SubScaleBatch sb;
    for (int j = 0; j < J; ++j) {
      sb.acc[sb.count] = P[s0 + j].acc;
      sb.conv[sb.count] = conv->p + (size_t)j * L1 * n;
      sb.addend[sb.count] = nullptr;
      sb.g[sb.count] = 0;
      sb.out[sb.count++] = P[s0 + j].out;
    }
    b_subscale(c, sb, L1, kd, kd + L1);
  }
}

void ks_jobs(Context& c, const ExtB& x, const std::vector<KsJob>& jobs, bool merged = false) {
  SF_HPROF("ks_jobs");
  const size_t n = c.n;
  const int limbs = x.limbs, nt = x.nt;
  const u64* kc = level_consts(c, limbs);
  std::vector<int> pidx, qidx;
  for (int k = 0; k < c.alpha; ++k) pidx.push_back(c.P_index(k));
  for (int l = 0; l < limbs; ++l) qidx.push_back(l);
  // fused rotations: keys with P^-1 on the Q limbs, ModDown without the final multiply
  const bool pre = fused_path(c) && x.col_only && !merged;
  const ConvPlan& down = conv_plan(c, pidx, qidx, pre);
  for (size_t s0 = 0; s0 < jobs.size(); s0 += kJobs) {
    const int J = (int)std::min<size_t>(kJobs, jobs.size() - s0);
    BufPtr acc = make_buf(c, (size_t)J * 2 * nt * n);
    auto accp = [&](int j, int poly) { return acc->p + ((size_t)j * 2 + poly) * nt * n; };
    if (x.col_only) {
      // fused: forward row pass of ext + automorphism + inner product + ModDown's
      // inverse row pass of the special primes, one launch (jobs grouped by source)
      KsRowArgs ka;
      ka.limbs = limbs;
      ka.nt = nt;
      ka.ndig = x.ndig;
      ka.alpha = x.dig;  // digit size (own-prime rows of each digit)
      ka.np = c.np;
      for (int t = 0; t < nt; ++t) ka.tprime[t] = x.tprime[t];
      std::vector<int> order(J);
      for (int j = 0; j < J; ++j) order[j] = j;
      std::stable_sort(order.begin(), order.end(),
                       [&](int a, int b) { return jobs[s0 + a].src < jobs[s0 + b].src; });
      // work units = (source, chunk of its jobs); a source with many hoisted
      // jobs is split so the grid still covers the GPU (each unit recomputes
      // the source rows' forward row pass, a small cost next to its jobs)
      int nsrc_present = 0;
      for (int k = 0; k < J; ++k)
        if (k == 0 || jobs[s0 + order[k]].src != jobs[s0 + order[k - 1]].src) ++nsrc_present;
      const int tiles = (1 << (c.logn / 2)) / 8;
      const int want_units = (1184 + nt * tiles - 1) / (nt * tiles);
      const int chunks = nsrc_present >= want_units ? 1 : (want_units + nsrc_present - 1) / nsrc_present;
      int prev = -1, run_begin = 0;
      for (int k = 0; k < J; ++k) {
        const int j = order[k];
        const KsJob& jb = jobs[s0 + j];
        if (jb.src != prev) {
          int run = 1;
          while (k + run < J && jobs[s0 + order[k + run]].src == jb.src) ++run;
          run_begin = k;
          prev = jb.src;
          (void)run;
          ka.c1[ka.nsrc] = x.src[jb.src];
          ka.ext[ka.nsrc] = x.ext(jb.src);
          ka.job_begin[ka.nsrc++] = k;
          ka.run_len = run;
        } else if (chunks > 1 && (k - run_begin) % ((ka.run_len + chunks - 1) / chunks) == 0) {
          ka.c1[ka.nsrc] = x.src[jb.src];
          ka.ext[ka.nsrc] = x.ext(jb.src);
          ka.job_begin[ka.nsrc++] = k;
        }
        ka.g[k] = jb.g;
        u64 gi = 1;  // g^-1 mod 2n = g^(n-1) (the unit group mod 2n has order n)
        if (jb.g > 1)
          for (u64 e = (u64)n - 1, b = jb.g, m2 = 2ull * n - 1; e; e >>= 1, b = (b * b) & m2)
            if (e & 1) gi = (gi * b) & m2;
        ka.ginv[k] = gi;
        ka.key[k] = get_key_mont(c, jb.g <= 1 ? (x.dig != c.alpha ? kRelinWide : 0) : jb.g, pre, x.ndig)->p;
        ka.acc[k] = accp(j, 0);
        ka.add0[k] = jb.add0;
        ka.add1[k] = jb.add1;
      }
      ka.job_begin[ka.nsrc] = J;
      if (merged) {
        ka.merged = 1;
        for (int l = 0; l < limbs; ++l) {
          u64 r = c.r64[l];  // P * R mod q (Montgomery-scaled like the keys)
          for (int k = 0; k < c.alpha; ++k) r = mulmod_h(r, c.primes[c.P_index(k)] % c.primes[l], c.primes[l]);
          ka.pm[l] = r;
        }
      }
      b_ks_row(c, ka);
    }
    KsBatch kb;
    kb.ndig = x.ndig;
    kb.nt = nt;
    kb.np = c.np;
    kb.logn = c.logn;
    for (int t = 0; t < nt; ++t) kb.tprime[t] = x.tprime[t];
    for (int j = 0; j < J; ++j) {
      const KsJob& jb = jobs[s0 + j];
      kb.ext[j] = x.ext(jb.src);
      kb.key[j] = get_key(c, jb.g <= 1 ? (x.dig != c.alpha ? kRelinWide : 0) : jb.g)->p;
      kb.g[j] = jb.g;
      kb.accb[j] = accp(j, 0);
      kb.acca[j] = accp(j, 1);
    }
    kb.count = J;
    if (!x.col_only) b_ks(c, kb);
    if (merged) {
      // X = acc + P (d0, d1) on the Q limbs, then one ModDown-and-rescale
      std::vector<MdPoly> md;
      if (!x.col_only) {
        const u64* kd = nullptr;
        (void)kd;
        std::vector<u64> pmh(limbs);
        for (int l = 0; l < limbs; ++l) {
          u64 r = 1 % c.primes[l];
          for (int k = 0; k < c.alpha; ++k) r = mulmod_h(r, c.primes[c.P_index(k)] % c.primes[l], c.primes[l]);
          pmh[l] = r;
        }
        BufPtr pmd = make_buf(c, limbs);
        SF_CUDA(cudaMemcpyAsync(pmd->p, pmh.data(), limbs * sizeof(u64), cudaMemcpyHostToDevice, c.stream));
        AxpyBatch ab;
        for (int j = 0; j < J; ++j)
          for (int poly = 0; poly < 2; ++poly) {
            ab.acc[ab.count] = accp(j, poly);
            ab.d[ab.count++] = poly ? jobs[s0 + j].add1 : jobs[s0 + j].add0;
          }
        b_axpy_pm(c, ab, limbs, pmd->p);
        host_sync(c);  // pmh outlives the copy (generic small-ring path only)
      }
      for (int j = 0; j < J; ++j)
        for (int poly = 0; poly < 2; ++poly) md.push_back({accp(j, poly), nullptr, 0, poly ? jobs[s0 + j].out1 : jobs[s0 + j].out0});
      mod_down_rescale_polys(c, limbs, md, x.col_only);
      continue;
    }
    if (fused_path(c)) {
      // ModDown of 2J polynomials: inverse row pass of the P limbs (in place),
      // fused [inverse column, P -> Q conversion, forward column], then the
      // forward row pass with the (acc - conv) * P^-1 (+ addend) epilogue
      const std::vector<u64>& kh = c.level_consts_h[limbs];
      LimbBatch lb;
      if (!x.col_only) {
        for (int j = 0; j < J; ++j)
          for (int poly = 0; poly < 2; ++poly)
            for (int k = 0; k < c.alpha; ++k) {
              lb.add(accp(j, poly) + (size_t)(limbs + k) * n, pidx[k]);
              if (lb.count == kMaxBatch) b_row(c, lb, true), lb.count = 0;
            }
        b_row(c, lb, true);
      }
      BufPtr conv = make_buf(c, (size_t)J * 2 * limbs * n);
      FusedColArgs A;
      A.ns = c.alpha;
      A.nd = limbs;
      A.set_plan(down.tab->p, down.nsrc, down.ndst);
      for (int k = 0; k < c.alpha; ++k) A.src_prime[k] = pidx[k];
      for (int l = 0; l < limbs; ++l) A.dst_prime[l] = l, A.out_slot[l] = l;
      for (int j = 0; j < J; ++j)
        for (int poly = 0; poly < 2; ++poly) {
          A.src[A.count] = accp(j, poly) + (size_t)limbs * n;
          A.dst[A.count++] = conv->p + ((size_t)j * 2 + poly) * limbs * n;
        }
      b_fused_col(c, A);
      EpiBatch E;
      E.nomul = pre;
      for (int j = 0; j < J; ++j) {
        const KsJob& jb = jobs[s0 + j];
        for (int poly = 0; poly < 2; ++poly) {
          const u64* add = poly ? jb.add1 : jb.add0;
          u64* out = poly ? jb.out1 : jb.out0;
          for (int l = 0; l < limbs; ++l) {
            E.buf[E.count] = conv->p + (((size_t)j * 2 + poly) * limbs + l) * n;
            E.acc[E.count] = accp(j, poly) + (size_t)l * n;
            E.addend[E.count] = add ? add + (size_t)l * n : nullptr;
            E.out[E.count] = out + (size_t)l * n;
            E.g[E.count] = jb.g;
            E.inv[E.count] = kh[2 * limbs + l];
            E.inv_s[E.count] = kh[3 * limbs + l];
            E.prime[E.count++] = (uint8_t)l;
            if (E.count == kJobsWide) b_row_epi(c, E), E.count = 0;
          }
        }
      }
      b_row_epi(c, E);
      continue;
    }
    // ModDown of 2J polynomials
    LimbBatch lb;
    for (int j = 0; j < J; ++j)
      for (int poly = 0; poly < 2; ++poly)
        for (int k = 0; k < c.alpha; ++k) ntt_push(c, lb, accp(j, poly) + (size_t)(limbs + k) * n, pidx[k], true);
    ntt_batch(c, lb, true);
    BufPtr conv = make_buf(c, (size_t)J * 2 * limbs * n);
    ConvBatch cv;
    fill_conv(cv, c, down);
    for (int l = 0; l < limbs; ++l) cv.out_slot[l] = l;
    for (int j = 0; j < J; ++j)
      for (int poly = 0; poly < 2; ++poly) {
        cv.in[cv.count] = accp(j, poly) + (size_t)limbs * n;
        cv.out[cv.count++] = conv->p + ((size_t)j * 2 + poly) * limbs * n;
      }
    b_conv(c, cv);
    for (int j = 0; j < J; ++j)
      for (int poly = 0; poly < 2; ++poly)
        for (int l = 0; l < limbs; ++l) ntt_push(c, lb, conv->p + (((size_t)j * 2 + poly) * limbs + l) * n, l, false);
    ntt_batch(c, lb, false);
    SubScaleBatch sb;
    for (int j = 0; j < J; ++j) {
      const KsJob& jb = jobs[s0 + j];
      for (int poly = 0; poly < 2; ++poly) {
        sb.acc[sb.count] = accp(j, poly);
        sb.conv[sb.count] = conv->p + ((size_t)j * 2 + poly) * limbs * n;
        sb.addend[sb.count] = poly ? jb.add1 : jb.add0;
        sb.g[sb.count] = jb.g;
        sb.out[sb.count++] = poly ? jb.out1 : jb.out0;
      }
    }
    b_subscale(c, sb, limbs, kc + 2 * limbs, kc + 3 * limbs);
  }
}

}  // namespace

// ---------------------------------------------------------- ModDown of polys
// out = (acc_Q - conv_{P->Q}(acc_P)) * P^-1 (+ addend permuted by g) for
// extended-basis polynomials acc = [nt][n]. p_rowpassed: the P limbs already
// had ModDown's inverse row pass (fused path); otherwise they are NTT domain.

void mod_down_polys(Context& c, int limbs, const std::vector<MdPoly>& P, bool p_rowpassed, bool prescaled = false) {
  SF_HPROF("mod_down_polys");
  const size_t n = c.n;
  std::vector<int> pidx, qidx;
  for (int k = 0; k < c.alpha; ++k) pidx.push_back(c.P_index(k));
  for (int l = 0; l < limbs; ++l) qidx.push_back(l);
  require(!prescaled || fused_path(c), kInternal, "mod_down_polys: P^-1-prescaled input needs the fused path");
  // prescaled: the Q limbs of acc already carry P^-1, so the conversion constants
  // do too and the combine is a plain subtraction
  const ConvPlan& down = conv_plan(c, pidx, qidx, prescaled);
  const u64* kc = level_consts(c, limbs);
  for (size_t s0 = 0; s0 < P.size(); s0 += kJobsWide) {
    const int J = (int)std::min<size_t>(kJobsWide, P.size() - s0);
    BufPtr conv = make_buf(c, (size_t)J * limbs * n);
    if (fused_path(c)) {
      LimbBatch lb;
      if (!p_rowpassed) {
        for (int j = 0; j < J; ++j)
          for (int k = 0; k < c.alpha; ++k) {
            lb.add(const_cast<u64*>(P[s0 + j].acc) + (size_t)(limbs + k) * n, pidx[k]);
            if (lb.count == kMaxBatch) b_row(c, lb, true), lb.count = 0;
          }
        b_row(c, lb, true);
      }
      const std::vector<u64>& kh = c.level_consts_h[limbs];
      FusedColArgs A;
      A.ns = c.alpha;
      A.nd = limbs;
      A.set_plan(down.tab->p, down.nsrc, down.ndst);
      for (int k = 0; k < c.alpha; ++k) A.src_prime[k] = pidx[k];
      for (int l = 0; l < limbs; ++l) A.dst_prime[l] = l, A.out_slot[l] = l;
      for (int j = 0; j < J; ++j) {
        A.src[A.count] = P[s0 + j].acc + (size_t)limbs * n;
        A.dst[A.count++] = conv->p + (size_t)j * limbs * n;
      }
      b_fused_col(c, A);
      EpiBatch E;
      E.nomul = prescaled;
      for (int j = 0; j < J; ++j) {
        const MdPoly& m = P[s0 + j];
        for (int l = 0; l < limbs; ++l) {
          E.buf[E.count] = conv->p + ((size_t)j * limbs + l) * n;
          E.acc[E.count] = m.acc + (size_t)l * n;
          E.addend[E.count] = m.addend ? m.addend + (size_t)l * n : nullptr;
          E.out[E.count] = m.out + (size_t)l * n;
          E.g[E.count] = m.g;
          E.inv[E.count] = kh[2 * limbs + l];
          E.inv_s[E.count] = kh[3 * limbs + l];
          E.post[E.count] = m.post ? m.post + (size_t)l * n : nullptr;
          E.prime[E.count++] = (uint8_t)l;
          if (E.count == kJobsWide) b_row_epi(c, E), E.count = 0;
        }
      }
      b_row_epi(c, E);
      continue;
    }
    require(!p_rowpassed, kInternal, "mod_down_polys: row-passed input on the generic path");
    for (const MdPoly& m : P) require(m.post == nullptr, kInternal, "mod_down_polys: post multiplier needs the fused path");
    LimbBatch lb;
    for (int j = 0; j < J; ++j)
      for (int k = 0; k < c.alpha; ++k)
        ntt_push(c, lb, const_cast<u64*>(P[s0 + j].acc) + (size_t)(limbs + k) * n, pidx[k], true);
    ntt_batch(c, lb, true);
    ConvBatch cv;
    fill_conv(cv, c, down);
    for (int l = 0; l < limbs; ++l) cv.out_slot[l] = l;
    for (int j = 0; j < J; ++j) {
      cv.in[cv.count] = P[s0 + j].acc + (size_t)limbs * n;
      cv.out[cv.count++] = conv->p + (size_t)j * limbs * n;
    }
    b_conv(c, cv);
    for (int j = 0; j < J; ++j)
      for (int l = 0; l < limbs; ++l) ntt_push(c, lb, conv->p + ((size_t)j * limbs + l) * n, l, false);
    ntt_batch(c, lb, false);
    SubScaleBatch sb;
    for (int j = 0; j < J; ++j) {
      sb.acc[sb.count] = P[s0 + j].acc;
      sb.conv[sb.count] = conv->p + (size_t)j * limbs * n;
      sb.addend[sb.count] = P[s0 + j].addend;
      sb.g[sb.count] = P[s0 + j].g;
      sb.out[sb.count++] = P[s0 + j].out;
    }
    b_subscale(c, sb, limbs, kc + 2 * limbs, kc + 3 * limbs);
  }
}

// ------------------------------------------------------------ rotation sums
// sum_i Rot(a_i, r_i) accumulated in the extended basis and
// brought back with one ModDown per part; the same function as the CPU
// oracle's rot_sum, charged as the reference's rotate/add chain.
std::vector<Ct> rot_sum_batch(Context& c, const std::vector<std::vector<SumTerm>>& groups, bool hoisted, bool count,
                              const std::vector<const Pt*>* post, bool rescale, int dig, std::vector<ExtPoly>* keep_b,
                              const std::map<const Ct*, const u64*>* ext_b) {
  SF_HPROF("rot_sum_batch");
  require(!(keep_b || ext_b) || (fused_path(c) && !rescale && dig == 0), kInternal, "rot_sum: double hoisting");
  if (keep_b) keep_b->assign(groups.size(), ExtPoly());
  require(!post || (post->size() == groups.size() && fused_path(c)), kInternal, "rot_sum: post multipliers");
  require(!(post && rescale), kInternal, "rot_sum: post multipliers with a merged rescale");
  std::vector<Ct> out(groups.size());
  std::map<int, std::vector<int>> by_limbs;
  for (size_t gi = 0; gi < groups.size(); ++gi) {
    const auto& G = groups[gi];
    require(!G.empty(), kShapeMismatch, "rot_sum: empty term list");
    int limbs = 1 << 30;
    const Ct* first = nullptr;
    OptLayout ly;
    for (size_t i = 0; i < G.size(); ++i) {
      const Ct& a = *G[i].ct;
      check_ct(c, a, "rotate");
      const bool rot = pos_mod(G[i].r, c.slots) != 0;
      if (count && rot) c.ledger.rot(hoisted);
      limbs = std::min(limbs, a.limbs);
      OptLayout t_ly = rot ? OptLayout() : a.layout;
      if (i == 0)
        ly = t_ly;
      else if (!(ly && t_ly && *ly == *t_ly))
        ly.reset();
      if (a.zero) continue;
      if (!first)
        first = &a;
      else
        check_scales(*first, a, "add");
    }
    if (count) c.ledger.add((long long)G.size() - 1);
    if (rescale) require(limbs > 1, kLevelUnderflow, "mul_plain: no multiplicative level left");
    if (!first) {
      Ct z = *G[0].ct;
      z.limbs = rescale ? limbs - 1 : limbs;
      z.layout = ly;
      out[gi] = z;
      continue;
    }
    out[gi] = rescale ? alloc_ct(c, limbs - 1, first->scale / (double)c.primes[limbs - 1])
                      : alloc_ct(c, limbs, first->scale);
    out[gi].layout = ly;
    by_limbs[limbs].push_back((int)gi);
  }
  const size_t n = c.n;
  for (auto& [limbs, gidx] : by_limbs) {
    std::vector<u64> pm(limbs);
    // fused path: Montgomery keys (R-scaled) with P^-1 on the
    // Q limbs (bit-identical results, fewer products); the merged ModDown +
    // rescale converts the unscaled sum (keys and pm times R only)
    const bool fused = fused_path(c);
    const bool pre = fused && !rescale;
    for (int l = 0; l < limbs; ++l) {
      u64 r = fused ? c.r64[l] : 1 % c.primes[l];
      for (int k = 0; k < c.alpha; ++k) r = mulmod_h(r, c.primes[c.P_index(k)] % c.primes[l], c.primes[l]);
      pm[l] = pre ? 1 : r;
    }
    size_t gpos = 0;
    while (gpos < gidx.size()) {
      // chunk: <= kSumOuts outputs, <= kSumJobs jobs, <= kSumSrcs sources
      std::map<const Ct*, int> src;
      std::vector<const Ct*> srcv;
      std::vector<int> chunk;
      int njobs = 0;
      while (gpos < gidx.size()) {
        const auto& G = groups[gidx[gpos]];
        int newsrc = 0;
        for (const auto& tm : G)
          if (!tm.ct->zero && !src.count(tm.ct)) ++newsrc;
        if (!chunk.empty() && ((int)chunk.size() == kSumOuts || njobs + (int)G.size() > kSumJobs ||
                               (int)srcv.size() + newsrc > kSumSrcs))
          break;
        require((int)G.size() <= kSumJobs && newsrc <= kSumSrcs, kShapeMismatch, "rot_sum: too many terms");
        for (const auto& tm : G)
          if (!tm.ct->zero && !src.count(tm.ct)) src[tm.ct] = (int)srcv.size(), srcv.push_back(tm.ct);
        njobs += (int)G.size();
        chunk.push_back(gidx[gpos++]);
      }
      std::vector<const u64*> d;
      for (const Ct* a : srcv) d.push_back(a->c1(c.n));
      ExtB x = mod_up_batch(c, d, limbs, true, dig);
      const int nt = x.nt;
      BufPtr acc = make_buf(c, chunk.size() * 2 * nt * n);
      KsSumArgs A;
      A.limbs = limbs;
      A.nt = nt;
      A.ndig = x.ndig;
      A.alpha = x.dig;  // digit size
      A.np = c.np;
      for (int t = 0; t < nt; ++t) A.tprime[t] = x.tprime[t];
      for (int l = 0; l < limbs; ++l) A.pm[l] = pm[l];
      A.pm_one = pre;
      if (rescale) A.inv_from = limbs - 1;
      A.keep_b = keep_b != nullptr;
      A.ext_c0 = ext_b != nullptr;
      for (size_t s = 0; s < srcv.size(); ++s) {
        if (ext_b) {
          auto e = ext_b->find(srcv[s]);
          require(e != ext_b->end(), kInternal, "rot_sum: source without its extended b part");
          A.c0[s] = e->second;
        } else {
          A.c0[s] = srcv[s]->c0();
        }
        A.c1[s] = srcv[s]->c1(c.n);
        A.ext[s] = x.ext((int)s);
      }
      int jb = 0;
      std::vector<MdPoly> md;
      for (size_t o = 0; o < chunk.size(); ++o) {
        A.out_begin[o] = jb;
        A.acc[o] = acc->p + o * 2 * nt * n;
        for (const auto& tm : groups[chunk[o]]) {
          if (tm.ct->zero) continue;
          const int r = pos_mod(tm.r, c.slots);
          A.jsrc[jb] = src[tm.ct];
          A.g[jb] = r == 0 ? 1 : galois_elt(c, r);
          const u64 kid = key_id(A.g[jb], x.dig, c.alpha);
          A.key[jb] = r == 0 ? nullptr : (fused ? get_key_mont(c, kid, pre, x.ndig) : get_key(c, kid))->p;
          ++jb;
        }
        const Ct& y = out[chunk[o]];
        const u64* pp = post ? (*post)[chunk[o]]->buf->p : nullptr;
        if (keep_b)
          (*keep_b)[chunk[o]] = ExtPoly{acc, A.acc[o]};
        else
          md.push_back({A.acc[o], nullptr, 0, y.c0(), pp});
        md.push_back({A.acc[o] + (size_t)nt * n, nullptr, 0, y.c1(c.n), pp});
      }
      A.out_begin[chunk.size()] = jb;
      A.nout = (int)chunk.size();
      b_ks_sum(c, A);
      if (rescale)
        mod_down_rescale_polys(c, limbs, md, fused_path(c));
      else
        mod_down_polys(c, limbs, md, fused_path(c), pre);
    }
  }
  return out;
}

// Doubling chains x <- x + Rot(x, r_i), i < m, of many ciphertexts (each with
// its own amounts): fold_within_head, replicate_lanes, fold_lanes and the VMM
// ladders (kv_attention.cpp:30-47, vmm.cpp:190-193, 226-230). The value is
// sum_{k < 2^m} Rot(x, sum_i bit_i(k) r_i), evaluated as the radix rotation sums
// of DESIGN.md §3.8 (m <= 3 bits in one sum, else ceil(m/2) then floor(m/2));
// charged as the reference's m rotate + add steps per ciphertext.
std::vector<Ct> fold_steps_batch(Context& c, const std::vector<const Ct*>& xs, const std::vector<std::vector<int>>& rots,
                                 bool count, bool lead, const std::vector<const Pt*>* post,
                                 const std::vector<int>* shift) {
  SF_HPROF("fold_steps_batch");
  std::vector<bool> posted(xs.size(), false);
  require(xs.size() == rots.size(), kShapeMismatch, "fold_steps: operand count");
  std::vector<Ct> cur;
  size_t mmax = 0;
  for (size_t i = 0; i < xs.size(); ++i) {
    check_ct(c, *xs[i], "rotate");
    if (count && lead) {
      for (int r : rots[i])
        if (pos_mod(r, c.slots) != 0) c.ledger.rot(false);
      c.ledger.add((long long)rots[i].size());
    }
    cur.push_back(*xs[i]);
    mmax = std::max(mmax, rots[i].size());
  }
  // all chains share the radix schedule of their own length; group by length
  std::map<int, std::vector<int>> by_len;
  for (size_t i = 0; i < xs.size(); ++i) by_len[(int)rots[i].size()].push_back((int)i);
  for (auto& [m, idx] : by_len) {
    if (m == 0 && !shift) continue;
    std::vector<int> steps;  // an empty chain with a shift: one single-term sum (the rotation)
    if (m <= 3)
      steps.push_back(m);
    else
      steps.push_back((m + 1) / 2), steps.push_back(m / 2);
    // double hoisting: the first radix sum's b part stays in the
    // extended basis and enters the second sum as its c0 terms -- one ModDown
    // (the first sum's b part) fewer; SF_VARIANT bit 8 turns it off (A/B only:
    // the CPU twin always hoists on this path)
    const bool dh = steps.size() == 2 && fused_path(c) && !(c.variant & 256);
    std::vector<ExtPoly> kept;
    std::map<const Ct*, const u64*> ext;
    int lo = 0;
    for (size_t si = 0; si < steps.size(); ++si) {
      const int bits = steps[si];
      const bool last = si + 1 == steps.size();
      std::vector<std::vector<SumTerm>> groups(idx.size());
      for (size_t g = 0; g < idx.size(); ++g) {
        const std::vector<int>& rs = rots[idx[g]];
        for (int k = 0; k < (1 << bits); ++k) {
          long long r = (shift && last) ? (*shift)[idx[g]] : 0;  // Rot(sum, s): every last-step term moves by s
          for (int i = 0; i < bits; ++i)
            if ((k >> i) & 1) r += rs[lo + i];
          groups[g].push_back({&cur[idx[g]], (int)pos_mod(r, c.slots)});
        }
      }
      std::vector<const Pt*> pg;  // the post multipliers ride the last step's ModDown epilogue
      if (post && last)
        for (int g : idx) pg.push_back((*post)[g]), posted[g] = true;
      std::vector<Ct> nxt = rot_sum_batch(c, groups, false, false, (post && last) ? &pg : nullptr, false, 0,
                                          (dh && si == 0) ? &kept : nullptr, (dh && si == 1) ? &ext : nullptr);
      for (size_t g = 0; g < idx.size(); ++g) cur[idx[g]] = std::move(nxt[g]);
      if (dh && si == 0) {
        ext.clear();
        for (size_t g = 0; g < idx.size(); ++g)
          if (kept[g].p) ext[&cur[idx[g]]] = kept[g].p;
      }
      lo += bits;
    }
  }
  for (size_t i = 0; i < xs.size(); ++i) {
    bool all0 = !shift || pos_mod((*shift)[i], c.slots) == 0;
    for (int r : rots[i]) all0 = all0 && pos_mod(r, c.slots) == 0;
    cur[i].layout = all0 ? xs[i]->layout : OptLayout();
    require(!post || posted[i], kInternal, "fold_steps: post multiplier on an empty chain");
  }
  return cur;
}

std::vector<Ct> fold_batch(Context& c, const std::vector<const Ct*>& xs, int d_head, int t, bool count,
                           const std::vector<const Pt*>* post, const std::vector<int>* shift) {
  std::vector<int> rs;
  for (int l = 0; (1 << l) < d_head; ++l) rs.push_back((1 << l) * t);
  return fold_steps_batch(c, xs, std::vector<std::vector<int>>(xs.size(), rs), count, true, post, shift);
}

// -------------------------------------------------------------------- rescale
std::vector<Ct> rescale_batch(Context& c, const std::vector<const Ct*>& xs) {
  SF_HPROF("rescale_batch");
  std::vector<Ct> out(xs.size());
  if (xs.empty()) return out;
  std::map<int, std::vector<int>> by_limbs;
  for (size_t i = 0; i < xs.size(); ++i) by_limbs[xs[i]->limbs].push_back((int)i);
  const size_t n = c.n;
  for (auto& [limbs, idx] : by_limbs) {
    const int L1 = limbs - 1;
    require(L1 >= 1, kLevelUnderflow, "rescale: no prime left to drop");
    const u64* kc = level_consts(c, limbs);
    if (fused_path(c)) {
      // inverse row pass of the top limb (out of place), fused [inverse column,
      // centred lift to the remaining primes, forward column], then the forward
      // row pass with the (c_i - lift_i) * q_top^-1 epilogue
      const std::vector<u64>& kh = c.level_consts_h[limbs];
      for (size_t s0 = 0; s0 < idx.size(); s0 += kJobs) {
        const int J = (int)std::min<size_t>(kJobs, idx.size() - s0);
        BufPtr last = make_buf(c, (size_t)2 * J * n);
        BufPtr lift = make_buf(c, (size_t)2 * J * L1 * n);
        LimbBatch lb;
        FusedColArgs A;
        A.ns = 1;
        A.nd = L1;
        A.mode = 1;
        A.q_last = c.primes[L1];
        A.src_prime[0] = L1;
        for (int l = 0; l < L1; ++l) A.dst_prime[l] = l, A.out_slot[l] = l;
        EpiBatch E;
        auto flush_epi = [&]() {
          b_row_epi(c, E);
          E.count = 0;
        };
        std::vector<std::array<const u64*, 2>> srcs(J);
        for (int j = 0; j < J; ++j) {
          const Ct& x = *xs[idx[s0 + j]];
          Ct r = alloc_ct(c, L1, x.scale / (double)c.primes[L1]);
          r.zero = x.zero;
          r.layout = x.layout;
          for (int poly = 0; poly < 2; ++poly) {
            const u64* src = poly ? x.c1(c.n) : x.c0();
            u64* lp = last->p + (size_t)(2 * j + poly) * n;
            lb.add(const_cast<u64*>(src) + (size_t)L1 * n, L1, lp);
            A.src[A.count] = lp;
            A.dst[A.count++] = lift->p + (size_t)(2 * j + poly) * L1 * n;
          }
          out[idx[s0 + j]] = r;
        }
        b_row(c, lb, true);
        b_fused_col(c, A);
        for (int j = 0; j < J; ++j) {
          const Ct& x = *xs[idx[s0 + j]];
          const Ct& r = out[idx[s0 + j]];
          for (int poly = 0; poly < 2; ++poly)
            for (int l = 0; l < L1; ++l) {
              E.buf[E.count] = lift->p + ((size_t)(2 * j + poly) * L1 + l) * n;
              E.acc[E.count] = (poly ? x.c1(c.n) : x.c0()) + (size_t)l * n;
              E.addend[E.count] = nullptr;
              E.out[E.count] = (poly ? r.c1(c.n) : r.c0()) + (size_t)l * n;
              E.g[E.count] = 0;
              E.inv[E.count] = kh[l];
              E.inv_s[E.count] = kh[limbs + l];
              E.prime[E.count++] = (uint8_t)l;
              if (E.count == kJobsWide) flush_epi();
            }
        }
        flush_epi();
      }
      continue;
    }
    for (size_t s0 = 0; s0 < idx.size(); s0 += kJobs) {
      const int J = (int)std::min<size_t>(kJobs, idx.size() - s0);
      BufPtr last = make_buf(c, (size_t)2 * J * n);
      BufPtr lift = make_buf(c, (size_t)2 * J * L1 * n);
      CopyBatch cb;
      LiftBatch lfb;
      LimbBatch lb;
      SubScaleBatch sb;
      for (int j = 0; j < J; ++j) {
        const Ct& x = *xs[idx[s0 + j]];
        Ct r = alloc_ct(c, L1, x.scale / (double)c.primes[L1]);
        r.zero = x.zero;
        r.layout = x.layout;
        for (int poly = 0; poly < 2; ++poly) {
          const u64* src = poly ? x.c1(c.n) : x.c0();
          u64* lp = last->p + (size_t)(2 * j + poly) * n;
          cb.src[cb.count] = src + (size_t)L1 * n;
          cb.dst[cb.count++] = lp;
          lb.add(lp, L1);
          lfb.x[lfb.count] = lp;
          lfb.out[lfb.count++] = lift->p + (size_t)(2 * j + poly) * L1 * n;
          sb.acc[sb.count] = src;
          sb.conv[sb.count] = lift->p + (size_t)(2 * j + poly) * L1 * n;
          sb.addend[sb.count] = nullptr;
          sb.g[sb.count] = 0;
          sb.out[sb.count++] = poly ? r.c1(c.n) : r.c0();
        }
        out[idx[s0 + j]] = r;
      }
      b_copy(c, cb, n);
      ntt_batch(c, lb, true);
      b_lift(c, lfb, L1, L1);
      for (int j = 0; j < 2 * J; ++j)
        for (int l = 0; l < L1; ++l) ntt_push(c, lb, lift->p + ((size_t)j * L1 + l) * n, l, false);
      ntt_batch(c, lb, false);
      b_subscale(c, sb, L1, kc, kc + limbs);
    }
  }
  return out;
}

Ct rescale(Context& c, const Ct& a) { return rescale_batch(c, {&a})[0]; }

// ------------------------------------------------------------------ rotations
std::vector<Ct> rotate_batch(Context& c, const std::vector<const Ct*>& srcs, const std::vector<RotJob>& jobs,
                             bool hoisted, bool count) {
  SF_HPROF("rotate_batch");
  std::vector<Ct> out(jobs.size());
  // group sources by limb count; one ModUp per distinct source that needs one
  std::map<int, std::vector<int>> need;  // limbs -> source indices
  std::vector<int> uses(srcs.size(), 0);
  for (size_t i = 0; i < jobs.size(); ++i) {
    const Ct& s = *srcs[jobs[i].src];
    check_ct(c, s, "rotate");
    if (pos_mod(jobs[i].r, c.slots) == 0) {
      out[i] = s;
      continue;
    }
    if (count) c.ledger.rot(hoisted);
    if (s.zero) {
      out[i] = s;
      out[i].layout.reset();
      continue;
    }
    if (uses[jobs[i].src]++ == 0) need[s.limbs].push_back(jobs[i].src);
  }
  for (auto& [limbs, sidx] : need) {
    const size_t chunk = c.rot_chunk > 0 ? (size_t)c.rot_chunk : (size_t)kJobs;
    for (size_t c0 = 0; c0 < sidx.size(); c0 += chunk) {  // bound the ModUp working set
      const size_t S = std::min<size_t>(chunk, sidx.size() - c0);
      std::vector<const u64*> d;
      std::map<int, int> local;
      for (size_t s = 0; s < S; ++s) {
        local[sidx[c0 + s]] = (int)s;
        d.push_back(srcs[sidx[c0 + s]]->c1(c.n));
      }
      ExtB x = mod_up_batch(c, d, limbs);
      std::vector<KsJob> kj;
      for (size_t i = 0; i < jobs.size(); ++i) {
        auto it = local.find(jobs[i].src);
        if (it == local.end() || out[i].buf) continue;
        const Ct& s = *srcs[jobs[i].src];
        if (pos_mod(jobs[i].r, c.slots) == 0 || s.zero) continue;
        out[i] = alloc_ct(c, limbs, s.scale);
        kj.push_back({it->second, galois_elt(c, jobs[i].r), s.c0(), nullptr, out[i].c0(), out[i].c1(c.n)});
      }
      ks_jobs(c, x, kj);
    }
  }
  return out;
}

Ct rotate(Context& c, const Ct& a, int r, bool hoisted, bool count) {
  SF_HPROF("rotate");
  return rotate_batch(c, {&a}, {{0, r}}, hoisted, count)[0];
}

std::vector<Ct> rotate_hoisted(Context& c, const Ct& a, const std::vector<int>& rs, bool count) {
  SF_HPROF("rotate_hoisted");
  std::vector<RotJob> jobs;
  for (int r : rs) jobs.push_back({0, r});
  return rotate_batch(c, {&a}, jobs, true, count);
}

// ------------------------------------------------------------- ct x ct mult
std::vector<Ct> mul_batch(Context& c, const std::vector<const Ct*>& a, const std::vector<const Ct*>& b, bool count) {
  SF_HPROF("mul_batch");
  require(a.size() == b.size(), kShapeMismatch, "mul_batch: operand count");
  std::vector<Ct> out(a.size());
  std::map<int, std::vector<int>> by_limbs;
  for (size_t i = 0; i < a.size(); ++i) {
    check_ct(c, *a[i], "mul");
    check_ct(c, *b[i], "mul");
    const int limbs = std::min(a[i]->limbs, b[i]->limbs);
    require(limbs - 1 > 0, kLevelUnderflow, "mul: no multiplicative level left");
    if (count) c.ledger.ctct();
    if (a[i]->zero || b[i]->zero) {
      out[i] = zeros(c, limbs - 2);
      out[i].layout = merge_layouts(*a[i], *b[i]);
      continue;
    }
    by_limbs[limbs].push_back((int)i);
  }
  const size_t n = c.n;
  for (auto& [limbs, idx] : by_limbs) {
    // one shared left operand (the QK^T query against every key ciphertext): its
    // Shoup companions once, then Shoup products (canonical, bit-identical)
    bool shared = idx.size() > 1;
    for (int i : idx) shared = shared && a[i] == a[idx[0]];
    BufPtr as;
    if (shared) {
      const Ct& x = *a[idx[0]];
      BufPtr ac = make_buf(c, (size_t)2 * limbs * n);  // c0, c1 at `limbs` limbs, contiguous
      SF_CUDA(cudaMemcpyAsync(ac->p, x.c0(), (size_t)limbs * n * 8, cudaMemcpyDeviceToDevice, c.stream));
      SF_CUDA(cudaMemcpyAsync(ac->p + (size_t)limbs * n, x.c1(c.n), (size_t)limbs * n * 8, cudaMemcpyDeviceToDevice,
                              c.stream));
      as = make_buf(c, (size_t)2 * limbs * n);
      b_shoup_companion(c, ac->p, as->p, limbs, 2);
    }
    for (size_t s0 = 0; s0 < idx.size(); s0 += kJobs) {
      const int J = (int)std::min<size_t>(kJobs, idx.size() - s0);
      BufPtr d = make_buf(c, (size_t)J * 3 * limbs * n);
      auto dp = [&](int j, int k) { return d->p + ((size_t)j * 3 + k) * limbs * n; };
      TensorBatch tb;
      std::vector<const u64*> d2;
      for (int j = 0; j < J; ++j) {
        const Ct &x = *a[idx[s0 + j]], &y = *b[idx[s0 + j]];
        tb.a0[j] = x.c0(), tb.a1[j] = x.c1(c.n), tb.b0[j] = y.c0(), tb.b1[j] = y.c1(c.n);
        tb.d0[j] = dp(j, 0), tb.d1[j] = dp(j, 1), tb.d2[j] = dp(j, 2);
        d2.push_back(dp(j, 2));
      }
      tb.count = J;
      tb.as = as ? as->p : nullptr;
      b_tensor(c, tb, limbs);
      ExtB x = mod_up_batch(c, d2, limbs, false, relin_digit(c, limbs));
      std::vector<Ct> t(J);
      std::vector<KsJob> kj;
      for (int j = 0; j < J; ++j) {  // relinearise + rescale in one conversion
        t[j] = alloc_ct(c, limbs - 1,
                        a[idx[s0 + j]]->scale * b[idx[s0 + j]]->scale / (double)c.primes[limbs - 1]);
        kj.push_back({j, 0, dp(j, 0), dp(j, 1), t[j].c0(), t[j].c1(c.n)});
      }
      ks_jobs(c, x, kj, true);
      for (int j = 0; j < J; ++j) {
        t[j].layout = merge_layouts(*a[idx[s0 + j]], *b[idx[s0 + j]]);
        out[idx[s0 + j]] = std::move(t[j]);
      }
    }
  }
  return out;
}

Ct mul(Context& c, const Ct& a, const Ct& b, bool count) { return mul_batch(c, {&a}, {&b}, count)[0]; }

// ------------------------------------------------- lazily relinearised sums
Ct3 tensor_sum(Context& c, const std::vector<const Ct*>& a, const std::vector<const Ct*>& b, bool count) {
  SF_HPROF("tensor_sum");
  require(a.size() == b.size() && !a.empty(), kShapeMismatch, "tensor_sum: operand count");
  int limbs = 1 << 30;
  double scale = 0.0;
  std::vector<int> live;
  for (size_t i = 0; i < a.size(); ++i) {
    check_ct(c, *a[i], "mul");
    check_ct(c, *b[i], "mul");
    const int l = std::min(a[i]->limbs, b[i]->limbs);
    require(l - 1 > 0, kLevelUnderflow, "mul: no multiplicative level left");
    limbs = std::min(limbs, l);
    if (a[i]->zero || b[i]->zero) continue;
    const double s = a[i]->scale * b[i]->scale;
    if (scale == 0.0)
      scale = s;
    else if (std::fabs(s / scale - 1.0) > 1e-9)
      fail(kScaleMismatch, "ScaleMismatch: add: operand scales differ");
    live.push_back((int)i);
  }
  if (count) {
    c.ledger.ctct((long long)a.size());
    c.ledger.add((long long)a.size() - 1);
  }
  Ct3 r;
  if (live.empty()) {
    r.d01 = zeros(c, limbs - 1);
    r.d2 = zeros(c, limbs - 1);
    return r;
  }
  r.zero = false;
  r.d01 = alloc_ct(c, limbs, scale);
  r.d2 = alloc_ct(c, limbs, scale);
  SF_CUDA(cudaMemsetAsync(r.d2.c1(c.n), 0, (size_t)limbs * c.n * 8, c.stream));
  TensorSumArgs A;
  A.d0 = r.d01.c0();
  A.d1 = r.d01.c1(c.n);
  A.d2 = r.d2.c0();
  for (size_t s = 0; s < live.size();) {
    A.k = 0;
    for (; s < live.size() && A.k < 512; ++s) {
      const Ct &x = *a[live[s]], &y = *b[live[s]];
      A.a0[A.k] = x.c0(), A.a1[A.k] = x.c1(c.n), A.b0[A.k] = y.c0(), A.b1[A.k] = y.c1(c.n);
      ++A.k;
    }
    b_tensor_sum(c, A, limbs);
    A.accumulate = true;
  }
  return r;
}

std::vector<Ct3> tensor_sum_multi(Context& c, const std::vector<std::vector<const Ct*>>& a,
                                  const std::vector<std::vector<const Ct*>>& b, bool count) {
  SF_HPROF("tensor_sum_multi");
  require(a.size() == b.size(), kShapeMismatch, "tensor_sum: operand count");
  std::vector<Ct3> out(a.size());
  std::vector<std::vector<int>> live(a.size());
  int limbs_all = 1 << 30;
  for (size_t o = 0; o < a.size(); ++o) {
    require(a[o].size() == b[o].size() && !a[o].empty(), kShapeMismatch, "tensor_sum: operand count");
    int limbs = 1 << 30;
    double scale = 0.0;
    for (size_t i = 0; i < a[o].size(); ++i) {
      check_ct(c, *a[o][i], "mul");
      check_ct(c, *b[o][i], "mul");
      const int l = std::min(a[o][i]->limbs, b[o][i]->limbs);
      require(l - 1 > 0, kLevelUnderflow, "mul: no multiplicative level left");
      limbs = std::min(limbs, l);
      if (a[o][i]->zero || b[o][i]->zero) continue;
      const double sc = a[o][i]->scale * b[o][i]->scale;
      if (scale == 0.0)
        scale = sc;
      else if (std::fabs(sc / scale - 1.0) > 1e-9)
        fail(kScaleMismatch, "ScaleMismatch: add: operand scales differ");
      live[o].push_back((int)i);
    }
    if (count) {
      c.ledger.ctct((long long)a[o].size());
      c.ledger.add((long long)a[o].size() - 1);
    }
    if (live[o].empty()) {
      out[o].d01 = zeros(c, limbs - 1);
      out[o].d2 = zeros(c, limbs - 1);
      continue;
    }
    out[o].zero = false;
    out[o].d01 = alloc_ct(c, limbs, scale);
    out[o].d2 = alloc_ct(c, limbs, scale);
    limbs_all = std::min(limbs_all, limbs);
  }
  // one launch per run of same-limb outputs that fits the parameter block
  std::map<int, std::vector<int>> by_limbs;
  for (size_t o = 0; o < a.size(); ++o)
    if (!out[o].zero) by_limbs[out[o].d01.limbs].push_back((int)o);
  (void)limbs_all;
  for (auto& [limbs_run, todo] : by_limbs) {
  size_t at = 0;
  while (at < todo.size()) {
    TensorSumMultiArgs A;
    int terms = 0;
    for (; at < todo.size() && A.nout < kTsmOuts; ++at) {
      const int o = todo[at];
      if (terms + (int)live[o].size() > kTsmTerms) break;
      require((int)live[o].size() <= kTsmTerms, kInternal, "tensor_sum_multi: too many terms");
      A.begin[A.nout] = terms;
      A.d0[A.nout] = out[o].d01.c0();
      A.d1[A.nout] = out[o].d01.c1(c.n);
      A.d2[A.nout] = out[o].d2.c0();
      for (int i : live[o]) {
        A.a0[terms] = a[o][i]->c0(), A.a1[terms] = a[o][i]->c1(c.n);
        A.b0[terms] = b[o][i]->c0(), A.b1[terms] = b[o][i]->c1(c.n);
        ++terms;
      }
      ++A.nout;
    }
    A.begin[A.nout] = terms;
    b_tensor_sum_multi(c, A, limbs_run);
  }
  }
  return out;
}

Ct3 add_ct3(Context& c, const std::vector<const Ct3*>& xs) {
  SF_HPROF("add_ct3");
  std::vector<const Ct*> a, b;
  for (const Ct3* x : xs)
    if (!x->zero) a.push_back(&x->d01), b.push_back(&x->d2);
  if (a.empty()) return *xs[0];
  Ct3 r;
  r.zero = false;
  r.d01 = sum_cts(c, a, false);
  r.d2 = sum_cts(c, b, false);
  return r;
}

Ct relin_rescale(Context& c, const Ct3& x) {
  SF_HPROF("relin_rescale");
  if (x.zero) return zeros(c, x.d01.level() - 1);
  const int limbs = std::min(x.d01.limbs, x.d2.limbs);
  ExtB e = mod_up_batch(c, {x.d2.c0()}, limbs, false, relin_digit(c, limbs));
  Ct t = alloc_ct(c, limbs - 1, x.d01.scale / (double)c.primes[limbs - 1]);
  ks_jobs(c, e, {KsJob{0, 0, x.d01.c0(), x.d01.c1(c.n), t.c0(), t.c1(c.n)}}, true);
  return t;
}

std::vector<Ct> relin_batch(Context& c, const std::vector<const Ct3*>& xs, bool rescale) {
  SF_HPROF("relin_batch");
  std::vector<Ct> out(xs.size());
  std::map<int, std::vector<int>> by_limbs;
  for (size_t i = 0; i < xs.size(); ++i) {
    if (xs[i]->zero)
      out[i] = zeros(c, xs[i]->d01.level() - (rescale ? 1 : 0));
    else
      by_limbs[std::min(xs[i]->d01.limbs, xs[i]->d2.limbs)].push_back((int)i);
  }
  for (auto& [limbs, idx] : by_limbs) {
    for (size_t s0 = 0; s0 < idx.size(); s0 += kJobs) {
      const int J = (int)std::min<size_t>(kJobs, idx.size() - s0);
      std::vector<const u64*> d2;
      for (int j = 0; j < J; ++j) d2.push_back(xs[idx[s0 + j]]->d2.c0());
      ExtB e = mod_up_batch(c, d2, limbs, false, relin_digit(c, limbs));
      std::vector<KsJob> kj;
      for (int j = 0; j < J; ++j) {
        const Ct3& x = *xs[idx[s0 + j]];
        Ct t = rescale ? alloc_ct(c, limbs - 1, x.d01.scale / (double)c.primes[limbs - 1])
                       : alloc_ct(c, limbs, x.d01.scale);
        kj.push_back({j, 0, x.d01.c0(), x.d01.c1(c.n), t.c0(), t.c1(c.n)});
        out[idx[s0 + j]] = std::move(t);
      }
      ks_jobs(c, e, kj, rescale);
    }
  }
  return out;
}

// ------------------------------------------------------------- ct x pt mult
std::vector<Ct> mul_plain_batch(Context& c, const std::vector<const Ct*>& xs, const std::vector<const Pt*>& ps,
                                bool count, bool rescale) {
  require(xs.size() == ps.size(), kShapeMismatch, "mul_plain_batch: operand count");
  std::vector<Ct> out(xs.size());
  std::vector<Ct> tmp(xs.size());
  std::vector<const Ct*> todo;
  std::vector<int> where;
  std::map<int, MulPtBatch> by_limbs;
  // ciphertexts feeding four or more products (value pieces of one v_open, RoPE):
  // Shoup companions once per (buffer, limbs)
  std::map<std::pair<const u64*, int>, int> uses;
  for (const Ct* x : xs)
    if (!x->zero) ++uses[{x->c0(), x->limbs}];
  std::map<std::pair<const u64*, int>, BufPtr> comp;
  for (auto& [key, cnt] : uses) {
    if (cnt < 4) continue;
    const Ct* x = nullptr;
    for (const Ct* y : xs)
      if (!y->zero && y->c0() == key.first && y->limbs == key.second) x = y;
    const size_t w = (size_t)x->limbs * c.n;
    BufPtr ac = make_buf(c, 2 * w);
    SF_CUDA(cudaMemcpyAsync(ac->p, x->c0(), w * 8, cudaMemcpyDeviceToDevice, c.stream));
    SF_CUDA(cudaMemcpyAsync(ac->p + w, x->c1(c.n), w * 8, cudaMemcpyDeviceToDevice, c.stream));
    BufPtr cs = make_buf(c, 2 * w);
    b_shoup_companion(c, ac->p, cs->p, x->limbs, 2);
    comp[key] = cs;
  }
  for (size_t i = 0; i < xs.size(); ++i) {
    const Ct& x = *xs[i];
    check_ct(c, x, "mul_plain");
    require(x.level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
    require(ps[i]->limbs >= x.limbs, kShapeMismatch, "mul_plain: plaintext has too few limbs");
    if (count) c.ledger.ctpt();
    if (x.zero) {
      out[i] = zeros(c, rescale ? x.level() - 1 : x.level());
      out[i].layout = x.layout;
      continue;
    }
    tmp[i] = alloc_ct(c, x.limbs, x.scale * (double)c.primes[x.limbs - 1]);
    tmp[i].layout = x.layout;
    MulPtBatch& B = by_limbs[x.limbs];
    B.c0[B.count] = x.c0(), B.c1[B.count] = x.c1(c.n), B.pt[B.count] = ps[i]->buf->p;
    B.o0[B.count] = tmp[i].c0(), B.o1[B.count] = tmp[i].c1(c.n);
    auto ci = comp.find({x.c0(), x.limbs});
    B.cs[B.count] = ci != comp.end() ? ci->second->p : nullptr;
    if (++B.count == kJobsWide) b_mulpt(c, B, x.limbs), B.count = 0, std::fill(B.cs, B.cs + kJobsWide, nullptr);
    todo.push_back(&tmp[i]);
    where.push_back((int)i);
  }
  for (auto& [limbs, B] : by_limbs) b_mulpt(c, B, limbs);
  if (!rescale) {  // the caller rescales later (e.g. merged into a rotation sum's ModDown)
    for (size_t k = 0; k < todo.size(); ++k) out[where[k]] = std::move(tmp[where[k]]);
    return out;
  }
  auto r = rescale_batch(c, todo);
  for (size_t k = 0; k < r.size(); ++k) {
    const Ct& x = *xs[where[k]];
    r[k].scale = x.scale;
    r[k].layout = x.layout;
    out[where[k]] = std::move(r[k]);
  }
  return out;
}

// ------------------------------------------------------------------ additions
std::vector<Ct> add_batch(Context& c, const std::vector<const Ct*>& a, const std::vector<const Ct*>& b, bool count) {
  SF_HPROF("add_batch");
  require(a.size() == b.size(), kShapeMismatch, "add_batch: operand count");
  std::vector<Ct> out(a.size());
  std::map<int, AddBatch> by_limbs;
  for (size_t i = 0; i < a.size(); ++i) {
    const Ct &x = *a[i], &y = *b[i];
    check_ct(c, x, "add");
    check_ct(c, y, "add");
    if (count) c.ledger.add();
    const int limbs = std::min(x.limbs, y.limbs);
    OptLayout ly = merge_layouts(x, y);
    if (y.zero || (x.zero && y.zero)) {
      if (!(x.zero && y.zero)) check_scales(x, y, "add");
      Ct r = x;
      r.limbs = limbs;
      r.layout = ly;
      out[i] = r;
      continue;
    }
    if (x.zero) {
      Ct r = y;
      r.limbs = limbs;
      r.layout = ly;
      out[i] = r;
      continue;
    }
    check_scales(x, y, "add");
    Ct r = alloc_ct(c, limbs, x.scale);
    r.layout = ly;
    AddBatch& B = by_limbs[limbs];
    B.a0[B.count] = x.c0(), B.a1[B.count] = x.c1(c.n), B.b0[B.count] = y.c0(), B.b1[B.count] = y.c1(c.n);
    B.o0[B.count] = r.c0(), B.o1[B.count] = r.c1(c.n);
    if (++B.count == kJobsWide) b_add(c, B, limbs), B.count = 0;
    out[i] = r;
  }
  for (auto& [limbs, B] : by_limbs) b_add(c, B, limbs);
  return out;
}

std::vector<Ct> sum_cts_multi(Context& c, const std::vector<std::vector<const Ct*>>& groups) {
  SF_HPROF("sum_cts_multi");
  std::vector<Ct> out(groups.size());
  std::map<int, std::vector<int>> by_limbs;  // groups needing a kernel, by limb count
  std::vector<std::vector<const Ct*>> live(groups.size());
  for (size_t g = 0; g < groups.size(); ++g) {
    require(!groups[g].empty(), kShapeMismatch, "sum: empty");
    int limbs = 1 << 30;
    for (const Ct* x : groups[g]) {
      check_ct(c, *x, "add");
      limbs = std::min(limbs, x->limbs);
      if (!x->zero) live[g].push_back(x);
    }
    for (const Ct* x : live[g]) check_scales(*live[g][0], *x, "add");
    if (live[g].size() <= 1) {  // as sum_cts: nothing to add
      Ct r = live[g].empty() ? *groups[g][0] : *live[g][0];
      r.limbs = limbs;
      r.layout.reset();
      out[g] = r;
      continue;
    }
    out[g] = alloc_ct(c, limbs, live[g][0]->scale);
    by_limbs[limbs].push_back((int)g);
  }
  for (auto& [limbs, gs] : by_limbs) {
    size_t at = 0;
    while (at < gs.size()) {
      SumMultiArgs A;
      int k = 0;
      for (; at < gs.size() && A.nout < 64; ++at) {
        const int g = gs[at];
        if (k + (int)live[g].size() > 512) break;
        A.begin[A.nout] = k;
        for (const Ct* x : live[g]) A.in0[k] = x->c0(), A.in1[k] = x->c1(c.n), ++k;
        A.out0[A.nout] = out[g].c0();
        A.out1[A.nout] = out[g].c1(c.n);
        ++A.nout;
      }
      A.begin[A.nout] = k;
      b_sum_multi(c, A, limbs);
    }
  }
  return out;
}

Ct sum_cts(Context& c, const std::vector<const Ct*>& xs, bool count) {
  SF_HPROF("sum_cts");
  require(!xs.empty(), kShapeMismatch, "sum: empty");
  if (count) c.ledger.add((long long)xs.size() - 1);
  int limbs = 1 << 30;
  std::vector<const Ct*> live;
  for (const Ct* x : xs) {
    check_ct(c, *x, "add");
    limbs = std::min(limbs, x->limbs);
    if (!x->zero) live.push_back(x);
  }
  OptLayout ly = xs[0]->layout;
  for (const Ct* x : xs)
    if (!(x->layout && ly && *x->layout == *ly)) ly.reset();
  if (live.empty()) {
    Ct z = *xs[0];
    z.limbs = limbs;
    z.layout = ly;
    return z;
  }
  for (const Ct* x : live) check_scales(*live[0], *x, "add");
  if (live.size() == 1) {
    Ct r = *live[0];
    r.limbs = limbs;
    r.layout = ly;
    return r;
  }
  Ct acc = alloc_ct(c, limbs, live[0]->scale);
  size_t s = 0;
  bool first = true;
  while (s < live.size()) {
    SumArgs A;
    if (!first) {
      A.in0[A.k] = acc.c0();
      A.in1[A.k++] = acc.c1(c.n);
    }
    for (; s < live.size() && A.k < 512; ++s) {
      A.in0[A.k] = live[s]->c0();
      A.in1[A.k++] = live[s]->c1(c.n);
    }
    Ct next = first ? acc : alloc_ct(c, limbs, acc.scale);
    A.out0 = next.c0();
    A.out1 = next.c1(c.n);
    b_sum(c, A, limbs);
    acc = next;
    first = false;
  }
  acc.layout = ly;
  return acc;
}

}  // namespace sf
