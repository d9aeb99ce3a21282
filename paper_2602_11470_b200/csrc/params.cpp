// Parameter generation, twiddle tables and the host CKKS encoder.
// Canonical definitions: DESIGN.md §3.1 (primes, roots) and §3.2 (encoder).
#include <algorithm>
#include <cmath>
#include <cstring>

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "context.h"

namespace sf {

namespace {
std::mutex g_hp_mu;
std::map<std::string, std::pair<double, long long>> g_hp;
}  // namespace
bool host_prof_on() {
  static const bool on = [] {
    const char* e = std::getenv("SF_HOST_PROF");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
void host_prof_add(const char* name, double us) {
  std::lock_guard<std::mutex> lk(g_hp_mu);
  auto& v = g_hp[name];
  v.first += us;
  v.second += 1;
}
std::string host_prof_dump(bool reset) {
  std::lock_guard<std::mutex> lk(g_hp_mu);
  std::string out;
  char line[160];
  for (auto& [k, v] : g_hp) {
    std::snprintf(line, sizeof line, "%s %.1f %lld\n", k.c_str(), v.first, v.second);
    out += line;
  }
  if (reset) g_hp.clear();
  return out;
}

namespace {

bool is_prime(u64 n) {
  if (n < 2) return false;
  static const u64 small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  for (u64 p : small)
    if (n % p == 0) return n == p;
  u64 d = n - 1;
  int s = 0;
  while ((d & 1) == 0) d >>= 1, ++s;
  for (u64 a : small) {  // deterministic for n < 3.3e24
    u64 x = powmod_h(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool composite = true;
    for (int r = 1; r < s && composite; ++r) {
      x = mulmod_h(x, x, n);
      if (x == n - 1) composite = false;
    }
    if (composite) return false;
  }
  return true;
}

constexpr double kPi = 3.14159265358979323846;

}  // namespace

// q0 = largest prime < 2^q0_bits, then L scale primes descending from
// 2^scale_bits, then alpha special primes descending from 2^special_bits; all
// == 1 mod 2n and pairwise distinct.
std::vector<u64> generate_primes(int logn, int L, int q0_bits, int scale_bits, int alpha, int special_bits) {
  const u64 m = 2ull << logn;
  std::vector<u64> used;
  auto take = [&](int bits, int count) {
    // <= 60 bits: the lazy kernels keep sums of up to 8 Shoup products in [0, 2q)
    // in one u64 (fused column conversion) and fold 128-bit inner products
    // every 64+ terms (ks_sum); both bounds need q < 2^60.
    require(bits >= 20 && bits <= 60, kDomain, "prime bits must be in [20, 60]");
    std::vector<u64> r;
    u64 c = ((1ull << bits) / m) * m + 1;
    if (c >= (1ull << bits)) c -= m;
    while ((int)r.size() < count) {
      require(c > m, kDomain, "ran out of NTT-friendly primes");
      if (is_prime(c) && std::find(used.begin(), used.end(), c) == used.end()) {
        r.push_back(c);
        used.push_back(c);
      }
      c -= m;
    }
    return r;
  };
  std::vector<u64> out = take(q0_bits, 1);
  auto sc = take(scale_bits, L);
  auto sp = take(special_bits, alpha);
  out.insert(out.end(), sc.begin(), sc.end());
  out.insert(out.end(), sp.begin(), sp.end());
  return out;
}

// The minimal primitive 2n-th root of unity mod q.
u64 min_primitive_root(u64 q, int n) {
  const u64 m = 2ull * (u64)n;
  u64 root = 0;
  for (u64 g = 2;; ++g) {
    const u64 c = powmod_h(g, (q - 1) / m, q);
    if (powmod_h(c, (u64)n, q) == q - 1) {
      root = c;
      break;
    }
  }
  u64 best = root, cur = root;
  const u64 r2 = mulmod_h(root, root, q);
  for (u64 k = 3; k < m; k += 2) {
    cur = mulmod_h(cur, r2, q);
    best = std::min(best, cur);
  }
  return best;
}

// --- layouts (layouts.cpp:50-64, 146-149) -------------------------------------
void validate_layout(const Layout& ly, int N) {
  require(is_pow2(N), kShapeMismatch, "layout: N must be a power of two");
  require(ly.d > 0 && is_pow2(ly.d), kShapeMismatch, "layout: d must be a positive power of two");
  require(ly.t > 0 && is_pow2(ly.t), kShapeMismatch, "layout: t must be a positive power of two");
  require((long long)ly.d * ly.t == N, kShapeMismatch, "layout: d*t must equal N");
  require(ly.offset >= 0 && ly.offset < ly.t, kShapeMismatch, "layout: offset out of range");
  require(ly.heads >= 1 && is_pow2(ly.heads) && ly.heads <= ly.d, kShapeMismatch,
          "layout: heads must be a power of two dividing d");
}
Layout make_interleaved(int d, int N, int offset, int heads) {
  Layout ly{LayoutKind::Interleaved, d, d > 0 ? N / d : 0, offset, heads, false};
  validate_layout(ly, N);
  return ly;
}
int padded_dim(int d) {
  require(d > 0, kShapeMismatch, "padded_dim: d must be positive");
  return (int)next_pow2(d);
}

// --- encoder ---------------------------------------------------------------------
// Inverse special FFT: Gentleman-Sande loop over zeta^{-br(k)}, the complex
// twin of the inverse NTT loop. Operation order is part of the
// spec: the CPU oracle performs exactly these IEEE operations.
static void fft_inverse(const Context& c, std::vector<double>& re, std::vector<double>& im) {
  int t = 1;
  for (int m = c.n; m > 1; m >>= 1) {
    const int h = m >> 1;
    int j1 = 0;
    for (int i = 0; i < h; ++i) {
      const double wr = c.fft_re[h + i], wi = -c.fft_im[h + i];
      for (int j = j1; j < j1 + t; ++j) {
        const double ur = re[j], ui = im[j], vr = re[j + t], vi = im[j + t];
        re[j] = ur + vr;
        im[j] = ui + vi;
        const double dr = ur - vr, di = ui - vi;
        re[j + t] = dr * wr - di * wi;
        im[j + t] = dr * wi + di * wr;
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
}

static void fft_forward(const Context& c, std::vector<double>& re, std::vector<double>& im) {
  int t = c.n;
  for (int m = 1; m < c.n; m <<= 1) {
    t >>= 1;
    for (int i = 0; i < m; ++i) {
      const int j1 = 2 * i * t;
      const double wr = c.fft_re[m + i], wi = c.fft_im[m + i];
      for (int j = j1; j < j1 + t; ++j) {
        const double xr = re[j + t], xi = im[j + t];
        const double vr = xr * wr - xi * wi, vi = xr * wi + xi * wr;
        const double ur = re[j], ui = im[j];
        re[j] = ur + vr;
        im[j] = ui + vi;
        re[j + t] = ur - vr;
        im[j + t] = ui - vi;
      }
    }
  }
}

std::vector<i64> encode_coeffs(const Context& c, const double* slots, double scale) {
  std::vector<double> re(c.n, 0.0), im(c.n, 0.0);
  const int half = c.n / 2;
  for (int j = 0; j < half; ++j) {
    const double v = slots[j % c.slots];
    re[c.slot_index[j]] = v;
    re[c.slot_index[half + j]] = v;  // conjugate root 2n - 5^j
  }
  fft_inverse(c, re, im);
  const double f = scale / (double)c.n;
  std::vector<i64> out(c.n);
  for (int k = 0; k < c.n; ++k) {
    const double v = re[k] * f;
    require(std::fabs(v) < 4.0e18, kDomain, "encode: value too large for the scale");
    out[k] = std::llround(v);
  }
  return out;
}

void decode_coeffs(const Context& c, const std::vector<double>& coeff, double scale, double* slots) {
  std::vector<double> re(coeff), im(c.n, 0.0);
  fft_forward(c, re, im);
  for (int j = 0; j < c.slots; ++j) slots[j] = re[c.slot_index[j]] / scale;
}

// Host-side table construction; device upload + secret key in evaluator.cu.
void build_host_tables(Context& c, std::vector<u64>& psi, std::vector<u64>& psi_s, std::vector<u64>& ipsi,
                       std::vector<u64>& ipsi_s, std::vector<u64>& ninv, std::vector<u64>& ninv_s) {
  const int n = c.n, np = c.np;
  psi.resize((size_t)np * n);
  psi_s.resize((size_t)np * n);
  ipsi.resize((size_t)np * n);
  ipsi_s.resize((size_t)np * n);
  ninv.resize(np);
  ninv_s.resize(np);
  c.mu_hi.resize(np);
  c.mu_lo.resize(np);
  c.qneg_inv.resize(np);
  c.r64.resize(np);
  std::vector<uint32_t> br(n);
  for (int k = 0; k < n; ++k) br[k] = (uint32_t)bitrev_h(k, c.logn);
  for (int m = 0; m < np; ++m) {
    const u64 q = c.primes[m];
    const u128 mu = (~(u128)0) / q;  // floor((2^128 - 1) / q) == floor(2^128 / q), q odd
    c.mu_hi[m] = (u64)(mu >> 64);
    c.mu_lo[m] = (u64)mu;
    u64 inv = q;  // q^-1 mod 2^64 by Newton (q odd: correct to 3 bits, doubling per step)
    for (int it = 0; it < 5; ++it) inv *= 2 - q * inv;
    c.qneg_inv[m] = 0 - inv;
    c.r64[m] = (u64)(((u128)1 << 64) % q);
    const u64 psi1 = min_primitive_root(q, n), ipsi1 = invmod_h(psi1, q);
    std::vector<u64> pw(n), ipw(n);
    pw[0] = ipw[0] = 1;
    for (int k = 1; k < n; ++k) {
      pw[k] = mulmod_h(pw[k - 1], psi1, q);
      ipw[k] = mulmod_h(ipw[k - 1], ipsi1, q);
    }
    for (int k = 0; k < n; ++k) {
      const size_t o = (size_t)m * n + k;
      psi[o] = pw[br[k]];
      ipsi[o] = ipw[br[k]];
      psi_s[o] = shoup_h(psi[o], q);
      ipsi_s[o] = shoup_h(ipsi[o], q);
    }
    ninv[m] = invmod_h((u64)n % q, q);
    ninv_s[m] = shoup_h(ninv[m], q);
  }
  c.fft_re.resize(n);
  c.fft_im.resize(n);
  for (int k = 0; k < n; ++k) {
    const double ang = kPi * (double)br[k] / (double)n;
    c.fft_re[k] = std::cos(ang);
    c.fft_im[k] = std::sin(ang);
  }
  // slot j <-> transform index br((5^j mod 2n - 1)/2); conjugates at n/2 + j
  const u64 m2 = 2ull * n;
  c.slot_index.resize(n);
  u64 e = 1;
  for (int j = 0; j < n / 2; ++j) {
    c.slot_index[j] = br[(e - 1) / 2];
    c.slot_index[n / 2 + j] = br[(m2 - e - 1) / 2];
    e = (e * 5) % m2;
  }
}

}  // namespace sf
