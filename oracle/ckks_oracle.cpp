// CPU RNS-CKKS oracle: the bit-exact twin the GPU product is held to.
// TEST INFRASTRUCTURE ONLY (loaded by tests/ and bench.py's cpu_baseline leg
// through oracle/ckks.py; never linked by the product).
//
// Parity status: the reference (/root/reference/proj) is a cleartext slot
// simulator and contains NO ciphertext arithmetic, so this
// file restates textbook full-RNS CKKS with hybrid key switching, following
// the canonical specification written down in DESIGN.md §3 ("CKKS spec"). Its
// ciphertext-level parity is therefore pinned only indirectly: decrypted slots
// are checked against the reference's golden slot vectors (tests/golden/) and
// op counts against the reference ledger. Everything here is deliberately
// "obviously correct" rather than fast: unsigned __int128 with % for every
// modular product, O(N log N) textbook NTT loops, OpenMP over limbs only.
//
// Semantics mirrored from the reference boundary (engine.hpp:102-111 level
// rules; engine.cpp:181-191 rotation direction out[i] = in[(i+r) mod N]).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

using u64 = uint64_t;
using u128 = unsigned __int128;
using i64 = int64_t;

thread_local std::string g_err;
constexpr double kPi = 3.14159265358979323846;

u64 mulmod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
u64 addmod(u64 a, u64 b, u64 m) {
  u64 s = a + b;
  return s >= m ? s - m : s;
}
u64 submod(u64 a, u64 b, u64 m) { return a >= b ? a - b : a + m - b; }
u64 powmod(u64 b, u64 e, u64 m) {
  u64 r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = mulmod(r, b, m);
    b = mulmod(b, b, m);
    e >>= 1;
  }
  return r;
}
u64 invmod(u64 a, u64 m) { return powmod(a, m - 2, m); }  // m prime

bool is_prime(u64 n) {
  if (n < 2) return false;
  for (u64 p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    if (n % p == 0) return n == p;
  }
  u64 d = n - 1;
  int s = 0;
  while ((d & 1) == 0) d >>= 1, ++s;
  for (u64 a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    u64 x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; ++r) {
      x = mulmod(x, x, n);
      if (x == n - 1) {
        comp = false;
        break;
      }
    }
    if (comp) return false;
  }
  return true;
}

u64 bitrev(u64 x, int bits) {
  u64 r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}

// --- PRNG: ChaCha20 counter stream ---------------------------
// Textbook ChaCha20 (D. J. Bernstein, 2008; RFC 8439 §2.3 block function with
// the original 64-bit counter / 64-bit nonce split): state = 4 constants,
// 8 key words, counter (2 words), nonce (2 words); 10 double rounds; output =
// final state + input state. Key = the 64-bit seed (2 words) followed by the
// domain words "sf_b200 ckks rng", 1, 0; nonce = the stream id; word i of a
// stream is 64-bit word i mod 8 of block i / 8. Pinned against the
// `cryptography` package's ChaCha20 (tests/test_ckks_oracle.py).
uint32_t rotl(uint32_t v, int c) { return (v << c) | (v >> (32 - c)); }
#define QR(a, b, c, d) \
  a += b; d ^= a; d = rotl(d, 16); c += d; b ^= c; b = rotl(b, 12); \
  a += b; d ^= a; d = rotl(d, 8);  c += d; b ^= c; b = rotl(b, 7);
void chacha20_block(const uint32_t key[8], u64 counter, u64 nonce, uint32_t out[16]) {
  const uint32_t in[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key[0], key[1], key[2], key[3],
                           key[4], key[5], key[6], key[7], (uint32_t)counter, (uint32_t)(counter >> 32),
                           (uint32_t)nonce, (uint32_t)(nonce >> 32)};
  uint32_t x[16];
  std::copy(in, in + 16, x);
  for (int i = 0; i < 10; ++i) {
    QR(x[0], x[4], x[8], x[12]) QR(x[1], x[5], x[9], x[13]) QR(x[2], x[6], x[10], x[14]) QR(x[3], x[7], x[11], x[15])
    QR(x[0], x[5], x[10], x[15]) QR(x[1], x[6], x[11], x[12]) QR(x[2], x[7], x[8], x[13]) QR(x[3], x[4], x[9], x[14])
  }
  for (int i = 0; i < 16; ++i) out[i] = x[i] + in[i];
}
#undef QR
u64 rand64(u64 seed, u64 stream, u64 ctr) {
  const uint32_t key[8] = {(uint32_t)seed, (uint32_t)(seed >> 32), 0x625f6673u, 0x20303032u,
                           0x736b6b63u, 0x676e7220u, 1u, 0u};
  uint32_t o[16];
  chacha20_block(key, ctr / 8, stream, o);
  const int w = (int)(ctr % 8);
  return (u64)o[2 * w] | ((u64)o[2 * w + 1] << 32);
}
// uniform residue k of a stream mod q: words 2k, 2k+1 as one 128-bit integer
u64 rand_mod(u64 seed, u64 stream, u64 k, u64 q) {
  const unsigned __int128 v = ((unsigned __int128)rand64(seed, stream, 2 * k + 1) << 64) | rand64(seed, stream, 2 * k);
  return (u64)(v % q);
}
u64 fmix(u64 z) {  // SplitMix64 finaliser: derives the seeds of counter-seeded encryptions
  z ^= z >> 30;
  z *= 0xbf58476d1ce4e5b9ull;
  z ^= z >> 27;
  z *= 0x94d049bb133111ebull;
  z ^= z >> 31;
  return z;
}
i64 cbd21(u64 r) {
  return (i64)__builtin_popcountll(r & 0x1FFFFFull) - (i64)__builtin_popcountll((r >> 21) & 0x1FFFFFull);
}
u64 to_mod(i64 v, u64 q) {
  if (v >= 0) return (u64)v % q;
  u64 r = (u64)(-(v + 1)) % q;  // careful with INT64_MIN
  r = (r + 1) % q;
  return r == 0 ? 0 : q - r;
}

struct Ct {
  std::vector<u64> d;   // [2][limbs][n]
  std::vector<u64> d2;  // degree-2 part [limbs][n] of a lazily relinearised sum (empty otherwise)
  int limbs = 0;
  double scale = 0.0;
  bool zero = false;
};

struct Ctx {
  int logn, n, slots, L, alpha, beta;
  double delta;
  std::vector<u64> primes;  // q0..qL, p0..p_{alpha-1}
  std::vector<std::vector<u64>> psi_rev, psi_inv_rev;
  std::vector<u64> n_inv;
  std::vector<double> fft_re, fft_im;  // zeta^{br(k)}
  std::vector<u64> sk;                 // [nprimes][n] NTT domain
  u64 seed;
  u64 enc_counter = 0;
  std::map<u64, std::vector<u64>> keys;  // galois elt (0 = relin) -> [beta][2][nprimes][n]
  std::mutex mu;

  int nq() const { return L + 1; }
  int np() const { return (int)primes.size(); }
  u64 P_index(int k) const { return (u64)(L + 1 + k); }
};

// minimal primitive 2n-th root of unity mod q
u64 min_psi(u64 q, int n) {
  const u64 m = 2 * (u64)n;
  u64 root = 0;
  for (u64 g = 2;; ++g) {
    u64 c = powmod(g, (q - 1) / m, q);
    if (powmod(c, (u64)n, q) == q - 1) {
      root = c;
      break;
    }
  }
  u64 best = root, cur = root;
  const u64 r2 = mulmod(root, root, q);
  for (u64 k = 3; k < m; k += 2) {
    cur = mulmod(cur, r2, q);
    best = std::min(best, cur);
  }
  return best;
}

std::vector<u64> gen_primes(int logn, int L, int q0_bits, int scale_bits, int alpha, int special_bits) {
  const u64 m = 2ull << logn;
  std::vector<u64> out;
  std::vector<u64> used;
  auto below = [&](int bits, int count) {
    std::vector<u64> r;
    u64 c = ((1ull << bits) / m) * m + 1;
    if (c >= (1ull << bits)) c -= m;
    while ((int)r.size() < count) {
      if (is_prime(c) && std::find(used.begin(), used.end(), c) == used.end()) {
        r.push_back(c);
        used.push_back(c);
      }
      c -= m;
    }
    return r;
  };
  auto q0 = below(q0_bits, 1);
  auto sc = below(scale_bits, L);
  auto sp = below(special_bits, alpha);
  out.push_back(q0[0]);
  out.insert(out.end(), sc.begin(), sc.end());
  out.insert(out.end(), sp.begin(), sp.end());
  return out;
}

void ntt_fwd(const Ctx& c, int pi, u64* a) {
  const u64 q = c.primes[pi];
  const auto& W = c.psi_rev[pi];
  int t = c.n;
  for (int m = 1; m < c.n; m <<= 1) {
    t >>= 1;
    for (int i = 0; i < m; ++i) {
      const int j1 = 2 * i * t;
      const u64 S = W[m + i];
      for (int j = j1; j < j1 + t; ++j) {
        const u64 U = a[j], V = mulmod(a[j + t], S, q);
        a[j] = addmod(U, V, q);
        a[j + t] = submod(U, V, q);
      }
    }
  }
}

void ntt_inv(const Ctx& c, int pi, u64* a) {
  const u64 q = c.primes[pi];
  const auto& W = c.psi_inv_rev[pi];
  int t = 1;
  for (int m = c.n; m > 1; m >>= 1) {
    const int h = m >> 1;
    int j1 = 0;
    for (int i = 0; i < h; ++i) {
      const u64 S = W[h + i];
      for (int j = j1; j < j1 + t; ++j) {
        const u64 U = a[j], V = a[j + t];
        a[j] = addmod(U, V, q);
        a[j + t] = mulmod(submod(U, V, q), S, q);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (int j = 0; j < c.n; ++j) a[j] = mulmod(a[j], c.n_inv[pi], q);
}

// NTT-domain automorphism X -> X^g: out[i] = in[idx(i)].
void automorph(const Ctx& c, const u64* in, u64* out, u64 g) {
  const u64 m2 = 2ull * c.n;
  for (int i = 0; i < c.n; ++i) {
    const u64 e = 2 * bitrev(i, c.logn) + 1;
    const u64 e2 = (e * g) % m2;
    out[i] = in[bitrev((e2 - 1) / 2, c.logn)];
  }
}

u64 galois_elt(const Ctx& c, int r) {
  const int rr = ((r % c.slots) + c.slots) % c.slots;
  return powmod(5, (u64)rr, 2ull * c.n);
}

// --- encoder ----------------------------------------------
void fft_inv(const Ctx& c, std::vector<double>& re, std::vector<double>& im) {
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

void fft_fwd(const Ctx& c, std::vector<double>& re, std::vector<double>& im) {
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

// slot j <-> transform index br((5^j mod 2n - 1)/2); conjugate at 2n - 5^j.
std::vector<i64> encode_coeffs(const Ctx& c, const double* slots, double scale) {
  std::vector<double> re(c.n, 0.0), im(c.n, 0.0);
  const u64 m2 = 2ull * c.n;
  u64 e = 1;
  for (int j = 0; j < c.n / 2; ++j) {
    const double v = slots[j % c.slots];
    re[bitrev((e - 1) / 2, c.logn)] = v;
    re[bitrev((m2 - e - 1) / 2, c.logn)] = v;
    e = (e * 5) % m2;
  }
  fft_inv(c, re, im);
  const double f = scale / (double)c.n;
  std::vector<i64> out(c.n);
  for (int k = 0; k < c.n; ++k) {
    const double v = re[k] * f;
    if (!(std::fabs(v) < 4.0e18)) throw std::runtime_error("DomainViolation: encode: value too large for scale");
    out[k] = std::llround(v);
  }
  return out;
}

void encode_ntt(const Ctx& c, const double* slots, double scale, int limbs, u64* out) {
  const auto co = encode_coeffs(c, slots, scale);
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) {
    const u64 q = c.primes[l];
    u64* o = out + (size_t)l * c.n;
    for (int k = 0; k < c.n; ++k) o[k] = to_mod(co[k], q);
    ntt_fwd(c, l, o);
  }
}

void decode_coeffs(const Ctx& c, const std::vector<double>& coeff, double scale, double* slots) {
  std::vector<double> re(coeff), im(c.n, 0.0);
  fft_fwd(c, re, im);
  const u64 m2 = 2ull * c.n;
  u64 e = 1;
  for (int j = 0; j < c.slots; ++j) {
    slots[j] = re[bitrev((e - 1) / 2, c.logn)] / scale;
    e = (e * 5) % m2;
  }
}

// --- key material -------------------------------------------
constexpr u64 kStreamSk = 1ull << 56, kStreamKeyA = 2ull << 56, kStreamKeyE = 3ull << 56,
              kStreamEncA = 4ull << 56, kStreamEncE = 5ull << 56;

void sample_sk(Ctx& c) {
  c.sk.assign((size_t)c.np() * c.n, 0);
  std::vector<i64> s(c.n);
  for (int k = 0; k < c.n; ++k) s[k] = (i64)(rand64(c.seed, kStreamSk, k) % 3) - 1;
#pragma omp parallel for
  for (int m = 0; m < c.np(); ++m) {
    u64* o = c.sk.data() + (size_t)m * c.n;
    for (int k = 0; k < c.n; ++k) o[k] = to_mod(s[k], c.primes[m]);
    ntt_fwd(c, m, o);
  }
}

u64 P_mod(const Ctx& c, u64 q) {
  u64 r = 1 % q;
  for (int k = 0; k < c.alpha; ++k) r = mulmod(r, c.primes[c.P_index(k)] % q, q);
  return r;
}

constexpr u64 kRelinWide = 1;  // the single-digit relinearisation key

// digit size of a relinearisation at `limbs` limbs: ONE digit over all limbs when
// log2(Q_l / P) <= 30 (the switch runs at the product scale), else alpha
int relin_digit(const Ctx& c, int limbs) {
  double lq = 0.0, lp = 0.0;
  for (int l = 0; l < limbs; ++l) lq += std::log2((double)c.primes[l]);
  for (int k = 0; k < c.alpha; ++k) lp += std::log2((double)c.primes[c.P_index(k)]);
  return (limbs > c.alpha && limbs <= 8 && lq - lp <= 30.0) ? limbs : c.alpha;
}

// key for target s' (NTT domain over all primes): [ndig][2 (b,a)][np][n], digits of
// `dig` Q primes (alpha; all Q primes for the wide relinearisation key)
constexpr u64 kKeyGalMask = (1ull << 40) - 1;  // key id: galois element | digit size (other than alpha) << 40

// largest digit size whose digits all stay within P 2^30 (at most 8 limbs): the key
// switches of ciphertexts at scale >= 2^80 (the HE-VMM giants before their rescale)
int scaled_digit(const Ctx& c, int limbs) {
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

std::vector<u64> make_ksk(const Ctx& c, u64 kid, const std::vector<u64>& sprime) {
  const int np = c.np(), n = c.n;
  const u64 gal = kid & kKeyGalMask, kd = kid >> 40;
  const int dig = kid == kRelinWide ? c.nq() : (kd ? (int)kd : c.alpha);
  const int ndig = (c.nq() + dig - 1) / dig;
  std::vector<u64> key((size_t)ndig * 2 * np * n);
  for (int j = 0; j < ndig; ++j) {
    std::vector<i64> e(n);
    const u64 tag = (gal << 16) | ((u64)j << 8) | (kd << 44);  // independent streams per digit layout
    for (int k = 0; k < n; ++k) e[k] = cbd21(rand64(c.seed, kStreamKeyE | tag, k));
    const int lo = j * dig, hi = std::min((j + 1) * dig, c.nq());
#pragma omp parallel for
    for (int m = 0; m < np; ++m) {
      const u64 q = c.primes[m];
      u64* b = key.data() + (((size_t)j * 2 + 0) * np + m) * n;
      u64* a = key.data() + (((size_t)j * 2 + 1) * np + m) * n;
      std::vector<u64> et(n);
      for (int k = 0; k < n; ++k) et[k] = to_mod(e[k], q);
      ntt_fwd(c, m, et.data());
      const u64 pm = (m >= lo && m < hi) ? P_mod(c, q) : 0;
      const u64* s = c.sk.data() + (size_t)m * n;
      const u64* sp = sprime.data() + (size_t)m * n;
      for (int k = 0; k < n; ++k) {
        a[k] = rand_mod(c.seed, kStreamKeyA | tag | (u64)m, k, q);
        u64 v = submod(et[k], mulmod(a[k], s[k], q), q);
        if (pm) v = addmod(v, mulmod(pm, sp[k], q), q);
        b[k] = v;
      }
    }
  }
  return key;
}

const std::vector<u64>& get_key(Ctx& c, u64 g) {
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.keys.find(g);
  if (it != c.keys.end()) return it->second;
  std::vector<u64> sp((size_t)c.np() * c.n);
  for (int m = 0; m < c.np(); ++m) {
    const u64* s = c.sk.data() + (size_t)m * c.n;
    u64* o = sp.data() + (size_t)m * c.n;
    const u64 gal = g & kKeyGalMask;
    if (gal == 0 || g == kRelinWide) {
      for (int k = 0; k < c.n; ++k) o[k] = mulmod(s[k], s[k], c.primes[m]);
    } else {
      automorph(c, s, o, gal);
    }
  }
  return c.keys.emplace(g, make_ksk(c, g, sp)).first->second;
}

// --- core ops ------------------------------------------------------------------
Ct* new_ct(const Ctx& c, int limbs, double scale) {
  auto* r = new Ct;
  r->limbs = limbs;
  r->scale = scale;
  r->d.assign((size_t)2 * limbs * c.n, 0);
  return r;
}
u64* poly(const Ctx& c, Ct* ct, int p, int l) { return ct->d.data() + ((size_t)p * ct->limbs + l) * c.n; }
const u64* poly(const Ctx& c, const Ct* ct, int p, int l) {
  return ct->d.data() + ((size_t)p * ct->limbs + l) * c.n;
}

Ct* encrypt(Ctx& c, const double* slots, int limbs, double scale, u64 seed) {
  Ct* r = new_ct(c, limbs, scale);
  std::vector<u64> m((size_t)limbs * c.n);
  encode_ntt(c, slots, scale, limbs, m.data());
  std::vector<i64> e(c.n);
  for (int k = 0; k < c.n; ++k) e[k] = cbd21(rand64(seed, kStreamEncE, k));
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) {
    const u64 q = c.primes[l];
    std::vector<u64> et(c.n);
    for (int k = 0; k < c.n; ++k) et[k] = to_mod(e[k], q);
    ntt_fwd(c, l, et.data());
    u64* c0 = poly(c, r, 0, l);
    u64* c1 = poly(c, r, 1, l);
    const u64* s = c.sk.data() + (size_t)l * c.n;
    const u64* mm = m.data() + (size_t)l * c.n;
    for (int k = 0; k < c.n; ++k) {
      const u64 a = rand_mod(seed, kStreamEncA | (u64)l, k, q);
      c1[k] = a;
      c0[k] = addmod(submod(et[k], mulmod(a, s[k], q), q), mm[k], q);
    }
  }
  return r;
}

void decrypt(const Ctx& c, const Ct* ct, double* slots) {
  if (ct->zero) {
    std::fill(slots, slots + c.slots, 0.0);
    return;
  }
  const u64 q = c.primes[0];
  std::vector<u64> mu(c.n);
  const u64* c0 = poly(c, ct, 0, 0);
  const u64* c1 = poly(c, ct, 1, 0);
  for (int k = 0; k < c.n; ++k) mu[k] = addmod(c0[k], mulmod(c1[k], c.sk[k], q), q);
  ntt_inv(c, 0, mu.data());
  std::vector<double> co(c.n);
  for (int k = 0; k < c.n; ++k) co[k] = mu[k] > q / 2 ? -(double)(q - mu[k]) : (double)mu[k];
  decode_coeffs(c, co, ct->scale, slots);
}

Ct* drop_to(const Ctx& c, const Ct* a, int limbs) {
  Ct* r = new_ct(c, limbs, a->scale);
  r->zero = a->zero;
  for (int p = 0; p < 2; ++p)
    std::memcpy(poly(c, r, p, 0), poly(c, a, p, 0), sizeof(u64) * limbs * c.n);
  return r;
}

void check_scales(const Ct* a, const Ct* b) {
  if (a->zero || b->zero) return;
  if (std::fabs(a->scale / b->scale - 1.0) > 1e-9) throw std::runtime_error("ScaleMismatch: add: operand scales differ");
}

Ct* rescale(const Ctx& c, const Ct* a);

// bring a (at more limbs) to `limbs` limbs and scale `target`
// -- drop to limbs+1, multiply by the integer m = round(target q / scale)
// (a constant polynomial), rescale by q = primes[limbs]. Part of add/sub's
// implicit level drop; no ledger charge.
Ct* align_scale(const Ctx& c, const Ct* a, int limbs, double target) {
  const u64 q = c.primes[limbs];
  const u64 m = (u64)std::llround(target * (double)q / a->scale);
  Ct* t = new_ct(c, limbs + 1, a->scale);
  for (int p = 0; p < 2; ++p)
    for (int l = 0; l <= limbs; ++l) {
      const u64 ql = c.primes[l], ml = m % ql;
      const u64* x = poly(c, a, p, l);
      u64* o = poly(c, t, p, l);
      for (int k = 0; k < c.n; ++k) o[k] = mulmod(x[k], ml, ql);
    }
  Ct* r = rescale(c, t);
  delete t;
  r->scale = a->scale * (double)m / (double)q;
  return r;
}

Ct* addsub(const Ctx& c, const Ct* a, const Ct* b, bool sub) {
  const int limbs = std::min(a->limbs, b->limbs);
  if (a->zero && b->zero) {
    Ct* r = new_ct(c, limbs, 0.0);
    r->zero = true;
    return r;
  }
  if (!a->zero && !b->zero && std::fabs(a->scale / b->scale - 1.0) > 1e-9 && a->limbs != b->limbs &&
      a->d2.empty() && b->d2.empty()) {
    const bool a_hi = a->limbs > b->limbs;
    Ct* al = align_scale(c, a_hi ? a : b, limbs, a_hi ? b->scale : a->scale);
    Ct* r = a_hi ? addsub(c, al, b, sub) : addsub(c, a, al, sub);
    delete al;
    return r;
  }
  check_scales(a, b);
  Ct* r = new_ct(c, limbs, a->zero ? b->scale : a->scale);
  const bool three = !a->d2.empty() || !b->d2.empty();
  if (three) r->d2.assign((size_t)limbs * c.n, 0);
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) {
    const u64 q = c.primes[l];
    for (int p = 0; p < 3; ++p) {
      if (p == 2 && !three) break;
      const u64* x = p < 2 ? poly(c, a, p, l) : (a->d2.empty() ? nullptr : a->d2.data() + (size_t)l * c.n);
      const u64* y = p < 2 ? poly(c, b, p, l) : (b->d2.empty() ? nullptr : b->d2.data() + (size_t)l * c.n);
      u64* o = p < 2 ? poly(c, r, p, l) : r->d2.data() + (size_t)l * c.n;
      for (int k = 0; k < c.n; ++k) {
        const u64 xv = x ? x[k] : 0, yv = y ? y[k] : 0;
        o[k] = sub ? submod(xv, yv, q) : addmod(xv, yv, q);
      }
    }
  }
  return r;
}

// divide by the top prime with rounding
Ct* rescale(const Ctx& c, const Ct* a) {
  const int L1 = a->limbs - 1;
  Ct* r = new_ct(c, L1, a->scale / (double)c.primes[L1]);
  r->zero = a->zero;
  const u64 ql = c.primes[L1];
  for (int p = 0; p < 2; ++p) {
    std::vector<u64> x(poly(c, a, p, L1), poly(c, a, p, L1) + c.n);
    ntt_inv(c, L1, x.data());
#pragma omp parallel for
    for (int l = 0; l < L1; ++l) {
      const u64 q = c.primes[l];
      std::vector<u64> t(c.n);
      const u64 qlm = ql % q;
      for (int k = 0; k < c.n; ++k) {
        const u64 v = x[k] % q;
        t[k] = x[k] > ql / 2 ? submod(v, qlm, q) : v;  // centred lift of x mod ql
      }
      ntt_fwd(c, l, t.data());
      const u64 inv = invmod(ql % q, q);
      const u64* in = poly(c, a, p, l);
      u64* o = poly(c, r, p, l);
      for (int k = 0; k < c.n; ++k) o[k] = mulmod(submod(in[k], t[k], q), inv, q);
    }
  }
  return r;
}

// Fast basis conversion of coefficient-domain limbs: from primes src[] to prime dst.
void conv_basis(const Ctx& c, const std::vector<int>& src, const std::vector<const u64*>& in, int dst, u64* out) {
  const u64 pd = c.primes[dst];
  const int s = (int)src.size();
  std::vector<u64> qhat_inv(s), qhat_mod(s);
  for (int i = 0; i < s; ++i) {
    const u64 qi = c.primes[src[i]];
    u64 h = 1, hm = 1 % pd;
    for (int k = 0; k < s; ++k)
      if (k != i) {
        h = mulmod(h, c.primes[src[k]] % qi, qi);
        hm = mulmod(hm, c.primes[src[k]] % pd, pd);
      }
    qhat_inv[i] = invmod(h, qi);
    qhat_mod[i] = hm;
  }
  for (int k = 0; k < c.n; ++k) {
    u64 acc = 0;
    for (int i = 0; i < s; ++i) {
      const u64 y = mulmod(in[i][k], qhat_inv[i], c.primes[src[i]]);
      acc = addmod(acc, mulmod(y % pd, qhat_mod[i], pd), pd);
    }
    out[k] = acc;
  }
}

// Key-switch inner product in the extended basis: ModUp of d
// (NTT, `limbs` limbs), the NTT-domain automorphism g applied to the ModUp
// output, and the inner product with key g, ADDED into (accb, acca) = nt limbs
// each over Q_l u P, NTT domain.
void key_switch_ext(Ctx& c, const u64* d, int limbs, u64 g, std::vector<u64>& accb, std::vector<u64>& acca,
                    int dig_in = 0) {
  const int n = c.n, np = c.np();
  // relinearisation: maybe one wide digit; rotations: alpha, or dig_in (scaled sums)
  const int dig = g == 0 ? relin_digit(c, limbs) : (dig_in ? dig_in : c.alpha);
  const u64 kid = g == 0 ? (dig != c.alpha ? kRelinWide : 0) : (dig != c.alpha ? g | ((u64)dig << 40) : g);
  const auto& key = get_key(c, kid);
  std::vector<int> T;  // extended basis, key limb indices
  for (int l = 0; l < limbs; ++l) T.push_back(l);
  for (int k = 0; k < c.alpha; ++k) T.push_back((int)c.P_index(k));
  const int nt = (int)T.size();
  std::vector<u64> dcoef(d, d + (size_t)limbs * n);
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) ntt_inv(c, l, dcoef.data() + (size_t)l * n);
  const int ndig = (limbs + dig - 1) / dig;
  for (int j = 0; j < ndig; ++j) {
    const int lo = j * dig, hi = std::min((j + 1) * dig, limbs);
    std::vector<int> src;
    std::vector<const u64*> in;
    for (int i = lo; i < hi; ++i) src.push_back(i), in.push_back(dcoef.data() + (size_t)i * n);
    std::vector<u64> ext((size_t)nt * n);
#pragma omp parallel for
    for (int t = 0; t < nt; ++t) {
      u64* e = ext.data() + (size_t)t * n;
      const int m = T[t];
      if (m >= lo && m < hi) {
        std::memcpy(e, d + (size_t)m * n, sizeof(u64) * n);
      } else {
        conv_basis(c, src, in, m, e);
        ntt_fwd(c, m, e);
      }
    }
#pragma omp parallel for
    for (int t = 0; t < nt; ++t) {
      const int m = T[t];
      const u64 q = c.primes[m];
      std::vector<u64> er(n);
      const u64* e = ext.data() + (size_t)t * n;
      if (g > 1)
        automorph(c, e, er.data(), g);
      else
        std::memcpy(er.data(), e, sizeof(u64) * n);
      const u64* b = key.data() + (((size_t)j * 2 + 0) * np + m) * n;
      const u64* a = key.data() + (((size_t)j * 2 + 1) * np + m) * n;
      u64* ob = accb.data() + (size_t)t * n;
      u64* oa = acca.data() + (size_t)t * n;
      for (int k = 0; k < n; ++k) {
        ob[k] = addmod(ob[k], mulmod(er[k], b[k], q), q);
        oa[k] = addmod(oa[k], mulmod(er[k], a[k], q), q);
      }
    }
  }
}

// ModDown of an extended-basis polynomial (nt = limbs + alpha limbs, NTT
// domain; the P limbs are consumed): out = (acc_Q - conv_{P->Q}(acc_P)) * P^-1.
void mod_down(Ctx& c, std::vector<u64>& acc, int limbs, u64* out) {
  const int n = c.n;
  std::vector<int> Pidx;
  for (int k = 0; k < c.alpha; ++k) Pidx.push_back((int)c.P_index(k));
#pragma omp parallel for
  for (int k = 0; k < c.alpha; ++k) ntt_inv(c, Pidx[k], acc.data() + (size_t)(limbs + k) * n);
  std::vector<const u64*> in;
  for (int k = 0; k < c.alpha; ++k) in.push_back(acc.data() + (size_t)(limbs + k) * n);
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) {
    const u64 q = c.primes[l];
    std::vector<u64> t(n);
    conv_basis(c, Pidx, in, l, t.data());
    ntt_fwd(c, l, t.data());
    const u64 pinv = invmod(P_mod(c, q), q);
    const u64* x = acc.data() + (size_t)l * n;
    u64* o = out + (size_t)l * n;
    for (int k = 0; k < n; ++k) o[k] = mulmod(submod(x[k], t[k], q), pinv, q);
  }
}

// ModDown and the rescale by the top prime as ONE fast basis conversion
// (DESIGN.md §3.6): X = [limbs + alpha][n] (NTT domain, Q limbs then P limbs;
// the M limbs are consumed); out (limbs - 1 limbs) =
// (X_i - conv_{M -> q_i}(X_M)) * M^-1 mod q_i, M = q_{limbs-1} * P.
void mod_down_rescale(Ctx& c, std::vector<u64>& X, int limbs, u64* out) {
  const int n = c.n;
  std::vector<int> M{limbs - 1};
  for (int k = 0; k < c.alpha; ++k) M.push_back((int)c.P_index(k));
  // coefficient forms of the M limbs: slot limbs-1 (q_top), then the P slots
  std::vector<u64> coef((size_t)M.size() * n);
#pragma omp parallel for
  for (int j = 0; j < (int)M.size(); ++j) {
    std::memcpy(coef.data() + (size_t)j * n, X.data() + (size_t)(limbs - 1 + j) * n, sizeof(u64) * n);
    ntt_inv(c, M[j], coef.data() + (size_t)j * n);
  }
  std::vector<const u64*> in;
  for (size_t j = 0; j < M.size(); ++j) in.push_back(coef.data() + j * n);
#pragma omp parallel for
  for (int l = 0; l < limbs - 1; ++l) {
    const u64 q = c.primes[l];
    std::vector<u64> t(n);
    conv_basis(c, M, in, l, t.data());
    ntt_fwd(c, l, t.data());
    const u64 minv = invmod(mulmod(P_mod(c, q), c.primes[limbs - 1] % q, q), q);
    const u64* x = X.data() + (size_t)l * n;
    u64* o = out + (size_t)l * n;
    for (int k = 0; k < n; ++k) o[k] = mulmod(submod(x[k], t[k], q), minv, q);
  }
}

// Relinearise-and-rescale in one basis conversion: for the
// degree-2 ciphertext (d0, d1, d2) at `limbs` limbs, (kb, ka) = the key-switch
// inner products of d2 under the relinearisation key (extended basis), and
// X = (kb + P d0, ka + P d1) on the Q limbs; the result, at limbs - 1 limbs, is
// (X_i - conv_{M -> q_i}(X_M)) * M^-1 mod q_i with M = q_{limbs-1} * P, i.e.
// ModDown and the rescale by the top prime as ONE fast basis conversion.
Ct* relin_rescale_merged(Ctx& c, const u64* d0, const u64* d1, const u64* d2, int limbs, double scale) {
  const int n = c.n;
  const size_t nt = (size_t)limbs + c.alpha;
  std::vector<u64> acc[2] = {std::vector<u64>(nt * n, 0), std::vector<u64>(nt * n, 0)};
  key_switch_ext(c, d2, limbs, 0, acc[0], acc[1]);
  const u64* dd[2] = {d0, d1};
  Ct* out = new_ct(c, limbs - 1, scale);
  for (int part = 0; part < 2; ++part) {
    std::vector<u64>& X = acc[part];
#pragma omp parallel for
    for (int l = 0; l < limbs; ++l) {  // X_Q = acc_Q + P d
      const u64 q = c.primes[l], pm = P_mod(c, q);
      u64* x = X.data() + (size_t)l * n;
      const u64* d = dd[part] + (size_t)l * n;
      for (int k = 0; k < n; ++k) x[k] = addmod(x[k], mulmod(d[k], pm, q), q);
    }
    mod_down_rescale(c, X, limbs, poly(c, out, part, 0));
  }
  return out;
}

// hybrid key switch of d under key `g` (ModUp, automorphism, inner product,
// ModDown of both parts). Returns (kb, ka), `limbs` limbs each.
void key_switch(Ctx& c, const u64* d, int limbs, u64 g, u64* kb, u64* ka) {
  const size_t nt = (size_t)limbs + c.alpha;
  std::vector<u64> accb(nt * c.n, 0), acca(nt * c.n, 0);
  key_switch_ext(c, d, limbs, g, accb, acca);
  mod_down(c, accb, limbs, kb);
  mod_down(c, acca, limbs, ka);
}

// Sum of rotations sum_i Rot(a_i, r_i) with ONE ModDown per part (DESIGN.md
// §3.8): every term is accumulated in the extended basis Q_l u P -- a
// rotation contributes its key-switch inner products plus P * sigma_g(c0) on
// the Q limbs, a zero rotation contributes P * (c0, c1) -- and the sum is
// brought back to Q_l once. Same value as the op-by-op sum up to the ModDown
// rounding of one instead of k terms.
// rescale: the sum is also rescaled by its top prime, in the ModDown's basis
// conversion (mod_down_rescale; the QK^T pack).
// Double hoisting (the two radix sums of fold_steps on the fused ring sizes,
// keyswitch.cu fold_steps_batch): keep_b receives the sum's b part in the
// extended basis (NTT domain, not ModDown'd; the returned b part is zero) and
// ext_b supplies it back as the c0 of every term of the next sum, sigma_g
// applied on all limbs with no P factor (it already carries it).
Ct* rot_sum(Ctx& c, const Ct* const* a, const int* rots, int k, bool rescale = false, int dig = 0,
            std::vector<u64>* keep_b = nullptr, const std::vector<u64>* ext_b = nullptr) {
  int limbs = 1 << 30;
  double scale = 0.0;
  bool any = false;
  for (int i = 0; i < k; ++i) {
    limbs = std::min(limbs, a[i]->limbs);
    if (a[i]->zero) continue;
    if (!any)
      scale = a[i]->scale, any = true;
    else if (std::fabs(a[i]->scale / scale - 1.0) > 1e-9)
      throw std::runtime_error("ScaleMismatch: add: operand scales differ");
  }
  if (rescale && limbs < 2) throw std::runtime_error("LevelUnderflow: mul_plain: no multiplicative level left");
  if (!any) return drop_to(c, a[0], rescale ? limbs - 1 : limbs);
  const int n = c.n;
  const size_t nt = (size_t)limbs + c.alpha;
  std::vector<u64> accb(nt * n, 0), acca(nt * n, 0);
  for (int i = 0; i < k; ++i) {
    if (a[i]->zero) continue;
    const int r = (int)(((long long)rots[i] % c.slots + c.slots) % c.slots);
    const u64 g = r == 0 ? 1 : galois_elt(c, r);
    if (r != 0) key_switch_ext(c, poly(c, a[i], 1, 0), limbs, g, accb, acca, dig);
    if (ext_b) {
#pragma omp parallel for
      for (int l = 0; l < (int)nt; ++l) {
        const u64 q = c.primes[l < limbs ? l : (int)c.P_index(l - limbs)];
        std::vector<u64> s0(n);
        const u64* e = ext_b->data() + (size_t)l * n;
        if (r != 0)
          automorph(c, e, s0.data(), g);
        else
          std::memcpy(s0.data(), e, sizeof(u64) * n);
        u64* ob = accb.data() + (size_t)l * n;
        for (int j = 0; j < n; ++j) ob[j] = addmod(ob[j], s0[j], q);
        if (r == 0 && l < limbs) {
          const u64 pm = P_mod(c, q);
          const u64* s1 = poly(c, a[i], 1, l);
          u64* oa = acca.data() + (size_t)l * n;
          for (int j = 0; j < n; ++j) oa[j] = addmod(oa[j], mulmod(s1[j], pm, q), q);
        }
      }
      continue;
    }
#pragma omp parallel for
    for (int l = 0; l < limbs; ++l) {
      const u64 q = c.primes[l];
      const u64 pm = P_mod(c, q);
      std::vector<u64> s0(n);
      if (r != 0)
        automorph(c, poly(c, a[i], 0, l), s0.data(), g);
      else
        std::memcpy(s0.data(), poly(c, a[i], 0, l), sizeof(u64) * n);
      u64* ob = accb.data() + (size_t)l * n;
      for (int j = 0; j < n; ++j) ob[j] = addmod(ob[j], mulmod(s0[j], pm, q), q);
      if (r == 0) {
        const u64* s1 = poly(c, a[i], 1, l);
        u64* oa = acca.data() + (size_t)l * n;
        for (int j = 0; j < n; ++j) oa[j] = addmod(oa[j], mulmod(s1[j], pm, q), q);
      }
    }
  }
  if (rescale) {
    Ct* out = new_ct(c, limbs - 1, scale / (double)c.primes[limbs - 1]);
    mod_down_rescale(c, accb, limbs, poly(c, out, 0, 0));
    mod_down_rescale(c, acca, limbs, poly(c, out, 1, 0));
    return out;
  }
  Ct* out = new_ct(c, limbs, scale);
  if (keep_b)
    *keep_b = accb;
  else
    mod_down(c, accb, limbs, poly(c, out, 0, 0));
  mod_down(c, acca, limbs, poly(c, out, 1, 0));
  return out;
}

// fold_steps' two radix sums with double hoisting (keyswitch.cu
// fold_steps_batch): the first sum's b part never leaves the extended basis.
// Ring sizes without the fused row kernels (logn < 12 or > 17, alpha > 7) and
// zero inputs take the plain two sums, as on the GPU.
Ct* fold2(Ctx& c, const Ct* a, const int* r1, int k1, const int* r2, int k2) {
  const bool dh = c.logn >= 12 && c.logn <= 17 && c.alpha <= 7 && !a->zero;
  std::vector<const Ct*> t1(k1, a);
  std::vector<u64> kb;
  Ct* mid = rot_sum(c, t1.data(), r1, k1, false, 0, dh ? &kb : nullptr);
  std::vector<const Ct*> t2(k2, mid);
  Ct* out = rot_sum(c, t2.data(), r2, k2, false, 0, nullptr, dh ? &kb : nullptr);
  delete mid;
  return out;
}

Ct* rotate(Ctx& c, const Ct* a, int r) {
  const u64 g = galois_elt(c, r);
  if (a->zero) return drop_to(c, a, a->limbs);
  Ct* out = new_ct(c, a->limbs, a->scale);
  const int n = c.n, limbs = a->limbs;
  std::vector<u64> kb((size_t)limbs * n), ka((size_t)limbs * n);
  key_switch(c, poly(c, a, 1, 0), limbs, g, kb.data(), ka.data());
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) {
    const u64 q = c.primes[l];
    automorph(c, poly(c, a, 0, l), poly(c, out, 0, l), g);
    u64* o0 = poly(c, out, 0, l);
    u64* o1 = poly(c, out, 1, l);
    for (int k = 0; k < n; ++k) {
      o0[k] = addmod(o0[k], kb[(size_t)l * n + k], q);
      o1[k] = ka[(size_t)l * n + k];
    }
  }
  return out;
}

Ct* mul(Ctx& c, const Ct* a, const Ct* b) {
  const int limbs = std::min(a->limbs, b->limbs);
  const int n = c.n;
  if (a->zero || b->zero) {
    Ct* r = new_ct(c, limbs - 1, 0.0);
    r->zero = true;
    return r;
  }
  std::vector<u64> d((size_t)3 * limbs * n);
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) {
    const u64 q = c.primes[l];
    const u64 *a0 = poly(c, a, 0, l), *a1 = poly(c, a, 1, l), *b0 = poly(c, b, 0, l), *b1 = poly(c, b, 1, l);
    u64* o0 = d.data() + (size_t)l * n;
    u64* o1 = d.data() + ((size_t)limbs + l) * n;
    u64* o2 = d.data() + ((size_t)2 * limbs + l) * n;
    for (int k = 0; k < n; ++k) {
      o0[k] = mulmod(a0[k], b0[k], q);
      o1[k] = addmod(mulmod(a0[k], b1[k], q), mulmod(a1[k], b0[k], q), q);
      o2[k] = mulmod(a1[k], b1[k], q);
    }
  }
  return relin_rescale_merged(c, d.data(), d.data() + (size_t)limbs * n, d.data() + (size_t)2 * limbs * n, limbs,
                              a->scale * b->scale / (double)c.primes[limbs - 1]);
}

// Lazily relinearised sum of ct x ct products: (d0, d1, d2) =
// sum_i tensor(a_i, b_i), kept as a degree-2 ciphertext until relin_rescale.
Ct* tensor_sum(Ctx& c, const Ct* const* a, const Ct* const* b, int k) {
  int limbs = 1 << 30;
  double scale = 0.0;
  for (int i = 0; i < k; ++i) {
    limbs = std::min(limbs, std::min(a[i]->limbs, b[i]->limbs));
    if (a[i]->zero || b[i]->zero) continue;
    const double s = a[i]->scale * b[i]->scale;
    if (scale == 0.0)
      scale = s;
    else if (std::fabs(s / scale - 1.0) > 1e-9)
      throw std::runtime_error("ScaleMismatch: add: operand scales differ");
  }
  Ct* r = new_ct(c, limbs, scale);
  r->d2.assign((size_t)limbs * c.n, 0);
  r->zero = scale == 0.0;
  const int n = c.n;
#pragma omp parallel for
  for (int l = 0; l < limbs; ++l) {
    const u64 q = c.primes[l];
    u64* o0 = poly(c, r, 0, l);
    u64* o1 = poly(c, r, 1, l);
    u64* o2 = r->d2.data() + (size_t)l * n;
    for (int i = 0; i < k; ++i) {
      if (a[i]->zero || b[i]->zero) continue;
      const u64 *a0 = poly(c, a[i], 0, l), *a1 = poly(c, a[i], 1, l), *b0 = poly(c, b[i], 0, l),
                *b1 = poly(c, b[i], 1, l);
      for (int j = 0; j < n; ++j) {
        o0[j] = addmod(o0[j], mulmod(a0[j], b0[j], q), q);
        o1[j] = addmod(o1[j], addmod(mulmod(a0[j], b1[j], q), mulmod(a1[j], b0[j], q), q), q);
        o2[j] = addmod(o2[j], mulmod(a1[j], b1[j], q), q);
      }
    }
  }
  return r;
}

Ct* relin_rescale(Ctx& c, const Ct* x) {
  const int limbs = x->limbs, n = c.n;
  if (x->zero) {
    Ct* z = new_ct(c, limbs - 1, 0.0);
    z->zero = true;
    return z;
  }
  if (x->d2.empty()) throw std::runtime_error("relin_rescale: not a degree-2 ciphertext");
  (void)n;
  return relin_rescale_merged(c, poly(c, x, 0, 0), poly(c, x, 1, 0), x->d2.data(), limbs,
                              x->scale / (double)c.primes[limbs - 1]);
}

// Relinearisation without the rescale (the Score*V giants):
// (d0, d1) + the hybrid key switch of d2 under the relinearisation key, same
// limbs and scale.
Ct* relin(Ctx& c, const Ct* x) {
  const int limbs = x->limbs, n = c.n;
  Ct* out = new_ct(c, limbs, x->scale);
  if (x->zero) {
    out->zero = true;
    return out;
  }
  if (x->d2.empty()) throw std::runtime_error("relin: not a degree-2 ciphertext");
  std::vector<u64> kb((size_t)limbs * n), ka((size_t)limbs * n);
  key_switch(c, x->d2.data(), limbs, 0, kb.data(), ka.data());
  for (int part = 0; part < 2; ++part) {
    const u64* k = part ? ka.data() : kb.data();
#pragma omp parallel for
    for (int l = 0; l < limbs; ++l) {
      const u64 q = c.primes[l];
      const u64* d = poly(c, x, part, l);
      u64* o = poly(c, out, part, l);
      for (int i = 0; i < n; ++i) o[i] = addmod(d[i], k[(size_t)l * n + i], q);
    }
  }
  return out;
}

// sum_k ct_k (*) pt_k with plaintexts encoded at scale q_top (so the scale is
// preserved), one rescale at the end (lazy rescale of a MAC).
Ct* mac_plain(Ctx& c, const Ct* const* cts, const double* slots, int k, bool rescale_out = true) {
  int limbs = 1 << 30;
  for (int i = 0; i < k; ++i) limbs = std::min(limbs, cts[i]->limbs);
  const u64 qtop = c.primes[limbs - 1];
  double scale = 0.0;
  for (int i = 0; i < k; ++i)
    if (!cts[i]->zero) {
      if (scale == 0.0)
        scale = cts[i]->scale;
      else if (std::fabs(cts[i]->scale / scale - 1.0) > 1e-9)
        throw std::runtime_error("ScaleMismatch: mac_plain: operand scales differ");
    }
  Ct* acc = new_ct(c, limbs, scale * (double)qtop);
  std::vector<u64> pt((size_t)limbs * c.n);
  bool any = false;
  for (int i = 0; i < k; ++i) {
    if (cts[i]->zero) continue;
    any = true;
    encode_ntt(c, slots + (size_t)i * c.slots, (double)qtop, limbs, pt.data());
#pragma omp parallel for
    for (int l = 0; l < limbs; ++l) {
      const u64 q = c.primes[l];
      for (int p = 0; p < 2; ++p) {
        const u64* x = poly(c, cts[i], p, l);
        const u64* y = pt.data() + (size_t)l * c.n;
        u64* o = poly(c, acc, p, l);
        for (int j = 0; j < c.n; ++j) o[j] = addmod(o[j], mulmod(x[j], y[j], q), q);
      }
    }
  }
  acc->zero = !any;
  if (!rescale_out) {  // the raw products at scale * q_top (the caller rescales later)
    if (acc->zero) acc->scale = 0.0;
    return acc;
  }
  Ct* r = rescale(c, acc);
  r->scale = acc->zero ? 0.0 : scale;
  delete acc;
  return r;
}

Ct* add_plain(Ctx& c, const Ct* a, const double* slots) {
  if (a->zero) throw std::runtime_error("InvalidTarget: add_plain on a trivial zero ciphertext");
  Ct* r = drop_to(c, a, a->limbs);
  std::vector<u64> pt((size_t)a->limbs * c.n);
  encode_ntt(c, slots, a->scale, a->limbs, pt.data());
  for (int l = 0; l < a->limbs; ++l) {
    const u64 q = c.primes[l];
    u64* o = poly(c, r, 0, l);
    for (int k = 0; k < c.n; ++k) o[k] = addmod(o[k], pt[(size_t)l * c.n + k], q);
  }
  return r;
}

template <class F>
void* guard(F f) {
  try {
    return f();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

}  // namespace

extern "C" {

const char* ock_last_error() { return g_err.c_str(); }

void* ock_context_new(int logn, int slots, int L, int q0_bits, int scale_bits, int alpha, int special_bits,
                      uint64_t seed) {
  return guard([&]() -> void* {
    auto* c = new Ctx;
    c->logn = logn;
    c->n = 1 << logn;
    c->slots = slots;
    c->L = L;
    c->alpha = alpha;
    c->beta = (L + 1 + alpha - 1) / alpha;
    c->delta = std::ldexp(1.0, scale_bits);
    c->seed = seed;
    c->primes = gen_primes(logn, L, q0_bits, scale_bits, alpha, special_bits);
    const int np = c->np();
    c->psi_rev.resize(np);
    c->psi_inv_rev.resize(np);
    c->n_inv.resize(np);
    for (int m = 0; m < np; ++m) {
      const u64 q = c->primes[m];
      const u64 psi = min_psi(q, c->n), psi_inv = invmod(psi, q);
      c->psi_rev[m].resize(c->n);
      c->psi_inv_rev[m].resize(c->n);
      for (int k = 0; k < c->n; ++k) {
        const u64 e = bitrev(k, logn);
        c->psi_rev[m][k] = powmod(psi, e, q);
        c->psi_inv_rev[m][k] = powmod(psi_inv, e, q);
      }
      c->n_inv[m] = invmod((u64)c->n, q);
    }
    c->fft_re.resize(c->n);
    c->fft_im.resize(c->n);
    for (int k = 0; k < c->n; ++k) {
      const double ang = kPi * (double)bitrev(k, logn) / (double)c->n;
      c->fft_re[k] = std::cos(ang);
      c->fft_im[k] = std::sin(ang);
    }
    sample_sk(*c);
    return c;
  });
}

void ock_context_free(void* c) { delete static_cast<Ctx*>(c); }
int ock_num_primes(void* c) { return static_cast<Ctx*>(c)->np(); }
void ock_primes(void* c, uint64_t* out) {
  auto* x = static_cast<Ctx*>(c);
  std::copy(x->primes.begin(), x->primes.end(), out);
}
void ock_secret_key(void* c, uint64_t* out) {
  auto* x = static_cast<Ctx*>(c);
  std::copy(x->sk.begin(), x->sk.end(), out);
}
// key for galois element g (0 = relinearisation): [beta][2][np][n]
void ock_key(void* c, uint64_t g, uint64_t* out) {
  const auto& k = get_key(*static_cast<Ctx*>(c), g);
  std::copy(k.begin(), k.end(), out);
}
uint64_t ock_galois_elt(void* c, int r) { return galois_elt(*static_cast<Ctx*>(c), r); }

void ock_ntt(void* c, int pi, uint64_t* a, int inverse) {
  auto* x = static_cast<Ctx*>(c);
  inverse ? ntt_inv(*x, pi, a) : ntt_fwd(*x, pi, a);
}
void ock_automorph(void* c, const uint64_t* in, uint64_t* out, uint64_t g) {
  automorph(*static_cast<Ctx*>(c), in, out, g);
}
int ock_encode(void* c, const double* slots, double scale, int limbs, uint64_t* out) {
  return guard([&]() -> void* {
           encode_ntt(*static_cast<Ctx*>(c), slots, scale, limbs, out);
           return (void*)1;
         }) != nullptr
             ? 0
             : -1;
}
int ock_encode_coeffs(void* c, const double* slots, double scale, int64_t* out) {
  return guard([&]() -> void* {
           auto v = encode_coeffs(*static_cast<Ctx*>(c), slots, scale);
           std::copy(v.begin(), v.end(), out);
           return (void*)1;
         }) != nullptr
             ? 0
             : -1;
}

void* ock_encrypt(void* c, const double* slots, int limbs, double scale, uint64_t seed) {
  return guard([&]() -> void* { return encrypt(*static_cast<Ctx*>(c), slots, limbs, scale, seed); });
}
void* ock_zero(void* c, int limbs) {
  Ct* r = new_ct(*static_cast<Ctx*>(c), limbs, 0.0);
  r->zero = true;
  return r;
}
void* ock_import(void* c, const uint64_t* data, int limbs, double scale, int zero) {
  Ct* r = new_ct(*static_cast<Ctx*>(c), limbs, scale);
  std::copy(data, data + r->d.size(), r->d.begin());
  r->zero = zero != 0;
  return r;
}
void ock_ct_free(void* ct) { delete static_cast<Ct*>(ct); }
void ock_ct_info(void* ct, int* limbs, double* scale, int* zero) {
  auto* x = static_cast<Ct*>(ct);
  *limbs = x->limbs;
  *scale = x->scale;
  *zero = x->zero ? 1 : 0;
}
void ock_ct_data(void* ct, uint64_t* out) {
  auto* x = static_cast<Ct*>(ct);
  std::copy(x->d.begin(), x->d.end(), out);
}
void ock_decrypt(void* c, void* ct, double* slots) { decrypt(*static_cast<Ctx*>(c), static_cast<Ct*>(ct), slots); }

void* ock_add(void* c, void* a, void* b) {
  return guard([&]() -> void* { return addsub(*static_cast<Ctx*>(c), (Ct*)a, (Ct*)b, false); });
}
void* ock_sub(void* c, void* a, void* b) {
  return guard([&]() -> void* { return addsub(*static_cast<Ctx*>(c), (Ct*)a, (Ct*)b, true); });
}
void* ock_add_plain(void* c, void* a, const double* slots) {
  return guard([&]() -> void* { return add_plain(*static_cast<Ctx*>(c), (Ct*)a, slots); });
}
void* ock_mac_plain(void* c, void** cts, const double* slots, int k) {
  return guard([&]() -> void* { return mac_plain(*static_cast<Ctx*>(c), (Ct* const*)cts, slots, k); });
}
void* ock_mul(void* c, void* a, void* b) {
  return guard([&]() -> void* { return mul(*static_cast<Ctx*>(c), (Ct*)a, (Ct*)b); });
}
void* ock_rotate(void* c, void* a, int r) {
  return guard([&]() -> void* { return rotate(*static_cast<Ctx*>(c), (Ct*)a, r); });
}
void* ock_rot_sum(void* c, void** a, const int* rots, int k) {
  return guard([&]() -> void* { return rot_sum(*static_cast<Ctx*>(c), (Ct* const*)a, rots, k); });
}
void* ock_fold2(void* c, void* a, const int* r1, int k1, const int* r2, int k2) {
  return guard([&]() -> void* { return fold2(*static_cast<Ctx*>(c), (const Ct*)a, r1, k1, r2, k2); });
}
void* ock_rot_sum_rescale(void* c, void** a, const int* rots, int k) {
  return guard([&]() -> void* { return rot_sum(*static_cast<Ctx*>(c), (Ct* const*)a, rots, k, true); });
}
// rot_sum of ciphertexts at scale >= 2^80 (the Score*V giants): scaled_digit digits
void* ock_rot_sum_scaled(void* c, void** a, const int* rots, int k) {
  return guard([&]() -> void* {
    Ctx& cx = *static_cast<Ctx*>(c);
    int limbs = 1 << 30;
    for (int i = 0; i < k; ++i) limbs = std::min(limbs, static_cast<Ct*>(a[i])->limbs);
    return rot_sum(cx, (Ct* const*)a, rots, k, false, scaled_digit(cx, limbs));
  });
}
// rot_sum_rescale of products still at scale >= 2^80 (the HE-VMM giants): the
// terms' decomposition uses scaled_digit(limbs)
void* ock_rot_sum_rescale_scaled(void* c, void** a, const int* rots, int k) {
  return guard([&]() -> void* {
    Ctx& cx = *static_cast<Ctx*>(c);
    int limbs = 1 << 30;
    for (int i = 0; i < k; ++i) limbs = std::min(limbs, static_cast<Ct*>(a[i])->limbs);
    return rot_sum(cx, (Ct* const*)a, rots, k, true, scaled_digit(cx, limbs));
  });
}
void* ock_mac_plain_lazy(void* c, void** cts, const double* slots, int k) {
  return guard([&]() -> void* { return mac_plain(*static_cast<Ctx*>(c), (Ct* const*)cts, slots, k, false); });
}
void* ock_tensor_sum(void* c, void** a, void** b, int k) {
  return guard([&]() -> void* { return tensor_sum(*static_cast<Ctx*>(c), (Ct* const*)a, (Ct* const*)b, k); });
}
void* ock_relin_rescale(void* c, void* a) {
  return guard([&]() -> void* { return relin_rescale(*static_cast<Ctx*>(c), (Ct*)a); });
}
void* ock_relin(void* c, void* a) {
  return guard([&]() -> void* { return relin(*static_cast<Ctx*>(c), (Ct*)a); });
}
int ock_ct_is_three(void* ct) { return static_cast<Ct*>(ct)->d2.empty() ? 0 : 1; }
void ock_ct_d2(void* ct, uint64_t* out) {
  auto* x = static_cast<Ct*>(ct);
  std::copy(x->d2.begin(), x->d2.end(), out);
}
void ock_ct_set_d2(void* ct, const uint64_t* in) {
  auto* x = static_cast<Ct*>(ct);
  x->d2.assign(in, in + (size_t)x->limbs * (x->d.size() / (2 * (size_t)x->limbs)));
}
void* ock_rescale(void* c, void* a) {
  return guard([&]() -> void* { return rescale(*static_cast<Ctx*>(c), (Ct*)a); });
}
void* ock_level_drop(void* c, void* a, int limbs) {
  return guard([&]() -> void* { return drop_to(*static_cast<Ctx*>(c), (Ct*)a, limbs); });
}
// One raw ChaCha20 block (the KAT hook of tests/test_ckks_oracle.py).
void ock_chacha20_block(const uint32_t* key, uint64_t counter, uint64_t nonce, uint32_t* out) {
  chacha20_block(key, counter, nonce, out);
}
uint64_t ock_rand64(uint64_t seed, uint64_t stream, uint64_t ctr) { return rand64(seed, stream, ctr); }
// The reference bench weight W[r][c] = sin(0.001 (31 r + c) + 0.25)
// (slotforge_cli.cpp:88-92), row-major rows x cols, evaluated with the same
// libm sin and operation order as the product's W = NULL plans.
void ock_bench_weight(int rows, int cols, double* out) {
#pragma omp parallel for
  for (int r = 0; r < rows; ++r)
    for (int cc = 0; cc < cols; ++cc) out[(size_t)r * cols + cc] = std::sin(0.001 * ((double)r * 31.0 + cc) + 0.25);
}

}  // extern "C"
