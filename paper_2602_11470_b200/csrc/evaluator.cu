// Context construction, key generation and the CKKS evaluator on one B200.
//
// Level / ledger semantics are the reference's (engine.hpp:102-111,
// engine.cpp:143-214); the arithmetic is full-RNS CKKS with hybrid key
// switching per DESIGN.md §3. Op sequences here are the spec the CPU oracle
// (oracle/ckks_oracle.cpp) restates, which is what makes every ciphertext word
// bit-identical between the two.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <functional>
#include <thread>
#include <unordered_map>

#include <cstdlib>

#include "context.h"
#include "kernels.cuh"

namespace sf {

void build_host_tables(Context& c, std::vector<u64>& psi, std::vector<u64>& psi_s, std::vector<u64>& ipsi,
                       std::vector<u64>& ipsi_s, std::vector<u64>& ninv, std::vector<u64>& ninv_s);

// ------------------------------------------------------------------ memory
namespace {
std::mutex g_live_mu;
std::unordered_map<const Context*, u64> g_live;
std::atomic<u64> g_next_gen{1};
}  // namespace
bool context_alive(const Context* c, u64 gen) {
  std::lock_guard<std::mutex> lk(g_live_mu);
  auto it = g_live.find(c);
  return it != g_live.end() && it->second == gen;
}

Buf::Buf(Context* c, size_t w) : words(w), ctx(c), gen(c->gen) {
  SF_HPROF("cudaMallocAsync");
  if (c->capturing) gm = c->capture_gm;
  if (!w) return;
  if (!c->capturing) {  // eager: reuse a released buffer of the same size (stream-ordered)
    std::lock_guard<std::mutex> lk(c->alloc_mu);
    auto it = c->free_bufs.find(w);
    if (it != c->free_bufs.end() && !it->second.empty()) {
      p = it->second.back();
      it->second.pop_back();
      c->cached_words -= w;
      return;
    }
  }
  SF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), w * sizeof(u64), c->stream));
}
Buf::~Buf() {
  SF_HPROF("cudaFreeAsync");
  if (!p) return;
  if (!context_alive(ctx, gen)) {  // released after its context: no stream, no free lists
    cudaFree(p);
    return;
  }
  if (gm) {  // a graph memory node
    if (ctx->capturing && ctx->capture_gm == gm) {
      cudaFreeAsync(p, ctx->stream);  // allocated and freed inside the same capture: a free node
      return;
    }
    std::lock_guard<std::mutex> lk(gm->mu);
    if (!gm->destroyed) {
      gm->dead.push_back(p);  // the graph still re-allocates it on replay; freed at sf_graph_destroy
    } else if (gm->launched) {
      cudaFreeAsync(p, ctx->stream);  // outstanding allocation of a destroyed graph
    }
    return;
  }
  if (ctx->capturing) {
    ctx->capture_deferred.push_back({p, words});  // a replay still reads it
    return;
  }
  {
    std::lock_guard<std::mutex> lk(ctx->alloc_mu);
    if (ctx->cached_words + words <= ctx->cache_cap_words) {
      ctx->free_bufs[words].push_back(p);
      ctx->cached_words += words;
      return;
    }
  }
  cudaFreeAsync(p, ctx->stream);
}

BufPtr make_buf(Context& c, size_t words) { return std::make_shared<Buf>(&c, words); }
static BufPtr buf(Context& c, size_t words) { return make_buf(c, words); }

Context::~Context() {
  if (stream) cudaStreamSynchronize(stream);
  p2p_destroy(*this);
  keys.clear();
  keys_pinv.clear();
  keys_r.clear();
  key_graveyard.clear();
  conv_plans.clear();
  pt_cache.clear();
  rot_memo.clear();
  level_consts.clear();
  merged_consts.clear();
  sk.reset();
  tab_store.reset();
  for (auto e : events) cudaEventDestroy(e);
  for (auto& [f, d] : stage_ev) cudaEventDestroy(f), cudaEventDestroy(d);
  if (copy_stream) cudaStreamSynchronize(copy_stream), cudaStreamDestroy(copy_stream);
  for (auto& st : stage) {
    if (st.ev) cudaEventDestroy(st.ev);
    if (st.p) cudaFreeHost(st.p);
  }
  stage.clear();
  for (auto& [w, v] : free_bufs)
    for (u64* q : v) cudaFreeAsync(q, stream);
  free_bufs.clear();
  {  // from here on, buffers still referenced elsewhere free themselves (Buf::~Buf)
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_live.erase(this);
  }
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

u64 Context::next_seed() {
  const u64 k = enc_counter++;
  return fmix64(seed ^ (0xE1C0000000000000ull + k));
}

std::unique_ptr<Context> make_context(int slots, int L, int log_n, int alpha, int q0_bits, int scale_bits,
                                      int special_bits, u64 seed, int device) {
  require(is_pow2(slots), kShapeMismatch, "engine: N must be a power of two");
  require(L >= 1, kInvalidTarget, "engine: level budget L must be >= 1");
  auto c = std::make_unique<Context>();
  c->gen = g_next_gen.fetch_add(1);
  {
    std::lock_guard<std::mutex> lk(g_live_mu);
    g_live[c.get()] = c->gen;
  }
  c->slots = slots;
  c->L = L;
  c->logn = log_n > 0 ? log_n : std::max(2, log2_exact(2LL * slots));
  c->n = 1 << c->logn;
  require(2LL * slots <= c->n, kShapeMismatch, "ckks: slot count exceeds ring degree / 2");
  require(c->logn <= 17, kShapeMismatch, "ckks: ring degree above 2^17 not supported");
  c->alpha = alpha > 0 ? alpha : std::min(L + 1, 5);
  c->beta = (L + 1 + c->alpha - 1) / c->alpha;
  c->seed = seed;
  c->device = device;
  if (const char* e = std::getenv("SF_KS_ROW")) c->ks_row = std::atoi(e) != 0;
  if (const char* e = std::getenv("SF_FUSED_CPW")) c->fused_cpw = std::atoi(e);
  if (const char* e = std::getenv("SF_VARIANT")) c->variant = std::atoi(e);
  if (const char* e = std::getenv("SF_FREE_CACHE_GIB")) c->cache_cap_words = (size_t)(std::atof(e) * (1u << 27));
  if (const char* e = std::getenv("SF_ROT_CHUNK")) c->rot_chunk = std::atoi(e);
  c->delta = std::ldexp(1.0, scale_bits > 0 ? scale_bits : 40);
  c->primes = generate_primes(c->logn, L, q0_bits > 0 ? q0_bits : 60, scale_bits > 0 ? scale_bits : 40, c->alpha,
                              special_bits > 0 ? special_bits : 60);
  c->np = (int)c->primes.size();
  require(c->np <= 64, kShapeMismatch, "ckks: at most 64 RNS primes");

  SF_CUDA(cudaSetDevice(device));
  SF_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  SF_CUDA(cudaDeviceGetDefaultMemPool(&c->pool, device));
  uint64_t thresh = UINT64_MAX;
  SF_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thresh));

  std::vector<u64> psi, psi_s, ipsi, ipsi_s, ninv, ninv_s;
  build_host_tables(*c, psi, psi_s, ipsi, ipsi_s, ninv, ninv_s);
  const size_t np = c->np, n = c->n;
  c->ipsi1_h.resize(np);
  std::vector<u64> ninvw(np), ninvw_s(np);
  for (size_t p = 0; p < np; ++p) {
    c->ipsi1_h[p] = ipsi[p * n + 1];
    ninvw[p] = mulmod_h(ninv[p], c->ipsi1_h[p], c->primes[p]);
    ninvw_s[p] = shoup_h(ninvw[p], c->primes[p]);
  }
  const size_t words = 5 * np + 4 * np * n + 4 * np;
  c->tab_store = buf(*c, words);
  std::vector<u64> host(words);
  u64* h = host.data();
  size_t off = 0;
  auto put = [&](const std::vector<u64>& v) {
    std::memcpy(h + off, v.data(), v.size() * sizeof(u64));
    const size_t o = off;
    off += v.size();
    return c->tab_store->p + o;
  };
  c->tabs.q = put(c->primes);
  c->tabs.mh = put(c->mu_hi);
  c->tabs.ml = put(c->mu_lo);
  c->tabs.qn = put(c->qneg_inv);
  c->tabs.r64 = put(c->r64);
  c->tabs.psi = put(psi);
  c->tabs.psi_s = put(psi_s);
  c->tabs.ipsi = put(ipsi);
  c->tabs.ipsi_s = put(ipsi_s);
  c->tabs.ninv = put(ninv);
  c->tabs.ninv_s = put(ninv_s);
  c->tabs.ninvw = put(ninvw);
  c->tabs.ninvw_s = put(ninvw_s);
  c->tabs.n = c->n;
  c->tabs.logn = c->logn;
  SF_CUDA(cudaMemcpyAsync(c->tab_store->p, host.data(), words * sizeof(u64), cudaMemcpyHostToDevice, c->stream));

  // secret key: ternary coefficients, NTT over every prime
  c->sk = buf(*c, np * n);
  k_ternary(*c, c->sk->p, stream_key(seed, kStreamSk), (int)np, 0);
  ntt_limbs(*c, c->sk->p, (int)np, 0, false);
  SF_CUDA(cudaStreamSynchronize(c->stream));
  return c;
}

// ------------------------------------------------------------------ helpers
u64 galois_elt(const Context& c, int r) {
  SF_HPROF("galois_elt");
  return powmod_h(5, (u64)pos_mod(r, c.slots), 2ull * c.n);
}

Ct alloc_ct(Context& c, int limbs, double scale) {
  SF_HPROF("alloc_ct");
  Ct r;
  r.buf = buf(c, (size_t)2 * limbs * c.n);
  r.limbs = limbs;
  r.stride = limbs;
  r.scale = scale;
  return r;
}

static Ct view(const Ct& a, int limbs) {
  SF_HPROF("view");
  Ct r = a;
  r.limbs = limbs;
  return r;
}

void check_ct(const Context& c, const Ct& a, const char* what) {
  SF_HPROF("check_ct");
  require(a.buf != nullptr, kInvalidTarget, std::string(what) + ": null ciphertext");
  require(a.level() >= 0 && a.level() <= c.L, kInvalidTarget,
          std::string(what) + ": ciphertext level " + std::to_string(a.level()) + " out of [0, L]");
}

void check_scales(const Ct& a, const Ct& b, const char* what) {
  SF_HPROF("check_scales");
  if (a.zero || b.zero) return;
  if (std::fabs(a.scale / b.scale - 1.0) > 1e-9)
    fail(kScaleMismatch, std::string("ScaleMismatch: ") + what + ": operand scales differ");
}

OptLayout merge_layouts(const Ct& a, const Ct& b) {
  if (a.layout && b.layout && *a.layout == *b.layout) return a.layout;
  return std::nullopt;
}

// device constants for `limbs` active limbs: rescale (drop limb limbs-1) and
// ModDown (P -> Q_limbs): [inv_ql, inv_ql_s, pinv, pinv_s] each `limbs` words
const u64* level_consts(Context& c, int limbs) {
  SF_HPROF("level_consts");
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.level_consts.find(limbs);
  if (it != c.level_consts.end()) return it->second->p;
  std::vector<u64> h(4 * (size_t)limbs, 0);
  const u64 ql = c.primes[limbs - 1];
  for (int i = 0; i < limbs; ++i) {
    const u64 q = c.primes[i];
    if (i < limbs - 1) {
      h[i] = invmod_h(ql % q, q);
      h[limbs + i] = shoup_h(h[i], q);
    }
    u64 pm = 1 % q;
    for (int k = 0; k < c.alpha; ++k) pm = mulmod_h(pm, c.primes[c.P_index(k)] % q, q);
    h[2 * limbs + i] = invmod_h(pm, q);
    h[3 * limbs + i] = shoup_h(h[2 * limbs + i], q);
  }
  BufPtr b = buf(c, h.size());
  SF_CUDA(cudaMemcpyAsync(b->p, h.data(), h.size() * sizeof(u64), cudaMemcpyHostToDevice, c.stream));
  host_sync(c);  // h goes out of scope
  c.level_consts[limbs] = b;
  c.level_consts_h[limbs] = h;
  return b->p;
}

const ConvPlan& conv_plan(Context& c, const std::vector<int>& src, const std::vector<int>& dst, bool pinv) {
  SF_HPROF("conv_plan");
  std::string key;
  for (int s : src) key += std::to_string(s) + ",";
  key += ">";
  for (int d : dst) key += std::to_string(d) + ",";
  if (pinv) key += ":pinv";  // destination constants times (prod src)^-1: ModDown with the P^-1 folded in
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.conv_plans.find(key);
  if (it != c.conv_plans.end()) return it->second;
  ConvPlan p;
  p.src = src;
  p.dst = dst;
  p.nsrc = (int)src.size();
  p.ndst = (int)dst.size();
  // [nsrc] qhat^-1, [nsrc] Shoup, [nsrc][ndst] qhat mod dst,
  // then for the fused column stage: [nsrc] n^-1 qhat^-1, [nsrc] Shoup, [nsrc][ndst] Shoup of qhat mod dst
  const size_t base2 = 2 * (size_t)p.nsrc + (size_t)p.nsrc * p.ndst;
  // + [nsrc] y-factor times the last inverse column stage's twiddle (ipsi[1]), [nsrc] Shoup
  std::vector<u64> h(2 * base2 + 2 * (size_t)p.nsrc);
  for (int i = 0; i < p.nsrc; ++i) {
    const u64 qi = c.primes[src[i]];
    u64 hat = 1 % qi;
    for (int k = 0; k < p.nsrc; ++k)
      if (k != i) hat = mulmod_h(hat, c.primes[src[k]] % qi, qi);
    h[i] = invmod_h(hat, qi);
    h[p.nsrc + i] = shoup_h(h[i], qi);
    for (int d = 0; d < p.ndst; ++d) {
      const u64 pd = c.primes[dst[d]];
      u64 hm = 1 % pd;
      for (int k = 0; k < p.nsrc; ++k)
        if (k != i) hm = mulmod_h(hm, c.primes[src[k]] % pd, pd);
      if (pinv) hm = invmod_h(c.primes[src[i]] % pd, pd);  // qhat_i * (prod src)^-1 = src_i^-1
      h[2 * p.nsrc + (size_t)i * p.ndst + d] = hm;
      h[base2 + 2 * p.nsrc + (size_t)i * p.ndst + d] = shoup_h(hm, pd);
    }
    const u64 ni = invmod_h((u64)c.n % qi, qi);
    h[base2 + i] = mulmod_h(ni, h[i], qi);
    h[base2 + p.nsrc + i] = shoup_h(h[base2 + i], qi);
    h[2 * base2 + i] = mulmod_h(h[base2 + i], c.ipsi1_h[src[i]], qi);
    h[2 * base2 + p.nsrc + i] = shoup_h(h[2 * base2 + i], qi);
  }
  p.tab = buf(c, h.size());
  SF_CUDA(cudaMemcpyAsync(p.tab->p, h.data(), h.size() * sizeof(u64), cudaMemcpyHostToDevice, c.stream));
  host_sync(c);
  return c.conv_plans.emplace(key, std::move(p)).first->second;
}

void upload_async(Context& c, void* dst, const void* src, size_t bytes) {
  require(!c.capturing, kInvalidTarget,
          "graph capture: a fresh plaintext / encryption upload is not capturable; run the step once eagerly "
          "before capturing it");
  constexpr size_t kSlots = 16;
  if (c.stage.empty()) c.stage.resize(kSlots);
  Context::StageSlot& st = c.stage[c.stage_next++ % kSlots];
  if (st.pending) SF_CUDA(cudaEventSynchronize(st.ev));  // the slot's previous copy has landed
  if (st.cap < bytes) {
    if (st.p) SF_CUDA(cudaFreeHost(st.p));
    st.p = nullptr;
    SF_CUDA(cudaMallocHost(&st.p, bytes));
    st.cap = bytes;
  }
  if (!st.ev) SF_CUDA(cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming));
  std::memcpy(st.p, src, bytes);
  SF_CUDA(cudaMemcpyAsync(dst, st.p, bytes, cudaMemcpyHostToDevice, c.stream));
  SF_CUDA(cudaEventRecord(st.ev, c.stream));
  st.pending = true;
}

// upload signed coefficients and reduce into `limbs` NTT-domain limbs (+ noise)
static BufPtr coeffs_to_ntt(Context& c, const std::vector<i64>& co, int limbs, bool noise, RngKey ekey) {
  SF_HPROF("coeffs_to_ntt");
  BufPtr tmp = buf(c, (size_t)c.n);
  upload_async(c, tmp->p, co.data(), co.size() * sizeof(i64));
  BufPtr out = buf(c, (size_t)limbs * c.n);
  std::vector<int> primes(limbs);
  for (int l = 0; l < limbs; ++l) primes[l] = l;
  k_small_rns(c, out->p, ekey, noise, reinterpret_cast<const i64*>(tmp->p), primes.data(), limbs);
  ntt_limbs(c, out->p, limbs, 0, false);
  return out;
}

Pt encode_pt(Context& c, const double* slots, double scale, int limbs) {
  SF_HPROF("encode_pt");
  Pt p;
  p.buf = coeffs_to_ntt(c, encode_coeffs(c, slots, scale), limbs, false, RngKey{0, 0});
  p.limbs = limbs;
  p.scale = scale;
  return p;
}

bool lookup_pt(Context& c, const std::string& key, int limbs, Pt* out) {
  std::lock_guard<std::mutex> lk(c.mu);
  auto it = c.pt_cache.find(key + "@" + std::to_string(limbs));
  if (it == c.pt_cache.end()) return false;
  *out = it->second;
  return true;
}

Pt cached_pt(Context& c, const std::string& key, const double* slots, double scale, int limbs) {
  SF_HPROF("cached_pt");
  const std::string k = key + "@" + std::to_string(limbs);
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.pt_cache.find(k);
    if (it != c.pt_cache.end()) return it->second;
  }
  Pt p = encode_pt(c, slots, scale, limbs);
  std::lock_guard<std::mutex> lk(c.mu);
  c.pt_cache[k] = p;
  return p;
}

// ------------------------------------------------------------------ client ops
Ct encrypt(Context& c, const double* slots, int level, u64 seed, OptLayout layout) {
  SF_HPROF("encrypt");
  if (level < 0) level = c.L;
  require(level <= c.L, kInvalidTarget, "encrypt: level exceeds budget L");
  if (layout) validate_layout(*layout, c.slots);
  const int limbs = level + 1;
  Ct r = alloc_ct(c, limbs, c.delta);
  r.layout = layout;
  BufPtr em = coeffs_to_ntt(c, encode_coeffs(c, slots, c.delta), limbs, true, stream_key(seed, kStreamEncE));
  std::vector<RngKey> keys(limbs);
  std::vector<int> primes(limbs);
  for (int l = 0; l < limbs; ++l) keys[l] = stream_key(seed, kStreamEncA | (u64)l), primes[l] = l;
  k_sample_uniform(c, r.c1(c.n), keys.data(), primes.data(), limbs);
  k_enc_combine(c, r.c0(), r.c1(c.n), c.sk->p, em->p, limbs);
  return r;
}

Ct zeros(Context& c, int level) {
  SF_HPROF("zeros");
  if (level < 0) level = c.L;
  require(level <= c.L, kInvalidTarget, "zeros: level exceeds budget L");
  Ct r = alloc_ct(c, level + 1, 0.0);
  SF_CUDA(cudaMemsetAsync(r.buf->p, 0, r.buf->words * sizeof(u64), c.stream));
  r.zero = true;
  return r;
}

void decrypt(Context& c, const Ct& a, double* out) {
  SF_HPROF("decrypt");
  if (a.zero) {
    std::fill(out, out + c.slots, 0.0);
    return;
  }
  BufPtr mu = buf(c, c.n);
  k_dec_combine(c, mu->p, a.c0(), a.c1(c.n), c.sk->p);
  ntt_limbs(c, mu->p, 1, 0, true);
  std::vector<u64> h(c.n);
  SF_CUDA(cudaMemcpyAsync(h.data(), mu->p, c.n * sizeof(u64), cudaMemcpyDeviceToHost, c.stream));
  host_sync(c);
  const u64 q = c.primes[0];
  std::vector<double> co(c.n);
  for (int k = 0; k < c.n; ++k) co[k] = h[k] > q / 2 ? -(double)(q - h[k]) : (double)h[k];
  decode_coeffs(c, co, a.scale, out);
}

// ------------------------------------------------------------------ evaluator
// bring a (at more limbs) to `limbs` limbs and scale
// `target`: drop to limbs+1, multiply by the integer m = round(target q /
// scale) (a constant polynomial: m mod q_i at every NTT point), rescale by
// q = primes[limbs]. Part of add/sub's implicit level drop (no ledger charge);
// it lets the residual adds of a decoder block combine a fresh chain input
// with a projection output whose scale went through ct x ct products.
Ct align_scale(Context& c, const Ct& a, int limbs, double target) {
  SF_HPROF("align_scale");
  require(a.limbs > limbs, kScaleMismatch, "ScaleMismatch: align needs a spare level");
  const u64 q = c.primes[limbs];
  const u64 m = (u64)std::llround(target * (double)q / a.scale);
  const std::string key = "const:" + std::to_string(m) + "@" + std::to_string(limbs + 1);
  Pt p;
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.pt_cache.find(key);
    if (it != c.pt_cache.end()) p = it->second;
  }
  if (!p.buf) {  // first use: upload the constant once (cached like the mask plaintexts)
    std::vector<u64> h((size_t)(limbs + 1) * c.n);
    for (int l = 0; l <= limbs; ++l)
      std::fill(h.begin() + (size_t)l * c.n, h.begin() + (size_t)(l + 1) * c.n, m % c.primes[l]);
    p.limbs = limbs + 1;
    p.scale = (double)m;
    p.buf = buf(c, h.size());
    SF_CUDA(cudaMemcpyAsync(p.buf->p, h.data(), h.size() * 8, cudaMemcpyHostToDevice, c.stream));
    host_sync(c);  // h is pageable and goes out of scope
    std::lock_guard<std::mutex> lk(c.mu);
    c.pt_cache[key] = p;
  }
  Ct t = view(a, limbs + 1);
  t.layout.reset();
  Ct r = mac_plain(c, {&t}, {&p}, false);
  r.scale = a.scale * (double)m / (double)q;
  r.layout = a.layout;
  return r;
}

Ct add(Context& c, const Ct& a, const Ct& b, bool sub, bool count) {
  SF_HPROF("add");
  check_ct(c, a, sub ? "sub" : "add");
  check_ct(c, b, sub ? "sub" : "add");
  const int limbs = std::min(a.limbs, b.limbs);
  if (!a.zero && !b.zero && std::fabs(a.scale / b.scale - 1.0) > 1e-9 && a.limbs != b.limbs) {
    const bool a_hi = a.limbs > b.limbs;
    const Ct al = align_scale(c, a_hi ? a : b, limbs, a_hi ? b.scale : a.scale);
    return a_hi ? add(c, al, b, sub, count) : add(c, a, al, sub, count);
  }
  if (count) c.ledger.add();
  OptLayout ly = merge_layouts(a, b);
  if (a.zero && b.zero) {
    Ct r = view(a, limbs);
    r.layout = ly;
    return r;
  }
  check_scales(a, b, sub ? "sub" : "add");
  if (b.zero) {  // x + 0 = x - 0 = x (exact on trivial ciphertexts)
    Ct r = view(a, limbs);
    r.layout = ly;
    return r;
  }
  Ct r = alloc_ct(c, limbs, a.zero ? b.scale : a.scale);
  r.layout = ly;
  k_addsub(c, r.c0(), a.c0(), b.c0(), limbs, sub);
  k_addsub(c, r.c1(c.n), a.c1(c.n), b.c1(c.n), limbs, sub);
  return r;
}

Ct add_plain(Context& c, const Ct& a, const double* slots) {
  SF_HPROF("add_plain");
  check_ct(c, a, "add_plain");
  require(!a.zero, kInvalidTarget, "add_plain on a trivial zero ciphertext");
  c.ledger.add();
  Pt p = encode_pt(c, slots, a.scale, a.limbs);
  Ct r = alloc_ct(c, a.limbs, a.scale);
  r.layout = a.layout;
  k_addsub(c, r.c0(), a.c0(), p.buf->p, a.limbs, false);
  k_copy(c, r.c1(c.n), a.c1(c.n), (size_t)a.limbs * c.n);
  return r;
}

Ct mac_plain(Context& c, const std::vector<const Ct*>& cts, const std::vector<const Pt*>& pts, bool count,
              bool rescale_out) {
  SF_HPROF("mac_plain");
  require(!cts.empty() && cts.size() == pts.size(), kShapeMismatch, "mac_plain: term count");
  int limbs = 1 << 30;
  for (const Ct* x : cts) {
    check_ct(c, *x, "mul_plain");
    require(x->level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
    limbs = std::min(limbs, x->limbs);
  }
  double scale = 0.0;
  for (const Ct* x : cts)
    if (!x->zero) {
      if (scale == 0.0)
        scale = x->scale;
      else if (std::fabs(x->scale / scale - 1.0) > 1e-9)
        fail(kScaleMismatch, "ScaleMismatch: mac_plain: operand scales differ");
    }
  if (count) {
    c.ledger.ctpt((long long)cts.size());
    c.ledger.add((long long)cts.size() - 1);
  }
  OptLayout ly = cts[0]->layout;
  for (const Ct* x : cts)
    if (!(x->layout == ly)) ly.reset();
  if (scale == 0.0) {  // every term trivially zero
    Ct z = zeros(c, rescale_out ? limbs - 2 : limbs - 1);
    z.layout = ly;
    return z;
  }
  Ct acc = alloc_ct(c, limbs, scale * (double)c.primes[limbs - 1]);
  for (size_t s = 0; s < cts.size(); s += kMaxTerms) {
    MacTerms t;
    t.k = 0;
    for (size_t i = s; i < cts.size() && t.k < kMaxTerms; ++i) {
      if (cts[i]->zero) continue;
      require(pts[i]->limbs >= limbs, kShapeMismatch, "mac_plain: plaintext has too few limbs");
      t.c0[t.k] = cts[i]->c0();
      t.c1[t.k] = cts[i]->c1(c.n);
      t.pt[t.k] = pts[i]->buf->p;
      ++t.k;
    }
    if (t.k == 0) continue;
    if (s == 0) {
      k_mac(c, acc.c0(), acc.c1(c.n), t, limbs);
    } else {  // chunk beyond 64 terms: accumulate into a scratch ct and add
      Ct part = alloc_ct(c, limbs, acc.scale);
      k_mac(c, part.c0(), part.c1(c.n), t, limbs);
      acc = add(c, acc, part, false, false);
    }
  }
  if (!rescale_out) {  // the raw sum at scale * q_top (the caller's rotation sum rescales)
    acc.layout = ly;
    return acc;
  }
  Ct r = rescale(c, acc);
  r.scale = scale;
  r.layout = ly;
  return r;
}

Ct mul_plain(Context& c, const Ct& a, const double* slots) {
  SF_HPROF("mul_plain");
  check_ct(c, a, "mul_plain");
  require(a.level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
  Pt p = encode_pt(c, slots, (double)c.primes[a.limbs - 1], a.limbs);
  return mac_plain(c, {&a}, {&p});
}

// ---------------------------------------------------------------- key switching
// The switching key for galois element g (0: relinearisation), DESIGN.md §3.4;
// deterministic in (seed, g), so it can be rebuilt instead of kept.
static BufPtr build_key(Context& c, u64 g, int ndig = 1 << 30) {
  const int np = c.np;
  const size_t n = c.n;
  const u64 gal = g & kKeyGalMask;
  const int kd = (int)(g >> 40);  // digit size encoded in the key id (0: alpha)
  // digit size: one digit over all Q primes for the wide relinearisation key
  const int dig = g == kRelinWide ? c.L + 1 : (kd ? kd : c.alpha);
  ndig = std::min(ndig, (c.L + 1 + dig - 1) / dig);
  BufPtr key = buf(c, (size_t)ndig * 2 * np * n);
  BufPtr sp = buf(c, (size_t)np * n);
  if (gal == 0 || g == kRelinWide)
    k_square(c, sp->p, c.sk->p, np);
  else
    k_automorph(c, sp->p, c.sk->p, nullptr, gal, np);
  BufPtr e = buf(c, (size_t)np * n);
  std::vector<int> primes(np);
  for (int m = 0; m < np; ++m) primes[m] = m;
  for (int j = 0; j < ndig; ++j) {
    // independent streams per digit layout (two keys sharing a and e but not their
    // gadgets would reveal the target)
    const u64 tag = (gal << 16) | ((u64)j << 8) | ((u64)kd << 44);
    k_small_rns(c, e->p, stream_key(c.seed, kStreamKeyE | tag), true, nullptr, primes.data(), np);
    ntt_limbs(c, e->p, np, 0, false);
    u64* b = key->p + ((size_t)j * 2 + 0) * np * n;
    u64* a = key->p + ((size_t)j * 2 + 1) * np * n;
    std::vector<RngKey> keys(np);
    std::vector<u64> pm(np, 0);
    const int lo = j * dig, hi = std::min((j + 1) * dig, c.L + 1);
    for (int m = 0; m < np; ++m) {
      keys[m] = stream_key(c.seed, kStreamKeyA | tag | (u64)m);
      if (m >= lo && m < hi) {
        const u64 q = c.primes[m];
        u64 v = 1 % q;
        for (int k = 0; k < c.alpha; ++k) v = mulmod_h(v, c.primes[c.P_index(k)] % q, q);
        pm[m] = v;
      }
    }
    k_sample_uniform(c, a, keys.data(), primes.data(), np);
    k_key_combine(c, b, a, c.sk->p, e->p, sp->p, pm.data(), primes.data(), np);
  }
  return key;
}

const BufPtr& get_key(Context& c, u64 g) {
  SF_HPROF("get_key");
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.keys.find(g);
    if (it != c.keys.end()) return it->second;
  }
  BufPtr key = build_key(c, g);
  std::lock_guard<std::mutex> lk(c.mu);
  return c.keys.emplace(g, key).first->second;
}

// Montgomery copies of the switching keys for the fused key-switch kernels
// (DESIGN.md §3.7b): every limb times R = 2^64 mod q, so the kernels' 128-bit
// inner-product sums T finish with one Montgomery reduction T R^-1 (a 64-bit
// low product and one high product) instead of a 128-bit Barrett reduction.
// With pinv the Q-prime limbs also carry P^-1: the
// rotation-sum inner products then land already divided by P on the Q primes,
// the P*sigma(c0) terms become plain additions and ModDown's final multiply
// disappears; the special-prime limbs (ModDown's conversion input) carry R
// only. Exact modular identities: results are bit-identical. The unscaled key
// is rebuilt (deterministic) rather than kept, unless something cached it.
const BufPtr& get_key_mont(Context& c, u64 g, bool pinv, int ndig) {
  SF_HPROF("get_key_mont");
  auto& cache = pinv ? c.keys_pinv : c.keys_r;
  auto& digs = pinv ? c.keys_pinv_dig : c.keys_r_dig;
  // at least two digits: the attention keys serve levels 1 and 2 (one and two
  // digits at alpha = 2); a one-digit key upgraded mid-stream cost a rebuild
  {
    const int kd = (int)(g >> 40);
    const int dmax = g == kRelinWide ? 1 : (c.L + 1 + (kd ? kd : c.alpha) - 1) / (kd ? kd : c.alpha);
    ndig = g == kRelinWide ? 1 : std::max(std::min(2, dmax), std::min(ndig, dmax));
  }
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = cache.find(g);
    if (it != cache.end()) {
      if (digs[g] >= ndig) return it->second;
      ndig = std::max(ndig, digs[g]);
      c.key_graveyard.push_back(it->second);  // a captured graph may still read it
      cache.erase(it);
    }
  }
  static const bool key_log = std::getenv("SF_KEY_LOG") != nullptr;
  if (key_log) std::fprintf(stderr, "[sf] build key g=%llu pinv=%d ndig=%d\n", (unsigned long long)g, (int)pinv, ndig);
  BufPtr out;
  {
    BufPtr cached;
    {
      std::lock_guard<std::mutex> lk(c.mu);
      auto it = c.keys.find(g);
      if (it != c.keys.end()) cached = it->second;
    }
    if (cached) {
      const size_t words = (size_t)ndig * 2 * c.np * c.n;
      out = buf(c, words);
      SF_CUDA(cudaMemcpyAsync(out->p, cached->p, words * sizeof(u64), cudaMemcpyDeviceToDevice, c.stream));
    } else {
      out = build_key(c, g, ndig);
    }
  }
  std::vector<u64> f(c.np);
  for (int m = 0; m < c.np; ++m) {
    const u64 q = c.primes[m];
    f[m] = c.r64[m];
    if (pinv && m <= c.L) {
      u64 pm = 1 % q;
      for (int kk = 0; kk < c.alpha; ++kk) pm = mulmod_h(pm, c.primes[c.P_index(kk)] % q, q);
      f[m] = mulmod_h(f[m], invmod_h(pm, q), q);
    }
  }
  BufPtr fd = buf(c, f.size());
  SF_CUDA(cudaMemcpyAsync(fd->p, f.data(), f.size() * sizeof(u64), cudaMemcpyHostToDevice, c.stream));
  k_scale_limbs(c, out->p, ndig * 2, fd->p);
  host_sync(c);  // f is pageable; keys are built once, off the timed path
  std::lock_guard<std::mutex> lk(c.mu);
  digs[g] = ndig;
  return cache.emplace(g, out).first->second;
}

Ct level_drop(Context& c, const Ct& a, int target) {
  SF_HPROF("level_drop");
  check_ct(c, a, "level_drop");
  require(target >= 0 && target <= a.level(), kInvalidTarget,
          "level_drop: target level " + std::to_string(target) + " outside [0, level]");
  return view(a, target + 1);
}

Ct bootstrap(Context& c, const Ct& a, int target) {
  SF_HPROF("bootstrap");
  check_ct(c, a, "bootstrap");
  require(target >= 1 && target <= c.L, kInvalidTarget,
          "bootstrap: target level " + std::to_string(target) + " outside [1, L]");
  c.ledger.boot();
  std::vector<double> s(c.slots);
  decrypt(c, a, s.data());
  return encrypt(c, s.data(), target, c.next_seed(), a.layout);
}

}  // namespace sf

namespace sf {

// Batch plaintext encoder for offline plans: slot vectors are
// synthesised and FFT-encoded on all host cores, uploaded in pinned chunks,
// reduced into RNS limbs and NTT'd on the device.
std::vector<Pt> encode_many(Context& c, const std::function<void(int, double*)>& gen, int count, double scale,
                            int limbs) {
  std::vector<Pt> out(count);
  const int chunk = 32;
  const size_t n = c.n;
  i64* pinned = nullptr;
  SF_CUDA(cudaMallocHost(reinterpret_cast<void**>(&pinned), (size_t)chunk * n * sizeof(i64)));
  std::vector<int> primes(limbs);
  for (int l = 0; l < limbs; ++l) primes[l] = l;
  const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
  try {
    for (int s = 0; s < count; s += chunk) {
      const int m = std::min(chunk, count - s);
      std::atomic<int> next{0};
      std::vector<std::thread> th;
      std::exception_ptr err;
      std::mutex emu;
      for (unsigned w = 0; w < std::min<unsigned>(hw, (unsigned)m); ++w)
        th.emplace_back([&]() {
          std::vector<double> slots(c.slots);
          for (int i = next++; i < m; i = next++) {
            try {
              gen(s + i, slots.data());
              auto co = encode_coeffs(c, slots.data(), scale);
              std::memcpy(pinned + (size_t)i * n, co.data(), n * sizeof(i64));
            } catch (...) {
              std::lock_guard<std::mutex> lk(emu);
              err = std::current_exception();
            }
          }
        });
      for (auto& t : th) t.join();
      if (err) std::rethrow_exception(err);
      BufPtr dev = buf(c, (size_t)m * n);
      SF_CUDA(cudaMemcpyAsync(dev->p, pinned, (size_t)m * n * sizeof(i64), cudaMemcpyHostToDevice, c.stream));
      BufPtr all = buf(c, (size_t)m * limbs * n);
      for (int i = 0; i < m; ++i)
        k_small_rns(c, all->p + (size_t)i * limbs * n, RngKey{0, 0}, false, reinterpret_cast<const i64*>(dev->p + (size_t)i * n),
                    primes.data(), limbs);
      std::vector<std::pair<u64*, int>> todo;
      for (int i = 0; i < m; ++i)
        for (int l = 0; l < limbs; ++l) todo.emplace_back(all->p + ((size_t)i * limbs + l) * n, l);
      ntt_list(c, todo, false);
      for (int i = 0; i < m; ++i) {
        // split the chunk buffer into per-plaintext buffers (copy keeps ownership simple)
        Pt p;
        p.buf = buf(c, (size_t)limbs * n);
        p.limbs = limbs;
        p.scale = scale;
        SF_CUDA(cudaMemcpyAsync(p.buf->p, all->p + (size_t)i * limbs * n, (size_t)limbs * n * 8,
                                cudaMemcpyDeviceToDevice, c.stream));
        out[s + i] = p;
      }
      host_sync(c);  // pinned buffer reused next chunk
    }
  } catch (...) {
    cudaFreeHost(pinned);
    throw;
  }
  cudaFreeHost(pinned);
  return out;
}

}  // namespace sf
