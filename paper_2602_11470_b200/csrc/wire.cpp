// Wire and on-disk formats:
//  * the reference's weight files (layouts.cpp:158-184): <name>.bin = rows x cols
//    row-major float64, <name>.json = {"name", "rows", "cols"};
//  * an encoded-plan cache: a VMM plan's NTT-domain diagonals (plus its weight
//    matrix) so a server skips the offline diagonal encoding on restart;
//  * the client <-> server ciphertext format: header + the RNS words.
// All integers little-endian; every file / buffer starts with a magic and a
// version and carries the ring fingerprint it was produced under.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>

#include "protocols.h"

namespace sf {

namespace {

constexpr uint32_t kCtMagic = 0x54434653u;    // "SFCT"
constexpr uint32_t kPlanMagic = 0x50564653u;  // "SFVP"
constexpr uint32_t kVersion = 2;

// FNV-1a over the whole prime chain (q0..qL, p0..p_{alpha-1}) plus a key-material
// id (a one-way mix of the key seed), so contexts that differ in any prime
// (e.g. scale_bits) or in the keys reject each other's ciphertexts. Plans hold
// plaintexts only and are key-independent: they carry key_id = 0.
u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
struct Fingerprint {
  uint32_t logn, np, alpha, L;
  uint64_t chain, key_id;
};
Fingerprint fingerprint(const Context& c, bool with_key) {
  u64 h = 0xCBF29CE484222325ull;
  for (u64 q : c.primes)
    for (int b = 0; b < 8; ++b) h = (h ^ ((q >> (8 * b)) & 0xFF)) * 0x100000001B3ull;
  return Fingerprint{(uint32_t)c.logn, (uint32_t)c.np, (uint32_t)c.alpha, (uint32_t)c.L, h,
                     with_key ? mix64(mix64(c.seed ^ 0x5F4B45595F494400ull) + 0x9E3779B97F4A7C15ull) : 0};
}
bool same(const Fingerprint& a, const Fingerprint& b) {
  return a.logn == b.logn && a.np == b.np && a.alpha == b.alpha && a.L == b.L && a.chain == b.chain &&
         a.key_id == b.key_id;
}

struct CtHeader {
  uint32_t magic, version;
  Fingerprint fp;
  int32_t limbs, zero;
  double scale;
  int32_t ly_valid, ly_kind, ly_d, ly_t, ly_offset, ly_heads, ly_deferred;
};

// {"rows": R, "cols": C} sidecar (the reference writes it with nlohmann::json)
long long json_int(const std::string& s, const std::string& key) {
  const size_t k = s.find("\"" + key + "\"");
  require(k != std::string::npos, kShapeMismatch, "load_weight: sidecar lacks \"" + key + "\"");
  size_t i = s.find(':', k);
  require(i != std::string::npos, kShapeMismatch, "load_weight: malformed sidecar");
  return std::stoll(s.substr(i + 1));
}

}  // namespace

std::vector<double> load_weight(const std::string& dir, const std::string& name, int* rows, int* cols) {
  std::ifstream js(dir + "/" + name + ".json");
  require((bool)js, kInvalidTarget, "load_weight: missing sidecar " + dir + "/" + name + ".json");
  std::stringstream ss;
  ss << js.rdbuf();
  const long long r = json_int(ss.str(), "rows"), cc = json_int(ss.str(), "cols");
  require(r > 0 && cc > 0, kShapeMismatch, "load_weight: bad shape");
  std::vector<double> w((size_t)r * cc);
  std::ifstream bin(dir + "/" + name + ".bin", std::ios::binary);
  require((bool)bin, kInvalidTarget, "load_weight: missing data " + dir + "/" + name + ".bin");
  bin.read(reinterpret_cast<char*>(w.data()), (std::streamsize)(w.size() * sizeof(double)));
  require(bin.gcount() == (std::streamsize)(w.size() * sizeof(double)), kShapeMismatch,
          "load_weight: truncated data for " + name);
  *rows = (int)r;
  *cols = (int)cc;
  return w;
}

size_t ct_wire_size(const Context& c, const Ct& a) {
  return sizeof(CtHeader) + (a.zero ? 0 : (size_t)2 * a.limbs * c.n * sizeof(u64));
}

void ct_serialize(Context& c, const Ct& a, uint8_t* out) {
  CtHeader h{};
  h.magic = kCtMagic;
  h.version = kVersion;
  h.fp = fingerprint(c, true);
  h.limbs = a.limbs;
  h.zero = a.zero ? 1 : 0;
  h.scale = a.scale;
  if (a.layout) {
    h.ly_valid = 1;
    h.ly_kind = (int)a.layout->kind;
    h.ly_d = a.layout->d;
    h.ly_t = a.layout->t;
    h.ly_offset = a.layout->offset;
    h.ly_heads = a.layout->heads;
    h.ly_deferred = a.layout->deferred_mask ? 1 : 0;
  }
  std::memcpy(out, &h, sizeof h);
  if (a.zero) return;
  const size_t w = (size_t)a.limbs * c.n;
  u64* words = reinterpret_cast<u64*>(out + sizeof h);
  SF_CUDA(cudaMemcpyAsync(words, a.c0(), w * 8, cudaMemcpyDeviceToHost, c.stream));
  SF_CUDA(cudaMemcpyAsync(words + w, a.c1(c.n), w * 8, cudaMemcpyDeviceToHost, c.stream));
  SF_CUDA(cudaStreamSynchronize(c.stream));
}

Ct ct_deserialize(Context& c, const uint8_t* in, size_t len) {
  require(len >= sizeof(CtHeader), kShapeMismatch, "ct_deserialize: buffer shorter than the header");
  CtHeader h;
  std::memcpy(&h, in, sizeof h);
  require(h.magic == kCtMagic, kShapeMismatch, "ct_deserialize: not a ciphertext (bad magic)");
  require(h.version == kVersion, kShapeMismatch, "ct_deserialize: unsupported version");
  require(same(h.fp, fingerprint(c, true)), kShapeMismatch,
          "ct_deserialize: produced under different parameters or keys");
  require(h.limbs >= 1 && h.limbs <= c.L + 1, kInvalidTarget, "ct_deserialize: level out of range");
  OptLayout ly;
  if (h.ly_valid) {
    Layout l;
    l.kind = (LayoutKind)h.ly_kind;
    l.d = h.ly_d;
    l.t = h.ly_t;
    l.offset = h.ly_offset;
    l.heads = h.ly_heads;
    l.deferred_mask = h.ly_deferred != 0;
    require(h.ly_kind >= 0 && h.ly_kind <= 2, kShapeMismatch, "ct_deserialize: bad layout kind");
    validate_layout(l, c.slots);  // untrusted header: same checks as Backend::encrypt (layouts.cpp:50-64)
    ly = l;
  }
  if (h.zero) {
    Ct z = zeros(c, h.limbs - 1);
    z.scale = h.scale;
    z.layout = ly;
    return z;
  }
  const size_t w = (size_t)h.limbs * c.n;
  require(len == sizeof h + 2 * w * sizeof(u64), kShapeMismatch, "ct_deserialize: truncated words");
  require(h.scale > 0 && std::isfinite(h.scale), kShapeMismatch, "ct_deserialize: bad scale");
  {  // every residue must be canonical (< its prime): the kernels assume it
    const u64* words = reinterpret_cast<const u64*>(in + sizeof h);
    for (int part = 0; part < 2; ++part)
      for (int i = 0; i < h.limbs; ++i) {
        const u64 q = c.primes[i];
        const u64* p = words + ((size_t)part * h.limbs + i) * c.n;
        u64 bad = 0;
        for (int j = 0; j < c.n; ++j) bad |= (u64)(p[j] >= q);
        require(!bad, kDomain, "ct_deserialize: non-canonical residue (word >= its prime)");
      }
  }
  Ct r = alloc_ct(c, h.limbs, h.scale);
  r.layout = ly;
  SF_CUDA(cudaMemcpyAsync(r.c0(), in + sizeof h, 2 * w * sizeof(u64), cudaMemcpyHostToDevice, c.stream));
  SF_CUDA(cudaStreamSynchronize(c.stream));
  return r;
}

// Plan cache: header, the weight matrix, then for every cached limb count the
// k diagonals' words. Loading reproduces the plan exactly (same words).
void vmm_plan_save(Context& c, VmmPlan& p, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  require((bool)f, kInvalidTarget, "vmm_plan_save: cannot open " + path);
  const Fingerprint fp = fingerprint(c, false);
  const int32_t hdr[9] = {p.rows, p.cols, p.level, p.s.tau_in, p.s.tau_out, p.bsgs ? 1 : 0, p.batch ? 1 : 0,
                          (int32_t)p.s.k, (int32_t)p.pts.size()};
  f.write(reinterpret_cast<const char*>(&kPlanMagic), 4);
  f.write(reinterpret_cast<const char*>(&kVersion), 4);
  f.write(reinterpret_cast<const char*>(&fp), sizeof fp);
  f.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
  std::vector<double> w((size_t)p.rows * p.cols);
  for (int r = 0; r < p.rows; ++r)
    for (int cc = 0; cc < p.cols; ++cc) w[(size_t)r * p.cols + cc] = p.w(r, cc);
  f.write(reinterpret_cast<const char*>(w.data()), (std::streamsize)(w.size() * sizeof(double)));
  std::vector<u64> host((size_t)c.n * (c.L + 1));
  for (auto& [limbs, pts] : p.pts) {
    const int32_t lb = limbs;
    f.write(reinterpret_cast<const char*>(&lb), 4);
    for (const Pt& pt : pts) {
      SF_CUDA(cudaMemcpyAsync(host.data(), pt.buf->p, (size_t)limbs * c.n * 8, cudaMemcpyDeviceToHost, c.stream));
      SF_CUDA(cudaStreamSynchronize(c.stream));
      f.write(reinterpret_cast<const char*>(host.data()), (std::streamsize)((size_t)limbs * c.n * 8));
    }
  }
  require((bool)f, kInvalidTarget, "vmm_plan_save: write failed for " + path);
}

std::unique_ptr<VmmPlan> vmm_plan_load(Context& c, const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  require((bool)f, kInvalidTarget, "vmm_plan_load: cannot open " + path);
  uint32_t magic = 0, version = 0;
  Fingerprint fp;
  int32_t hdr[9];
  f.read(reinterpret_cast<char*>(&magic), 4);
  f.read(reinterpret_cast<char*>(&version), 4);
  f.read(reinterpret_cast<char*>(&fp), sizeof fp);
  f.read(reinterpret_cast<char*>(hdr), sizeof hdr);
  require((bool)f && magic == kPlanMagic, kShapeMismatch, "vmm_plan_load: not a plan file (bad magic)");
  require(version == kVersion, kShapeMismatch, "vmm_plan_load: unsupported version");
  require(same(fp, fingerprint(c, false)), kShapeMismatch, "vmm_plan_load: plan encoded under different parameters");
  const int rows = hdr[0], cols = hdr[1], level = hdr[2];
  std::vector<double> w((size_t)rows * cols);
  f.read(reinterpret_cast<char*>(w.data()), (std::streamsize)(w.size() * sizeof(double)));
  require((bool)f, kShapeMismatch, "vmm_plan_load: truncated weights");
  // build the plan shell from the weights without encoding, then fill the words
  std::unique_ptr<VmmPlan> p = hdr[6] ? make_vmm_batch_plan(c, w.data(), rows, cols, level, hdr[5] != 0, false)
                                      : make_vmm_plan(c, w.data(), rows, cols, level, hdr[3], hdr[4], hdr[5] != 0, false);
  require(p->s.k == hdr[7], kShapeMismatch, "vmm_plan_load: diagonal count differs");
  std::vector<u64> host;
  for (int i = 0; i < hdr[8]; ++i) {
    int32_t limbs = 0;
    f.read(reinterpret_cast<char*>(&limbs), 4);
    require((bool)f && limbs >= 1 && limbs <= c.L + 1, kShapeMismatch, "vmm_plan_load: bad limb count");
    std::vector<Pt> pts(p->s.k);
    host.resize((size_t)limbs * c.n);
    for (auto& pt : pts) {
      f.read(reinterpret_cast<char*>(host.data()), (std::streamsize)(host.size() * 8));
      require((bool)f, kShapeMismatch, "vmm_plan_load: truncated diagonals");
      pt.buf = make_buf(c, host.size());
      pt.limbs = limbs;
      pt.scale = (double)c.primes[limbs - 1];
      SF_CUDA(cudaMemcpyAsync(pt.buf->p, host.data(), host.size() * 8, cudaMemcpyHostToDevice, c.stream));
      SF_CUDA(cudaStreamSynchronize(c.stream));
    }
    p->pts.emplace(limbs, std::move(pts));
  }
  return p;
}

}  // namespace sf
