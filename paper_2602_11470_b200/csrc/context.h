// Device-resident CKKS context, ciphertext values and the evaluator.
// DESIGN.md §3 is the canonical specification these routines implement
// (shared, as a spec only, with the CPU oracle under oracle/).
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.h"

namespace sf {

struct Context;

void cuda_check(cudaError_t e, const char* what);
#define SF_CUDA(x) ::sf::cuda_check((x), #x)

// Stream-ordered device allocation (cudaMallocAsync pool; frees are enqueued on
// the context stream so in-flight kernels that still read a buffer are safe).
// Allocations a captured graph owns (graph memory nodes). A graph instantiated
// with AutoFreeOnLaunch frees and re-allocates them on every replay; those still
// outstanding when the graph is destroyed are freed then (if their Buf already
// died) or when their Buf dies (sf_graph_destroy / ~Buf).
struct GraphMem {
  std::mutex mu;
  bool destroyed = false;
  bool launched = false;
  std::vector<u64*> dead;  // Bufs gone while the graph lives: free at destroy
};
struct Buf {
  u64* p = nullptr;
  size_t words = 0;
  Context* ctx = nullptr;
  u64 gen = 0;  // the context's generation: a Buf outliving its context frees itself directly
  std::shared_ptr<GraphMem> gm;  // set: allocated while capturing that graph (a graph memory node)
  Buf(Context* c, size_t w);
  ~Buf();
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};
using BufPtr = std::shared_ptr<Buf>;

// Ciphertext value: c0 at p, c1 at p + stride*n, `limbs` active limbs each
// (level = limbs - 1); level_drop is an O(1) view.
struct Ct {
  BufPtr buf;
  int limbs = 0;
  int stride = 0;
  double scale = 0.0;
  bool zero = false;  // trivial (0, 0) ciphertext: Backend::zeros (engine.cpp:123)
  OptLayout layout;
  // value-cache piece only (make_v_pieces): Rot(this, aligned_r), computed from the
  // rotated input, for v_append's giant-aligned variants
  std::shared_ptr<const Ct> aligned;
  int aligned_r = 0;
  int level() const { return limbs - 1; }
  u64* c0() const { return buf ? buf->p : nullptr; }
  u64* c1(int n) const { return buf ? buf->p + (size_t)stride * n : nullptr; }
};

// NTT-domain plaintext (limbs x n words), encoded at `scale`.
struct Pt {
  BufPtr buf;
  int limbs = 0;
  double scale = 0.0;
};

// Fast basis conversion tables for src primes -> dst primes.
struct ConvPlan {
  int nsrc = 0, ndst = 0;
  std::vector<int> src, dst;  // prime indices
  BufPtr tab;                 // [nsrc] qhat_inv, [nsrc] qhat_inv_shoup, [nsrc][ndst] qhat mod dst
};

struct OpCounts {
  long long rotations = 0, hoisted_rotations = 0, ct_pt_mults = 0, ct_ct_mults = 0, additions = 0,
            bootstraps = 0;
};

// CostLedger (engine.hpp:54-96): totals + first-use-ordered phases.
struct Ledger {
  std::mutex mu;
  OpCounts total;
  std::vector<std::string> order;
  std::map<std::string, OpCounts> by_phase;
  std::vector<std::string> stack{"(unphased)"};
  template <class F>
  void bump(F f) {
    std::lock_guard<std::mutex> lk(mu);
    f(total);
    auto it = by_phase.find(stack.back());
    if (it == by_phase.end()) {
      order.push_back(stack.back());
      it = by_phase.emplace(stack.back(), OpCounts{}).first;
    }
    f(it->second);
  }
  void rot(bool hoisted, long long k = 1) {
    bump([&](OpCounts& c) {
      c.rotations += k;
      if (hoisted) c.hoisted_rotations += k;
    });
  }
  void ctpt(long long k = 1) { bump([&](OpCounts& c) { c.ct_pt_mults += k; }); }
  void ctct(long long k = 1) { bump([&](OpCounts& c) { c.ct_ct_mults += k; }); }
  void add(long long k = 1) {
    if (k) bump([&](OpCounts& c) { c.additions += k; });
  }
  void boot() { bump([&](OpCounts& c) { c.bootstraps += 1; }); }
  void reset() {
    std::lock_guard<std::mutex> lk(mu);
    total = {};
    order.clear();
    by_phase.clear();
    stack = {"(unphased)"};
  }
};

// Device-side prime / twiddle tables (one array per quantity, indexed by prime).
struct Tabs {
  const u64 *q, *mh, *ml;          // prime, Barrett mu = floor(2^128 / q)
  const u64 *qn, *r64;             // Montgomery: -q^-1 mod 2^64, R = 2^64 mod q
  const u64 *psi, *psi_s;          // [np][n] psi^{br(k)} (+ Shoup)
  const u64 *ipsi, *ipsi_s;        // [np][n] psi^{-br(k)} (+ Shoup)
  const u64 *ninv, *ninv_s;        // [np]
  const u64 *ninvw, *ninvw_s;      // [np] n^-1 * ipsi[1]: the last inverse column stage's twiddle with n^-1 folded in
  int n, logn;
};

// A batch of limbs for one kernel launch: entry b -> (limb pointer, prime
// index). Travels as a kernel parameter (> 4 KB kernel parameters: CUDA 12.1+
// on sm_70+), so one launch can cover every limb of a whole batch of
// ciphertexts without a staging copy.
constexpr int kMaxBatch = 1024;
struct LimbBatch {
  int count = 0;
  u64* ptr[kMaxBatch];
  u64* optr[kMaxBatch];  // out-of-place destination (nullptr: in place); row passes only
  uint8_t prime[kMaxBatch];
  void add(u64* p, int prime_idx, u64* out = nullptr) {
    ptr[count] = p;
    optr[count] = out;
    prime[count] = (uint8_t)prime_idx;
    ++count;
  }
};

// Live per-family kernel timing (sf_profile_begin / end).
enum Family : int { kFamNtt = 0, kFamKs = 1, kFamMac = 2, kFamConv = 3, kFamElem = 4, kFamSample = 5, kFamCount = 6 };
struct ProfRec {
  int family;
  cudaEvent_t a, b;
  double bytes;
  double bfly;  // radix-2 NTT butterflies the launch executes (0 for non-NTT kernels)
};

// Live-context registry: handles (ciphertexts, plans, caches, graphs) may be
// released after their context (e.g. a garbage-collected cycle that finalises
// the context first); their buffers then bypass the dead context.
bool context_alive(const Context* c, u64 gen);

struct Context {
  u64 gen = 0;  // unique per context (context_alive)
  // profiling
  int prof_mask = 0;
  std::vector<ProfRec> prof_recs;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_pool_next = 0;
  double prof_bfly[kFamCount] = {};  // butterflies per family of the last profile window

  // parameters
  int logn = 0, n = 0, slots = 0, L = 0, alpha = 0, beta = 0, np = 0;
  double delta = 0.0;
  u64 seed = 0;
  int device = 0;
  // CUDA-graph capture of whole decode steps (sf_graph_*): allocations made while
  // capturing become graph memory nodes; frees of older buffers are deferred
  // to graph destruction (a replay still reads them).
  bool capturing = false;
  std::shared_ptr<GraphMem> capture_gm;  // the graph being captured
  // sharded ops (comm.cpp): NCCL communicator on this context's stream
  void* comm = nullptr;
  int rank = 0, world = 1;
  // the Score*V giant groups this process owns ((G mod 8) mod sv_world == sv_rank,
  // DESIGN.md §3.9): make_v_pieces builds aligned companions for those only (set by
  // sf_comm_init / sf_p2p_init / sf_set_value_shard)
  int sv_rank = 0, sv_world = 1;
  std::map<std::string, std::vector<u64>> comm_hdr, comm_meta;
  void* p2p = nullptr;  // peer-memory exchange state (p2p.cu)
  // exact-size free lists of device buffers (eager path only): every kernel runs
  // on `stream`, so a buffer released after its last use was enqueued can back
  // the next same-size allocation (stream order); saves the per-op
  // cudaMallocAsync / cudaFreeAsync host cost
  std::mutex alloc_mu;
  std::unordered_map<size_t, std::vector<u64*>> free_bufs;
  // 24 GiB (SF_FREE_CACHE_GIB): the decode step's whole temporary working set, so a
  // steady-state eager step never reaches cudaMallocAsync (an 8 GiB cap overflowed
  // and stalled single allocations for 100-400 ms)
  size_t cached_words = 0, cache_cap_words = (size_t)3 << 30;
  std::vector<std::pair<u64*, size_t>> capture_deferred;
  long long graph_launch_base = 0;
  bool ks_row = true;  // fused key-switch row stage
  int variant = 0;     // SF_VARIANT bit mask: kernel variants under A/B evaluation
  int rot_chunk = 0;   // SF_ROT_CHUNK: sources per ModUp batch in rotate_batch (0: kJobs), for A/B timing
  int fused_cpw = 1;   // columns per warp in batched fused column stages (SF_FUSED_CPW=1|2, for A/B timing) (SF_KS_ROW=0: separate passes, for A/B timing)
  std::vector<u64> primes;  // q0..qL, p0..p_{alpha-1}
  std::vector<u64> ipsi1_h;  // per prime: ipsi table index 1 (the last inverse column stage's twiddle)
  cudaStream_t stream = nullptr;
  cudaMemPool_t pool = nullptr;

  // device tables
  BufPtr tab_store;  // owns all table memory below
  Tabs tabs{};
  std::vector<u64> mu_hi, mu_lo, qneg_inv, r64;

  // host copies needed by the encoder
  std::vector<double> fft_re, fft_im;  // zeta^{br(k)}
  std::vector<uint32_t> slot_index;    // transform index of slot j (n/2 entries)

  BufPtr sk;  // [np][n] NTT domain
  std::map<u64, BufPtr> keys;  // galois element (0 = relin) -> [beta][2][np][n]
  std::map<std::string, ConvPlan> conv_plans;
  // Montgomery copies of the switching keys for the fused kernels (get_key_mont):
  // every limb times R = 2^64, the Q limbs of the rotation-sum copy also times P^-1
  std::map<u64, BufPtr> keys_pinv, keys_r;
  std::map<u64, int> keys_pinv_dig, keys_r_dig;  // digits built per key (level-truncated keys)
  std::vector<BufPtr> key_graveyard;              // superseded truncated keys (captured graphs may read them)
  std::map<std::string, Pt> pt_cache;  // semantic-key plaintext cache (masks)
  std::map<int, BufPtr> level_consts;  // per-limb-count rescale / moddown constants
  std::map<int, std::vector<u64>> level_consts_h;
  std::map<int, BufPtr> merged_consts;               // (q_top P)^-1 per limb count (merged relin + rescale)
  std::map<int, std::vector<u64>> merged_consts_h;  // host copies (row-pass epilogue parameters)
  // Rot(V, r) of value-cache ciphertexts for the BSGS Score*V:
  // kept while the source buffer lives (a completed cache group's variants are
  // rotated once, not once per decode step); never filled while capturing
  struct RotMemo {
    std::weak_ptr<Buf> src;
    int limbs, r;
    Ct out;
  };
  std::unordered_multimap<const Buf*, RotMemo> rot_memo;

  // pinned staging ring for host -> device uploads of fresh plaintexts and
  // encryptions (upload_async): the copy is stream-ordered and the host returns
  // at once; a slot is reused only after its previous copy has completed
  struct StageSlot {
    void* p = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;
    bool pending = false;
  };
  std::vector<StageSlot> stage;
  size_t stage_next = 0;
  int live_graphs = 0;  // instantiated graphs of this context (they may read cached plaintexts)

  Ledger ledger;
  u64 enc_counter = 0;
  std::atomic<long long> launches{0};
  std::vector<cudaEvent_t> events;
  // sf_ct_stage: host->device input copies on a side stream (overlapping the
  // stages before the input's first use); per slot: fork and done events
  cudaStream_t copy_stream = nullptr;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stage_ev;

  std::mutex mu;  // guards key / plan caches

  ~Context();

  int P_index(int k) const { return L + 1 + k; }
  u64 next_seed();  // DESIGN.md §3.4 auto seed
};

// RAII bracket for one profiled launch (no-op unless the family is enabled).
struct ProfScope {
  Context& c;
  int fam;
  double bytes;
  bool on;
  cudaEvent_t b{};
  ProfScope(Context& ctx, int family, double algorithmic_bytes, double butterflies = 0.0);
  ~ProfScope();
};

std::string host_prof_dump(bool reset);

// --- construction ------------------------------------------------------------
std::unique_ptr<Context> make_context(int slots, int L, int log_n, int alpha, int q0_bits, int scale_bits,
                                      int special_bits, u64 seed, int device);
std::vector<u64> generate_primes(int logn, int L, int q0_bits, int scale_bits, int alpha, int special_bits);
u64 min_primitive_root(u64 q, int n);

// --- encoder (host) ------------------------------------------
std::vector<i64> encode_coeffs(const Context& c, const double* slots, double scale);
void decode_coeffs(const Context& c, const std::vector<double>& coeff, double scale, double* slots);

// --- device primitives (kernels.cu) -----------------------------------------
void launch_ntt(Context& c, const LimbBatch& b, bool inverse);
bool ntt_two_pass(Context& c, const LimbBatch& b, bool inverse);
void ntt_limbs(Context& c, u64* base, int count, int first_prime, bool inverse);  // contiguous limbs
void ntt_list(Context& c, const std::vector<std::pair<u64*, int>>& limbs, bool inverse);

// --- evaluator (evaluator.cu) -------------------------------------------------
BufPtr make_buf(Context& c, size_t words);
Ct alloc_ct(Context& c, int limbs, double scale);
void p2p_destroy(Context& c);  // p2p.cu
Pt encode_pt(Context& c, const double* slots, double scale, int limbs);
std::vector<Pt> encode_many(Context& c, const std::function<void(int, double*)>& gen, int count, double scale,
                            int limbs);
Pt cached_pt(Context& c, const std::string& key, const double* slots, double scale, int limbs);
bool lookup_pt(Context& c, const std::string& key, int limbs, Pt* out);  // cached_pt's cache, no encode
Ct encrypt(Context& c, const double* slots, int level, u64 seed, OptLayout layout);
Ct zeros(Context& c, int level);
void decrypt(Context& c, const Ct& a, double* out);
Ct add(Context& c, const Ct& a, const Ct& b, bool sub = false, bool count = true);
Ct add_plain(Context& c, const Ct& a, const double* slots);
Ct rescale(Context& c, const Ct& a);
Ct mac_plain(Context& c, const std::vector<const Ct*>& cts, const std::vector<const Pt*>& pts, bool count = true,
              bool rescale_out = true);
Ct mul_plain(Context& c, const Ct& a, const double* slots);
Ct mul(Context& c, const Ct& a, const Ct& b, bool count = true);
Ct rotate(Context& c, const Ct& a, int r, bool hoisted, bool count = true);
std::vector<Ct> rotate_hoisted(Context& c, const Ct& a, const std::vector<int>& rs, bool count = true);
Ct level_drop(Context& c, const Ct& a, int target);
Ct bootstrap(Context& c, const Ct& a, int target);
u64 galois_elt(const Context& c, int r);
const BufPtr& get_key(Context& c, u64 g);
// Montgomery key copy: limbs times R = 2^64 mod q, and with
// pinv the Q limbs also times P^-1 (rotation sums / hoisted rotations, §3.7a)
// ndig: the key is built (and kept) for its first ndig digits only -- a key used
// at level l needs ceil((l + 1) / alpha) digits; a later use
// with more digits rebuilds it (the old buffer stays alive for captured graphs)
const BufPtr& get_key_mont(Context& c, u64 g, bool pinv, int ndig = 1 << 30);
// Key id of the single-digit relinearisation key (target s^2, ONE digit over all
// Q primes; galois element 1 is never a rotation key). A relinearisation at limbs
// l uses it when log2(Q_l / P) <= 30 (relin_digit): the switch runs at the product
// scale (>= 2^80), where Q_l / P * e * n is far below the rescale rounding
// -- half the ModUp NTTs and inner products at levels 1-2.
constexpr u64 kRelinWide = 1;
int relin_digit(const Context& c, int limbs);  // digit size of a relinearisation at `limbs` limbs
// Switching-key ids: the galois element in the low 40 bits, a digit size other
// than alpha in bits 40-47 (keys for key switches at a product scale >= 2^80,
// e.g. the HE-VMM giant rotations before their rescale: DESIGN.md §3.6b)
constexpr u64 kKeyGalMask = (1ull << 40) - 1;
inline u64 key_id(u64 gal, int dig, int alpha) { return dig == alpha ? gal : gal | ((u64)dig << 40); }
// largest digit size whose digits all stay within P 2^30 (at most 8 limbs): the
// key switches of ciphertexts at scale >= 2^80 use it
int scaled_digit(const Context& c, int limbs);
void check_ct(const Context& c, const Ct& a, const char* what);
void check_scales(const Ct& a, const Ct& b, const char* what);

// Host synchronisation of the lazy builders (constant tables, keys, cached
// plaintexts uploaded from pageable memory on first use). Not allowed inside a
// graph capture: the caller must run the step once eagerly first.
// Stream-ordered upload of `bytes` host bytes to device memory through the
// pinned staging ring (no stream synchronisation; `src` may be released on
// return). Not allowed inside a graph capture (the staging slot is reused).
void upload_async(Context& c, void* dst, const void* src, size_t bytes);

inline void host_sync(Context& c) {
  require(!c.capturing, kInvalidTarget,
          "graph capture: a lazily built table / key / plaintext is not warm yet; run the step once eagerly "
          "before capturing it");
  SF_CUDA(cudaStreamSynchronize(c.stream));
}

}  // namespace sf
