// extern "C" boundary (include/sf_b200.h): opaque refcounted handles over the
// C++ evaluator and protocols; every exception is mapped 1:1 onto an sf_status
// code matching the reference's exception types (types.hpp:16-46).
#include "../../include/sf_b200.h"

#include <cstring>
#include <string>

#include "context.h"
#include "protocols.h"
#include "batch.cuh"

struct sf_context {
  std::unique_ptr<sf::Context> c;
};
struct sf_ct {
  std::atomic<int> rc{1};
  sf::Ct v;
};
struct sf_vmm_plan {
  std::unique_ptr<sf::VmmPlan> p;
};
struct sf_graph {
  sf_context* ctx = nullptr;
  sf::Context* cp = nullptr;  // the context and its generation (sf_graph_destroy may run after it died)
  sf::u64 gen = 0;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t x = nullptr;
  long long launches = 0;  // library kernels per replay
  std::vector<std::pair<sf::u64*, size_t>> deferred;
  std::shared_ptr<sf::GraphMem> gm;
};
struct sf_kvcache {
  std::atomic<int> rc{1};
  sf::KV kv;
};

namespace {

thread_local std::string g_err;

template <class F>
sf_status guard(F&& f) {
  try {
    f();
    return SF_OK;
  } catch (const sf::Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SF_ERR_INTERNAL;
  } catch (...) {
    g_err = "unknown error";
    return SF_ERR_INTERNAL;
  }
}

sf::OptLayout to_layout(const sf_layout* l) {
  if (!l || !l->valid) return std::nullopt;
  sf::Layout ly;
  ly.kind = static_cast<sf::LayoutKind>(l->kind);
  ly.d = l->d;
  ly.t = l->t;
  ly.offset = l->offset;
  ly.heads = l->heads;
  ly.deferred_mask = l->deferred_mask != 0;
  return ly;
}

void from_layout(const sf::OptLayout& ly, sf_layout* out) {
  std::memset(out, 0, sizeof(*out));
  if (!ly) return;
  out->valid = 1;
  out->kind = static_cast<int>(ly->kind);
  out->d = ly->d;
  out->t = ly->t;
  out->offset = ly->offset;
  out->heads = ly->heads;
  out->deferred_mask = ly->deferred_mask ? 1 : 0;
}

sf_ct* wrap(sf::Ct v) {
  auto* h = new sf_ct;
  h->v = std::move(v);
  return h;
}
sf_kvcache* wrap_kv(sf::KV kv) {
  auto* h = new sf_kvcache;
  h->kv = std::move(kv);
  return h;
}

void need(const void* p, const char* what) { sf::require(p != nullptr, sf::kInvalidTarget, std::string(what) + ": null"); }

void counts_out(const sf::OpCounts& c, sf_op_counts* o) {
  o->rotations = c.rotations;
  o->hoisted_rotations = c.hoisted_rotations;
  o->ct_pt_mults = c.ct_pt_mults;
  o->ct_ct_mults = c.ct_ct_mults;
  o->additions = c.additions;
  o->bootstraps = c.bootstraps;
}

}  // namespace

extern "C" {

const char* sf_last_error(void) { return g_err.c_str(); }

sf_status sf_context_create(const sf_params* p, sf_context** out) {
  return guard([&] {
    need(p, "params");
    auto* h = new sf_context;
    try {
      h->c = sf::make_context(p->slots, p->L, p->log_n, p->alpha, p->q0_bits, p->scale_bits, p->special_bits,
                              p->seed, p->device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void sf_context_destroy(sf_context* ctx) { delete ctx; }

sf_status sf_context_info(const sf_context* ctx, int* n, int* slots, int* L, int* alpha, int* num_primes,
                          uint64_t* primes) {
  return guard([&] {
    need(ctx, "ctx");
    const auto& c = *ctx->c;
    if (n) *n = c.n;
    if (slots) *slots = c.slots;
    if (L) *L = c.L;
    if (alpha) *alpha = c.alpha;
    if (num_primes) *num_primes = c.np;
    if (primes) std::copy(c.primes.begin(), c.primes.end(), primes);
  });
}

sf_status sf_synchronize(sf_context* ctx) {
  return guard([&] { SF_CUDA(cudaStreamSynchronize(ctx->c->stream)); });
}

sf_status sf_gen_rotation_keys(sf_context* ctx, const int* rotations, int count) {
  return guard([&] {
    for (int i = 0; i < count; ++i)
      if (sf::pos_mod(rotations[i], ctx->c->slots) != 0) sf::get_key(*ctx->c, sf::galois_elt(*ctx->c, rotations[i]));
  });
}

sf_status sf_secret_key_export(sf_context* ctx, uint64_t* out) {
  return guard([&] {
    auto& c = *ctx->c;
    SF_CUDA(cudaMemcpyAsync(out, c.sk->p, (size_t)c.np * c.n * 8, cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
  });
}

sf_status sf_switching_key_export(sf_context* ctx, uint64_t g, uint64_t* out) {
  return guard([&] {
    auto& c = *ctx->c;
    const auto& k = sf::get_key(c, g);
    SF_CUDA(cudaMemcpyAsync(out, k->p, k->words * 8, cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
  });
}

uint64_t sf_galois_elt(const sf_context* ctx, int r) { return sf::galois_elt(*ctx->c, r); }

// --- handles
sf_ct* sf_ct_retain(sf_ct* ct) {
  if (ct) ct->rc.fetch_add(1);
  return ct;
}
void sf_ct_release(sf_ct* ct) {
  if (ct && ct->rc.fetch_sub(1) == 1) delete ct;
}

sf_status sf_ct_info(const sf_ct* ct, int* level, double* scale, int* is_zero, sf_layout* layout) {
  return guard([&] {
    need(ct, "ct");
    if (level) *level = ct->v.level();
    if (scale) *scale = ct->v.scale;
    if (is_zero) *is_zero = ct->v.zero ? 1 : 0;
    if (layout) from_layout(ct->v.layout, layout);
  });
}

sf_status sf_ct_with_layout(sf_context*, const sf_ct* ct, const sf_layout* layout, sf_ct** out) {
  return guard([&] {
    need(ct, "ct");
    sf::Ct v = ct->v;
    v.layout = to_layout(layout);
    *out = wrap(std::move(v));
  });
}

sf_status sf_ct_export(sf_context* ctx, const sf_ct* ct, uint64_t* out) {
  return guard([&] {
    auto& c = *ctx->c;
    const sf::Ct& v = ct->v;
    const size_t w = (size_t)v.limbs * c.n;
    SF_CUDA(cudaMemcpyAsync(out, v.c0(), w * 8, cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaMemcpyAsync(out + w, v.c1(c.n), w * 8, cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
  });
}

sf_status sf_ct_import(sf_context* ctx, const uint64_t* words, int level, double scale, int is_zero,
                       const sf_layout* layout, sf_ct** out) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(level >= 0 && level <= c.L, sf::kInvalidTarget, "import: level out of range");
    sf::Ct v = sf::alloc_ct(c, level + 1, scale);
    v.zero = is_zero != 0;
    v.layout = to_layout(layout);
    SF_CUDA(cudaMemcpyAsync(v.c0(), words, v.buf->words * 8, cudaMemcpyHostToDevice, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
    *out = wrap(std::move(v));
  });
}

// --- client side
sf_status sf_encrypt(sf_context* ctx, const double* slots, int level, const sf_layout* layout, uint64_t seed,
                     int use_seed, sf_ct** out) {
  return guard([&] {
    auto& c = *ctx->c;
    need(slots, "slots");
    const uint64_t s = use_seed ? seed : c.next_seed();
    *out = wrap(sf::encrypt(c, slots, level, s, to_layout(layout)));
  });
}

sf_status sf_zeros(sf_context* ctx, int level, sf_ct** out) {
  return guard([&] { *out = wrap(sf::zeros(*ctx->c, level)); });
}

sf_status sf_decrypt(sf_context* ctx, const sf_ct* ct, double* slots_out) {
  return guard([&] {
    need(ct, "ct");
    sf::decrypt(*ctx->c, ct->v, slots_out);
  });
}

sf_status sf_encode(sf_context* ctx, const double* slots, double scale, int limbs, uint64_t* out) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::Pt p = sf::encode_pt(c, slots, scale, limbs);
    SF_CUDA(cudaMemcpyAsync(out, p.buf->p, (size_t)limbs * c.n * 8, cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
  });
}

// --- evaluator
sf_status sf_add(sf_context* ctx, const sf_ct* a, const sf_ct* b, sf_ct** out) {
  return guard([&] { *out = wrap(sf::add(*ctx->c, a->v, b->v, false)); });
}
sf_status sf_sub(sf_context* ctx, const sf_ct* a, const sf_ct* b, sf_ct** out) {
  return guard([&] { *out = wrap(sf::add(*ctx->c, a->v, b->v, true)); });
}
sf_status sf_add_plain(sf_context* ctx, const sf_ct* a, const double* slots, sf_ct** out) {
  return guard([&] { *out = wrap(sf::add_plain(*ctx->c, a->v, slots)); });
}
sf_status sf_mul(sf_context* ctx, const sf_ct* a, const sf_ct* b, sf_ct** out) {
  return guard([&] { *out = wrap(sf::mul(*ctx->c, a->v, b->v)); });
}
sf_status sf_mul_plain(sf_context* ctx, const sf_ct* a, const double* slots, sf_ct** out) {
  return guard([&] { *out = wrap(sf::mul_plain(*ctx->c, a->v, slots)); });
}
sf_status sf_mac_plain(sf_context* ctx, const sf_ct* const* cts, const double* slots, int k, sf_ct** out) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(k >= 1, sf::kShapeMismatch, "mac_plain: need at least one term");
    int limbs = 1 << 30;
    for (int i = 0; i < k; ++i) {
      sf::check_ct(c, cts[i]->v, "mul_plain");
      sf::require(cts[i]->v.level() > 0, sf::kLevelUnderflow, "mul_plain: no multiplicative level left");
      limbs = std::min(limbs, cts[i]->v.limbs);
    }
    std::vector<sf::Pt> pts;
    pts.reserve(k);
    for (int i = 0; i < k; ++i)
      pts.push_back(sf::encode_pt(c, slots + (size_t)i * c.slots, (double)c.primes[limbs - 1], limbs));
    std::vector<const sf::Ct*> cv;
    std::vector<const sf::Pt*> pv;
    for (int i = 0; i < k; ++i) cv.push_back(&cts[i]->v), pv.push_back(&pts[i]);
    *out = wrap(sf::mac_plain(c, cv, pv));
  });
}
sf_status sf_rotate(sf_context* ctx, const sf_ct* a, int r, int hoisted, sf_ct** out) {
  return guard([&] { *out = wrap(sf::rotate(*ctx->c, a->v, r, hoisted != 0)); });
}
sf_status sf_rotate_hoisted(sf_context* ctx, const sf_ct* a, const int* r, int k, sf_ct** outs) {
  return guard([&] {
    auto v = sf::rotate_hoisted(*ctx->c, a->v, std::vector<int>(r, r + k));
    for (int i = 0; i < k; ++i) outs[i] = wrap(std::move(v[i]));
  });
}
sf_status sf_rotate_many(sf_context* ctx, const sf_ct* const* a, int k, int r, sf_ct** outs) {
  return guard([&] {
    std::vector<const sf::Ct*> src(k);
    std::vector<sf::RotJob> jobs(k);
    for (int i = 0; i < k; ++i) src[i] = &a[i]->v, jobs[i] = {i, r};
    auto v = sf::rotate_batch(*ctx->c, src, jobs, false);
    for (int i = 0; i < k; ++i) outs[i] = wrap(std::move(v[i]));
  });
}
sf_status sf_bench_ntt(sf_context* ctx, int limbs, int count, int reps, double* ms_per_limb_ntt) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(limbs >= 1 && limbs <= c.L + 1 && count >= 1 && reps >= 1, sf::kInvalidTarget, "bench_ntt: bad sizes");
    sf::BufPtr b = sf::make_buf(c, (size_t)count * limbs * c.n);
    SF_CUDA(cudaMemsetAsync(b->p, 0x11, (size_t)count * limbs * c.n * 8, c.stream));
    std::vector<std::pair<sf::u64*, int>> lst;
    for (int j = 0; j < count; ++j)
      for (int l = 0; l < limbs; ++l) lst.push_back({b->p + ((size_t)j * limbs + l) * c.n, l});
    sf::ntt_list(c, lst, false);  // warm-up (both directions: lazy module loading)
    sf::ntt_list(c, lst, true);
    cudaEvent_t e0, e1;
    SF_CUDA(cudaEventCreate(&e0));
    SF_CUDA(cudaEventCreate(&e1));
    SF_CUDA(cudaEventRecord(e0, c.stream));
    for (int i = 0; i < reps; ++i) sf::ntt_list(c, lst, (i & 1) != 0);
    SF_CUDA(cudaEventRecord(e1, c.stream));
    SF_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SF_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms_per_limb_ntt = ms / ((double)reps * count * limbs);
  });
}
sf_status sf_level_drop(sf_context* ctx, const sf_ct* a, int target, sf_ct** out) {
  return guard([&] { *out = wrap(sf::level_drop(*ctx->c, a->v, target)); });
}
sf_status sf_bootstrap(sf_context* ctx, const sf_ct* a, int target, sf_ct** out) {
  return guard([&] { *out = wrap(sf::bootstrap(*ctx->c, a->v, target)); });
}

// --- ledger
sf_status sf_ledger_totals(const sf_context* ctx, sf_op_counts* out) {
  return guard([&] {
    auto& l = ctx->c->ledger;
    std::lock_guard<std::mutex> lk(l.mu);
    counts_out(l.total, out);
  });
}
sf_status sf_ledger_phase_totals(const sf_context* ctx, const char* phase, sf_op_counts* out) {
  return guard([&] {
    auto& l = ctx->c->ledger;
    std::lock_guard<std::mutex> lk(l.mu);
    auto it = l.by_phase.find(phase);
    counts_out(it == l.by_phase.end() ? sf::OpCounts{} : it->second, out);
  });
}
sf_status sf_ledger_reset(sf_context* ctx) {
  return guard([&] { ctx->c->ledger.reset(); });
}
sf_status sf_phase_push(sf_context* ctx, const char* phase) {
  return guard([&] {
    auto& l = ctx->c->ledger;
    std::lock_guard<std::mutex> lk(l.mu);
    l.stack.push_back(phase);
  });
}
sf_status sf_phase_pop(sf_context* ctx) {
  return guard([&] {
    auto& l = ctx->c->ledger;
    std::lock_guard<std::mutex> lk(l.mu);
    if (l.stack.size() > 1) l.stack.pop_back();
  });
}

// --- VMM
sf_status sf_vmm_plan_create(sf_context* ctx, const double* W, int rows, int cols, int level, int in_offset,
                             int out_offset, int bsgs, sf_vmm_plan** out) {
  return guard([&] {
    auto* h = new sf_vmm_plan;
    try {
      h->p = sf::make_vmm_plan(*ctx->c, W, rows, cols, level, in_offset, out_offset, bsgs != 0);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
void sf_vmm_plan_destroy(sf_vmm_plan* plan) { delete plan; }

sf_status sf_vmm_predict(const sf_context* ctx, int rows, int cols, int bsgs, int mask_output, long long* rotations,
                         long long* ct_pt_mults, int* depth) {
  return guard([&] {
    sf::predict_interleaved_cost(ctx->c->slots, rows, cols, bsgs != 0, mask_output != 0, rotations, ct_pt_mults,
                                 depth);
  });
}

sf_status sf_vmm_interleaved(sf_context* ctx, const sf_ct* x, const sf_vmm_plan* plan, int mask_output,
                             sf_ct** out) {
  return guard([&] { *out = wrap(sf::vmm_interleaved(*ctx->c, x->v, *plan->p, mask_output != 0)); });
}

sf_status sf_vmm_interleaved_multi(sf_context* ctx, const sf_ct* x, sf_vmm_plan* const* plans, int k,
                                   int mask_output, sf_ct** outs) {
  return guard([&] {
    std::vector<sf::VmmPlan*> ps(k);
    for (int i = 0; i < k; ++i) ps[i] = plans[i]->p.get();
    auto v = sf::vmm_interleaved_multi(*ctx->c, x->v, ps, mask_output != 0);
    for (int i = 0; i < k; ++i) outs[i] = wrap(std::move(v[i]));
  });
}

sf_status sf_vmm_interleaved_many(sf_context* ctx, const sf_ct* const* xs, int k, const sf_vmm_plan* plan,
                                  int mask_output, sf_ct** outs) {
  return guard([&] {
    std::vector<const sf::Ct*> v;
    for (int i = 0; i < k; ++i) v.push_back(&xs[i]->v);
    auto r = sf::vmm_interleaved_many(*ctx->c, v, *plan->p, mask_output != 0);
    for (int i = 0; i < k; ++i) outs[i] = wrap(std::move(r[i]));
  });
}
sf_status sf_vmm_multi_partial(sf_context* ctx, const sf_ct* x, sf_vmm_plan* const* plans, int k, int rank,
                               int world, sf_ct** outs) {
  return guard([&] {
    std::vector<sf::VmmPlan*> ps(k);
    for (int i = 0; i < k; ++i) ps[i] = plans[i]->p.get();
    auto v = sf::vmm_multi_partial(*ctx->c, x->v, ps, rank, world);
    for (int i = 0; i < k; ++i) outs[i] = wrap(std::move(v[i]));
  });
}
sf_status sf_vmm_multi_finish(sf_context* ctx, const sf_ct* const* accs, sf_vmm_plan* const* plans, int k,
                              int mask_output, sf_ct** outs) {
  return guard([&] {
    std::vector<sf::VmmPlan*> ps(k);
    std::vector<sf::Ct> a;
    for (int i = 0; i < k; ++i) ps[i] = plans[i]->p.get(), a.push_back(accs[i]->v);
    auto v = sf::vmm_multi_finish(*ctx->c, a, ps, mask_output != 0);
    for (int i = 0; i < k; ++i) outs[i] = wrap(std::move(v[i]));
  });
}
sf_status sf_vmm_multi_sharded(sf_context* ctx, const sf_ct* x, sf_vmm_plan* const* plans, int k, int mask_output,
                               sf_ct** outs) {
  return guard([&] {
    std::vector<sf::VmmPlan*> ps(k);
    for (int i = 0; i < k; ++i) ps[i] = plans[i]->p.get();
    auto v = sf::vmm_multi_sharded(*ctx->c, x->v, ps, mask_output != 0);
    for (int i = 0; i < k; ++i) outs[i] = wrap(std::move(v[i]));
  });
}

// --- wire / on-disk formats (wire.cpp)
sf_status sf_vmm_plan_create_from_file(sf_context* ctx, const char* dir, const char* name, int level, int in_offset,
                                       int out_offset, int bsgs, sf_vmm_plan** out) {
  return guard([&] {
    int rows = 0, cols = 0;
    const std::vector<double> w = sf::load_weight(dir, name, &rows, &cols);
    auto* h = new sf_vmm_plan;
    try {
      h->p = sf::make_vmm_plan(*ctx->c, w.data(), rows, cols, level, in_offset, out_offset, bsgs != 0);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
sf_status sf_vmm_plan_save(sf_context* ctx, sf_vmm_plan* plan, const char* path) {
  return guard([&] { sf::vmm_plan_save(*ctx->c, *plan->p, path); });
}
sf_status sf_vmm_plan_load(sf_context* ctx, const char* path, sf_vmm_plan** out) {
  return guard([&] {
    auto* h = new sf_vmm_plan;
    try {
      h->p = sf::vmm_plan_load(*ctx->c, path);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
sf_status sf_ct_wire_size(sf_context* ctx, const sf_ct* ct, size_t* bytes) {
  return guard([&] { *bytes = sf::ct_wire_size(*ctx->c, ct->v); });
}
sf_status sf_ct_serialize(sf_context* ctx, const sf_ct* ct, uint8_t* buf, size_t cap, size_t* len) {
  return guard([&] {
    const size_t need = sf::ct_wire_size(*ctx->c, ct->v);
    sf::require(cap >= need, sf::kShapeMismatch, "ct_serialize: buffer too small");
    sf::ct_serialize(*ctx->c, ct->v, buf);
    *len = need;
  });
}
sf_status sf_ct_deserialize(sf_context* ctx, const uint8_t* buf, size_t len, sf_ct** out) {
  return guard([&] { *out = wrap(sf::ct_deserialize(*ctx->c, buf, len)); });
}

// --- prefill (kv_attention.cpp:119-129, 245-376; vmm.cpp:30-43, 417-467)
sf_status sf_vmm_batch_plan_create(sf_context* ctx, const double* W, int rows, int cols, int level, int bsgs,
                                   sf_vmm_plan** out) {
  return guard([&] {
    auto* h = new sf_vmm_plan;
    try {
      h->p = sf::make_vmm_batch_plan(*ctx->c, W, rows, cols, level, bsgs != 0);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
sf_status sf_vmm_batch(sf_context* ctx, const sf_ct* x, sf_vmm_plan* plan, sf_ct** out) {
  return guard([&] { *out = wrap(sf::vmm_batch(*ctx->c, x->v, *plan->p)); });
}
sf_status sf_inner_rotate(sf_context* ctx, const sf_ct* x, int r, int block, int hoisted, sf_ct** out) {
  return guard([&] { *out = wrap(sf::inner_rotate(*ctx->c, x->v, r, block, hoisted != 0)); });
}
sf_status sf_rope_apply_batch(sf_context* ctx, const sf_ct* x, int d, int H, long long first_pos, double base,
                              sf_ct** out) {
  return guard([&] {
    sf::AttnCfg cfg{ctx->c->slots, d, H, 0, 1};
    sf::validate_attention_config(cfg, ctx->c->slots);
    *out = wrap(sf::rope_apply_batch(*ctx->c, x->v, cfg, first_pos, base));
  });
}
sf_status sf_prefill_scores(sf_context* ctx, const sf_ct* const* xs, int P, sf_vmm_plan* wq, sf_vmm_plan* wk,
                            sf_vmm_plan* wv, int d, int H, int n0, int n_max, double base, sf_kvcache** cache_out,
                            sf_ct** maps_out, int maps_cap, int* n_maps) {
  return guard([&] {
    sf::AttnCfg cfg{ctx->c->slots, d, H, n0, n_max};
    sf::validate_attention_config(cfg, ctx->c->slots);
    std::vector<sf::Ct> x;
    for (int p = 0; p < P; ++p) x.push_back(xs[p]->v);
    sf::PrefillScores r = sf::prefill_scores(*ctx->c, x, *wq->p, *wk->p, *wv->p, cfg, base);
    int k = 0;
    for (auto& mp : r.maps)
      for (auto& row : mp) k += (int)row.size();
    sf::require(k <= maps_cap, sf::kShapeMismatch, "prefill: map buffer too small");
    k = 0;
    for (auto& mp : r.maps)
      for (auto& row : mp)
        for (auto& m : row) maps_out[k++] = wrap(std::move(m));
    *n_maps = k;
    *cache_out = wrap_kv(std::move(r.cache));
  });
}
sf_status sf_prefill_attend(sf_context* ctx, const sf_ct* const* probs, int n_probs, const sf_kvcache* cache,
                            sf_ct** att_out, int att_cap, int* n_att) {
  return guard([&] {
    const sf::KV& kv = cache->kv;
    const int t = kv.cfg.t(), gt = kv.cfg.group_tokens();
    const int P = (kv.n_prime + t - 1) / t;
    std::vector<std::vector<std::vector<sf::Ct>>> pm(P);
    int k = 0;
    for (int p = 0; p < P; ++p) {
      pm[p].resize((p * t) / gt + 1);
      for (auto& row : pm[p])
        for (int rho = 0; rho < t; ++rho) {
          sf::require(k < n_probs, sf::kShapeMismatch, "prefill: softmax changed the map shape");
          row.push_back(probs[k++]->v);
        }
    }
    sf::require(k == n_probs, sf::kShapeMismatch, "prefill: softmax changed the map shape");
    sf::require(P <= att_cap, sf::kShapeMismatch, "prefill: attention buffer too small");
    auto att = sf::prefill_attend(*ctx->c, pm, kv);
    for (int p = 0; p < P; ++p) att_out[p] = wrap(std::move(att[p]));
    *n_att = P;
  });
}

// --- KV attention
sf_status sf_kv_create(sf_context* ctx, int d, int H, int n0, int n_max, sf_kvcache** out) {
  return guard([&] {
    sf::KV kv;
    kv.cfg = sf::AttnCfg{ctx->c->slots, d, H, n0, n_max};
    sf::validate_attention_config(kv.cfg, ctx->c->slots);
    *out = wrap_kv(std::move(kv));
  });
}
sf_kvcache* sf_kv_retain(sf_kvcache* kv) {
  if (kv) kv->rc.fetch_add(1);
  return kv;
}
void sf_kv_release(sf_kvcache* kv) {
  if (kv && kv->rc.fetch_sub(1) == 1) delete kv;
}
sf_status sf_kv_info(const sf_kvcache* kv, int* n_prime, int* n_k, int* n_groups, int* n_variants) {
  return guard([&] {
    if (n_prime) *n_prime = kv->kv.n_prime;
    if (n_k) *n_k = (int)kv->kv.k.size();
    if (n_groups) *n_groups = (int)kv->kv.v.size();
    if (n_variants) *n_variants = sf::v_variant_count(kv->kv.cfg);
  });
}
sf_status sf_kv_get(const sf_kvcache* kv, int which, int g, int idx, sf_ct** out) {
  return guard([&] {
    const auto& k = kv->kv;
    if (which == 0) {
      sf::require(idx >= 0 && idx < (int)k.k.size(), sf::kShapeMismatch, "kv_get: key index");
      *out = wrap(k.k[idx]);
    } else {
      sf::require(g >= 0 && g < (int)k.v.size() && idx >= 0 && idx < (int)k.v[g].size(), sf::kShapeMismatch,
                  "kv_get: value index");
      *out = wrap(k.v[g][idx]);
    }
  });
}
sf_status sf_kv_from_cts(sf_context* ctx, int d, int H, int n0, int n_max, int n_prime, const sf_ct* const* k_cts,
                         int n_k, const sf_ct* const* v_cts, int n_groups, sf_kvcache** out) {
  return guard([&] {
    sf::KV kv;
    kv.cfg = sf::AttnCfg{ctx->c->slots, d, H, n0, n_max};
    sf::validate_attention_config(kv.cfg, ctx->c->slots);
    kv.n_prime = n_prime;
    for (int i = 0; i < n_k; ++i) kv.k.push_back(k_cts[i]->v);
    const int nv = sf::v_variant_count(kv.cfg);
    for (int g = 0; g < n_groups; ++g) {
      kv.v.emplace_back();
      for (int i = 0; i < nv; ++i) kv.v.back().push_back(v_cts[(size_t)g * nv + i]->v);
    }
    *out = wrap_kv(std::move(kv));
  });
}
sf_status sf_rope_apply(sf_context* ctx, const sf_ct* x, int d, int H, long long position, double base,
                        sf_ct** out) {
  return guard([&] {
    sf::AttnCfg cfg{ctx->c->slots, d, H, 0, 1};
    *out = wrap(sf::rope_apply(*ctx->c, x->v, cfg, position, base));
  });
}
sf_status sf_rope_prepare(sf_context* ctx, int d, int H, int offset, int level, long long position, double base) {
  return guard([&] {
    sf::AttnCfg cfg{ctx->c->slots, d, H, 0, 1};
    sf::rope_prepare(*ctx->c, cfg, offset, level, position, base);
  });
}
sf_status sf_fused_extract_mask(sf_context* ctx, const sf_ct* x, const double* coeff, sf_ct** out) {
  return guard([&] { *out = wrap(sf::fused_extract_mask(*ctx->c, x->v, coeff)); });
}
sf_status sf_k_append(sf_context* ctx, const sf_kvcache* cache, const sf_ct* k_new, sf_kvcache** out) {
  return guard([&] { *out = wrap_kv(sf::k_append(*ctx->c, cache->kv, k_new->v)); });
}
sf_status sf_make_v_pieces(sf_context* ctx, const sf_kvcache* cache, const sf_ct* v_open, int position,
                           sf_ct** parts_out) {
  return guard([&] {
    auto parts = sf::make_v_pieces(*ctx->c, cache->kv, v_open->v, position);
    for (size_t i = 0; i < parts.size(); ++i) parts_out[i] = wrap(std::move(parts[i]));
  });
}
sf_status sf_v_append(sf_context* ctx, const sf_kvcache* cache, const sf_ct* const* parts, int n_parts,
                      sf_kvcache** out) {
  return guard([&] {
    std::vector<sf::Ct> p;
    for (int i = 0; i < n_parts; ++i) p.push_back(parts[i]->v);
    *out = wrap_kv(sf::v_append(*ctx->c, cache->kv, p));
  });
}
sf_status sf_qk_dot(sf_context* ctx, const sf_ct* q, const sf_kvcache* cache, sf_ct** maps_out, int* n_maps) {
  return guard([&] {
    auto maps = sf::qk_dot(*ctx->c, q->v, cache->kv);
    *n_maps = (int)maps.size();
    for (size_t i = 0; i < maps.size(); ++i) maps_out[i] = wrap(std::move(maps[i]));
  });
}
sf_status sf_softmax_times_v(sf_context* ctx, const sf_ct* const* probs, int n_probs, const sf_kvcache* cache,
                             sf_ct** out) {
  return guard([&] {
    std::vector<sf::Ct> p;
    for (int i = 0; i < n_probs; ++i) p.push_back(probs[i]->v);
    *out = wrap(sf::softmax_times_v(*ctx->c, p, cache->kv));
  });
}

// --- sharded hot path
sf_status sf_vmm_partial(sf_context* ctx, const sf_ct* x, const sf_vmm_plan* plan, int rank, int world,
                         sf_ct** out) {
  return guard([&] { *out = wrap(sf::vmm_partial(*ctx->c, x->v, *plan->p, rank, world)); });
}
sf_status sf_vmm_finish(sf_context* ctx, const sf_ct* acc, const sf_vmm_plan* plan, int mask_output, sf_ct** out) {
  return guard([&] { *out = wrap(sf::vmm_finish(*ctx->c, acc->v, *plan->p, mask_output != 0)); });
}
sf_status sf_qk_dot_partial(sf_context* ctx, const sf_ct* q, const sf_kvcache* cache, int rank, int world,
                            sf_ct** maps_out, int* n_maps) {
  return guard([&] {
    auto maps = sf::qk_dot_partial(*ctx->c, q->v, cache->kv, rank, world);
    *n_maps = (int)maps.size();
    for (size_t i = 0; i < maps.size(); ++i) maps_out[i] = wrap(std::move(maps[i]));
  });
}
sf_status sf_softmax_times_v_partial(sf_context* ctx, const sf_ct* const* probs, int n_probs,
                                     const sf_kvcache* cache, int rank, int world, sf_ct** out) {
  return guard([&] {
    std::vector<sf::Ct> p;
    for (int i = 0; i < n_probs; ++i) p.push_back(probs[i]->v);
    *out = wrap(sf::softmax_times_v_partial(*ctx->c, p, cache->kv, rank, world));
  });
}
sf_status sf_softmax_times_v_finish(sf_context* ctx, const sf_ct* const* parts, int n, const sf_kvcache* cache,
                                    sf_ct** out) {
  return guard([&] {
    sf::require(n >= 1, sf::kShapeMismatch, "softmax_times_v_finish: need at least one part");
    std::vector<const sf::Ct*> pp;
    for (int i = 0; i < n; ++i) pp.push_back(&parts[i]->v);
    *out = wrap(sf::softmax_times_v_finish(*ctx->c, pp, cache->kv));
  });
}
sf_status sf_sum_partials(sf_context* ctx, const sf_ct* const* parts, int n, sf_ct** out) {
  return guard([&] {
    sf::require(n >= 1, sf::kShapeMismatch, "sum_partials: need at least one part");
    std::vector<const sf::Ct*> p;
    for (int i = 0; i < n; ++i) p.push_back(&parts[i]->v);
    *out = wrap(sf::sum_partials(*ctx->c, p));
  });
}
sf_status sf_p2p_init(sf_context* ctx, int rank, int world, size_t cap_words, uint8_t handle_out[64]) {
  return guard([&] {
    need(ctx, "ctx");
    need(handle_out, "handle_out");
    sf::p2p_init(*ctx->c, rank, world, cap_words, handle_out);
  });
}
sf_status sf_p2p_open(sf_context* ctx, const uint8_t* handles, int world) {
  return guard([&] {
    need(ctx, "ctx");
    need(handles, "handles");
    int r, w;
    sf::p2p_rank_world(*ctx->c, r, w);
    sf::require(w == world, sf::kShapeMismatch, "p2p_open: world size differs from sf_p2p_init");
    sf::p2p_open(*ctx->c, handles);
  });
}
sf_status sf_p2p_destroy(sf_context* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    sf::p2p_destroy(*ctx->c);
  });
}
sf_status sf_comm_unique_id(uint8_t id_out[128]) {
  return guard([&] {
    need(id_out, "id_out");
    sf::comm_unique_id(id_out);
  });
}
sf_status sf_comm_init(sf_context* ctx, const uint8_t id[128], int rank, int world) {
  return guard([&] {
    need(ctx, "ctx");
    need(id, "id");
    sf::comm_init(*ctx->c, id, rank, world);
  });
}
sf_status sf_comm_destroy(sf_context* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    sf::comm_destroy(*ctx->c);
  });
}
sf_status sf_vmm_sharded(sf_context* ctx, const sf_ct* x, const sf_vmm_plan* plan, int mask_output, sf_ct** out) {
  return guard([&] { *out = wrap(sf::vmm_sharded(*ctx->c, x->v, *plan->p, mask_output != 0)); });
}
sf_status sf_qk_dot_sharded(sf_context* ctx, const sf_ct* q, const sf_kvcache* cache, sf_ct** maps_out,
                            int* n_maps) {
  return guard([&] {
    auto maps = sf::qk_dot_sharded(*ctx->c, q->v, cache->kv);
    *n_maps = (int)maps.size();
    for (size_t i = 0; i < maps.size(); ++i) maps_out[i] = wrap(std::move(maps[i]));
  });
}
sf_status sf_softmax_times_v_sharded(sf_context* ctx, const sf_ct* const* probs, int n_probs,
                                     const sf_kvcache* cache, sf_ct** out) {
  return guard([&] {
    std::vector<sf::Ct> p;
    for (int i = 0; i < n_probs; ++i) p.push_back(probs[i]->v);
    *out = wrap(sf::softmax_times_v_sharded(*ctx->c, p, cache->kv));
  });
}
sf_status sf_ct_device_view(const sf_ct* ct, uint64_t** c0, uint64_t** c1, size_t* words_per_poly) {
  return guard([&] {
    need(ct, "ct");
    const auto& v = ct->v;
    const int n = (int)(v.buf->words / (2 * (size_t)v.stride));
    *c0 = v.c0();
    *c1 = v.c1(n);
    *words_per_poly = (size_t)v.limbs * n;
  });
}
sf_status sf_ct_from_device(sf_context* ctx, const uint64_t* c0, const uint64_t* c1, int level, double scale,
                            int is_zero, const sf_layout* layout, sf_ct** out) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(level >= 0 && level <= c.L, sf::kInvalidTarget, "from_device: level out of range");
    sf::Ct v = sf::alloc_ct(c, level + 1, scale);
    v.zero = is_zero != 0;
    v.layout = to_layout(layout);
    const size_t w = (size_t)v.limbs * c.n;
    SF_CUDA(cudaMemcpyAsync(v.c0(), c0, w * 8, cudaMemcpyDeviceToDevice, c.stream));
    SF_CUDA(cudaMemcpyAsync(v.c1(c.n), c1, w * 8, cudaMemcpyDeviceToDevice, c.stream));
    *out = wrap(std::move(v));
  });
}

// --- timing
sf_status sf_event_record(sf_context* ctx, int slot) {
  return guard([&] {
    auto& c = *ctx->c;
    while ((int)c.events.size() <= slot) {
      cudaEvent_t e;
      SF_CUDA(cudaEventCreate(&e));
      c.events.push_back(e);
    }
    // inside a graph capture the record must be an external event node, so
    // the event is really recorded (and timed) on every replay
    if (c.capturing)
      SF_CUDA(cudaEventRecordWithFlags(c.events[slot], c.stream, cudaEventRecordExternal));
    else
      SF_CUDA(cudaEventRecord(c.events[slot], c.stream));
  });
}
sf_status sf_event_elapsed_ms(sf_context* ctx, int a, int b, float* ms) {
  return guard([&] {
    auto& c = *ctx->c;
    SF_CUDA(cudaEventSynchronize(c.events[b]));
    SF_CUDA(cudaEventElapsedTime(ms, c.events[a], c.events[b]));
  });
}
long long sf_kernel_launches(const sf_context* ctx) { return ctx->c->launches.load(); }

sf_status sf_profile_begin(sf_context* ctx, int mask) {
  return guard([&] {
    auto& c = *ctx->c;
    SF_CUDA(cudaStreamSynchronize(c.stream));
    c.prof_recs.clear();
    c.prof_pool_next = 0;
    c.prof_mask = mask;
  });
}

sf_status sf_profile_end(sf_context* ctx, double* ms, double* bytes, long long* launches) {
  return guard([&] {
    auto& c = *ctx->c;
    c.prof_mask = 0;
    SF_CUDA(cudaStreamSynchronize(c.stream));
    for (int f = 0; f < SF_PROF_FAMILIES; ++f) ms[f] = 0.0, bytes[f] = 0.0, launches[f] = 0, c.prof_bfly[f] = 0.0;
    for (const auto& r : c.prof_recs) {
      c.prof_bfly[r.family] += r.bfly;
      float t = 0.f;
      SF_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
      ms[r.family] += t;
      bytes[r.family] += r.bytes;
      launches[r.family] += 1;
    }
    c.prof_recs.clear();
    c.prof_pool_next = 0;
  });
}

sf_status sf_graph_capture_begin(sf_context* ctx) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(!c.capturing, sf::kInvalidTarget, "graph capture already in progress");
    SF_CUDA(cudaStreamSynchronize(c.stream));
    c.capture_deferred.clear();
    c.capture_gm = std::make_shared<sf::GraphMem>();
    c.capturing = true;
    c.graph_launch_base = c.launches.load();
    const cudaError_t e = cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) c.capturing = false;
    SF_CUDA(e);
  });
}

sf_status sf_graph_capture_end(sf_context* ctx, sf_graph** out) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(c.capturing, sf::kInvalidTarget, "no graph capture in progress");
    auto g = std::make_unique<sf_graph>();
    g->ctx = ctx;
    g->cp = ctx->c.get();
    g->gen = ctx->c->gen;
    const cudaError_t e = cudaStreamEndCapture(c.stream, &g->g);
    c.capturing = false;
    g->deferred.swap(c.capture_deferred);
    g->gm = std::move(c.capture_gm);
    g->launches = c.launches.load() - c.graph_launch_base;
    cudaError_t ie = e;
    if (e == cudaSuccess) ie = cudaGraphInstantiateWithFlags(&g->x, g->g, cudaGraphInstantiateFlagAutoFreeOnLaunch);
    if (ie != cudaSuccess) {  // failed capture: nothing will replay; release what it deferred
      cudaGetLastError();
      if (g->g) cudaGraphDestroy(g->g);
      g->g = nullptr;
      {
        std::lock_guard<std::mutex> lk(g->gm->mu);
        g->gm->destroyed = true;  // never launched: its Bufs own nothing outstanding
        g->gm->dead.clear();
      }
      for (auto& d : g->deferred) cudaFreeAsync(d.first, c.stream);
      g->deferred.clear();
    }
    SF_CUDA(e);
    SF_CUDA(ie);
    ++c.live_graphs;
    *out = g.release();
  });
}

sf_status sf_graph_launch(sf_context* ctx, sf_graph* g) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(g && g->ctx == ctx, sf::kInvalidTarget, "graph belongs to another context");
    SF_CUDA(cudaGraphLaunch(g->x, c.stream));
    { std::lock_guard<std::mutex> lk(g->gm->mu); g->gm->launched = true; }
    c.launches.fetch_add(g->launches);
  });
}

long long sf_graph_kernel_launches(const sf_graph* g) { return g ? g->launches : 0; }

void sf_graph_destroy(sf_graph* g) {
  if (!g) return;
  const bool alive = sf::context_alive(g->cp, g->gen);
  cudaStream_t st = alive ? g->cp->stream : nullptr;
  if (alive) cudaStreamSynchronize(st);
  if (alive && g->x) --g->cp->live_graphs;
  if (g->x) cudaGraphExecDestroy(g->x);
  if (g->g) cudaGraphDestroy(g->g);
  auto free_ = [&](sf::u64* p) { alive ? (void)cudaFreeAsync(p, st) : (void)cudaFree(p); };
  for (auto& d : g->deferred) free_(d.first);
  {
    std::lock_guard<std::mutex> lk(g->gm->mu);
    g->gm->destroyed = true;
    if (g->gm->launched)
      for (sf::u64* p : g->gm->dead) free_(p);  // outstanding allocations of dead Bufs
    g->gm->dead.clear();
  }
  if (alive) cudaStreamSynchronize(st);
  delete g;
}

sf_status sf_ct_refill(sf_context* ctx, sf_ct* ct, const uint64_t* words) {
  return guard([&] {
    auto& c = *ctx->c;
    const sf::Ct& v = ct->v;
    sf::require(v.buf && !v.zero, sf::kInvalidTarget, "refill: ciphertext has no device words");
    const size_t w = (size_t)v.limbs * c.n;
    SF_CUDA(cudaMemcpyAsync(v.c0(), words, w * 8, cudaMemcpyHostToDevice, c.stream));
    SF_CUDA(cudaMemcpyAsync(v.c1(c.n), words + w, w * 8, cudaMemcpyHostToDevice, c.stream));
  });
}

// Staged input upload: the copy runs on a side stream forked from the library
// stream at this point, so it overlaps whatever the library stream runs until
// sf_ct_stage_wait(slot) joins it back (inside a capture: memcpy nodes on a
// parallel branch of the graph, re-read from the host words on every replay).
sf_status sf_ct_stage(sf_context* ctx, sf_ct* ct, const uint64_t* words, int slot) {
  return guard([&] {
    auto& c = *ctx->c;
    const sf::Ct& v = ct->v;
    sf::require(v.buf && !v.zero, sf::kInvalidTarget, "stage: ciphertext has no device words");
    sf::require(slot >= 0 && slot < 64, sf::kInvalidTarget, "stage: slot out of range");
    if (!c.copy_stream) SF_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    while ((int)c.stage_ev.size() <= slot) {
      cudaEvent_t f, d;
      SF_CUDA(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
      SF_CUDA(cudaEventCreateWithFlags(&d, cudaEventDisableTiming));
      c.stage_ev.push_back({f, d});
    }
    auto [fork, done] = c.stage_ev[slot];
    const size_t w = (size_t)v.limbs * c.n;
    SF_CUDA(cudaEventRecord(fork, c.stream));
    SF_CUDA(cudaStreamWaitEvent(c.copy_stream, fork, 0));
    SF_CUDA(cudaMemcpyAsync(v.c0(), words, w * 8, cudaMemcpyHostToDevice, c.copy_stream));
    SF_CUDA(cudaMemcpyAsync(v.c1(c.n), words + w, w * 8, cudaMemcpyHostToDevice, c.copy_stream));
    SF_CUDA(cudaEventRecord(done, c.copy_stream));
  });
}
// The read-back counterpart: device words -> (pinned) host memory on the side
// stream, forked here (after everything enqueued so far, i.e. once ct is final),
// overlapping what follows until sf_ct_stage_wait(slot).
sf_status sf_ct_stage_out(sf_context* ctx, const sf_ct* ct, uint64_t* words, int slot) {
  return guard([&] {
    auto& c = *ctx->c;
    const sf::Ct& v = ct->v;
    sf::require(v.buf && !v.zero, sf::kInvalidTarget, "stage_out: ciphertext has no device words");
    sf::require(slot >= 0 && slot < 64, sf::kInvalidTarget, "stage_out: slot out of range");
    if (!c.copy_stream) SF_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    while ((int)c.stage_ev.size() <= slot) {
      cudaEvent_t f, d;
      SF_CUDA(cudaEventCreateWithFlags(&f, cudaEventDisableTiming));
      SF_CUDA(cudaEventCreateWithFlags(&d, cudaEventDisableTiming));
      c.stage_ev.push_back({f, d});
    }
    auto [fork, done] = c.stage_ev[slot];
    const size_t w = (size_t)v.limbs * c.n;
    SF_CUDA(cudaEventRecord(fork, c.stream));
    SF_CUDA(cudaStreamWaitEvent(c.copy_stream, fork, 0));
    SF_CUDA(cudaMemcpyAsync(words, v.c0(), w * 8, cudaMemcpyDeviceToHost, c.copy_stream));
    SF_CUDA(cudaMemcpyAsync(words + w, v.c1(c.n), w * 8, cudaMemcpyDeviceToHost, c.copy_stream));
    SF_CUDA(cudaEventRecord(done, c.copy_stream));
  });
}
sf_status sf_ct_stage_wait(sf_context* ctx, int slot) {
  return guard([&] {
    auto& c = *ctx->c;
    sf::require(slot >= 0 && slot < (int)c.stage_ev.size(), sf::kInvalidTarget, "stage_wait: slot never staged");
    SF_CUDA(cudaStreamWaitEvent(c.stream, c.stage_ev[slot].second, 0));
  });
}

sf_status sf_mem_stats(sf_context* ctx, size_t* graph_bytes, size_t* pool_bytes) {
  return guard([&] {
    auto& c = *ctx->c;
    unsigned long long g = 0, p = 0;
    SF_CUDA(cudaStreamSynchronize(c.stream));
    SF_CUDA(cudaDeviceGetGraphMemAttribute(c.device, cudaGraphMemAttrUsedMemCurrent, &g));
    SF_CUDA(cudaMemPoolGetAttribute(c.pool, cudaMemPoolAttrUsedMemCurrent, &p));
    if (graph_bytes) *graph_bytes = (size_t)g;
    if (pool_bytes) *pool_bytes = (size_t)p;
  });
}

sf_status sf_key_stats(sf_context* ctx, int* count, size_t* bytes, size_t* full_bytes) {
  return guard([&] {
    auto& c = *ctx->c;
    std::lock_guard<std::mutex> lk(c.mu);
    size_t b = 0, f = 0;
    int k = 0;
    const size_t per_digit = (size_t)2 * c.np * c.n * sizeof(sf::u64);
    for (auto* m : {&c.keys_pinv_dig, &c.keys_r_dig})
      for (auto& [g, d] : *m) b += per_digit * d, f += per_digit * c.beta, ++k;
    for (auto& [g, p] : c.keys) b += p->words * sizeof(sf::u64), f += per_digit * c.beta, ++k;
    if (count) *count = k;
    if (bytes) *bytes = b;
    if (full_bytes) *full_bytes = f;
  });
}

sf_status sf_set_value_shard(sf_context* ctx, int rank, int world) {
  return guard([&] {
    sf::require(world >= 1 && rank >= 0 && rank < world, sf::kInvalidTarget, "set_value_shard: bad rank/world");
    ctx->c->sv_rank = rank;
    ctx->c->sv_world = world;
  });
}

sf_status sf_mem_reserve(sf_context* ctx, size_t bytes) {
  return guard([&] {
    auto& c = *ctx->c;
    void* p = nullptr;
    SF_CUDA(cudaMallocAsync(&p, bytes, c.stream));  // grows the pool once (its release threshold is unbounded)
    SF_CUDA(cudaFreeAsync(p, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
  });
}

sf_status sf_host_profile(char* buf, int len, int reset) {
  return guard([&] {
    const std::string s = sf::host_prof_dump(reset != 0);
    if (buf && len > 0) {
      const size_t k = std::min<size_t>(s.size(), (size_t)len - 1);
      std::memcpy(buf, s.data(), k);
      buf[k] = 0;
    }
  });
}

sf_status sf_profile_butterflies(sf_context* ctx, double* out) {
  return guard([&] {
    for (int f = 0; f < SF_PROF_FAMILIES; ++f) out[f] = ctx->c->prof_bfly[f];
  });
}

}  // extern "C"
