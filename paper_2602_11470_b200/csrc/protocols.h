// Hot-path protocols over the GPU evaluator: the packed HE-VMM
// (vmm.hpp:74-75 / vmm.cpp:179-236) and the KV-cache attention decode step
// (kv_attention.hpp:32-109 / kv_attention.cpp:80-241).
#pragma once
#include <functional>

#include "batch.cuh"
#include "context.h"

namespace sf {

// vmm.cpp:124-153 (InterleavedShape)
struct VmmShape {
  int N = 0, d_in = 0, d_out = 0, t_in = 0, t_out = 0;
  long long k = 0;
  int alpha_up = 0, ladder_T = 0, tau_in = 0, tau_out = 0, tau_u = 0, carry = 0, delta = 0;
};
VmmShape vmm_shape(int N, int rows, int cols, int tau_in, int tau_out);
struct BsgsSplit {
  int baby, giant;
};
BsgsSplit bsgs_split(long long k);
void predict_interleaved_cost(int N, int rows, int cols, bool bsgs, bool mask, long long* rot, long long* ctpt,
                              int* depth);

struct VmmPlan {
  Context* ctx = nullptr;
  int rows = 0, cols = 0, level = 0;
  bool bsgs = false;
  VmmShape s;
  BsgsSplit bg{1, 1};
  std::function<double(int, int)> w;  // weight_at (vmm.cpp:17-19 semantics: 0 outside)
  std::vector<double> w_store;
  std::map<int, std::vector<Pt>> pts;  // limbs -> k diagonals (NTT, scale q_top)
  bool batch = false;                   // token-batched square diagonals (vmm.cpp:426-433, vmm_batch)
  const std::vector<Pt>& diagonals(int limbs);
};

std::unique_ptr<VmmPlan> make_vmm_plan(Context& c, const double* W, int rows, int cols, int level, int in_offset,
                                       int out_offset, bool bsgs, bool encode = true);
Ct vmm_interleaved(Context& c, const Ct& x, VmmPlan& plan, bool mask_output);
// several VMMs of the same input (shared ladder + babies, batched tails)
std::vector<Ct> vmm_multi_partial(Context& c, const Ct& x, const std::vector<VmmPlan*>& plans, int rank, int world);
std::vector<Ct> vmm_multi_finish(Context& c, const std::vector<Ct>& accs, const std::vector<VmmPlan*>& plans,
                                 bool mask_output);
std::vector<Ct> vmm_interleaved_many(Context& c, const std::vector<const Ct*>& xs, VmmPlan& plan, bool mask_output);
std::vector<Ct> vmm_interleaved_multi(Context& c, const Ct& x, const std::vector<VmmPlan*>& plans, bool mask_output);
// sharded form: partial over the giant steps g2 = rank mod world, then (after
// the exchange's modular sum) the reduce ladder + mask
Ct vmm_partial(Context& c, const Ct& x, VmmPlan& plan, int rank, int world);
Ct vmm_finish(Context& c, const Ct& acc, VmmPlan& plan, bool mask_output);
Ct sum_partials(Context& c, const std::vector<const Ct*>& parts);

// --- attention ---------------------------------------------------------------
struct AttnCfg {
  int N = 0, d = 0, H = 1, n0 = 0, n_max = 0;
  int d_head() const { return d / H; }
  int t() const { return N / d; }
  int group_tokens() const { return N / H; }
};
void validate_attention_config(const AttnCfg& cfg, int N_backend);

struct KV {
  AttnCfg cfg;
  int n_prime = 0;
  std::vector<Ct> k;
  std::vector<std::vector<Ct>> v;  // [group][variant]
  // giant-aligned variants Rot(v[g][w], G B t) for the BSGS Score*V (DESIGN.md
  // §3.9), kept current by v_append from the pieces' aligned companions;
  // va_ok[g][w] = 0: not tracked (softmax_times_v rotates v[g][w] itself)
  std::vector<std::vector<Ct>> va;
  std::vector<std::vector<char>> va_ok;
};
int v_variant_count(const AttnCfg& cfg);
int v_variant_index(const AttnCfg& cfg, int w);
int v_variant_of(const AttnCfg& cfg, int e, int u_local);

Ct rope_apply(Context& c, const Ct& x, const AttnCfg& cfg, long long position, double base);
void rope_prepare(Context& c, const AttnCfg& cfg, int offset, int level, long long position, double base);
Ct fused_extract_mask(Context& c, const Ct& x, const double* coeff);
KV k_append(Context& c, const KV& cache, const Ct& k_new);
std::vector<Ct> make_v_pieces(Context& c, const KV& cache, const Ct& v_open, int position);
KV v_append(Context& c, const KV& cache, const std::vector<Ct>& parts);
std::vector<Ct> qk_dot(Context& c, const Ct& q, const KV& cache);
std::vector<Ct> qk_dot_partial(Context& c, const Ct& q, const KV& cache, int rank, int world);
// Score*V: the rank's baby-step / giant-step partial (whole
// giant groups), then the sum of the partials, fold_lanes and the stride mask
int sv_baby(const AttnCfg& cfg);
Ct softmax_times_v_partial(Context& c, const std::vector<Ct>& probs, const KV& cache, int rank, int world);
Ct softmax_times_v_finish(Context& c, const std::vector<const Ct*>& parts, const KV& cache);
Ct softmax_times_v(Context& c, const std::vector<Ct>& probs, const KV& cache);

// --- prefill (kv_attention.cpp:119-129, 245-376; vmm.cpp:30-43, 417-467) ------
Ct inner_rotate(Context& c, const Ct& x, int r, int block, bool hoisted);
std::unique_ptr<VmmPlan> make_vmm_batch_plan(Context& c, const double* W, int rows, int cols, int level, bool bsgs,
                                             bool encode = true);
Ct vmm_batch(Context& c, const Ct& x, VmmPlan& plan);
Ct rope_apply_batch(Context& c, const Ct& x, const AttnCfg& cfg, long long first_pos, double base);
// prefill up to the caller's softmax: the cache and the score maps [p][g][rho]
struct PrefillScores {
  KV cache;
  std::vector<std::vector<std::vector<Ct>>> maps;
};
PrefillScores prefill_scores(Context& c, const std::vector<Ct>& xs, VmmPlan& wq, VmmPlan& wk, VmmPlan& wv,
                             const AttnCfg& cfg, double base);
// the probability-weighted values per prompt ct (after the caller's softmax)
std::vector<Ct> prefill_attend(Context& c, const std::vector<std::vector<std::vector<Ct>>>& probs, const KV& cache);

// --- sharded ops with the exchange on the library stream (comm.cpp) ------------
void comm_unique_id(uint8_t* out128);
void comm_init(Context& c, const uint8_t* id128, int rank, int world);
void comm_destroy(Context& c);
Ct vmm_sharded(Context& c, const Ct& x, VmmPlan& plan, bool mask_output);
std::vector<Ct> vmm_multi_sharded(Context& c, const Ct& x, const std::vector<VmmPlan*>& plans, bool mask_output);
std::vector<Ct> qk_dot_sharded(Context& c, const Ct& q, const KV& cache);
Ct softmax_times_v_sharded(Context& c, const std::vector<Ct>& probs, const KV& cache);

// --- sharded ops with the exchange over peer memory (p2p.cu) --------------------
void p2p_init(Context& c, int rank, int world, size_t cap_words, uint8_t* handle_out64);
void p2p_open(Context& c, const uint8_t* handles);  // world x 64 bytes
void p2p_destroy(Context& c);
void p2p_rank_world(Context& c, int& rank, int& world);
std::vector<Ct> p2p_sum_cts(Context& c, const std::vector<const Ct*>& cts, const std::string& tag, bool charge = true,
                            std::vector<int>* live_out = nullptr);

// --- wire / on-disk formats (wire.cpp) ---------------------------------------
std::vector<double> load_weight(const std::string& dir, const std::string& name, int* rows, int* cols);
size_t ct_wire_size(const Context& c, const Ct& a);
void ct_serialize(Context& c, const Ct& a, uint8_t* out);
Ct ct_deserialize(Context& c, const uint8_t* in, size_t len);
void vmm_plan_save(Context& c, VmmPlan& p, const std::string& path);
std::unique_ptr<VmmPlan> vmm_plan_load(Context& c, const std::string& path);

}  // namespace sf
