/* sf_b200.h — C ABI of the B200-native encrypted-decode hot path.
 *
 * Drop-in boundary for the reference's `slotforge` C++ API
 * (/root/reference/proj/include/slotforge/*.hpp). Plain pointers, sizes and
 * opaque handles only; no C++ or torch types. Every entry point returns an
 * sf_status (0 = OK); on failure sf_last_error() holds the message and the code
 * maps 1:1 onto the reference exception types (types.hpp:16-46), so a C++ or
 * Python host layer can rethrow the same types the reference tests expect.
 *
 * Ciphertexts are immutable, reference-counted device values (engine.hpp:102-104:
 * "Operations return fresh ciphertext values"); an op never mutates its inputs.
 * All work is enqueued on the context's CUDA stream; only decrypt / export /
 * sf_synchronize block the host.
 *
 * Reference interface each entry point replaces is cited per declaration.
 */
#ifndef SF_B200_H
#define SF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* --- status codes: 1:1 with slotforge exception types (types.hpp:16-46) --- */
typedef int sf_status;
#define SF_OK 0
#define SF_ERR_LEVEL_UNDERFLOW 1 /* slotforge::LevelUnderflow */
#define SF_ERR_INVALID_TARGET 2  /* slotforge::InvalidTarget  */
#define SF_ERR_SHAPE_MISMATCH 3  /* slotforge::ShapeMismatch  */
#define SF_ERR_LAYOUT_MISMATCH 4 /* slotforge::LayoutMismatch */
#define SF_ERR_CACHE_FULL 5      /* slotforge::CacheFull      */
#define SF_ERR_CACHE_EMPTY 6     /* slotforge::CacheEmpty     */
#define SF_ERR_DOMAIN 7          /* slotforge::DomainViolation */
#define SF_ERR_SCALE_MISMATCH 8  /* CKKS: adding ciphertexts at different scales (slotforge::Error) */
#define SF_ERR_CUDA 9            /* device failure (slotforge::Error) */
#define SF_ERR_INTERNAL 10       /* anything else (slotforge::Error) */

typedef struct sf_context sf_context;
typedef struct sf_ct sf_ct;
typedef struct sf_vmm_plan sf_vmm_plan;
typedef struct sf_kvcache sf_kvcache;

/* layouts.hpp:22-33 (Layout). kind: 0 contiguous, 1 replicated, 2 interleaved.
 * valid = 0 means "no layout tag" (std::optional<Layout> empty). */
typedef struct {
  int valid;
  int kind;
  int d;
  int t;
  int offset;
  int heads;
  int deferred_mask;
} sf_layout;

/* engine.hpp:19-22 (EngineParams{N, L}) extended with the CKKS parameters the
 * reference leaves "unhoused by design". slots = the reference N.
 * log_n = ring degree exponent (0: 2*slots). alpha = special primes per digit
 * (0: min(L+1, 5)). Bits of q0 / scale primes / special primes (0: 60/40/60),
 * each in [20, 60] (the lazy kernels need q < 2^60; SF_ERR_DOMAIN otherwise). */
typedef struct {
  int slots;
  int L;
  int log_n;
  int alpha;
  int q0_bits;
  int scale_bits;
  int special_bits;
  int device;
  uint64_t seed; /* secret-key / evaluation-key seed */
} sf_params;

/* engine.hpp:30-49 (OpCounts) */
typedef struct {
  long long rotations;
  long long hoisted_rotations;
  long long ct_pt_mults;
  long long ct_ct_mults;
  long long additions;
  long long bootstraps;
} sf_op_counts;

/* --- errors ---------------------------------------------------------------- */
const char* sf_last_error(void);

/* --- context: Backend::Backend(EngineParams) (engine.cpp:92-95) + keygen ----- */
sf_status sf_context_create(const sf_params* params, sf_context** out);
void sf_context_destroy(sf_context* ctx);
/* ring degree, slots, L, alpha, number of primes (q0..qL, p0..p_{alpha-1});
 * primes may be NULL, else receives num_primes words. */
sf_status sf_context_info(const sf_context* ctx, int* n, int* slots, int* L, int* alpha, int* num_primes,
                          uint64_t* primes);
sf_status sf_synchronize(sf_context* ctx);
/* Galois keys are generated lazily on first use; this pre-generates a set. */
sf_status sf_gen_rotation_keys(sf_context* ctx, const int* rotations, int count);
/* secret key (NTT domain, all primes: num_primes*n words) and one switching
 * key (galois element g, 0 = relinearisation; beta*2*num_primes*n words):
 * exported for bit-exact parity tests only. */
sf_status sf_secret_key_export(sf_context* ctx, uint64_t* out);
sf_status sf_switching_key_export(sf_context* ctx, uint64_t galois_elt, uint64_t* out);
uint64_t sf_galois_elt(const sf_context* ctx, int rotation);

/* --- ciphertext handles ---------------------------------------------------- */
sf_ct* sf_ct_retain(sf_ct* ct);
void sf_ct_release(sf_ct* ct);
/* Ciphertext{slots, level, layout} (engine.hpp:24-28) + CKKS scale. */
sf_status sf_ct_info(const sf_ct* ct, int* level, double* scale, int* is_zero, sf_layout* layout);
/* same value, new layout tag (the reference assigns `ct.layout = ...`) */
sf_status sf_ct_with_layout(sf_context* ctx, const sf_ct* ct, const sf_layout* layout, sf_ct** out);
/* raw RNS words, limb-major [2][level+1][n] (NTT domain) */
sf_status sf_ct_export(sf_context* ctx, const sf_ct* ct, uint64_t* out);
sf_status sf_ct_import(sf_context* ctx, const uint64_t* words, int level, double scale, int is_zero,
                       const sf_layout* layout, sf_ct** out);

/* --- client side, off-ledger: Backend::encrypt / zeros (engine.cpp:109-123),
 *     encode/decode (layouts.cpp:66-104 composed with CKKS encoding) -------- */
/* level < 0: L. use_seed = 0: seed from the context's encryption counter. */
sf_status sf_encrypt(sf_context* ctx, const double* slots, int level, const sf_layout* layout, uint64_t seed,
                     int use_seed, sf_ct** out);
sf_status sf_zeros(sf_context* ctx, int level, sf_ct** out);
sf_status sf_decrypt(sf_context* ctx, const sf_ct* ct, double* slots_out);
/* CKKS encode of `slots` at `scale` into `limbs` RNS limbs, NTT domain. */
sf_status sf_encode(sf_context* ctx, const double* slots, double scale, int limbs, uint64_t* out);

/* --- evaluator: virtual ops of slotforge::Backend (engine.hpp:112-149) ------ */
sf_status sf_add(sf_context* ctx, const sf_ct* a, const sf_ct* b, sf_ct** out);       /* engine.cpp:143 */
sf_status sf_sub(sf_context* ctx, const sf_ct* a, const sf_ct* b, sf_ct** out);       /* engine.cpp:150 */
sf_status sf_add_plain(sf_context* ctx, const sf_ct* a, const double* slots, sf_ct** out); /* :157 */
sf_status sf_mul(sf_context* ctx, const sf_ct* a, const sf_ct* b, sf_ct** out);       /* engine.cpp:164 */
sf_status sf_mul_plain(sf_context* ctx, const sf_ct* a, const double* slots, sf_ct** out); /* :173 */
/* sum_k cts[k] * slots[k*N..] with one rescale; charged as k ct-pt mults and
 * k-1 additions (the reference's mul_plain/add chain, vmm.cpp:214-219). */
sf_status sf_mac_plain(sf_context* ctx, const sf_ct* const* cts, const double* slots, int k, sf_ct** out);
sf_status sf_rotate(sf_context* ctx, const sf_ct* a, int r, int hoisted, sf_ct** out); /* :181 */
/* k rotations of one ciphertext sharing one ModUp (RotationHint{hoisted}). */
sf_status sf_rotate_hoisted(sf_context* ctx, const sf_ct* a, const int* r, int k, sf_ct** outs);
/* k independent rotations Rot(a[i], r) (same Galois key), batched into one
   key-switching pass; charged k rotations. Extension (no reference twin):
   the throughput form of Backend::rotate used by the C5 sweep. */
sf_status sf_rotate_many(sf_context* ctx, const sf_ct* const* a, int k, int r, sf_ct** outs);
/* Microbenchmark: batched two-pass NTT of count x limbs scratch limbs (forward
   and inverse alternating), device time per limb transform. Diagnostics. */
sf_status sf_bench_ntt(sf_context* ctx, int limbs, int count, int reps, double* ms_per_limb_ntt);
sf_status sf_level_drop(sf_context* ctx, const sf_ct* a, int target, sf_ct** out); /* engine.cpp:201 */
/* oracle hook (engine.cpp:193): client round trip decrypt -> encrypt at target */
sf_status sf_bootstrap(sf_context* ctx, const sf_ct* a, int target, sf_ct** out);

/* --- ledger: CostLedger (engine.hpp:54-96) -------------------------------- */
sf_status sf_ledger_totals(const sf_context* ctx, sf_op_counts* out);
sf_status sf_ledger_phase_totals(const sf_context* ctx, const char* phase, sf_op_counts* out);
sf_status sf_ledger_reset(sf_context* ctx);
sf_status sf_phase_push(sf_context* ctx, const char* phase);
sf_status sf_phase_pop(sf_context* ctx);

/* --- packed HE-VMM: vmm_interleaved (vmm.hpp:74-75, vmm.cpp:179-236) ------
 * A plan holds the k interleaved diagonals (vmm.cpp:159-175) pre-encoded on
 * the device at `level` (offline, not charged). W is row-major
 * rows x cols with y = x^T W; W == NULL selects the reference bench weight
 * sin(0.001*(31 r + c) + 0.25) (slotforge_cli.cpp:88-92). */
sf_status sf_vmm_plan_create(sf_context* ctx, const double* W, int rows, int cols, int level, int in_offset,
                             int out_offset, int bsgs, sf_vmm_plan** out);
void sf_vmm_plan_destroy(sf_vmm_plan* plan);
/* predict_interleaved_cost (vmm.cpp:473-488) */
sf_status sf_vmm_predict(const sf_context* ctx, int rows, int cols, int bsgs, int mask_output,
                         long long* rotations, long long* ct_pt_mults, int* depth);
sf_status sf_vmm_interleaved(sf_context* ctx, const sf_ct* x, const sf_vmm_plan* plan, int mask_output,
                             sf_ct** out);
/* k VMMs of the same input (e.g. Q/K/V): outs[i] is word-for-word the result of
   sf_vmm_interleaved(x, plans[i]) and the ledger is charged as k such calls;
   the input-only ladder and baby steps run once, the rest as batched launches. */
sf_status sf_vmm_interleaved_multi(sf_context* ctx, const sf_ct* x, sf_vmm_plan* const* plans, int k,
                                   int mask_output, sf_ct** outs);
/* [vmm_interleaved(x_i, plan) for each of k independent inputs], word for word
 * and in the ledger, every stage batched across the inputs (HE-VMM throughput) */
sf_status sf_vmm_interleaved_many(sf_context* ctx, const sf_ct* const* xs, int k, const sf_vmm_plan* plan,
                                  int mask_output, sf_ct** outs);

/* ---- wire and on-disk formats ---------------------------------
   Weights in the reference's files (layouts.cpp:158-184: <dir>/<name>.bin =
   rows x cols row-major float64, <name>.json = {"name","rows","cols"}); an
   encoded-plan cache (the plan's NTT-domain diagonals + weights, so a restart
   skips the offline encode); and the client <-> server ciphertext format
   (header with magic, version, ring fingerprint, level, scale, layout; then the
   2 x limbs x n RNS words). Loading checks the ring fingerprint. */
sf_status sf_vmm_plan_create_from_file(sf_context* ctx, const char* dir, const char* name, int level, int in_offset,
                                       int out_offset, int bsgs, sf_vmm_plan** out);
sf_status sf_vmm_plan_save(sf_context* ctx, sf_vmm_plan* plan, const char* path);
sf_status sf_vmm_plan_load(sf_context* ctx, const char* path, sf_vmm_plan** out);
sf_status sf_ct_wire_size(sf_context* ctx, const sf_ct* ct, size_t* bytes);
sf_status sf_ct_serialize(sf_context* ctx, const sf_ct* ct, uint8_t* buf, size_t cap, size_t* len);
sf_status sf_ct_deserialize(sf_context* ctx, const uint8_t* buf, size_t len, sf_ct** out);

/* ---- prefill (kv_attention.hpp:111-150; kv_attention.cpp:245-376) -------------
   vmm_batch (vmm.cpp:417-467) with its own plan type (token-batched square
   diagonals), inner_rotate (vmm.cpp:30-43), rope_apply_batch (kv_attention.cpp:
   119-129). The reference's prefill takes a softmax callback; across the ABI it
   is split at that callback: sf_prefill_scores returns the cache (slot-identical
   to sequential appends) and the score maps flattened in [p][g][rho] order
   (g < p*t/(N/H) + 1, rho < t); the caller applies its softmax and hands the
   probability maps, same order and count, to sf_prefill_attend. */
sf_status sf_vmm_batch_plan_create(sf_context* ctx, const double* W, int rows, int cols, int level, int bsgs,
                                   sf_vmm_plan** out);
sf_status sf_vmm_batch(sf_context* ctx, const sf_ct* x, sf_vmm_plan* plan, sf_ct** out);
sf_status sf_inner_rotate(sf_context* ctx, const sf_ct* x, int r, int block, int hoisted, sf_ct** out);
sf_status sf_rope_apply_batch(sf_context* ctx, const sf_ct* x, int d, int H, long long first_pos, double base,
                              sf_ct** out);
sf_status sf_prefill_scores(sf_context* ctx, const sf_ct* const* xs, int P, sf_vmm_plan* wq, sf_vmm_plan* wk,
                            sf_vmm_plan* wv, int d, int H, int n0, int n_max, double base, sf_kvcache** cache_out,
                            sf_ct** maps_out, int maps_cap, int* n_maps);
sf_status sf_prefill_attend(sf_context* ctx, const sf_ct* const* probs, int n_probs, const sf_kvcache* cache,
                            sf_ct** att_out, int att_cap, int* n_att);

/* --- KV-cache attention (kv_attention.hpp:32-109) --------------------------- */
/* AttentionConfig{N = slots, d, H, n0, n_max}; validate_attention_config */
sf_status sf_kv_create(sf_context* ctx, int d, int H, int n0, int n_max, sf_kvcache** out);
sf_kvcache* sf_kv_retain(sf_kvcache* kv);
void sf_kv_release(sf_kvcache* kv);
/* n_prime, #k cts, #groups, variants per group */
sf_status sf_kv_info(const sf_kvcache* kv, int* n_prime, int* n_k, int* n_groups, int* n_variants);
/* which = 0: K ct idx; which = 1: V handle (group g, variant index idx) */
sf_status sf_kv_get(const sf_kvcache* kv, int which, int g, int idx, sf_ct** out);
/* build a cache directly from ciphertexts (the reference tests' direct_cache):
 * k_cts[n_k], v_cts[n_groups * variants] */
sf_status sf_kv_from_cts(sf_context* ctx, int d, int H, int n0, int n_max, int n_prime, const sf_ct* const* k_cts,
                         int n_k, const sf_ct* const* v_cts, int n_groups, sf_kvcache** out);
/* rope_apply (kv_attention.cpp:111-117 -> fused_extract Rope, vmm.cpp:85-100) */
sf_status sf_rope_apply(sf_context* ctx, const sf_ct* x, int d, int H, long long position, double base,
                        sf_ct** out);
/* encode + upload (stream-ordered, no host wait) the RoPE plaintexts that
 * sf_rope_apply will use for an input interleaved at `offset` with `level` at
 * `position`: a decode loop issues it for the next token while the current one
 * runs, taking the host encode off the token's critical path. No ledger charge. */
sf_status sf_rope_prepare(sf_context* ctx, int d, int H, int offset, int level, long long position, double base);
/* fused_extract with a mask successor (vmm.cpp:102-108); coeff may be NULL */
sf_status sf_fused_extract_mask(sf_context* ctx, const sf_ct* x, const double* coeff, sf_ct** out);
sf_status sf_k_append(sf_context* ctx, const sf_kvcache* cache, const sf_ct* k_new, sf_kvcache** out);
/* parts_out receives d/H handles */
sf_status sf_make_v_pieces(sf_context* ctx, const sf_kvcache* cache, const sf_ct* v_open, int position,
                           sf_ct** parts_out);
sf_status sf_v_append(sf_context* ctx, const sf_kvcache* cache, const sf_ct* const* parts, int n_parts,
                      sf_kvcache** out);
/* maps_out must hold ceil(n_prime / (N/H)) handles */
sf_status sf_qk_dot(sf_context* ctx, const sf_ct* q, const sf_kvcache* cache, sf_ct** maps_out, int* n_maps);
sf_status sf_softmax_times_v(sf_context* ctx, const sf_ct* const* probs, int n_probs, const sf_kvcache* cache,
                             sf_ct** out);

/* --- sharded hot path (one process per GPU) ------------------
 * Each rank computes its share (VMM giant steps g2 = rank mod world; QK^T key
 * ciphertexts j = rank mod world; Score*V (group, variant) pairs by index mod
 * world), the partial ciphertexts are exchanged (all-gather over NVLink) and
 * summed mod q with sf_sum_partials, then the replicated tail runs.
 * Modular sums are exact: the result is bit-identical to world = 1. */
sf_status sf_vmm_partial(sf_context* ctx, const sf_ct* x, const sf_vmm_plan* plan, int rank, int world,
                         sf_ct** out);
sf_status sf_vmm_finish(sf_context* ctx, const sf_ct* acc, const sf_vmm_plan* plan, int mask_output, sf_ct** out);
sf_status sf_qk_dot_partial(sf_context* ctx, const sf_ct* q, const sf_kvcache* cache, int rank, int world,
                            sf_ct** maps_out, int* n_maps);
/* Score*V partial = the rank's share of the baby-step / giant-step product
 * sum (whole giant groups G mod 8 with (G mod 8) mod world ==
 * rank), one relinearised ciphertext one level below the maps. finish sums the
 * n ranks' partials, folds the lanes and masks (kv_attention.cpp:227-238). */
sf_status sf_softmax_times_v_partial(sf_context* ctx, const sf_ct* const* probs, int n_probs,
                                     const sf_kvcache* cache, int rank, int world, sf_ct** out);
sf_status sf_softmax_times_v_finish(sf_context* ctx, const sf_ct* const* parts, int n, const sf_kvcache* cache,
                                    sf_ct** out);
sf_status sf_sum_partials(sf_context* ctx, const sf_ct* const* parts, int n, sf_ct** out);
/* multi-VMM of one input (sf_vmm_interleaved_multi) split the same way: one
 * partial accumulator per plan; finish = batched reduce ladders + masks */
sf_status sf_vmm_multi_partial(sf_context* ctx, const sf_ct* x, sf_vmm_plan* const* plans, int k, int rank,
                               int world, sf_ct** outs);
sf_status sf_vmm_multi_finish(sf_context* ctx, const sf_ct* const* accs, sf_vmm_plan* const* plans, int k,
                              int mask_output, sf_ct** outs);
/* Sharded operators with the exchange on the library stream: NCCL (resolved at
 * run time from the process's libnccl.so.2) all-gathers the partials on the
 * context's stream, so partial -> exchange -> mod-add -> tail is one stream of
 * work and a whole sharded step can be captured by sf_graph_begin/end (run the
 * step once eagerly first: the exchange caches each call site's metadata).
 * sf_comm_unique_id (rank 0) fills 128 bytes the caller broadcasts; every
 * rank then calls sf_comm_init with its rank and the world size.
 * Results are bit-identical to the unsharded sf_vmm / sf_qk_dot /
 * sf_softmax_times_v. */
/* Exchange over peer memory instead of NCCL (SURVEY §8(e) "fused P2P"): each
 * rank allocates a symmetric buffer of 2 x cap_words words (sf_p2p_init returns
 * its 64-byte CUDA IPC handle), the caller all-gathers the handles (any
 * transport) and passes world x 64 bytes to sf_p2p_open. The sharded
 * operators then publish their partials into the buffer and ONE kernel per
 * exchange reads every rank's partial over NVLink and sums them mod q --
 * graph-capturable (device-side epochs, release/acquire flags). Takes
 * precedence over sf_comm_init when both are set. */
sf_status sf_p2p_init(sf_context* ctx, int rank, int world, size_t cap_words, uint8_t handle_out[64]);
sf_status sf_p2p_open(sf_context* ctx, const uint8_t* handles, int world);
sf_status sf_p2p_destroy(sf_context* ctx);
sf_status sf_comm_unique_id(uint8_t id_out[128]);
sf_status sf_comm_init(sf_context* ctx, const uint8_t id[128], int rank, int world);
sf_status sf_comm_destroy(sf_context* ctx);
sf_status sf_vmm_sharded(sf_context* ctx, const sf_ct* x, const sf_vmm_plan* plan, int mask_output, sf_ct** out);
sf_status sf_vmm_multi_sharded(sf_context* ctx, const sf_ct* x, sf_vmm_plan* const* plans, int k, int mask_output,
                               sf_ct** outs);
sf_status sf_qk_dot_sharded(sf_context* ctx, const sf_ct* q, const sf_kvcache* cache, sf_ct** maps_out,
                            int* n_maps);
sf_status sf_softmax_times_v_sharded(sf_context* ctx, const sf_ct* const* probs, int n_probs,
                                     const sf_kvcache* cache, sf_ct** out);
/* device words of a ciphertext for peer/NCCL exchange: c0 and c1 each
 * (level+1)*n words; the view stays valid while the handle is alive */
sf_status sf_ct_device_view(const sf_ct* ct, uint64_t** c0, uint64_t** c1, size_t* words_per_poly);
/* new ciphertext from device words (copied on the context stream) */
sf_status sf_ct_from_device(sf_context* ctx, const uint64_t* c0, const uint64_t* c1, int level, double scale,
                            int is_zero, const sf_layout* layout, sf_ct** out);

/* --- device timing of the last enqueued work (CUDA events on the ctx stream) */
sf_status sf_event_record(sf_context* ctx, int slot);
sf_status sf_event_elapsed_ms(sf_context* ctx, int slot_begin, int slot_end, float* ms);
/* number of kernels this context has launched since creation */
long long sf_kernel_launches(const sf_context* ctx);

/* Per-kernel-family live timing: between begin and end, every launch of a
 * family whose bit is set in `mask` is bracketed by CUDA events on the context
 * stream and charged its algorithmic bytes. Families:
 * 0 NTT (both passes of one batched transform), 1 key-switch inner product,
 * 2 ct x pt multiply-accumulate, 3 basis conversion, 4 other elementwise,
 * 5 sampling. end() synchronises and fills SF_PROF_FAMILIES entries. */
#define SF_PROF_FAMILIES 6
sf_status sf_profile_begin(sf_context* ctx, int mask);
sf_status sf_profile_end(sf_context* ctx, double* ms, double* bytes, long long* launches);
/* Radix-2 NTT butterflies each family executed in the last profile window
   (the INT-pipe work measure behind bench.py's int_roofline). */
sf_status sf_profile_butterflies(sf_context* ctx, double* butterflies);
/* ---- CUDA graphs of whole decode steps ----------------------------------------
   Everything the library enqueues between begin and end (on this thread) is
   captured into one graph instead of running; replaying it re-executes every
   kernel of the step on the same device buffers. Handles created during the
   capture stay valid and hold the latest replay's results; inputs are fed by
   sf_ct_refill on handles created before the capture. */
typedef struct sf_graph sf_graph;
sf_status sf_graph_capture_begin(sf_context* ctx);
sf_status sf_graph_capture_end(sf_context* ctx, sf_graph** out);
sf_status sf_graph_launch(sf_context* ctx, sf_graph* g);
long long sf_graph_kernel_launches(const sf_graph* g);
void sf_graph_destroy(sf_graph* g);
/* Overwrite a ciphertext's words from host memory (stream-ordered; pinned host
   memory makes it asynchronous): the input slots of a captured graph. */
sf_status sf_ct_refill(sf_context* ctx, sf_ct* ct, const uint64_t* words);
/* The same copy issued on a side stream, forked from the library stream here:
   it overlaps the work enqueued until sf_ct_stage_wait(slot) joins it (call the
   wait before the ciphertext's first use; inside a capture, before the capture
   ends). Host words must be pinned for the overlap (and stay valid for every
   replay of a captured graph, which re-reads them). Slots 0..63. */
sf_status sf_ct_stage(sf_context* ctx, sf_ct* ct, const uint64_t* words, int slot);
sf_status sf_ct_stage_wait(sf_context* ctx, int slot);
/* Read-back counterpart: ct's words -> pinned host memory [2][limbs][n] on the side
   stream, forked here (ct final at this point), overlapping the work enqueued until
   sf_ct_stage_wait(slot); the host words are valid once the stream is synchronised. */
sf_status sf_ct_stage_out(sf_context* ctx, const sf_ct* ct, uint64_t* words, int slot);

/* Device memory in use (diagnostics): bytes currently allocated by CUDA-graph
   memory nodes on the context's device (outstanding step outputs of live
   graphs) and by the context's stream-ordered pool (live buffers + free lists). */
sf_status sf_mem_stats(sf_context* ctx, size_t* graph_bytes, size_t* pool_bytes);
/* grow the context's stream-ordered pool by `bytes` once (allocate + free): later
 * allocations up to that peak never map new device memory mid-step */
sf_status sf_mem_reserve(sf_context* ctx, size_t bytes);
/* the Score*V giant groups this process owns ((G mod 8) mod world == rank): sf_make_v_pieces
 * builds aligned companions for those only (set automatically by sf_comm_init / sf_p2p_init).
 * Sharded results stay word-identical to the single-device ones; a single-device
 * sf_softmax_times_v on such a process rotates the other giants' variants instead
 * (same decryption, other words) */
sf_status sf_set_value_shard(sf_context* ctx, int rank, int world);
/* switching keys held: count, bytes, and the bytes they would take untruncated
 * (every digit; keys are kept for the digits their levels use) */
sf_status sf_key_stats(sf_context* ctx, int* count, size_t* bytes, size_t* full_bytes);

/* Host-side wall time per internal scope ("name total_us calls" lines), collected
   when SF_HOST_PROF=1 is set in the environment; diagnostics only. */
sf_status sf_host_profile(char* buf, int len, int reset);

#ifdef __cplusplus
}
#endif
#endif /* SF_B200_H */
