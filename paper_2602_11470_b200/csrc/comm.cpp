// Sharded decode-step operators with the exchange on the library stream
// (DESIGN.md §7): NCCL is resolved at run time (dlopen; the process's already
// loaded libnccl -- e.g. torch's -- is preferred) and its all-gather is issued
// on the context stream, so a sharded step -- partial compute, all-gather of
// the partial ciphertexts, GPU mod-add, replicated tail -- is one stream of
// work that a CUDA graph captures whole (no host synchronisation inside).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>

#include "protocols.h"

namespace sf {

namespace {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  if (api.loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy already in the process
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  require(h != nullptr, kInternal, "sharded ops: libnccl.so.2 not found");
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
  require(api.get_unique_id && api.comm_init_rank && api.all_gather && api.comm_destroy, kInternal,
          "sharded ops: incomplete NCCL symbols");
  api.loaded = true;
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    fail(kCuda, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

constexpr size_t kHdr = 4;  // per-ciphertext header words: zero flag, limbs, scale bits, reserved

// All-gather of k ciphertexts from every rank (each rank passes its own k, in
// the same order): returns [rank][i]. Every slot carries a header (zero flag,
// limbs, scale) so the receivers rebuild the metadata; the headers of a call
// site (`tag`) are read back once, eagerly, and cached -- a decode step has the
// same shapes every token -- so later calls (and CUDA-graph captures) run
// without any host synchronisation.
std::vector<std::vector<Ct>> allgather_cts(Context& c, const std::vector<const Ct*>& cts, const std::string& tag) {
  require(c.comm != nullptr, kInvalidTarget, "sharded ops: call sf_comm_init first");
  const size_t n = c.n;
  const int k = (int)cts.size();
  int limbs = 0;
  for (const Ct* x : cts) limbs = std::max(limbs, x->limbs);
  const size_t W = kHdr + 2 * (size_t)limbs * n;  // words per ciphertext slot
  BufPtr send = make_buf(c, (size_t)k * W);
  BufPtr recv = make_buf(c, (size_t)c.world * k * W);
  std::vector<u64>& hdr = c.comm_hdr[tag];
  hdr.assign((size_t)k * kHdr, 0);
  for (int i = 0; i < k; ++i) {
    const Ct& x = *cts[i];
    std::memcpy(&hdr[(size_t)i * kHdr + 2], &x.scale, 8);
    hdr[(size_t)i * kHdr + 0] = x.zero ? 1 : 0;
    hdr[(size_t)i * kHdr + 1] = (u64)x.limbs;
    u64* dst = send->p + (size_t)i * W + kHdr;
    if (x.zero) {
      SF_CUDA(cudaMemsetAsync(dst, 0, 2 * (size_t)limbs * n * 8, c.stream));
    } else {
      SF_CUDA(cudaMemcpyAsync(dst, x.c0(), (size_t)x.limbs * n * 8, cudaMemcpyDeviceToDevice, c.stream));
      SF_CUDA(cudaMemcpyAsync(dst + (size_t)limbs * n, x.c1(c.n), (size_t)x.limbs * n * 8, cudaMemcpyDeviceToDevice,
                              c.stream));
    }
  }
  auto it = c.comm_meta.find(tag);
  const bool cached = it != c.comm_meta.end() && it->second.size() == (size_t)c.world * k * kHdr;
  if (!cached) {  // first (eager) call of this site: ship the headers too
    require(!c.capturing, kInvalidTarget, "sharded ops: run the step once eagerly before capturing it");
    for (int i = 0; i < k; ++i)
      SF_CUDA(cudaMemcpyAsync(send->p + (size_t)i * W, hdr.data() + (size_t)i * kHdr, kHdr * 8,
                              cudaMemcpyHostToDevice, c.stream));
  }
  nccl_check(nccl().all_gather(send->p, recv->p, (size_t)k * W, ncclUint64, (ncclComm_t)c.comm, c.stream),
             "ncclAllGather");
  if (!cached) {
    std::vector<u64> meta((size_t)c.world * k * kHdr);
    for (int r = 0; r < c.world; ++r)
      for (int i = 0; i < k; ++i)
        SF_CUDA(cudaMemcpyAsync(meta.data() + ((size_t)r * k + i) * kHdr, recv->p + ((size_t)r * k + i) * W,
                                kHdr * 8, cudaMemcpyDeviceToHost, c.stream));
    SF_CUDA(cudaStreamSynchronize(c.stream));
    it = c.comm_meta.insert_or_assign(tag, std::move(meta)).first;
  }
  const std::vector<u64>& meta = it->second;
  std::vector<std::vector<Ct>> out(c.world);
  for (int r = 0; r < c.world; ++r)
    for (int i = 0; i < k; ++i) {
      const u64* m = meta.data() + ((size_t)r * k + i) * kHdr;
      double scale;
      std::memcpy(&scale, &m[2], 8);
      const int lb = (int)m[1];
      if (r == c.rank) {  // own slots: the cached shape must still hold
        require(lb == cts[i]->limbs && (m[0] != 0) == cts[i]->zero, kInternal,
                "sharded ops: step shape changed since the metadata was cached (" + tag + ")");
        out[r].push_back(*cts[i]);
        continue;
      }
      if (m[0]) {
        Ct z = zeros(c, lb - 1);
        z.scale = scale;
        z.layout = cts[i]->layout;
        out[r].push_back(z);
        continue;
      }
      Ct y = alloc_ct(c, lb, scale);
      y.layout = cts[i]->layout;  // layouts are a function of the protocol, identical on every rank
      const u64* src = recv->p + ((size_t)r * k + i) * W + kHdr;
      SF_CUDA(cudaMemcpyAsync(y.c0(), src, (size_t)lb * n * 8, cudaMemcpyDeviceToDevice, c.stream));
      SF_CUDA(cudaMemcpyAsync(y.c1(c.n), src + (size_t)limbs * n, (size_t)lb * n * 8, cudaMemcpyDeviceToDevice,
                              c.stream));
      out[r].push_back(y);
    }
  return out;
}

}  // namespace

static void rank_world(Context& c, int& rank, int& world) {
  if (c.p2p) {
    p2p_rank_world(c, rank, world);
    return;
  }
  require(c.comm != nullptr, kInvalidTarget, "sharded ops: initialise an exchange (sf_comm_init or sf_p2p_init)");
  rank = c.rank;
  world = c.world;
}

void comm_unique_id(uint8_t* out) {
  ncclUniqueId id;
  nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
}

void comm_init(Context& c, const uint8_t* id_bytes, int rank, int world) {
  require(world >= 1 && rank >= 0 && rank < world, kInvalidTarget, "comm_init: bad rank/world");
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof id);
  ncclComm_t comm;
  SF_CUDA(cudaSetDevice(c.device));
  nccl_check(nccl().comm_init_rank(&comm, world, id, rank), "ncclCommInitRank");
  c.comm = comm;
  c.rank = rank;
  c.world = world;
  c.sv_rank = rank;
  c.sv_world = world;
}

void comm_destroy(Context& c) {
  if (c.comm) nccl().comm_destroy((ncclComm_t)c.comm);
  c.comm = nullptr;
}

// rank / world of the active exchange: peer memory (p2p.cu) when initialised, else NCCL
static void rank_world(Context& c, int& rank, int& world);

Ct vmm_sharded(Context& c, const Ct& x, VmmPlan& plan, bool mask_output) {
  SF_HPROF("vmm_sharded");
  int rank, world;
  rank_world(c, rank, world);
  Ct part = vmm_partial(c, x, plan, rank, world);
  char tag[64];
  std::snprintf(tag, sizeof tag, "vmm:%p", (const void*)&plan);
  if (c.p2p) return vmm_finish(c, p2p_sum_cts(c, {&part}, tag)[0], plan, mask_output);
  auto got = allgather_cts(c, {&part}, tag);
  std::vector<const Ct*> ps;
  for (int r = 0; r < c.world; ++r) ps.push_back(&got[r][0]);
  return vmm_finish(c, sum_partials(c, ps), plan, mask_output);
}

std::vector<Ct> vmm_multi_sharded(Context& c, const Ct& x, const std::vector<VmmPlan*>& plans, bool mask_output) {
  SF_HPROF("vmm_multi_sharded");
  int rank, world;
  rank_world(c, rank, world);
  std::vector<Ct> parts = vmm_multi_partial(c, x, plans, rank, world);
  std::vector<const Ct*> pp;
  for (auto& p : parts) pp.push_back(&p);
  char tag[64];
  std::snprintf(tag, sizeof tag, "vmm_multi:%p", (const void*)plans[0]);
  if (c.p2p) return vmm_multi_finish(c, p2p_sum_cts(c, pp, tag), plans, mask_output);
  auto got = allgather_cts(c, pp, tag);
  std::vector<Ct> accs;
  for (size_t i = 0; i < parts.size(); ++i) {
    std::vector<const Ct*> ps;
    for (int r = 0; r < c.world; ++r) ps.push_back(&got[r][i]);
    accs.push_back(sum_partials(c, ps));
  }
  return vmm_multi_finish(c, accs, plans, mask_output);
}

std::vector<Ct> qk_dot_sharded(Context& c, const Ct& q, const KV& cache) {
  SF_HPROF("qk_dot_sharded");
  int rank, world;
  rank_world(c, rank, world);
  std::vector<Ct> maps = qk_dot_partial(c, q, cache, rank, world);
  std::vector<const Ct*> mp;
  for (auto& m : maps) mp.push_back(&m);
  if (c.p2p) return p2p_sum_cts(c, mp, "qk:" + std::to_string(cache.n_prime));
  auto got = allgather_cts(c, mp, "qk:" + std::to_string(cache.n_prime));
  std::vector<Ct> out;
  for (size_t m = 0; m < maps.size(); ++m) {
    std::vector<const Ct*> ps;
    for (int r = 0; r < c.world; ++r) ps.push_back(&got[r][m]);
    out.push_back(sum_partials(c, ps));
  }
  return out;
}

Ct softmax_times_v_sharded(Context& c, const std::vector<Ct>& probs, const KV& cache) {
  SF_HPROF("softmax_times_v_sharded");
  int rank, world;
  rank_world(c, rank, world);
  Ct part = softmax_times_v_partial(c, probs, cache, rank, world);
  if (c.p2p) {  // the parts' sum over peer memory; finish charges the exchange additions once
    std::vector<int> live;
    std::vector<Ct> sum = p2p_sum_cts(c, {&part}, "sv:" + std::to_string(cache.n_prime), false, &live);
    if (live[0] > 1) c.ledger.add(live[0] - 1);
    return softmax_times_v_finish(c, {&sum[0]}, cache);
  }
  auto got = allgather_cts(c, {&part}, "sv:" + std::to_string(cache.n_prime));
  std::vector<const Ct*> pp;
  for (int r = 0; r < c.world; ++r) pp.push_back(&got[r][0]);
  return softmax_times_v_finish(c, pp, cache);
}

}  // namespace sf
