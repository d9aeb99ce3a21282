// Peer-memory exchange for the sharded operators (SURVEY §8(e)
// "fused P2P kernel"): instead of an NCCL all-gather followed by a separate
// mod-q add, every rank publishes its partial ciphertexts into a symmetric
// buffer and ONE reduction kernel reads all ranks' partials straight from
// peer memory (NVLink loads through CUDA IPC mappings) and sums them mod q
// into the local result -- the all-gather and the mod-add in one pass, no
// collective library, no mod-q-unaware ncclSum.
//
// Protocol (all device-side, so a sharded step captured into a CUDA graph
// replays correctly): each rank's region = two data slots + control words
// {flag[2], ack[2], epoch}. Op number e (the local epoch + 1) uses slot
// s = e & 1:
//   begin   wait until ack[s] >= world * ((e - 1) >> 1): every rank has
//           finished reading this slot's previous use;
//   pack    write the headers + words of this rank's partials into slot s;
//   release __threadfence_system(); flag[s] = e (release, system scope);
//   reduce  each CTA waits for flag[s] >= e on every peer (acquire), then
//           sums the peers' words mod q_limb into the outputs;
//   ack     atomically bump ack[s] on every peer; epoch = e.
// Every rank issues the same sequence of exchanges (the sharded operators are
// SPMD), so the waits always make progress. With world == 1 the peer is the
// rank itself.
#include <cuda_runtime.h>

#include <cstring>

#include "protocols.h"

namespace sf {

namespace {

constexpr int kMaxRanks = 8;
constexpr int kMaxCts = 16;
constexpr size_t kHdrW = 4;    // zero flag, limbs, scale bits, reserved
constexpr size_t kCtrlW = 16;  // flag[2], ack[2], epoch, padding

struct P2P {
  int rank = 0, world = 1;
  size_t cap = 0;  // words per data slot
  u64* region = nullptr;
  u64* peers[kMaxRanks] = {};
  std::vector<void*> opened;
  std::map<std::string, std::vector<u64>> meta;  // headers of every rank per call site
};

inline void launched(Context& c) {  // count the library's kernels (sf_kernel_launches)
  c.launches.fetch_add(1, std::memory_order_relaxed);
  SF_CUDA(cudaGetLastError());
}

P2P& state(Context& c) {
  require(c.p2p != nullptr, kInvalidTarget, "peer exchange: call sf_p2p_init / sf_p2p_open first");
  return *static_cast<P2P*>(c.p2p);
}

__device__ __forceinline__ u64 ld_acquire_sys(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(u64* p, u64 v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ u64 ld_volatile(const u64* p) {
  u64 v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

struct PackArgs {
  int k = 0;
  size_t cap = 0;
  u64* region = nullptr;
  const u64* c0[kMaxCts];
  const u64* c1[kMaxCts];
  size_t off[kMaxCts];    // word offset of ct j in the slot (its header)
  size_t words[kMaxCts];  // limbs * n (per polynomial); 0 for a zero partial
  size_t pad[kMaxCts];    // the slot's per-polynomial width (max limbs * n)
  u64 hdr[kMaxCts][kHdrW];
};

struct ReduceArgs {
  int k = 0, world = 1, n = 0;
  size_t cap = 0, pw = 0;  // pw: per-polynomial width of every slot
  const u64* peers[kMaxRanks];
  u64* out0[kMaxCts];
  u64* out1[kMaxCts];
  size_t off[kMaxCts];
  size_t words[kMaxCts];  // limbs * n of the published polynomials
};

__device__ __forceinline__ u64* ctrl(u64* region, size_t cap) { return region + 2 * cap; }

__global__ void p2p_begin_kernel(u64* region, size_t cap, int world) {
  u64* cw = ctrl(region, cap);
  const u64 e = ld_volatile(cw + 4) + 1, s = e & 1;
  const u64 need = (u64)world * ((e - 1) >> 1);
  while (ld_acquire_sys(cw + 2 + s) < need) __nanosleep(64);
}

__global__ void p2p_pack_kernel(PackArgs A) {
  const u64 e = ld_volatile(ctrl(A.region, A.cap) + 4) + 1;
  u64* slot = A.region + (e & 1) * A.cap;
  const int j = blockIdx.y;
  u64* dst = slot + A.off[j];
  if (blockIdx.x == 0 && threadIdx.x < kHdrW) dst[threadIdx.x] = A.hdr[j][threadIdx.x];
  const size_t w = A.words[j], pw = A.pad[j];
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < pw; i += (size_t)gridDim.x * blockDim.x) {
    dst[kHdrW + i] = i < w ? A.c0[j][i] : 0;
    dst[kHdrW + pw + i] = i < w ? A.c1[j][i] : 0;
  }
}

__global__ void p2p_release_kernel(u64* region, size_t cap) {
  u64* cw = ctrl(region, cap);
  const u64 e = ld_volatile(cw + 4) + 1;
  __threadfence_system();
  st_release_sys(cw + (e & 1), e);
}

__device__ __forceinline__ ulonglong2 ld_volatile2(const u64* p) {
  ulonglong2 v;
  asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

// One thread per PAIR of words (16-byte peer loads over NVLink): the slot
// layout keeps every polynomial at an even word offset (header 4 words,
// widths limbs*n), and a pair never straddles a limb (n is even).
__global__ void p2p_reduce_kernel(ReduceArgs A, const u64* Q, u64* own_region) {
  const u64 e = ld_volatile(ctrl(own_region, A.cap) + 4) + 1, s = e & 1;
  if (threadIdx.x == 0)
    for (int r = 0; r < A.world; ++r)
      while (ld_acquire_sys(ctrl(const_cast<u64*>(A.peers[r]), A.cap) + s) < e) __nanosleep(64);
  __syncthreads();
  const int j = blockIdx.y;
  const size_t w2 = A.words[j] >> 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < 2 * w2; i += (size_t)gridDim.x * blockDim.x) {
    const int poly = i >= w2;
    const size_t ii = 2 * (i - poly * w2);
    const u64 q = Q[ii / A.n];
    const size_t at = s * A.cap + A.off[j] + kHdrW + poly * A.pw + ii;
    ulonglong2 acc = ld_volatile2(A.peers[0] + at);
    for (int r = 1; r < A.world; ++r) {
      const ulonglong2 v = ld_volatile2(A.peers[r] + at);
      acc.x += v.x;
      acc.x = acc.x >= q ? acc.x - q : acc.x;
      acc.y += v.y;
      acc.y = acc.y >= q ? acc.y - q : acc.y;
    }
    *reinterpret_cast<ulonglong2*>((poly ? A.out1[j] : A.out0[j]) + ii) = acc;
  }
}

// Release our reads of every peer's slot: the fence orders them before the
// system-scope release atomics that let each peer overwrite the slot.
__global__ void p2p_ack_kernel(ReduceArgs A, u64* own_region) {
  u64* cw = ctrl(own_region, A.cap);
  const u64 e = ld_volatile(cw + 4) + 1, s = e & 1;
  __threadfence_system();
  for (int r = 0; r < A.world; ++r) {
    u64* ack = ctrl(const_cast<u64*>(A.peers[r]), A.cap) + 2 + s;
    asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(ack) : "memory");
  }
  cw[4] = e;
}

}  // namespace

void p2p_init(Context& c, int rank, int world, size_t cap_words, uint8_t* handle_out) {
  require(world >= 1 && world <= kMaxRanks && rank >= 0 && rank < world, kInvalidTarget,
          "p2p_init: bad rank/world (at most 8 ranks)");
  require(c.p2p == nullptr, kInvalidTarget, "p2p_init: already initialised");
  auto* p = new P2P;
  p->rank = rank, p->world = world, p->cap = cap_words;
  c.sv_rank = rank, c.sv_world = world;
  SF_CUDA(cudaSetDevice(c.device));
  SF_CUDA(cudaMalloc(&p->region, (2 * cap_words + kCtrlW) * sizeof(u64)));  // plain allocation: IPC-exportable
  SF_CUDA(cudaMemset(p->region, 0, (2 * cap_words + kCtrlW) * sizeof(u64)));
  cudaIpcMemHandle_t h;
  SF_CUDA(cudaIpcGetMemHandle(&h, p->region));
  std::memcpy(handle_out, &h, sizeof h);
  c.p2p = p;
}

void p2p_open(Context& c, const uint8_t* handles) {
  P2P& p = state(c);
  for (int r = 0; r < p.world; ++r) {
    if (r == p.rank) {
      p.peers[r] = p.region;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + (size_t)r * sizeof h, sizeof h);
    void* ptr = nullptr;
    SF_CUDA(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    p.peers[r] = static_cast<u64*>(ptr);
    p.opened.push_back(ptr);
  }
  SF_CUDA(cudaDeviceSynchronize());
}

void p2p_rank_world(Context& c, int& rank, int& world) {
  const P2P& p = state(c);
  rank = p.rank;
  world = p.world;
}

void p2p_destroy(Context& c) {
  if (!c.p2p) return;
  auto* p = static_cast<P2P*>(c.p2p);
  cudaStreamSynchronize(c.stream);
  for (void* ptr : p->opened) cudaIpcCloseMemHandle(ptr);
  cudaFree(p->region);
  delete p;
  c.p2p = nullptr;
}

// Sum over ranks (mod q) of each of the k partial ciphertexts every rank
// passes, in the same order (sum_partials semantics and ledger charge: the
// additions of the live partials); returns the k sums.
std::vector<Ct> p2p_sum_cts(Context& c, const std::vector<const Ct*>& cts, const std::string& tag, bool charge,
                            std::vector<int>* live_out) {
  P2P& p = state(c);
  const int k = (int)cts.size();
  require(k >= 1 && k <= kMaxCts, kShapeMismatch, "peer exchange: 1..16 ciphertexts per call");
  const size_t n = c.n;
  int limbs = 0;
  for (const Ct* x : cts) limbs = std::max(limbs, x->limbs);
  const size_t pw = (size_t)limbs * n;  // every slot's per-polynomial width (same on every rank)
  PackArgs P;
  ReduceArgs R;
  P.k = R.k = k;
  P.cap = R.cap = p.cap;
  P.region = p.region;
  R.world = p.world;
  R.n = (int)n;
  R.pw = pw;
  for (int r = 0; r < p.world; ++r) R.peers[r] = p.peers[r];
  size_t off = 0;
  for (int j = 0; j < k; ++j) {
    const Ct& x = *cts[j];
    P.off[j] = R.off[j] = off;
    P.c0[j] = x.zero ? nullptr : x.c0();
    P.c1[j] = x.zero ? nullptr : x.c1(c.n);
    P.words[j] = x.zero ? 0 : (size_t)x.limbs * n;
    P.pad[j] = pw;
    P.hdr[j][0] = x.zero ? 1 : 0;
    P.hdr[j][1] = (u64)x.limbs;
    std::memcpy(&P.hdr[j][2], &x.scale, 8);
    P.hdr[j][3] = pw;
    off += kHdrW + 2 * pw;
  }
  require(off <= p.cap, kShapeMismatch, "peer exchange: partials exceed the symmetric buffer (raise cap_words)");
  auto it = p.meta.find(tag);
  const bool cached = it != p.meta.end() && it->second.size() == (size_t)p.world * k * kHdrW;
  require(cached || !c.capturing, kInvalidTarget, "peer exchange: run the step once eagerly before capturing it");
  // outputs at the own partials' shapes (SPMD: every rank's partial j has the same limbs)
  std::vector<Ct> out(k);
  for (int j = 0; j < k; ++j) {
    out[j] = alloc_ct(c, cts[j]->limbs, cts[j]->scale);
    R.out0[j] = out[j].c0();
    R.out1[j] = out[j].c1(c.n);
    R.words[j] = (size_t)cts[j]->limbs * n;
  }
  p2p_begin_kernel<<<1, 1, 0, c.stream>>>(p.region, p.cap, p.world);
  launched(c);
  {
    const unsigned gx = (unsigned)std::max<size_t>(1, std::min<size_t>(148, (pw + 255) / 256));
    p2p_pack_kernel<<<dim3(gx, k), 256, 0, c.stream>>>(P);
    launched(c);
  }
  p2p_release_kernel<<<1, 1, 0, c.stream>>>(p.region, p.cap);
  launched(c);
  {
    const unsigned gx = (unsigned)std::max<size_t>(1, std::min<size_t>(148 * 4, (pw + 255) / 256));
    p2p_reduce_kernel<<<dim3(gx, k), 256, 0, c.stream>>>(R, c.tabs.q, p.region);
    launched(c);
  }
  if (!cached) {  // headers of every rank, read from the peers' slots before the ack releases them
    SF_CUDA(cudaStreamSynchronize(c.stream));
    u64 e = 0;
    SF_CUDA(cudaMemcpy(&e, p.region + 2 * p.cap + 4, 8, cudaMemcpyDeviceToHost));
    const u64 s = (e + 1) & 1;
    std::vector<u64> meta((size_t)p.world * k * kHdrW);
    for (int r = 0; r < p.world; ++r)
      for (int j = 0; j < k; ++j)
        SF_CUDA(cudaMemcpy(meta.data() + ((size_t)r * k + j) * kHdrW, p.peers[r] + s * p.cap + P.off[j],
                           kHdrW * 8, cudaMemcpyDeviceToHost));
    it = p.meta.insert_or_assign(tag, std::move(meta)).first;
  }
  p2p_ack_kernel<<<1, 1, 0, c.stream>>>(R, p.region);
  launched(c);
  const std::vector<u64>& meta = it->second;
  for (int j = 0; j < k; ++j) {
    int live = 0;
    double sc = 0.0;
    for (int r = 0; r < p.world; ++r) {
      const u64* m = meta.data() + ((size_t)r * k + j) * kHdrW;
      if (r == p.rank)
        require((m[0] != 0) == cts[j]->zero && (int)m[1] == cts[j]->limbs && m[3] == pw, kInternal,
                "peer exchange: step shape changed since the metadata was cached (" + tag + ")");
      require((int)m[1] == cts[j]->limbs && m[3] == pw, kShapeMismatch, "peer exchange: partial shapes differ");
      if (m[0]) continue;
      double v;
      std::memcpy(&v, &m[2], 8);
      if (live == 0) sc = v;
      ++live;
    }
    if (charge && live > 1) c.ledger.add(live - 1);  // sum_partials' additions
    if (live_out) live_out->push_back(live);
    if (live == 0) {
      Ct z = *cts[j];
      out[j] = z;
      continue;
    }
    out[j].scale = sc;
    out[j].layout = cts[j]->layout;
  }
  return out;
}

}  // namespace sf
