// Packed HE-VMM and KV-cache attention over the GPU evaluator.
//
// The op sequences restate the reference algorithms (file:line cited per
// function) and charge the ledger exactly as the reference does; the CKKS
// arithmetic underneath is bit-identical to the CPU oracle running the same
// sequence (oracle/protocols.py over oracle/ckks.py).
#include "protocols.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "batch.cuh"

namespace sf {

// ct (.) mask with the mask plaintext encoded once per (key, limb count) and
// kept resident: numerically identical to mul_plain (same encode, same scale
// q_top), without re-running the host FFT every decode step.
static Ct mul_plain_cached(Context& c, const Ct& a, const std::string& key, const std::vector<double>& slots) {
  SF_HPROF("mul_plain_cached");
  check_ct(c, a, "mul_plain");
  require(a.level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
  Pt p = cached_pt(c, key, slots.data(), (double)c.primes[a.limbs - 1], a.limbs);
  return mac_plain(c, {&a}, {&p});
}

// ============================================================== VMM (vmm.cpp)

BsgsSplit bsgs_split(long long k) {  // vmm.cpp:10-28
  require(k >= 1, kShapeMismatch, "bsgs_split: k must be >= 1");
  long long b = (long long)std::sqrt((double)k);
  while (b * b < k) ++b;
  while (b > 1 && (b - 1) * (b - 1) >= k) --b;
  return {(int)b, (int)((k + b - 1) / b)};
}

VmmShape vmm_shape(int N, int rows, int cols, int tau_in, int tau_out) {  // vmm.cpp:135-153
  VmmShape s;
  s.N = N;
  s.d_in = padded_dim(rows);
  s.d_out = padded_dim(cols);
  require(s.d_in <= N && s.d_out <= N, kShapeMismatch, "vmm_interleaved: padded dimension exceeds N");
  s.t_in = N / s.d_in;
  s.t_out = N / s.d_out;
  s.k = std::max<long long>((long long)s.d_in * s.d_out / N, 1);
  s.alpha_up = std::max(1, s.t_out / s.t_in);
  s.ladder_T = std::max(s.t_in, s.t_out);
  require(tau_in >= 0 && tau_in < s.t_in, kShapeMismatch, "vmm_interleaved: input offset out of range");
  require(tau_out >= 0 && tau_out < s.t_out, kShapeMismatch, "vmm_interleaved: output offset out of range");
  s.tau_in = tau_in;
  s.tau_out = tau_out;
  s.tau_u = tau_in % s.t_out;
  s.carry = tau_out < s.tau_u ? 1 : 0;
  s.delta = (int)pos_mod(tau_out - s.tau_u, s.t_out);
  return s;
}

void predict_interleaved_cost(int N, int rows, int cols, bool bsgs, bool mask, long long* rot, long long* ctpt,
                              int* depth) {  // vmm.cpp:473-488
  const int d_in = padded_dim(rows), d_out = padded_dim(cols);
  const long long k = std::max<long long>((long long)d_in * d_out / N, 1);
  long long r = log2_exact(N / d_in) + log2_exact(N / d_out);
  if (bsgs) {
    const auto bg = bsgs_split(k);
    r += (bg.baby - 1) + (bg.giant - 1);
  } else {
    r += k - 1;
  }
  *rot = r;
  *ctpt = k + (mask ? 1 : 0);
  *depth = 1 + (mask ? 1 : 0);
}

// Generalised interleaved diagonal g at slot j of the pre-giant frame
// (vmm.cpp:159-168; Appendix B).
static double diag_value(const VmmShape& s, const std::function<double(int, int)>& w, long long g, long long j) {
  const long long N = s.N;
  const long long i0 = pos_mod(j + g * s.t_in * s.t_out - s.tau_in, N);
  const int row = (int)((i0 / s.t_in + (i0 % s.t_in) * s.alpha_up) % s.d_in);
  const long long rel = pos_mod(j - s.tau_u, N);
  const long long u = rel % s.t_out;
  const long long within = u / s.t_in + (u % s.t_in) * s.alpha_up;
  if (g * s.t_out + within >= s.d_in) return 0.0;
  const int col = (int)((rel / s.t_out + s.carry) % s.d_out);
  return w(row, col);
}

const std::vector<Pt>& VmmPlan::diagonals(int limbs) {
  auto it = pts.find(limbs);
  if (it != pts.end()) return it->second;
  Context& c = *ctx;
  const long long unit = (long long)s.t_in * s.t_out;
  const double scale = (double)c.primes[limbs - 1];  // scale-preserving ct-pt
  auto gen = [&](int g, double* slots) {
    // BSGS diagonals are pre-shifted by their giant step (vmm.cpp:170-175, 217)
    const long long shift = bsgs ? (long long)(g / bg.baby) * bg.baby * unit : 0;
    if (batch) {  // vmm.cpp:426-433: p[i] = W[(e + j) mod d][e], e = ((i - pre) mod N) / t
      const int d = s.d_in, t = s.t_in;
      for (int i = 0; i < s.N; ++i) {
        const int e = (int)(pos_mod(i - shift, s.N) / t);
        slots[i] = w((e + g) % d, e);
      }
      return;
    }
    for (int i = 0; i < s.N; ++i) slots[i] = diag_value(s, w, g, pos_mod(i - shift, s.N));
  };
  return pts.emplace(limbs, encode_many(c, gen, (int)s.k, scale, limbs)).first->second;
}

std::unique_ptr<VmmPlan> make_vmm_plan(Context& c, const double* W, int rows, int cols, int level, int in_offset,
                                       int out_offset, bool bsgs, bool encode) {
  require(rows > 0 && cols > 0, kShapeMismatch, "vmm plan: empty weight");
  require(level >= 1 && level <= c.L, kInvalidTarget, "vmm plan: level must be in [1, L]");
  auto p = std::make_unique<VmmPlan>();
  p->ctx = &c;
  p->rows = rows;
  p->cols = cols;
  p->level = level;
  p->bsgs = bsgs;
  p->s = vmm_shape(c.slots, rows, cols, in_offset, out_offset);
  p->bg = bsgs ? bsgs_split(p->s.k) : BsgsSplit{1, (int)p->s.k};
  if (W) {
    p->w_store.assign(W, W + (size_t)rows * cols);
    const double* d = p->w_store.data();
    p->w = [d, rows, cols](int r, int cc) { return (r < rows && cc < cols) ? d[(size_t)r * cols + cc] : 0.0; };
  } else {  // slotforge_cli.cpp:88-92 bench weight
    p->w = [rows, cols](int r, int cc) {
      return (r < rows && cc < cols) ? std::sin(0.001 * ((double)r * 31.0 + cc) + 0.25) : 0.0;
    };
  }
  if (encode) p->diagonals(level + 1);
  return p;
}

static void vmm_check_input(Context& c, const Ct& x, const VmmPlan& plan) {
  SF_HPROF("vmm_check_input");
  require(x.layout && x.layout->kind == LayoutKind::Interleaved, kLayoutMismatch,
          "vmm_interleaved: input must carry an interleaved layout");
  require(!x.layout->deferred_mask, kLayoutMismatch,
          "vmm_interleaved: mask (or fuse) deferred garbage before feeding a VMM");
  require(x.layout->offset == plan.s.tau_in, kLayoutMismatch, "vmm_interleaved: input offset differs from the plan");
  require(x.layout->d == plan.s.d_in, kShapeMismatch,
          "vmm_interleaved: layout d=" + std::to_string(x.layout->d) + " but weights want " +
              std::to_string(plan.s.d_in));
  check_ct(c, x, "vmm_interleaved");
  require(x.level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
}

static std::vector<int> ladder_rots(const VmmShape& s) {  // vmm.cpp:190-193
  std::vector<int> r;
  for (int step = 1; step < s.t_in; step <<= 1) r.push_back(step * (s.ladder_T - 1));
  return r;
}
static std::vector<int> reduce_rots(const VmmShape& s) {  // vmm.cpp:226-230
  std::vector<int> r;
  for (int m = 0; (1 << m) < s.t_out; ++m) r.push_back(((s.delta >> m) & 1) ? -(1 << m) : (1 << m));
  return r;
}

constexpr int kGiantGroups = 8;  // giant-step groups of the BSGS rotation sums
constexpr int kPackGroups = 8;   // key-ct groups of the QK^T pack rotation sums

// Steps 1-2 of vmm.cpp:179-236 for the giant steps this rank owns
// (g2 = rank mod world; world = 1 is the whole VMM): preprocess ladder,
// hoisted babies, the giants' lazy MACs (one rescale each), giant rotations and
// their sum. Work every rank repeats (ladder, babies) is charged on rank 0 only,
// so the ledgers of all ranks sum to the reference's counts.
Ct vmm_partial(Context& c, const Ct& x, VmmPlan& plan, int rank, int world) {
  SF_HPROF("vmm_partial");
  vmm_check_input(c, x, plan);
  require(world >= 1 && rank >= 0 && rank < world, kInvalidTarget, "vmm: bad rank/world");
  const bool lead = rank == 0;
  const VmmShape& s = plan.s;
  const std::vector<Pt>& diag = plan.diagonals(x.limbs);
  Ct stair = fold_steps_batch(c, {&x}, {ladder_rots(s)}, true, lead)[0];  // ladder (vmm.cpp:190-193)
  const long long unit = (long long)s.t_in * s.t_out;
  const int limbs = x.limbs;
  if (!plan.bsgs) {
    std::vector<Ct> xs;
    std::vector<long long> own;
    for (long long g = rank; g < s.k; g += world) own.push_back(g), xs.push_back(rotate(c, stair, (int)(g * unit), false));
    if (own.empty()) return zeros(c, x.level() - 1);
    std::vector<const Ct*> cts;
    std::vector<const Pt*> pts;
    for (size_t i = 0; i < own.size(); ++i) cts.push_back(&xs[i]), pts.push_back(&diag[own[i]]);
    return mac_plain(c, cts, pts);
  }
  const int b = plan.bg.baby, giants = plan.bg.giant;
  std::vector<int> mine;  // whole giant groups r = g2 mod kGiantGroups with r mod world == rank
  for (int g2 = 0; g2 < giants; ++g2)
    if ((g2 % kGiantGroups) % world == rank) mine.push_back(g2);
  if (mine.empty()) return zeros(c, x.level() - 1);
  std::vector<RotJob> jobs;
  for (int g1 = 1; g1 < b; ++g1) jobs.push_back({0, (int)(g1 * unit)});
  std::vector<Ct> baby{stair};
  for (Ct& r : rotate_batch(c, {&stair}, jobs, true, lead)) baby.push_back(std::move(r));
  std::vector<Ct> resc;
  if (!stair.zero && b <= 64 && giants <= 64 && s.k <= 2048 && c.n >= 64) {
    // every owned giant's partial sum in ONE fused MAC launch (babies staged
    // on-chip once, each diagonal streamed once), then one batched rescale
    VmmMacArgs A;
    A.n = c.n;
    A.b = b;
    A.giants = (int)mine.size();
    A.k = (int)s.k;
    for (int g1 = 0; g1 < b; ++g1) A.baby0[g1] = baby[g1].c0(), A.baby1[g1] = baby[g1].c1(c.n);
    for (long long g = 0; g < s.k; ++g) A.pt[g] = diag[g].buf->p;
    std::vector<Ct> partial(mine.size());
    for (size_t i = 0; i < mine.size(); ++i) {
      const int cnt = (int)std::min<long long>(b, s.k - (long long)mine[i] * b);
      c.ledger.ctpt(cnt);
      c.ledger.add(cnt - 1);  // the reference's partial-sum additions (vmm.cpp:214-219)
      partial[i] = alloc_ct(c, limbs, stair.scale * (double)c.primes[limbs - 1]);
      A.gidx[i] = mine[i];
      A.out0[i] = partial[i].c0();
      A.out1[i] = partial[i].c1(c.n);
    }
    b_vmm_mac(c, A, limbs);
    resc = std::move(partial);  // unrescaled (scale * q_top): the group sums rescale
    for (auto& r : resc) r.layout.reset();
  } else {
    for (int g2 : mine) {
      std::vector<const Ct*> cts;
      std::vector<const Pt*> pts;
      for (int g1 = 0; g1 < b && (long long)g2 * b + g1 < s.k; ++g1)
        cts.push_back(&baby[g1]), pts.push_back(&diag[(long long)g2 * b + g1]);
      resc.push_back(mac_plain(c, cts, pts, true, false));
    }
  }
  // giant alignment + sum (vmm.cpp:221-222): one rotation sum per giant group
  // (ModDown once per group instead of once per giant), on the
  // unrescaled partials with the rescale merged into the ModDown: at scale >= 2^80
  // the giant rotations decompose with the wider digits of scaled_digit (§3.6b)
  std::vector<std::vector<SumTerm>> groups;
  std::map<int, int> gpos;
  for (size_t i = 0; i < mine.size(); ++i) {
    const int r = mine[i] % kGiantGroups;
    if (!gpos.count(r)) gpos[r] = (int)groups.size(), groups.emplace_back();
    groups[gpos[r]].push_back({&resc[i], (int)(((long long)mine[i] * b * unit) % c.slots)});
  }
  std::vector<Ct> gs = rot_sum_batch(c, groups, false, true, nullptr, true, scaled_digit(c, limbs));
  std::vector<const Ct*> ap;
  for (auto& a : gs) ap.push_back(&a);
  return sum_cts(c, ap);
}

// Steps 3-4 of vmm.cpp:179-236 on the summed partials: the reduce ladder
// folding each t_out window onto its output offset, then mask or defer.
Ct vmm_finish(Context& c, const Ct& acc_in, VmmPlan& plan, bool mask_output) {
  SF_HPROF("vmm_finish");
  const VmmShape& s = plan.s;
  Ct acc = fold_steps_batch(c, {&acc_in}, {reduce_rots(s)})[0];  // reduce (vmm.cpp:226-230)
  if (mask_output) {
    std::vector<double> mk(c.slots, 0.0);
    for (int i = s.tau_out; i < c.slots; i += s.t_out) mk[i] = 1.0;
    acc = mul_plain_cached(c, acc, "stride:" + std::to_string(s.t_out) + ":" + std::to_string(s.tau_out), mk);
  }
  acc.layout = Layout{LayoutKind::Interleaved, s.d_out, s.t_out, s.tau_out, 1, !mask_output};
  return acc;
}

// The same VMM (one plan) of several independent inputs: identical to separate
// vmm_interleaved calls word for word and in the ledger, with every stage
// batched across the inputs (ladders, hoisted babies, rescales, giant rotation
// sums, reduce ladders, masks) so small rings fill the GPU (the HE-VMM
// throughput configuration, BASELINE configs[0]).
std::vector<Ct> vmm_interleaved_many(Context& c, const std::vector<const Ct*>& xs, VmmPlan& plan, bool mask_output) {
  SF_HPROF("vmm_interleaved_many");
  require(!xs.empty(), kShapeMismatch, "vmm_many: no inputs");
  bool batched = plan.bsgs && !(plan.bg.baby > 64 || plan.bg.giant > 64 || plan.s.k > 2048 || c.n < 64);
  for (const Ct* x : xs) {
    vmm_check_input(c, *x, plan);
    batched = batched && !x->zero && x->limbs == xs[0]->limbs;
  }
  std::vector<Ct> out;
  if (!batched) {
    for (const Ct* x : xs) out.push_back(vmm_interleaved(c, *x, plan, mask_output));
    return out;
  }
  const int B = (int)xs.size();
  const VmmShape& s = plan.s;
  const std::vector<Pt>& diag = plan.diagonals(xs[0]->limbs);
  const long long unit = (long long)s.t_in * s.t_out;
  const int limbs = xs[0]->limbs, b = plan.bg.baby, giants = plan.bg.giant;
  // 1. ladders (vmm.cpp:190-193)
  std::vector<Ct> stair = fold_steps_batch(c, xs, std::vector<std::vector<int>>(B, ladder_rots(s)), true, true);
  // 2. hoisted babies (vmm.cpp:208-209), every input's in one batch
  std::vector<const Ct*> sp;
  for (auto& st : stair) sp.push_back(&st);
  std::vector<RotJob> jobs;
  for (int i = 0; i < B; ++i)
    for (int g1 = 1; g1 < b; ++g1) jobs.push_back({i, (int)(g1 * unit)});
  std::vector<Ct> rots = rotate_batch(c, sp, jobs, true, true);
  // 3. per input: the fused MAC over all giants; then one batched rescale
  std::vector<Ct> partial((size_t)B * giants);
  for (int i = 0; i < B; ++i) {
    VmmMacArgs A;
    A.n = c.n;
    A.b = b;
    A.giants = giants;
    A.k = (int)s.k;
    A.baby0[0] = stair[i].c0(), A.baby1[0] = stair[i].c1(c.n);
    for (int g1 = 1; g1 < b; ++g1) {
      const Ct& r = rots[(size_t)i * (b - 1) + g1 - 1];
      A.baby0[g1] = r.c0(), A.baby1[g1] = r.c1(c.n);
    }
    for (long long g = 0; g < s.k; ++g) A.pt[g] = diag[g].buf->p;
    for (int g2 = 0; g2 < giants; ++g2) {
      const int cnt = (int)std::min<long long>(b, s.k - (long long)g2 * b);
      c.ledger.ctpt(cnt);
      c.ledger.add(cnt - 1);
      Ct& pt = partial[(size_t)i * giants + g2];
      pt = alloc_ct(c, limbs, stair[i].scale * (double)c.primes[limbs - 1]);
      A.gidx[g2] = g2;
      A.out0[g2] = pt.c0();
      A.out1[g2] = pt.c1(c.n);
    }
    b_vmm_mac(c, A, limbs);
  }
  std::vector<Ct> resc = std::move(partial);  // unrescaled: the group sums rescale (§3.6b)
  for (auto& r : resc) r.layout.reset();
  // 4. giant alignment + sum: every input's groups in one batch
  std::vector<std::vector<SumTerm>> groups;
  std::vector<int> gowner;
  for (int i = 0; i < B; ++i)
    for (int r = 0; r < std::min(kGiantGroups, giants); ++r) {
      groups.emplace_back();
      gowner.push_back(i);
      for (int g2 = r; g2 < giants; g2 += kGiantGroups)
        groups.back().push_back({&resc[(size_t)i * giants + g2], (int)(((long long)g2 * b * unit) % c.slots)});
    }
  std::vector<Ct> gs = rot_sum_batch(c, groups, false, true, nullptr, true, scaled_digit(c, limbs));
  std::vector<Ct> acc;
  for (int i = 0; i < B; ++i) {
    std::vector<const Ct*> ap;
    for (size_t k = 0; k < gs.size(); ++k)
      if (gowner[k] == i) ap.push_back(&gs[k]);
    acc.push_back(sum_cts(c, ap));
  }
  // 5-6. reduce ladders and masks, batched (the multi-plan finish with one plan per input)
  return vmm_multi_finish(c, acc, std::vector<VmmPlan*>(B, &plan), mask_output);
}

// Several VMMs of the SAME input x (the decode step's Q/K/V and gate/up
// projections): identical to separate vmm_interleaved calls word for word and
// in the ledger (each call's charges are applied), but the input-only work --
// the preprocess ladder and the hoisted baby steps, which depend on x, t_in,
// t_out and b alone -- runs once, and the per-call work (MACs, rescales, giant
// rotation sums, reduce ladders, masks) runs as batched launches.
static bool vmm_multi_shares(Context& c, const Ct& x, const std::vector<VmmPlan*>& plans) {
  require(!plans.empty(), kShapeMismatch, "vmm_multi: no plans");
  bool share = !x.zero;
  for (VmmPlan* p : plans) {
    vmm_check_input(c, x, *p);
    const VmmShape &a = p->s, &b0 = plans[0]->s;
    share = share && p->bsgs && a.t_in == b0.t_in && a.t_out == b0.t_out && a.ladder_T == b0.ladder_T &&
            a.k == b0.k && p->bg.baby == plans[0]->bg.baby && p->bg.giant == plans[0]->bg.giant &&
            !(p->bg.baby > 64 || p->bg.giant > 64 || a.k > 2048 || c.n < 64);
  }
  return share;
}

// Steps 1-4 of every call (ladder, babies, MACs, giant rotation sums) for the
// giant groups rank owns; the ladder and babies are input-only (shared by the
// calls, replicated on every rank and charged on rank 0).
std::vector<Ct> vmm_multi_partial(Context& c, const Ct& x, const std::vector<VmmPlan*>& plans, int rank, int world) {
  SF_HPROF("vmm_multi_partial");
  require(world >= 1 && rank >= 0 && rank < world, kInvalidTarget, "vmm: bad rank/world");
  const int P = (int)plans.size();
  std::vector<Ct> out;
  if (!vmm_multi_shares(c, x, plans)) {
    for (VmmPlan* p : plans) out.push_back(vmm_partial(c, x, *p, rank, world));
    return out;
  }
  const bool lead = rank == 0;
  const VmmShape& s0 = plans[0]->s;
  const long long unit = (long long)s0.t_in * s0.t_out;
  const int limbs = x.limbs, b = plans[0]->bg.baby, giants = plans[0]->bg.giant;
  // 1. ladder (vmm.cpp:190-193), charged once per call
  const std::vector<int> lr = ladder_rots(s0);
  if (lead) {
    for (int r : lr)
      if (pos_mod(r, c.slots) != 0) c.ledger.rot(false, P);
    c.ledger.add((long long)P * lr.size());
  }
  Ct stair = fold_steps_batch(c, {&x}, {lr}, false)[0];
  // 2. hoisted babies (vmm.cpp:208-209), charged once per call
  std::vector<RotJob> jobs;
  for (int g1 = 1; g1 < b; ++g1) {
    jobs.push_back({0, (int)(g1 * unit)});
    if (lead && pos_mod(g1 * unit, c.slots) != 0) c.ledger.rot(true, P);
  }
  std::vector<int> mine;  // whole giant groups r = g2 mod kGiantGroups with r mod world == rank
  for (int g2 = 0; g2 < giants; ++g2)
    if ((g2 % kGiantGroups) % world == rank) mine.push_back(g2);
  if (mine.empty()) {
    for (int pi = 0; pi < P; ++pi) out.push_back(zeros(c, x.level() - 1));
    return out;
  }
  std::vector<Ct> baby{stair};
  for (Ct& r : rotate_batch(c, {&stair}, jobs, true, false)) baby.push_back(std::move(r));
  // 3. every call's fused MAC over the owned giants, then one batched rescale
  const int G = (int)mine.size();
  std::vector<Ct> partial((size_t)P * G);
  for (int pi = 0; pi < P; ++pi) {
    const std::vector<Pt>& diag = plans[pi]->diagonals(limbs);
    VmmMacArgs A;
    A.n = c.n;
    A.b = b;
    A.giants = G;
    A.k = (int)s0.k;
    for (int g1 = 0; g1 < b; ++g1) A.baby0[g1] = baby[g1].c0(), A.baby1[g1] = baby[g1].c1(c.n);
    for (long long g = 0; g < s0.k; ++g) A.pt[g] = diag[g].buf->p;
    for (int i = 0; i < G; ++i) {
      const int cnt = (int)std::min<long long>(b, s0.k - (long long)mine[i] * b);
      c.ledger.ctpt(cnt);
      c.ledger.add(cnt - 1);
      Ct& pt = partial[(size_t)pi * G + i];
      pt = alloc_ct(c, limbs, stair.scale * (double)c.primes[limbs - 1]);
      A.gidx[i] = mine[i];
      A.out0[i] = pt.c0();
      A.out1[i] = pt.c1(c.n);
    }
    b_vmm_mac(c, A, limbs);
  }
  std::vector<Ct> resc = std::move(partial);  // unrescaled: the group sums rescale (§3.6b)
  for (auto& r : resc) r.layout.reset();
  // 4. giant alignment + sum: the owned groups of every call in one batch
  std::vector<std::vector<SumTerm>> groups;
  std::vector<int> gowner;
  for (int pi = 0; pi < P; ++pi)
    for (int r = 0; r < std::min(kGiantGroups, giants); ++r) {
      if (r % world != rank) continue;
      groups.emplace_back();
      gowner.push_back(pi);
      for (int i = 0; i < G; ++i)
        if (mine[i] % kGiantGroups == r)
          groups.back().push_back({&resc[(size_t)pi * G + i], (int)(((long long)mine[i] * b * unit) % c.slots)});
    }
  std::vector<Ct> gs = rot_sum_batch(c, groups, false, true, nullptr, true, scaled_digit(c, limbs));
  for (int pi = 0; pi < P; ++pi) {
    std::vector<const Ct*> ap;
    for (size_t i = 0; i < gs.size(); ++i)
      if (gowner[i] == pi) ap.push_back(&gs[i]);
    out.push_back(sum_cts(c, ap));
  }
  return out;
}

// Steps 5-6 of every call on the summed partials: batched reduce ladders, masks.
std::vector<Ct> vmm_multi_finish(Context& c, const std::vector<Ct>& accs, const std::vector<VmmPlan*>& plans,
                                 bool mask_output) {
  SF_HPROF("vmm_multi_finish");
  const int P = (int)plans.size();
  require((int)accs.size() == P, kShapeMismatch, "vmm_multi_finish: one accumulator per plan");
  std::vector<Ct> acc;
  {  // reduce ladders (vmm.cpp:226-230), one batched rotation + addition per step
    std::vector<const Ct*> src;
    std::vector<std::vector<int>> rr;
    for (int pi = 0; pi < P; ++pi) src.push_back(&accs[pi]), rr.push_back(reduce_rots(plans[pi]->s));
    acc = fold_steps_batch(c, src, rr);
  }
  if (mask_output) {  // masks (vmm.cpp:233)
    std::vector<Pt> mk;
    std::vector<const Ct*> xs;
    for (int pi = 0; pi < P; ++pi) {
      const VmmShape& sp = plans[pi]->s;
      std::vector<double> m(c.slots, 0.0);
      for (int i = sp.tau_out; i < c.slots; i += sp.t_out) m[i] = 1.0;
      mk.push_back(cached_pt(c, "stride:" + std::to_string(sp.t_out) + ":" + std::to_string(sp.tau_out), m.data(),
                             (double)c.primes[acc[pi].limbs - 1], acc[pi].limbs));
      xs.push_back(&acc[pi]);
    }
    std::vector<const Pt*> ps;
    for (auto& m : mk) ps.push_back(&m);
    acc = mul_plain_batch(c, xs, ps);
  }
  for (int pi = 0; pi < P; ++pi) {
    const VmmShape& sp = plans[pi]->s;
    acc[pi].layout = Layout{LayoutKind::Interleaved, sp.d_out, sp.t_out, sp.tau_out, 1, !mask_output};
  }
  return acc;
}

// Several VMMs of the SAME input x (the decode step's Q/K/V and gate/up
// projections): identical to separate vmm_interleaved calls word for word and
// in the ledger (each call's charges are applied), but the input-only work --
// the preprocess ladder and the hoisted baby steps, which depend on x, t_in,
// t_out and b alone -- runs once, and the per-call work (MACs, rescales, giant
// rotation sums, reduce ladders, masks) runs as batched launches.
std::vector<Ct> vmm_interleaved_multi(Context& c, const Ct& x, const std::vector<VmmPlan*>& plans, bool mask_output) {
  SF_HPROF("vmm_interleaved_multi");
  if (!vmm_multi_shares(c, x, plans)) {
    std::vector<Ct> out;
    for (VmmPlan* p : plans) out.push_back(vmm_interleaved(c, x, *p, mask_output));
    return out;
  }
  return vmm_multi_finish(c, vmm_multi_partial(c, x, plans, 0, 1), plans, mask_output);
}

// vmm.cpp:179-236: the whole VMM on one GPU.
Ct vmm_interleaved(Context& c, const Ct& x, VmmPlan& plan, bool mask_output) {
  SF_HPROF("vmm_interleaved");
  return vmm_finish(c, vmm_partial(c, x, plan, 0, 1), plan, mask_output);
}

// Sum of per-rank partial results (the exchange's modular reduction; NCCL has
// no mod-q sum). Charges one addition per non-trivial operand beyond the first.
Ct sum_partials(Context& c, const std::vector<const Ct*>& parts) {
  SF_HPROF("sum_partials");
  std::vector<const Ct*> live;
  for (const Ct* p : parts)
    if (!p->zero) live.push_back(p);
  if (live.empty()) return *parts[0];
  return sum_cts(c, live);
}

// ======================================================= attention (kv_attention.cpp)

void validate_attention_config(const AttnCfg& cfg, int N_backend) {  // kv_attention.cpp:80-88
  require(cfg.N == N_backend, kShapeMismatch,
          "attention config N " + std::to_string(cfg.N) + " != backend slot count " + std::to_string(N_backend));
  require(is_pow2(cfg.N) && is_pow2(cfg.d) && is_pow2(cfg.H), kShapeMismatch,
          "attention config: N, d and H must be powers of two");
  require(cfg.H <= cfg.d && cfg.d <= cfg.N, kShapeMismatch, "attention config: need H <= d <= N");
  require(cfg.n0 >= 0 && cfg.n_max >= std::max(cfg.n0, 1), kShapeMismatch,
          "attention config: need 0 <= n0 <= n_max, n_max >= 1");
}

int v_variant_count(const AttnCfg& cfg) { return cfg.H == 1 ? cfg.d_head() : 2 * cfg.d_head() - 1; }
int v_variant_index(const AttnCfg& cfg, int w) {
  const int dh = cfg.d_head();
  if (cfg.H == 1) {
    require(w >= 0 && w < dh, kShapeMismatch, "v_variant_index: merged variant out of range");
    return w;
  }
  require(w > -dh && w < dh, kShapeMismatch, "v_variant_index: variant out of range");
  return w + dh - 1;
}
int v_variant_of(const AttnCfg& cfg, int e, int u_local) {
  const int raw = e - u_local / cfg.t();
  return cfg.H == 1 ? (int)pos_mod(raw, cfg.d_head()) : raw;
}

static void require_clean_interleaved(const Ct& x, const AttnCfg& cfg, int offset, const char* who) {
  SF_HPROF("require_clean_interleaved");
  require(x.layout && x.layout->kind == LayoutKind::Interleaved, kLayoutMismatch,
          std::string(who) + ": input must carry an interleaved layout");
  require(x.layout->d == cfg.d, kShapeMismatch, std::string(who) + ": layout width mismatch");
  require(x.layout->offset == offset, kLayoutMismatch,
          std::string(who) + ": expected slot offset " + std::to_string(offset) + ", got " +
              std::to_string(x.layout->offset));
  require(!x.layout->deferred_mask, kLayoutMismatch, std::string(who) + ": input garbage must be cleared first");
}

static std::vector<double> valid_mask(const Layout& ly, int N) {  // vmm.cpp:45-56
  std::vector<double> m(N, 0.0);
  switch (ly.kind) {
    case LayoutKind::Interleaved:
      for (int i = ly.offset; i < N; i += ly.t) m[i] = 1.0;
      break;
    case LayoutKind::Contiguous:
      for (int i = 0; i < ly.d; ++i) m[i] = 1.0;
      break;
    case LayoutKind::Replicated:
      std::fill(m.begin(), m.end(), 1.0);
      break;
  }
  return m;
}

// The RoPE plaintexts depend on the token position, so a decode stream encodes
// fresh ones every token; keep those of the last few positions only (a graph
// may read cached plaintexts, so nothing is dropped while one is alive).
static void prune_rope_plaintexts(Context& c, long long position) {
  constexpr long long kKeep = 8;
  std::lock_guard<std::mutex> lk(c.mu);
  if (c.live_graphs > 0 || c.capturing) return;
  for (auto it = c.pt_cache.lower_bound("rope:"); it != c.pt_cache.end() && it->first.compare(0, 5, "rope:") == 0;) {
    const long long p = std::atoll(it->first.c_str() + 5);
    if (p < position - kKeep || p > position + kKeep)
      it = c.pt_cache.erase(it);
    else
      ++it;
  }
}

// The three RoPE plaintexts of (layout, limb count, position) (vmm.cpp:66-83),
// encoded once at scale q_top and cached (pruned to recent positions).
static std::vector<Pt> rope_plaintexts(Context& c, const Layout& ly, int limbs, int dh, long long position,
                                       double base) {
  SF_HPROF("rope_plaintexts");
  require(dh > 0 && dh % 2 == 0, kShapeMismatch, "rope_plaintexts: d_head must be positive and even");
  require(limbs > 1, kLevelUnderflow, "mul_plain: no multiplicative level left");
  prune_rope_plaintexts(c, position);
  char key[160];
  std::snprintf(key, sizeof key, "rope:%lld:%d:%d:%d:%d:%a:", position, ly.d, ly.t, ly.offset, dh, base);
  std::vector<Pt> pts(3);
  bool warm = true;
  for (int i = 0; i < 3 && warm; ++i) warm = lookup_pt(c, key + std::to_string(i), limbs, &pts[i]);
  if (warm) return pts;
  const int N = c.slots;
  std::vector<double> p0(N, 0.0), p1(N, 0.0), p2(N, 0.0);
  for (int e = 0; e < ly.d; ++e) {  // vmm.cpp:66-83
    const int pair = (e % dh) / 2;
    const double angle = (double)position * std::pow(base, -2.0 * pair / (double)dh);
    const int i = e * ly.t + ly.offset;
    p0[i] = std::cos(angle);
    if (e % 2 == 0)
      p1[i] = std::sin(angle);
    else
      p2[i] = -std::sin(angle);
  }
  const double* v[3] = {p0.data(), p1.data(), p2.data()};
  for (int i = 0; i < 3; ++i) pts[i] = cached_pt(c, key + std::to_string(i), v[i], (double)c.primes[limbs - 1], limbs);
  return pts;
}

// fused_extract, Rope successor (vmm.cpp:85-100) via rope_apply
// (kv_attention.cpp:111-117): y = x.p0 + Rot(x.p1, -s) + Rot(x.p2, s), s = t.
Ct rope_apply(Context& c, const Ct& x, const AttnCfg& cfg, long long position, double base) {
  SF_HPROF("rope_apply");
  require(x.layout && x.layout->kind == LayoutKind::Interleaved && x.layout->d == cfg.d, kLayoutMismatch,
          "rope_apply: input must be interleaved at the configured width");
  const Layout ly = *x.layout;
  const int dh = cfg.d_head();
  check_ct(c, x, "mul_plain");
  require(x.level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
  const std::vector<Pt> pts = rope_plaintexts(c, ly, x.limbs, dh, position, base);
  const int s = cfg.t();
  // p0 x + Rot(p1 x, -s) + Rot(p2 x, s) as ONE rotation sum of the unrescaled
  // products with the rescale merged into its ModDown: one
  // conversion instead of three rescales and two ModDowns; charged as the
  // reference's 3 mul_plain + 2 rotations + 2 additions
  Ct y;
  if (!x.zero) {
    std::vector<Ct> u = mul_plain_batch(c, {&x, &x, &x}, {&pts[0], &pts[1], &pts[2]}, false, false);
    for (auto& v : u) v.layout.reset();
    y = rot_sum_batch(c, {{{&u[0], 0}, {&u[1], -s}, {&u[2], s}}}, false, false, nullptr, true,
                      scaled_digit(c, x.limbs))[0];  // products at scale >= 2^80: wider digits (§3.6b)
  } else {
    y = zeros(c, x.level() - 1);
  }
  c.ledger.ctpt(3);
  c.ledger.rot(false, 2);
  c.ledger.add(2);
  Layout out = ly;
  out.deferred_mask = false;
  y.layout = out;
  return y;
}

// Encode (and upload, stream-ordered) the RoPE plaintexts rope_apply will use
// for an input of this layout and level at `position`, ahead of time: a decode
// loop calls it for the next token while the current one runs on the GPU, so
// the host encode leaves the token's critical path. No ledger charge.
void rope_prepare(Context& c, const AttnCfg& cfg, int offset, int level, long long position, double base) {
  SF_HPROF("rope_prepare");
  require(level >= 0 && level <= c.L, kInvalidTarget, "rope_prepare: level outside [0, L]");
  Layout ly = make_interleaved(cfg.d, c.slots, offset, cfg.H);
  rope_plaintexts(c, ly, level + 1, cfg.d_head(), position, base);
}

Ct fused_extract_mask(Context& c, const Ct& x, const double* coeff) {  // vmm.cpp:102-108
  require(x.layout.has_value(), kLayoutMismatch, "fused_extract: input must carry a layout");
  std::vector<double> m = valid_mask(*x.layout, c.slots);
  if (coeff)
    for (int i = 0; i < c.slots; ++i) m[i] *= coeff[i];
  Ct y = mul_plain(c, x, m.data());
  Layout out = *x.layout;
  out.deferred_mask = false;
  y.layout = out;
  return y;
}

KV k_append(Context& c, const KV& cache, const Ct& k_new) {  // kv_attention.cpp:131-143
  require(cache.n_prime < cache.cfg.n_max, kCacheFull, "k_append: cache at capacity");
  const int t = cache.cfg.t();
  require_clean_interleaved(k_new, cache.cfg, cache.n_prime % t, "k_append");
  KV out = cache;
  if (cache.n_prime % t == 0)
    out.k.push_back(k_new);
  else
    out.k.back() = add(c, out.k.back(), k_new);
  out.n_prime = cache.n_prime + 1;
  return out;
}

constexpr int kSvGroups = 8;  // Score*V giant groups
static std::vector<Ct> rotate_memo(Context& c, const std::vector<const Ct*>& xs, const std::vector<int>& rs,
                                   const std::vector<char>& keep);
static bool cache_v_zero(const KV& cache, int g, int idx) {
  return g >= (int)cache.v.size() || cache.v[g][idx].zero;
}
// the tracked giant-aligned copy of v[g][idx], or null
static const Ct* aligned_of(const KV& cache, int g, int idx) {
  if (g >= (int)cache.va_ok.size() || idx >= (int)cache.va_ok[g].size() || !cache.va_ok[g][idx]) return nullptr;
  return &cache.va[g][idx];
}

std::vector<Ct> make_v_pieces(Context& c, const KV& cache, const Ct& v_open, int position) {  // :145-163
  const AttnCfg& cfg = cache.cfg;
  require(position >= 0 && position < cfg.n_max, kShapeMismatch, "make_v_pieces: position outside cache capacity");
  require(v_open.layout && v_open.layout->kind == LayoutKind::Interleaved && v_open.layout->d == cfg.d,
          kLayoutMismatch, "make_v_pieces: input must be interleaved at the configured width");
  const int t = cfg.t(), dh = cfg.d_head(), j0 = position % t;
  require(v_open.layout->offset == j0, kLayoutMismatch,
          "make_v_pieces: value ct offset does not match the token position");
  std::vector<Ct> parts;
  parts.reserve(dh);
  std::vector<double> m(c.slots);
  const std::vector<double> valid = valid_mask(*v_open.layout, c.slots);
  Layout out = *v_open.layout;
  out.deferred_mask = false;
  check_ct(c, v_open, "mul_plain");
  require(v_open.level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
  std::vector<Pt> masks;
  for (int e = 0; e < dh; ++e) {  // fused_extract(VcacheMask) with the piece mask (vmm.cpp:102-108)
    char key[96];
    std::snprintf(key, sizeof key, "vpiece:%d:%d:%d:%d:%d", cfg.d, cfg.H, t, e, j0);
    Pt hit;
    if (lookup_pt(c, key, v_open.limbs, &hit)) {  // warm: no host mask synthesis
      masks.push_back(std::move(hit));
      continue;
    }
    std::fill(m.begin(), m.end(), 0.0);
    for (int h = 0; h < cfg.H; ++h) m[(h * dh + e) * t + j0] = 1.0;
    for (int i = 0; i < c.slots; ++i) m[i] *= valid[i];
    masks.push_back(cached_pt(c, key, m.data(), (double)c.primes[v_open.limbs - 1], v_open.limbs));
  }
  std::vector<const Ct*> xs(dh, &v_open);
  std::vector<const Pt*> ps;
  for (auto& p : masks) ps.push_back(&p);
  parts = mul_plain_batch(c, xs, ps);
  for (auto& y : parts) y.layout = out;
  // aligned companions: piece e lands in variant w of giant
  // G = floor(w / B); Rot(piece, G B t) = RS(Rot(mask_e, G B t) (.) Rot(v_open, G B t))
  // and Rot(mask_e, G B t) = mask_{(e - G B) mod d_head} when the valid slots are
  // invariant under a lane-block shift -- one hoisted rotation of v_open per giant
  bool periodic = true;
  for (int i = 0; i < c.slots && periodic; ++i) periodic = valid[i] == valid[(i + t) % c.slots];
  if (periodic && !v_open.zero) {
    const int B = sv_baby(cfg), gt = cfg.group_tokens(), u_local = position % gt;
    std::vector<int> shift(dh), esrc(dh);
    std::vector<RotJob> jobs;
    std::map<int, int> job_of;
    for (int e = 0; e < dh; ++e) {
      const int w = v_variant_of(cfg, e, u_local);
      const int G = w >= 0 ? w / B : -((-w + B - 1) / B);
      // a sharded process builds companions for its own giant groups only (the
      // others' aligned variants are never read here): the appends shard too
      shift[e] = (int)pos_mod(G, kSvGroups) % c.sv_world == c.sv_rank ? G * B * t : 0;
      esrc[e] = (int)pos_mod(e - G * B, dh);
      if (pos_mod(shift[e], c.slots) && !job_of.count(shift[e]))
        job_of[shift[e]] = (int)jobs.size(), jobs.push_back({0, shift[e]});
    }
    std::vector<Ct> rv = rotate_batch(c, {&v_open}, jobs, true, false);
    std::vector<const Ct*> ax;
    std::vector<const Pt*> ap;
    std::vector<int> which;
    for (int e = 0; e < dh; ++e) {
      if (!pos_mod(shift[e], c.slots)) continue;  // giant 0: the piece itself
      ax.push_back(&rv[job_of[shift[e]]]);
      ap.push_back(&masks[esrc[e]]);
      which.push_back(e);
    }
    std::vector<Ct> al = mul_plain_batch(c, ax, ap, false);
    for (size_t k = 0; k < which.size(); ++k) {
      parts[which[k]].aligned = std::make_shared<const Ct>(std::move(al[k]));
      parts[which[k]].aligned_r = shift[which[k]];
    }
  }
  return parts;
}

KV v_append(Context& c, const KV& cache, const std::vector<Ct>& parts) {  // kv_attention.cpp:165-182
  const AttnCfg& cfg = cache.cfg;
  require(cache.n_prime < cfg.n_max, kCacheFull, "v_append: cache at capacity");
  const int dh = cfg.d_head();
  require((int)parts.size() == dh, kShapeMismatch,
          "v_append: expected d/H pieces, got " + std::to_string(parts.size()));
  const int gt = cfg.group_tokens();
  const int g = cache.n_prime / gt;
  const int u_local = cache.n_prime - g * gt;
  KV out = cache;
  if (g == (int)out.v.size()) out.v.emplace_back(v_variant_count(cfg), zeros(c, -1));
  std::vector<int> idx(dh);
  std::vector<const Ct*> a, b;
  for (int e = 0; e < dh; ++e) {  // distinct variant per element: independent additions
    idx[e] = v_variant_index(cfg, v_variant_of(cfg, e, u_local));
    a.push_back(&out.v[g][idx[e]]);
    b.push_back(&parts[e]);
  }
  // giant-aligned variants: aligned' = (aligned, or Rot(V_old)
  // when untracked, or 0 for an empty variant) + the piece's aligned companion
  const int B = sv_baby(cfg), t = cfg.t();
  if ((int)out.va.size() <= g) out.va.resize(g + 1), out.va_ok.resize(g + 1);
  out.va[g].resize(v_variant_count(cfg));
  out.va_ok[g].resize(v_variant_count(cfg), 0);
  std::vector<const Ct*> base_rot;
  std::vector<int> base_r, base_e;
  std::vector<int> r_of(dh, 0);
  for (int e = 0; e < dh; ++e) {
    const int w = v_variant_of(cfg, e, u_local);
    const int G = w >= 0 ? w / B : -((-w + B - 1) / B);
    r_of[e] = G * B * t;
    const Ct* p = &parts[e];
    const bool comp = pos_mod(r_of[e], c.slots) && p->aligned && p->aligned_r == r_of[e] &&
                      p->aligned->limbs == p->limbs && !p->zero;
    if (!comp) {
      out.va_ok[g][idx[e]] = 0;
      r_of[e] = 0;
      continue;
    }
    if (!out.va_ok[g][idx[e]] && !cache_v_zero(cache, g, idx[e]))
      base_rot.push_back(&cache.v[g][idx[e]]), base_r.push_back(r_of[e]), base_e.push_back(e);
  }
  std::vector<Ct> based = rotate_memo(c, base_rot, base_r, std::vector<char>(base_rot.size(), 1));
  std::vector<const Ct*> xa, xb;
  std::vector<int> tgt;
  for (size_t k = 0; k < base_e.size(); ++k) out.va[g][idx[base_e[k]]] = std::move(based[k]), out.va_ok[g][idx[base_e[k]]] = 1;
  for (int e = 0; e < dh; ++e) {
    if (!r_of[e]) continue;
    if (!out.va_ok[g][idx[e]]) {  // empty variant: the companion alone
      out.va[g][idx[e]] = *parts[e].aligned;
      out.va_ok[g][idx[e]] = 1;
      continue;
    }
    xa.push_back(&out.va[g][idx[e]]);
    xb.push_back(parts[e].aligned.get());
    tgt.push_back(idx[e]);
  }
  std::vector<Ct> asum = add_batch(c, xa, xb, false);
  for (size_t k = 0; k < tgt.size(); ++k) out.va[g][tgt[k]] = std::move(asum[k]);
  std::vector<Ct> sums = add_batch(c, a, b);
  for (int e = 0; e < dh; ++e) {
    out.v[g][idx[e]] = std::move(sums[e]);
    out.v[g][idx[e]].aligned.reset();
  }
  return out;
}

static int ceil_div(int a, int b) { return (a + b - 1) / b; }

// kv_attention.cpp:184-214 for the K ciphertexts this rank owns (j = rank
// mod world; world = 1 is the whole QK^T). Every K ciphertext runs the same op
// sequence (mul, fold_within_head 38-41, mask, pack rotation), so each step is
// one batched call over all owned ciphertexts. Returns per-map partial sums
// (trivial zeros for maps this rank has no keys for); the lane replication of
// q (30-34), repeated on every rank, is charged on rank 0 only.
std::vector<Ct> qk_dot_partial(Context& c, const Ct& q, const KV& cache, int rank, int world) {
  SF_HPROF("qk_dot_partial");
  const AttnCfg& cfg = cache.cfg;
  require(cache.n_prime != 0, kCacheEmpty, "qk_dot: no cached keys");
  require_clean_interleaved(q, cfg, 0, "qk_dot");
  require(world >= 1 && rank >= 0 && rank < world, kInvalidTarget, "qk_dot: bad rank/world");
  const int t = cfg.t(), dh = cfg.d_head(), gt = cfg.group_tokens(), N = cfg.N;
  require((int)cache.k.size() == ceil_div(cache.n_prime, t), kShapeMismatch,
          "qk_dot: key ct count does not match n_prime");
  const bool lead = rank == 0;
  std::vector<int> rep;  // replicate_lanes (30-34)
  for (int step = 1; step < t; step <<= 1) rep.push_back(-step);
  Ct q_rep = fold_steps_batch(c, {&q}, {rep}, true, lead)[0];
  std::vector<double> head_mask(N, 0.0);  // ReplicateExtract (layouts.cpp:134-138)
  const int hb = N / cfg.H;
  for (int h = 0; h < cfg.H; ++h)
    for (int i = 0; i < t; ++i) head_mask[h * hb + i] = 1.0;
  std::vector<int> own;  // whole pack groups r = j mod kPackGroups with r mod world == rank
  for (int j = 0; j < (int)cache.k.size(); ++j)
    if ((j % kPackGroups) % world == rank) own.push_back(j);
  // key ciphertexts with the same pack shift (j t mod gt) use the same shifted
  // fold keys: processed next to each other, their key rows are L2 hits
  std::stable_sort(own.begin(), own.end(), [&](int a, int b) { return (a * t) % gt < (b * t) % gt; });
  const int J = (int)own.size();
  const int n_maps = ceil_div(cache.n_prime, gt);
  std::vector<Ct> out;
  if (J == 0) {
    for (int m = 0; m < n_maps; ++m) out.push_back(zeros(c, q.level() - 2));
    return out;
  }
  std::vector<const Ct*> qs(J, &q_rep), ks;
  for (int j : own) ks.push_back(&cache.k[j]);
  std::vector<Ct> prod0 = mul_batch(c, qs, ks);
  std::vector<const Ct*> pp0;
  for (auto& p : prod0) pp0.push_back(&p);
  const std::string hkey = "headmask:" + std::to_string(cfg.H) + ":" + std::to_string(t);
  // the pack rotation (kv_attention.cpp:201-204) rides the fold: Rot(mask (.) F, r)
  // = Rot(mask, r) (.) Rot(F, r), and Rot(fold(x), r) is the fold's last radix sum
  // with every term moved by r -- no key switch of its own
  std::vector<int> shift(J);
  for (int i = 0; i < J; ++i) shift[i] = -((own[i] * t) % gt);
  std::map<std::pair<int, int>, Pt> mask_pt;  // (shift, limbs) -> Rot(mask, shift), encoded once per context
  auto mask_of = [&](int i, int limbs) {
    auto it = mask_pt.find({shift[i], limbs});
    if (it != mask_pt.end()) return it->second;
    const std::string key = hkey + ":" + std::to_string(shift[i]);
    Pt p;
    if (!lookup_pt(c, key, limbs, &p)) {
      std::vector<double> m(N);
      for (int k = 0; k < N; ++k) m[k] = head_mask[pos_mod((long long)k + shift[i], N)];  // Rot(mask, r)
      p = cached_pt(c, key, m.data(), (double)c.primes[limbs - 1], limbs);
    }
    mask_pt[{shift[i], limbs}] = p;
    return p;
  };
  std::vector<Ct> masked;
  bool fused_mask = fused_path(c);
  for (int i = 0; i < J; ++i) fused_mask = fused_mask && !prod0[i].zero && prod0[i].limbs == prod0[0].limbs;
  // the masked products stay unrescaled (scale * q_top): each (map, pack group)
  // sum is rescaled once instead of J separate rescales
  if (fused_mask) {
    // fold_within_head (38-41), shifted by the pack rotation, with the rotated
    // ReplicateExtract mask (layouts.cpp:134-138) multiplied in the fold's last
    // ModDown epilogue (a fused ct x pt)
    const int lb = prod0[0].limbs;
    require(lb - 1 > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
    std::vector<Pt> hm;
    for (int i = 0; i < J; ++i) hm.push_back(mask_of(i, lb));
    std::vector<const Pt*> post;
    for (auto& p : hm) post.push_back(&p);
    masked = fold_batch(c, pp0, dh, t, true, &post, &shift);
    for (int i = 0; i < J; ++i) {
      c.ledger.ctpt();
      masked[i].scale *= (double)c.primes[lb - 1];  // the product's scale before its rescale
      masked[i].layout.reset();
    }
  } else {
    std::vector<Ct> prod = fold_batch(c, pp0, dh, t, true, nullptr, &shift);  // fold_within_head (38-41)
    std::vector<const Ct*> pp;
    std::vector<Pt> hm;
    for (int i = 0; i < J; ++i) {
      require(prod[i].level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
      hm.push_back(mask_of(i, prod[i].limbs));
    }
    std::vector<const Pt*> hp;
    for (int i = 0; i < J; ++i) pp.push_back(&prod[i]), hp.push_back(&hm[i]);
    masked = mul_plain_batch(c, pp, hp, true, false);
    for (auto& m : masked) m.layout.reset();
  }
  // pack + accumulate (kv_attention.cpp:202-206): per (map, key-ct group j mod
  // kPackGroups) the plain sum of the already aligned masked products and one
  // rescale, then the groups' sum; charged as the reference's rotate/add chain
  std::vector<std::vector<const Ct*>> groups;
  std::vector<std::pair<int, int>> gid;  // (map, group) of each group sum
  std::map<std::pair<int, int>, int> where;
  for (int i = 0; i < J; ++i) {
    const std::pair<int, int> key{(own[i] * t) / gt, own[i] % kPackGroups};
    if (!where.count(key)) where[key] = (int)groups.size(), groups.emplace_back(), gid.push_back(key);
    groups[where[key]].push_back(&masked[i]);
    if (pos_mod(shift[i], c.slots)) c.ledger.rot(false);
  }
  for (auto& g : groups) c.ledger.add((long long)g.size() - 1);
  std::vector<Ct> sums = sum_cts_multi(c, groups);  // every group's sum in one launch
  std::vector<const Ct*> sp;
  for (auto& x : sums) sp.push_back(&x);
  std::vector<Ct> gs = rescale_batch(c, sp);
  std::vector<std::vector<const Ct*>> per_map(n_maps);
  for (int m = 0; m < n_maps; ++m)
    for (int r = 0; r < kPackGroups; ++r) {
      auto it = where.find({m, r});
      if (it != where.end()) per_map[m].push_back(&gs[it->second]);
    }
  for (auto& m : per_map) {
    if (m.empty()) {
      out.push_back(zeros(c, q.level() - 2));
      continue;
    }
    Ct s = sum_cts(c, m);
    s.layout.reset();
    out.push_back(std::move(s));
  }
  return out;
}

std::vector<Ct> qk_dot(Context& c, const Ct& q, const KV& cache) { return qk_dot_partial(c, q, cache, 0, 1); }

// Score*V as a baby-step / giant-step sum. The reference's
// sum over (group g, variant w) of Rot(P_g, -w t) (x) V[g][w]
// (kv_attention.cpp:216-241) is regrouped with w = G B + b (G = floor(w / B),
// 0 <= b < B) and Rot(X, -G B t) (x) V = Rot(X (x) Rot(V, G B t), -G B t):
//   sum_G Rot( sum_(g, b) Rot(P_g, -b t) (x) Rot(V[g][G B + b], G B t), -G B t ).
// The babies Rot(P_g, -b t) share one hoisted ModUp per map, the inner sums are
// lazily relinearised degree-2 accumulations (one relinearisation per giant,
// both maps together), and the giants run as rotation sums, one per giant
// group G mod kSvGroups, at the products' scale (one rescale in finish, so the
// groups' ModDown roundings are divided by q_top): B + #giants key switches per map instead of one
// per variant (255 at d_head 128). Rot(V, G B t) of a cache ciphertext is kept
// with the ciphertext (Context::rot_memo): a completed group's variants are
// rotated once. A rank owns whole giant groups (group mod world == rank), so
// the partials summed mod q are the single-device result for any world size
// dividing kSvGroups; each rank charges the reference's rotations / ct-ct
// mults / additions of the (group, variant) pairs it owns.
int sv_baby(const AttnCfg& cfg) {
  const int nv = v_variant_count(cfg);
  int b = 1;
  while ((long long)b * b < nv) b <<= 1;
  return b;
}

static int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

// Rot(x, r) of value-cache ciphertexts through the context's memo; results are
// kept only where keep[i] (a completed group's variants: the growing group's
// change with every append)
static std::vector<Ct> rotate_memo(Context& c, const std::vector<const Ct*>& xs, const std::vector<int>& rs,
                                   const std::vector<char>& keep) {
  std::vector<Ct> out(xs.size());
  for (auto it = c.rot_memo.begin(); it != c.rot_memo.end();)  // drop entries of dead sources
    it = it->second.src.expired() ? c.rot_memo.erase(it) : std::next(it);
  std::vector<const Ct*> miss;
  std::vector<RotJob> jobs;
  std::vector<int> where;
  for (size_t i = 0; i < xs.size(); ++i) {
    const Ct& x = *xs[i];
    if (x.zero || pos_mod(rs[i], c.slots) == 0 || !x.buf) {
      out[i] = x;
      continue;
    }
    bool hit = false;
    auto range = c.rot_memo.equal_range(x.buf.get());
    for (auto it = range.first; it != range.second; ++it) {
      const Context::RotMemo& m = it->second;
      if (m.limbs == x.limbs && m.r == rs[i] && m.src.lock() == x.buf && m.out.scale == x.scale) {
        out[i] = m.out;
        hit = true;
        break;
      }
    }
    if (hit) continue;
    where.push_back((int)i);
    jobs.push_back({(int)miss.size(), rs[i]});
    miss.push_back(xs[i]);
  }
  if (!miss.empty()) {
    std::vector<Ct> r = rotate_batch(c, miss, jobs, false, false);
    for (size_t k = 0; k < r.size(); ++k) {
      const Ct& x = *xs[where[k]];
      if (!c.capturing && keep[where[k]])
        c.rot_memo.emplace(x.buf.get(), Context::RotMemo{x.buf, x.limbs, jobs[k].r, r[k]});
      out[where[k]] = std::move(r[k]);
    }
  }
  return out;
}

Ct softmax_times_v_partial(Context& c, const std::vector<Ct>& probs, const KV& cache, int rank, int world) {
  SF_HPROF("softmax_times_v_partial");
  const AttnCfg& cfg = cache.cfg;
  require(cache.n_prime != 0, kCacheEmpty, "softmax_times_v: no cached values");
  require(world >= 1 && rank >= 0 && rank < world, kInvalidTarget, "softmax_times_v: bad rank/world");
  const int t = cfg.t(), gt = cfg.group_tokens();
  const int n_maps = ceil_div(cache.n_prime, gt);
  require((int)probs.size() == n_maps, kShapeMismatch,
          "softmax_times_v: expected " + std::to_string(n_maps) + " probability maps, got " +
              std::to_string(probs.size()));
  require((int)cache.v.size() >= n_maps, kShapeMismatch, "softmax_times_v: value cache is missing groups");
  const int B = sv_baby(cfg);
  struct Pair {
    int g, w, G, b;
  };
  std::vector<Pair> own;
  int limbs = 1 << 30;
  for (int g = 0; g < n_maps; ++g) {
    const int tokens = std::min(gt, cache.n_prime - g * gt);
    const int u_max = (tokens - 1) / t;  // touched_variants (53-57)
    const int w_lo = cfg.H == 1 ? 0 : -u_max, w_hi = cfg.d_head();
    for (int w = w_lo; w < w_hi; ++w) {
      const int G = floor_div(w, B);
      if ((int)pos_mod(G, kSvGroups) % world != rank) continue;
      own.push_back({g, w, G, w - G * B});
      const Ct& v = cache.v[g][v_variant_index(cfg, w)];
      check_ct(c, probs[g], "mul");
      check_ct(c, v, "mul");
      const int l = std::min(probs[g].limbs, v.limbs);
      require(l - 1 > 0, kLevelUnderflow, "mul: no multiplicative level left");
      limbs = std::min(limbs, l);
    }
  }
  // the reference's charges for the owned pairs (kv_attention.cpp:227-235)
  for (const Pair& p : own)
    if (pos_mod((long long)-p.w * t, c.slots)) c.ledger.rot(false);
  c.ledger.ctct((long long)own.size());
  if (own.size() > 1) c.ledger.add((long long)own.size() - 1);
  if (own.empty()) return zeros(c, std::min(probs[0].level(), cache.v[0][0].level()));
  // babies: Rot(P_g, -b t), one hoisted ModUp per map
  std::vector<const Ct*> src;
  for (const Ct& p : probs) src.push_back(&p);
  std::map<std::pair<int, int>, int> baby_of;
  std::vector<RotJob> bj;
  for (const Pair& p : own)
    if (!baby_of.count({p.g, p.b})) baby_of[{p.g, p.b}] = (int)bj.size(), bj.push_back({p.g, -p.b * t});
  std::vector<Ct> babies = rotate_batch(c, src, bj, true, false);
  // giant-aligned values Rot(V, G B t)
  std::vector<const Ct*> vs;
  std::vector<int> vr;
  std::vector<char> keep;
  std::vector<const Ct*> vsel(own.size(), nullptr);
  std::vector<int> vpos;
  for (size_t i = 0; i < own.size(); ++i) {  // tracked aligned copies first, else Rot(V) (memo)
    const Pair& p = own[i];
    const int vi = v_variant_index(cfg, p.w);
    if (p.G != 0) vsel[i] = aligned_of(cache, p.g, vi);
    if (vsel[i]) continue;
    vs.push_back(&cache.v[p.g][vi]);
    vr.push_back(p.G * B * t);
    keep.push_back(cache.n_prime - p.g * gt >= gt);
    vpos.push_back((int)i);
  }
  std::vector<Ct> vrot = rotate_memo(c, vs, vr, keep);
  std::vector<Ct> va(own.size());
  for (size_t i = 0; i < own.size(); ++i)
    if (vsel[i]) va[i] = *vsel[i];
  for (size_t k = 0; k < vpos.size(); ++k) va[vpos[k]] = std::move(vrot[k]);
  // inner sums per giant (both maps), lazily relinearised
  std::map<int, std::pair<std::vector<const Ct*>, std::vector<const Ct*>>> inner;
  for (size_t i = 0; i < own.size(); ++i) {
    auto& [a, b] = inner[own[i].G];
    a.push_back(&babies[baby_of[{own[i].g, own[i].b}]]);
    b.push_back(&va[i]);
  }
  std::vector<int> giants;
  std::vector<Ct3> sums;
  {
    std::vector<int> gs;
    std::vector<std::vector<const Ct*>> ta, tb;
    for (auto& [G, ab] : inner) gs.push_back(G), ta.push_back(ab.first), tb.push_back(ab.second);
    std::vector<Ct3> all = tensor_sum_multi(c, ta, tb, false);
    for (size_t i = 0; i < all.size(); ++i) {
      if (all[i].zero) continue;
      giants.push_back(gs[i]);
      sums.push_back(std::move(all[i]));
    }
  }
  if (giants.empty()) return zeros(c, limbs - 1);
  std::vector<const Ct3*> sp;
  for (auto& s : sums) sp.push_back(&s);
  std::vector<Ct> rel = relin_batch(c, sp, false);
  // giant rotation sums, one per giant group, still at the products' scale:
  // their ModDown roundings are then divided by q_top in finish's single rescale
  std::map<int, std::vector<SumTerm>> grp;
  for (size_t i = 0; i < giants.size(); ++i)
    grp[(int)pos_mod(giants[i], kSvGroups)].push_back({&rel[i], -giants[i] * B * t});
  std::vector<std::vector<SumTerm>> groups;
  for (auto& [r, terms] : grp) groups.push_back(terms);
  // at the products' scale (>= 2^80): the wider digits of scaled_digit
  std::vector<Ct> gs = rot_sum_batch(c, groups, false, false, nullptr, false, scaled_digit(c, limbs));
  std::vector<const Ct*> gp;
  for (auto& x : gs) gp.push_back(&x);
  Ct acc = sum_cts(c, gp, false);
  acc.layout.reset();
  return acc;
}

// Sum of the ranks' partials, the rescale, then fold_lanes
// (kv_attention.cpp:44-47) and the final stride mask (238).
Ct softmax_times_v_finish(Context& c, const std::vector<const Ct*>& parts, const KV& cache) {
  SF_HPROF("softmax_times_v_finish");
  const AttnCfg& cfg = cache.cfg;
  const int t = cfg.t();
  long long live = 0;
  for (const Ct* p : parts) live += p->zero ? 0 : 1;
  if (live > 1) c.ledger.add(live - 1);
  Ct folded = sum_cts(c, parts, false);
  if (!folded.zero) folded = rescale(c, folded);
  else folded = zeros(c, folded.level() - 1);
  {
    std::vector<int> fl;  // fold_lanes (44-47)
    for (int step = 1; step < t; step <<= 1) fl.push_back(step);
    folded = fold_steps_batch(c, {&folded}, {fl})[0];
  }
  std::vector<double> sm(cfg.N, 0.0);
  for (int i = 0; i < cfg.N; i += t) sm[i] = 1.0;
  Ct out = mul_plain_cached(c, folded, "stride:" + std::to_string(t) + ":0", sm);
  out.layout = make_interleaved(cfg.d, cfg.N, 0, cfg.H);
  return out;
}

Ct softmax_times_v(Context& c, const std::vector<Ct>& probs, const KV& cache) {
  SF_HPROF("softmax_times_v");
  Ct p = softmax_times_v_partial(c, probs, cache, 0, 1);
  return softmax_times_v_finish(c, {&p}, cache);
}

// ============================================================== prefill
// kv_attention.cpp:245-376 and the helpers it uses. Every op is the reference's
// op on the batched evaluator; the plaintexts (masks, batched RoPE, batched
// diagonals) are encoded once and cached like the decode step's.

Ct inner_rotate(Context& c, const Ct& x, int r, int block, bool hoisted) {  // vmm.cpp:30-43
  SF_HPROF("inner_rotate");
  const int N = c.slots;
  require(block > 0 && N % block == 0, kShapeMismatch, "inner_rotate: block must divide N");
  const int s = (int)pos_mod(r, block);
  if (s == 0) return x;
  std::vector<double> keep(N), wrap(N);
  for (int i = 0; i < N; ++i) keep[i] = (i % block < block - s) ? 1.0 : 0.0, wrap[i] = 1.0 - keep[i];
  // the two rotations of x share one ModUp (same ciphertexts as two calls)
  std::vector<Ct> rot = rotate_batch(c, {&x}, {{0, s}, {0, s - block}}, hoisted);
  const std::string k = "irot:" + std::to_string(block) + ":" + std::to_string(s) + ":";
  Ct lo = mul_plain_cached(c, rot[0], k + "keep", keep);
  Ct hi = mul_plain_cached(c, rot[1], k + "wrap", wrap);
  return add(c, lo, hi);
}

std::unique_ptr<VmmPlan> make_vmm_batch_plan(Context& c, const double* W, int rows, int cols, int level, bool bsgs,
                                             bool encode) {
  require(rows > 0 && cols > 0 && W, kShapeMismatch, "vmm_batch plan: empty weight");
  require(level >= 1 && level <= c.L, kInvalidTarget, "vmm plan: level must be in [1, L]");
  const int d = padded_dim(rows);
  require(padded_dim(cols) == d, kShapeMismatch, "vmm_batch: square weights only");
  require(d <= c.slots, kShapeMismatch, "vmm_batch: dimension exceeds N");
  auto p = std::make_unique<VmmPlan>();
  p->ctx = &c;
  p->rows = rows;
  p->cols = cols;
  p->level = level;
  p->bsgs = bsgs;
  p->batch = true;
  VmmShape& s = p->s;
  s.N = c.slots;
  s.d_in = s.d_out = d;
  s.t_in = c.slots / d;
  s.t_out = 1;  // giant unit = t_in * t_out = t (vmm.cpp:450)
  s.k = d;
  p->bg = bsgs ? bsgs_split(d) : BsgsSplit{1, d};
  p->w_store.assign(W, W + (size_t)rows * cols);
  const double* wd = p->w_store.data();
  p->w = [wd, rows, cols](int r, int cc) { return (r < rows && cc < cols) ? wd[(size_t)r * cols + cc] : 0.0; };
  if (encode) p->diagonals(level + 1);
  return p;
}

Ct vmm_batch(Context& c, const Ct& x, VmmPlan& plan) {  // vmm.cpp:417-467
  SF_HPROF("vmm_batch");
  require(plan.batch, kInvalidTarget, "vmm_batch: plan is not a token-batched plan");
  require(x.layout && x.layout->kind == LayoutKind::Interleaved, kLayoutMismatch,
          "vmm_batch: input must carry an interleaved layout");
  require(!x.layout->deferred_mask, kLayoutMismatch, "vmm_batch: input garbage must be cleared first");
  const int d = plan.s.d_in, t = plan.s.t_in;
  require(x.layout->d == d, kShapeMismatch, "vmm_batch: layout/weight dimension mismatch");
  check_ct(c, x, "vmm_batch");
  require(x.level() > 0, kLevelUnderflow, "mul_plain: no multiplicative level left");
  const std::vector<Pt>& diag = plan.diagonals(x.limbs);
  Ct acc;
  if (!plan.bsgs) {
    std::vector<RotJob> jobs;
    for (int j = 0; j < d; ++j) jobs.push_back({0, j * t});
    std::vector<Ct> rx = rotate_batch(c, {&x}, jobs, false);
    std::vector<const Ct*> cts;
    std::vector<const Pt*> pts;
    for (int j = 0; j < d; ++j) cts.push_back(&rx[j]), pts.push_back(&diag[j]);
    acc = mac_plain(c, cts, pts);
  } else {
    const int b = plan.bg.baby, giants = plan.bg.giant;
    std::vector<RotJob> jobs;
    for (int g1 = 1; g1 < b; ++g1) jobs.push_back({0, g1 * t});
    std::vector<Ct> baby{x};
    for (Ct& r : rotate_batch(c, {&x}, jobs, true)) baby.push_back(std::move(r));
    std::vector<Ct> partial(giants);
    for (int g2 = 0; g2 < giants; ++g2) {
      std::vector<const Ct*> cts;
      std::vector<const Pt*> pts;
      for (int g1 = 0; g1 < b && g2 * b + g1 < d; ++g1) cts.push_back(&baby[g1]), pts.push_back(&diag[g2 * b + g1]);
      partial[g2] = mac_plain(c, cts, pts);
    }
    std::vector<std::vector<SumTerm>> groups;
    for (int r = 0; r < std::min(kGiantGroups, giants); ++r) {
      groups.emplace_back();
      for (int g2 = r; g2 < giants; g2 += kGiantGroups)
        groups.back().push_back({&partial[g2], (int)(((long long)g2 * b * t) % c.slots)});
    }
    std::vector<Ct> gs = rot_sum_batch(c, groups, false);
    std::vector<const Ct*> ap;
    for (auto& a : gs) ap.push_back(&a);
    acc = sum_cts(c, ap);
  }
  acc.layout = Layout{LayoutKind::Interleaved, d, t, 0, 1, false};
  return acc;
}

Ct rope_apply_batch(Context& c, const Ct& x, const AttnCfg& cfg, long long first_pos, double base) {
  SF_HPROF("rope_apply_batch");  // kv_attention.cpp:119-129 (plaintexts: 59-76)
  require_clean_interleaved(x, cfg, 0, "rope_apply_batch");
  const int N = cfg.N, t = cfg.t(), dh = cfg.d_head();
  require(dh % 2 == 0, kShapeMismatch, "rope_apply_batch: d_head must be even");
  std::vector<double> p[3] = {std::vector<double>(N, 0.0), std::vector<double>(N, 0.0), std::vector<double>(N, 0.0)};
  for (int i = 0; i < N; ++i) {
    const int e = (i / t) % dh;
    const double angle = (double)(first_pos + i % t) * std::pow(base, -2.0 * (e / 2) / (double)dh);
    p[0][i] = std::cos(angle);
    if (e % 2 == 0)
      p[1][i] = std::sin(angle);
    else
      p[2][i] = -std::sin(angle);
  }
  char key[160];
  std::snprintf(key, sizeof key, "ropeb:%lld:%d:%d:%d:%a:", first_pos, N, t, dh, base);
  const int s = t;
  Ct y = mul_plain_cached(c, x, std::string(key) + "0", p[0]);
  y = add(c, y, rotate(c, mul_plain_cached(c, x, std::string(key) + "1", p[1]), -s, false));
  y = add(c, y, rotate(c, mul_plain_cached(c, x, std::string(key) + "2", p[2]), s, false));
  y.layout = x.layout;
  return y;
}

PrefillScores prefill_scores(Context& c, const std::vector<Ct>& xs, VmmPlan& wq, VmmPlan& wk, VmmPlan& wv,
                             const AttnCfg& cfg, double base) {
  SF_HPROF("prefill_scores");  // kv_attention.cpp:245-333
  const int t = cfg.t(), dh = cfg.d_head(), gt = cfg.group_tokens(), N = cfg.N, n0 = cfg.n0;
  require(n0 >= 1, kShapeMismatch, "prefill: need a nonempty prompt");
  require(n0 <= cfg.n_max, kCacheFull, "prefill: prompt exceeds cache capacity");
  const int P = ceil_div(n0, t);
  require((int)xs.size() == P, kShapeMismatch,
          "prefill: expected " + std::to_string(P) + " prompt cts, got " + std::to_string(xs.size()));
  PrefillScores out;
  KV& cache = out.cache;
  cache.cfg = cfg;
  std::vector<Ct> q_cts;
  for (int p = 0; p < P; ++p) {
    q_cts.push_back(rope_apply_batch(c, vmm_batch(c, xs[p], wq), cfg, (long long)p * t, base));
    cache.k.push_back(rope_apply_batch(c, vmm_batch(c, xs[p], wk), cfg, (long long)p * t, base));
  }
  for (int p = 0; p < P; ++p) {
    const Ct v_raw = vmm_batch(c, xs[p], wv);
    const int g = (p * t) / gt;
    const int u_cap = p - g * dh;
    if (g == (int)cache.v.size()) cache.v.emplace_back(v_variant_count(cfg), zeros(c, -1));
    std::vector<Pt> masks;
    for (int e = 0; e < dh; ++e) {
      std::vector<double> m(N, 0.0);
      for (int h = 0; h < cfg.H; ++h)
        for (int j = 0; j < t; ++j) m[(h * dh + e) * t + j] = 1.0;
      masks.push_back(cached_pt(c, "vblk:" + std::to_string(cfg.H) + ":" + std::to_string(dh) + ":" +
                                       std::to_string(t) + ":" + std::to_string(e),
                                m.data(), (double)c.primes[v_raw.limbs - 1], v_raw.limbs));
    }
    std::vector<const Ct*> vx(dh, &v_raw);
    std::vector<const Pt*> ps;
    for (auto& m : masks) ps.push_back(&m);
    std::vector<Ct> pieces = mul_plain_batch(c, vx, ps);
    for (int e = 0; e < dh; ++e) {
      const int idx = v_variant_index(cfg, v_variant_of(cfg, e, u_cap * t));
      cache.v[g][idx] = add(c, cache.v[g][idx], pieces[e]);
    }
  }
  cache.n_prime = n0;
  std::vector<std::vector<Ct>> k_rot(P);
  for (int j = 0; j < P; ++j) {
    k_rot[j].push_back(cache.k[j]);
    for (int rho = 1; rho < t; ++rho) k_rot[j].push_back(inner_rotate(c, cache.k[j], rho, t, false));
  }
  std::vector<std::vector<std::vector<std::optional<Ct>>>> acc(P);
  for (int p = 0; p < P; ++p) acc[p].assign((p * t) / gt + 1, std::vector<std::optional<Ct>>(t));
  for (int p = 0; p < P; ++p)
    for (int j = 0; j <= p; ++j) {
      const int g_key = (j * t) / gt, local = (j * t) % gt;
      for (int rho = 0; rho < t; ++rho) {
        std::vector<double> m(N, 0.0);
        bool any = false;
        std::string mk = "causal:" + std::to_string(cfg.H) + ":" + std::to_string(gt) + ":";
        for (int tau = 0; tau < t; ++tau) {
          const int key = j * t + (tau + rho) % t, query = p * t + tau;
          if (key <= query && key < n0 && query < n0) {
            for (int h = 0; h < cfg.H; ++h) m[h * gt + tau] = 1.0;
            any = true;
            mk += std::to_string(tau) + ",";
          }
        }
        if (!any) continue;
        Ct prod = mul(c, q_cts[p], k_rot[j][rho]);
        prod = fold_batch(c, {&prod}, dh, t)[0];  // fold_within_head (38-41)
        Ct masked = mul_plain_cached(c, prod, mk, m);
        Ct packed = local ? rotate(c, masked, -local, false) : masked;
        auto& cell = acc[p][g_key][rho];
        cell = cell ? add(c, *cell, packed) : packed;
      }
    }
  out.maps.resize(P);
  for (int p = 0; p < P; ++p) {
    for (size_t g = 0; g < acc[p].size(); ++g) {
      const int ref_level = acc[p][g][0]->level();
      std::vector<Ct> row;
      for (int rho = 0; rho < t; ++rho) {
        Ct cell = acc[p][g][rho] ? *acc[p][g][rho] : zeros(c, ref_level);
        cell.layout.reset();
        row.push_back(cell);
      }
      out.maps[p].push_back(std::move(row));
    }
  }
  return out;
}

std::vector<Ct> prefill_attend(Context& c, const std::vector<std::vector<std::vector<Ct>>>& probs, const KV& cache) {
  SF_HPROF("prefill_attend");  // kv_attention.cpp:340-376
  const AttnCfg& cfg = cache.cfg;
  const int t = cfg.t(), gt = cfg.group_tokens(), n0 = cache.n_prime;
  const int groups = (int)cache.v.size();
  std::vector<int> w_lo(groups);
  std::vector<std::vector<std::vector<Ct>>> v_rot(groups);
  for (int g = 0; g < groups; ++g) {
    const int tokens = std::min(gt, n0 - g * gt);
    const int u_max = (tokens - 1) / t;  // touched_variants (53-57)
    const int lo = cfg.H == 1 ? 0 : -u_max, hi = cfg.d_head();
    w_lo[g] = lo;
    for (int w = lo; w < hi; ++w) {
      const Ct& base = cache.v[g][v_variant_index(cfg, w)];
      std::vector<Ct> row{base};
      for (int rho = 1; rho < t; ++rho) row.push_back(inner_rotate(c, base, rho, t, false));
      v_rot[g].push_back(std::move(row));
    }
  }
  std::vector<Ct> att;
  for (size_t p = 0; p < probs.size(); ++p) {
    std::vector<Ct> scores;
    std::vector<std::pair<int, int>> who;  // (g, w index, rho) flattened below
    std::vector<const Ct*> vv;
    scores.reserve(probs[p].size() * t * (2 * cfg.d_head()));
    for (size_t g = 0; g < probs[p].size(); ++g) {
      const int tokens = std::min(gt, n0 - (int)g * gt);
      const int u_max = (tokens - 1) / t;
      const int lo = cfg.H == 1 ? 0 : -u_max, hi = cfg.d_head();
      for (int rho = 0; rho < t; ++rho) {
        const Ct& pm = probs[p][g][rho];
        // the map's alignment rotations share one ModUp (same words as separate calls)
        std::vector<RotJob> jobs;
        for (int w = lo; w < hi; ++w) jobs.push_back({0, -w * t});
        std::vector<Ct> rs = rotate_batch(c, {&pm}, jobs, false);
        for (int w = lo; w < hi; ++w) {
          scores.push_back(std::move(rs[w - lo]));
          vv.push_back(&v_rot[g][w - w_lo[g]][rho]);
        }
      }
    }
    std::vector<const Ct*> sp;
    for (auto& x : scores) sp.push_back(&x);
    // sum of the products (kv_attention.cpp:358-368) relinearised once
    Ct3 s3 = tensor_sum(c, sp, vv);
    Ct a = relin_rescale(c, s3);
    a.layout = make_interleaved(cfg.d, cfg.N, 0, cfg.H);
    att.push_back(std::move(a));
  }
  return att;
}

}  // namespace sf
