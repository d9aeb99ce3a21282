"""Benchmark: one encrypted Llama-3-8B-shaped decoder-layer hot path per token
(BASELINE.json configs[3]) on B200, through the C ABI.

Step (= one decode token, Table-4 stage levels):
  Q,K,V   3x vmm_interleaved 4096x4096 at level 4           (vmm.cpp:179-236)
  RoPE&Cache  rope_apply(q), rope_apply(k), make_v_pieces, v_append, k_append
                                                            (kv_attention.cpp:111-182)
  QK^T    qk_dot over the cache at n' = 2048                (kv_attention.cpp:184-214)
  Score*V softmax_times_v on fresh level-2 probability maps (kv_attention.cpp:216-241)
  Out     vmm 4096x4096 at level 7 (post-bootstrap input)
  Up/Gate 2x vmm 4096->14336 at level 3
  Down    vmm 14336->4096 at level 1
Excluded (stated): softmax, norms, SiLU and bootstrapping; every stage that
follows one of them starts from a fresh encryption at its Table-4 level.

`value` = ms per decode token (device time, CUDA events on the library
stream, inputs resident); `e2e` = the same step through the public API with
inputs imported from pinned host words and the outputs read back each step.
--impl reference runs the reference's own CPU implementation
(oracle/_ref/ref_bench: the unmodified slotforge SimBackend) on this host.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Encrypted decode-step latency (ms/token) at N=2^16; HE-VMM ciphertexts/sec"
SLOTS = 32768          # ring N' = 2^16
D, H, FF, NP = 4096, 32, 14336, 2048
LEVELS = dict(qkv=4, cache=2, probs=2, out=7, up=3, down=1)


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


# ------------------------------------------------------------------ clocks sampling
class Clocks:
    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        if os.environ.get("SF_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def wait_first(self, timeout=5.0):
        """nvidia-smi's start-up is not allowed to overlap the timed region."""
        t = time.time()
        while self.proc and not self.rows and time.time() - t < timeout:
            time.sleep(0.05)

    def mark(self):
        self.start = len(self.rows)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows[getattr(self, "start", 0):] or self.rows[-1:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > i + 2 and r[i + 2] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------------ workload
class LlamaLayer:
    def __init__(self, be, sf, log=print):
        self.be, self.sf = be, sf
        t0 = time.time()
        cfg = sf.AttentionConfig(SLOTS, D, H, 0, NP)
        self.cfg = cfg
        t = cfg.t
        self.pos = NP - 1
        # plans: offline diagonal encoding (not charged)
        mk = lambda r, c, lvl, off=0: sf.VmmPlan(be, None, r, c, lvl, 0, off, True)
        self.wq = mk(D, D, LEVELS["qkv"])
        self.wk = mk(D, D, LEVELS["qkv"], self.pos % t)
        self.wv = mk(D, D, LEVELS["qkv"], self.pos % t)
        self.wo = mk(D, D, LEVELS["out"])
        self.wg = mk(D, FF, LEVELS["up"])
        self.wu = mk(D, FF, LEVELS["up"])
        self.wd = mk(FF, D, LEVELS["down"])
        log(f"[bench] plans encoded in {time.time() - t0:.1f}s")
        # cache at n' = 2047 tokens, built directly in cache layout (the
        # reference tests' direct_cache; tokens stand in for the prefill)
        t1 = time.time()
        rng = np.random.default_rng(7)
        n = NP - 1
        gt, dh = cfg.group_tokens, cfg.d_head
        k_cts = []
        self.v_sum = np.zeros(D)  # sum over cached tokens of V[u, h*dh+e] (the attention parity check)
        self.k_vals = np.zeros((n, D))  # cached keys (the QK^T parity check)
        for j in range((n + t - 1) // t):
            s = np.zeros(SLOTS)
            for tau in range(min(t, n - j * t)):
                self.k_vals[j * t + tau] = rng.normal(size=D)
                s[np.arange(D) * t + tau] = self.k_vals[j * t + tau]
            k_cts.append(be.encrypt(s, LEVELS["cache"]))
        nv = 2 * dh - 1
        v_cts = []
        for g in range((n + gt - 1) // gt):
            rows = np.zeros((nv, SLOTS))
            for u in range(g * gt, min(n, (g + 1) * gt)):
                ul = u - g * gt
                j0 = ul % t
                e = np.arange(dh)
                w = e - ul // t
                idx = w + dh - 1
                for h in range(H):
                    vals = rng.normal(size=dh)
                    rows[idx, (h * dh + e) * t + j0] = vals
                    self.v_sum[h * dh + e] += vals
            v_cts.append([be.encrypt(r, LEVELS["cache"]) for r in rows])
        self.cache = sf.kv_from_cts(be, cfg, n, k_cts, v_cts)
        log(f"[bench] cache n'={n}: {len(k_cts)} K cts + {len(v_cts)}x{nv} V handles in {time.time() - t1:.1f}s")
        # per-step fresh inputs (client-encrypted activations at each stage's level)
        self.vals = {}

        def fresh(d, lvl, seed, name):
            s = np.zeros(SLOTS)
            self.vals[name] = np.random.default_rng(seed).normal(size=d)
            s[np.arange(d) * (SLOTS // d)] = self.vals[name]
            return be.encrypt(s, lvl, sf.make_interleaved(d, SLOTS, 0))
        self.x = fresh(D, LEVELS["qkv"], 42, "x")
        self.h7 = fresh(D, LEVELS["out"], 43, "h7")
        self.h3 = fresh(D, LEVELS["up"], 44, "h3")
        self.h1 = fresh(16384, LEVELS["down"], 45, "h1")
        probs = np.zeros(SLOTS)
        for h in range(H):
            probs[h * gt:h * gt + min(gt, NP)] = 1.0 / NP
        self.probs = [be.encrypt(probs, LEVELS["probs"]), be.encrypt(probs, LEVELS["probs"])]
        self.inputs = [self.x, self.h7, self.h3, self.h1] + self.probs

    PHASES = ["Q, K, V", "RoPE & Cache", "QK^T", "Score*V", "Output projection", "Up & Gate projection",
              "Down projection"]

    def phase_ms(self, steps):
        """Device time per phase: CUDA events between phases, recorded inside a
        captured graph of the marked step (host issue time cannot leak in)."""
        be = self.be
        graph, _ = be.capture(self.step, marks=True)
        graph.launch()
        be.synchronize()
        tot = [0.0] * len(self.PHASES)
        for _ in range(steps):
            graph.launch()
            be.synchronize()
            for i in range(len(self.PHASES)):
                tot[i] += be.event_elapsed_ms(10 + i, 11 + i)
        del graph
        return {p: round(t / steps, 3) for p, t in zip(self.PHASES, tot)}

    def step(self, inputs=None, marks=False, staged=None, staged_out=None):
        """One decode step. staged (e2e): the six inputs' pinned host words; their
        uploads start at the step's beginning on a side stream (sf_ct_stage) and each
        joins right before its stage, so the later stages' uploads overlap Q/K/V,
        RoPE and QK^T (the stage inputs are independent client data)."""
        be, sf = self.be, self.sf
        x, h7, h3, h1, p0, p1 = inputs or self.inputs
        wait = (lambda *slots: [be.stage_wait(i) for i in slots]) if staged else (lambda *slots: None)
        if staged:
            for i, (ct, w) in enumerate(zip((x, h7, h3, h1, p0, p1), staged)):
                be.stage(ct, w, i)
        mark = (lambda i: be.event_record(10 + i)) if marks else (lambda i: None)
        mark(0)
        wait(0)
        with be.phase("Q, K, V"):  # three VMMs of one input: shared ladder + babies
            q, k, v = sf.vmm_interleaved_multi(be, x, [self.wq, self.wk, self.wv])
        mark(1)
        with be.phase("RoPE & Cache"):
            qr = sf.rope_apply(be, q, self.cfg, self.pos)
            kr = sf.rope_apply(be, k, self.cfg, self.pos)
            cache = sf.v_append(be, self.cache, sf.make_v_pieces(be, self.cache, v, self.pos))
            cache = sf.k_append(be, cache, kr)
        mark(2)
        with be.phase("QK^T"):
            maps = sf.qk_dot(be, qr, cache)
        mark(3)
        wait(4, 5)
        with be.phase("Score*V"):
            att = sf.softmax_times_v(be, [p0, p1], cache)
        if staged_out:  # the attention output's read-back overlaps the projections
            be.stage_out(att, staged_out[0], 6)
        mark(4)
        wait(1)
        with be.phase("Output projection"):
            o = sf.vmm_interleaved(be, h7, None, plan=self.wo)
        mark(5)
        wait(2)
        with be.phase("Up & Gate projection"):
            g, u = sf.vmm_interleaved_multi(be, h3, [self.wg, self.wu])
        mark(6)
        wait(3)
        with be.phase("Down projection"):
            dn = sf.vmm_interleaved(be, h1, None, plan=self.wd)
        if staged_out:
            be.stage_out(dn, staged_out[1], 7)
            be.stage_wait(6)
            be.stage_wait(7)
        mark(7)
        return [q, k, v, maps[0], att, o, g, u, dn, qr]


    def step_sharded(self, sh, inputs=None):
        """One decode token split over the ranks of `sh` (paper_2602_11470_b200.shard,
        DESIGN.md §7): VMM giant groups, QK^T key-ct groups and Score*V giant groups per
        rank, partial ciphertexts all-gathered over NCCL and mod-added on the GPU;
        RoPE, the appends and the replicated tails (reduce ladders, lane fold) on
        every rank. Word-identical to step() for any world size."""
        be, sf = self.be, self.sf
        x, h7, h3, h1, p0, p1 = inputs or self.inputs
        q, k, v = sh.vmm_multi(x, [self.wq, self.wk, self.wv])
        qr = sf.rope_apply(be, q, self.cfg, self.pos)
        kr = sf.rope_apply(be, k, self.cfg, self.pos)
        cache = sf.v_append(be, self.cache, sf.make_v_pieces(be, self.cache, v, self.pos))
        cache = sf.k_append(be, cache, kr)
        maps = sh.qk_dot(qr, cache)
        att = sh.softmax_times_v([p0, p1], cache)
        o = sh.vmm(h7, self.wo)
        g, u = sh.vmm_multi(h3, [self.wg, self.wu])
        dn = sh.vmm(h1, self.wd)
        return [q, k, v, maps[0], att, o, g, u, dn, qr]


def bench_config(alpha, world, sharded):
    """The workload's config, identical on both arms (the reference arm runs the
    same decode step on the host cores)."""
    par = "single" if world == 1 else (
        f"sharded{world} (one token split over the ranks: VMM giant groups, QK^T key-ct groups, Score*V giant groups; "
        "fused peer-memory exchange)" if sharded else f"replicas{world}")
    return {"workload": "llama3-8b-layer-decode@n'=2048", "ring_degree": 2 * SLOTS, "slots": SLOTS, "d": D,
            "heads": H, "ffn": FF, "context": NP, "levels": LEVELS, "L": 7, "alpha": alpha, "parallelism": par,
            "l2": "working set (plaintext diagonals + keys ~30 GB) >> 126 MB L2; no flush needed"}


def bench_weight(rows, cols):
    r = np.arange(rows, dtype=np.float64)[:, None]
    c = np.arange(cols, dtype=np.float64)[None, :]
    return np.sin(0.001 * (31.0 * r + c) + 0.25)  # slotforge_cli.cpp:88-92


def decrypt_parity(be, layer, outs):
    """The step's outputs decrypted and compared with float64 linear algebra on
    the same inputs: Q (= V's new token, same bench weight), the attention
    output (uniform probabilities over the n' = 2048 cached + appended values),
    the output / gate / down projections. Relative max error over the valid
    lanes of each output."""
    q, _k, _v, maps0, att, o, g, _u, dn, qr = outs[:10]
    Wdd = bench_weight(D, D)
    x, h7, h3, h1 = (layer.vals[k] for k in ("x", "h7", "h3", "h1"))
    xw = x @ Wdd
    want = {"q": (q, xw, SLOTS // D),
            "att": (att, (layer.v_sum + xw) / NP, SLOTS // D),
            "o": (o, h7 @ Wdd, SLOTS // D),
            "gate": (g, h3 @ bench_weight(D, FF), SLOTS // 16384),
            "down": (dn, h1[:FF] @ bench_weight(FF, D), SLOTS // D)}
    errs = {}
    for name, (ct, w, t) in want.items():
        got = be.decrypt(ct)[np.arange(len(w)) * t]
        errs[name] = float(np.max(np.abs(got - w)) / max(np.max(np.abs(w)), 1e-30))
    # QK^T: score map 0 (tokens 0..gt-1, slot h*gt + u) against float64 dot products of
    # the decrypted RoPE'd query with the cached keys, per head
    gt, dh = SLOTS // H, D // H
    qv = be.decrypt(qr)[np.arange(D) * (SLOTS // D)]
    kk = layer.k_vals[:gt]
    want_s = np.stack([kk[:, h * dh:(h + 1) * dh] @ qv[h * dh:(h + 1) * dh] for h in range(H)])  # [H, gt]
    got_s = be.decrypt(maps0).reshape(H, gt)
    errs["scores"] = float(np.max(np.abs(got_s - want_s)) / max(np.max(np.abs(want_s)), 1e-30))
    return errs


def reduce_ranks(dist, v, op):
    """All-reduce one float over the ranks (a CUDA tensor over NCCL, a CPU one
    over gloo when ranks share a device)."""
    import torch
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(v)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return float(t.item())


def run_sharded(args, be, sf, layer, dist, rank, world, clk):
    """--shard: strong scaling of ONE token over the ranks (latency). Default:
    the exchange on the library stream (shard.StreamSharded, csrc/comm.cpp) and
    the whole sharded step captured into one CUDA graph; --shard-host: the
    torch-stream exchange (shard.Sharded), eager."""
    from paper_2602_11470_b200 import shard
    import torch
    stream = not args.shard_host
    # the single-device step on every rank, for the bit-exactness check -- before the
    # exchange is set up (that restricts the appends' aligned companions to the rank's
    # own Score*V giant groups, sf_set_value_shard)
    ref = layer.step()
    if args.shard_host:
        sh = shard.Sharded(be)
    elif args.shard_nccl:
        sh = shard.StreamSharded(be)
    else:  # default: the fused peer-memory exchange (csrc/p2p.cu)
        sh = shard.PeerSharded(be)
    got = layer.step_sharded(sh)
    exact = all(np.array_equal(a.data(), b.data()) for a, b in zip(ref, got))
    for _ in range(args.warmup):
        layer.step_sharded(sh)
    be.synchronize()
    torch.cuda.synchronize()

    def max_over_ranks(v):
        return reduce_ranks(dist, v, dist.ReduceOp.MAX)

    # eager (host-issued) timing, for the record
    dist.barrier()
    be.event_record(0)
    t_w = time.perf_counter()
    for _ in range(args.steps):
        layer.step_sharded(sh)
    be.event_record(1)
    ms_eager = max_over_ranks(be.event_elapsed_ms(0, 1) / args.steps)
    be.synchronize()
    wall = (time.perf_counter() - t_w) * 1e3 / args.steps

    graph = None
    if stream:  # the whole sharded step (NCCL all-gathers included) in one graph
        graph, gouts = be.capture(layer.step_sharded, sh)
        graph.launch()
        be.synchronize()
        exact = exact and all(np.array_equal(a.data(), b.data()) for a, b in zip(ref, gouts))
    run = graph.launch if graph else (lambda: layer.step_sharded(sh))
    be.synchronize()
    torch.cuda.synchronize()
    dist.barrier()
    clk.mark()
    l0 = be.kernel_launches()
    be.event_record(0)
    for _ in range(args.steps):
        run()
    be.event_record(1)
    ms = max_over_ranks(be.event_elapsed_ms(0, 1) / args.steps)
    be.synchronize()
    launches = (be.kernel_launches() - l0) // args.steps
    clk.__exit__()
    ex_all = reduce_ranks(dist, 1.0 if exact else 0.0, dist.ReduceOp.MIN)

    # e2e: inputs from host memory every step, results read back
    host_in = [c.data() for c in layer.inputs]
    outs = gouts if graph else None
    be.synchronize()
    dist.barrier()
    t_e = time.perf_counter()
    for _ in range(args.steps):
        for slot, w in zip(layer.inputs, host_in):
            be.refill(slot, w)
        if graph:
            graph.launch()
        else:
            outs = layer.step_sharded(sh)
        res = [outs[4].data(), outs[8].data()]
    be.synchronize()
    e2e = max_over_ranks((time.perf_counter() - t_e) * 1e3 / args.steps)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(ms, 3), "unit": "ms/token", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64",
            "data": "synthetic: reference bench weights sin(0.001(31r+c)+0.25), N(0,1) activations/cache, seeded",
            "config": bench_config(args.alpha, world, True),
            "exchange": ("torch-stream NCCL all-gather + mod-add" if args.shard_host else
                         "NCCL all-gather on the library stream + mod-add" if args.shard_nccl else
                         "fused peer-memory read + mod-add kernel (CUDA IPC / NVLink)"),
            "sharded_bit_exact_vs_single_device": bool(ex_all == 1.0),
            "eager_ms_per_step": round(ms_eager, 3), "wall_ms_per_step_rank0_eager": round(wall, 3),
            "e2e": {"value": round(e2e, 3), "unit": "ms/token",
                    "h2d_bytes_per_step": int(sum(w.nbytes for w in host_in)),
                    "d2h_bytes_per_step": int(sum(r.nbytes for r in res))},
            "gpu_launches": int(launches) if graph else None, "clocks": clk.summary(), "cpu_baseline": None,
            "execution": ("one CUDA graph per step; the exchanges on the library stream inside it" if graph else
                          "eager (host-issued; NCCL exchanges on torch's stream between library launches)"),
        }
        print(json.dumps(line), flush=True)
    if stream:
        sh.close()


# ---------------------------------------------------------------- reference arm
def run_reference(args, rank):
    """The reference's own CPU implementation of the step (oracle/_ref/ref_bench:
    the unmodified slotforge SimBackend, single-threaded) on this host: every
    warm-up and timed step is one process, run concurrently on all host cores
    (W untimed, then K timed); value = the mean per-step latency the processes
    measure themselves. Same metric, unit and config as our arm. Under torchrun
    only rank 0 runs."""
    if rank != 0:
        return
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    cores = os.cpu_count() or 1

    def batch(n):
        res, running, todo = [], [], n
        while todo or running:
            while todo and len(running) < cores:
                running.append(subprocess.Popen([exe, "--workload", "llama", "--steps", "1", "--warmup", "0"],
                                                stdout=subprocess.PIPE, text=True))
                todo -= 1
            p = running.pop(0)
            outp, _ = p.communicate()
            if p.returncode:
                raise RuntimeError(f"ref_bench exited {p.returncode}")
            res.append(json.loads(outp.strip().splitlines()[-1]))
        return res

    batch(args.warmup)
    t0 = time.perf_counter()
    res = batch(args.steps)
    wall = time.perf_counter() - t0
    v = round(float(np.mean([r["ms_per_step"] for r in res])), 3)
    used = min(cores, args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "ms/token", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
        "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: reference bench weights sin(0.001(31r+c)+0.25) (slotforge_cli.cpp:88-92), "
                "mt19937_64-seeded activations",
        "config": bench_config(args.alpha, args.gpus, args.gpus > 1 and not args.replicas),
        "cpu_baseline": {"value": v, "unit": "ms/token", "cores": used, "kind": "reference",
                         "sample": f"{args.steps} full decode steps of the unmodified reference SimBackend "
                                   f"(cleartext slot simulator), one single-threaded process per step, "
                                   f"{used} concurrently on {cores} host cores; wall {wall:.1f} s"},
        "e2e": {"value": v, "unit": "ms/token", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "counts": res[0].get("counts"),
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_sample():
    """Reference CPU path timed on this host: one full decode step of the
    unmodified reference (oracle/_ref/ref_bench), ~19 s on one core."""
    exe = os.path.join(ROOT, "oracle", "_ref", "ref_bench")
    if not os.path.exists(exe):
        return None
    try:
        out = subprocess.run([exe, "--workload", "llama", "--steps", "1", "--warmup", "0"], capture_output=True,
                             text=True, timeout=300, check=True).stdout.strip().splitlines()[-1]
        r = json.loads(out)
        return {"value": r["ms_per_step"], "unit": "ms/token", "cores": 1, "kind": "reference",
                "sample": "1 full Llama-layer decode step of the unmodified reference SimBackend "
                          "(cleartext slot simulator, single-threaded)"}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "ms/token", "cores": 1, "kind": "reference", "sample": f"failed: {e}"}


def token_stream(be, sf, layer, T=16):
    """A real decode stream through the public API: T consecutive tokens at
    positions 2047, 2048, ... (n' grows 2047 -> 2047 + T): every token uploads
    the stage inputs from pinned host words (H2D, staged: each overlaps the
    stages before its first use), runs Q/K/V with the K/V
    plans of its lane offset pos mod t (vmm.cpp:66-83 out_offset), RoPE at its
    own position (its RoPE plaintexts are encoded on the host inside the timed
    region -- for token p+1 while token p runs, sf_rope_prepare), appends k and
    v to the persistent cache (a new K-ct every t tokens, a third V group and
    score map at n' = 2049: later tokens do more attention work than the
    n' = 2048 bench step), QK^T and Score*V over the grown cache, the output /
    up / gate / down projections, and reads the attention and down-projection
    outputs back (D2H). Eager (the cache changes shape every token, so no single
    graph fits); two untimed warm-up tokens first. Wall clock per token,
    synchronised by the read-back."""
    t = layer.cfg.t
    mk = lambda off: sf.VmmPlan(be, None, D, D, LEVELS["qkv"], 0, off, True)  # noqa: E731
    wk = {o: (layer.wk if o == layer.pos % t else mk(o)) for o in range(t)}
    wv = {o: (layer.wv if o == layer.pos % t else mk(o)) for o in range(t)}
    gt = layer.cfg.group_tokens
    pmap = np.zeros(SLOTS)
    for h in range(H):
        pmap[h * gt:(h + 1) * gt] = 1.0 / (NP + T)
    probs = [be.encrypt(pmap, LEVELS["probs"], seed=700 + i) for i in range(3)]
    import torch
    host_in = []
    for c in layer.inputs[:4]:
        w = c.data()
        tt = torch.empty(w.shape, dtype=torch.uint64 if hasattr(torch, "uint64") else torch.int64, pin_memory=True)
        a = tt.numpy().view(np.uint64)
        a[...] = w
        host_in.append((a, tt))
    # the same cache (n' = 2047) under a config with room for the T new tokens
    cfg = sf.AttentionConfig(SLOTS, D, H, 0, NP + T)
    cache = sf.kv_from_cts(be, cfg, layer.cache.n_prime, layer.cache.k_cts, layer.cache.v_cts)
    x, h7, h3, h1 = layer.inputs[:4]
    # setup (untimed): the value-piece masks depend on the lane offset pos mod t
    # only -- position-independent constants like the plans -- so every offset's
    # set is encoded once here, as a deployment does before its first token
    for o in range(t):
        _, _, v_o = sf.vmm_interleaved_multi(be, x, [layer.wq, wk[o], wv[o]])
        sf.make_v_pieces(be, cache, v_o, o)
    rope_level = v_o.level
    sf.rope_prepare(be, cfg, layer.pos, rope_level, 0)
    sf.rope_prepare(be, cfg, layer.pos, rope_level, layer.pos % t)
    # setup: grow the device pool past the stream's peak once (a deployment sizes
    # its pool at start-up; otherwise the first token that raises the peak maps
    # new device memory inside its step)
    be.mem_reserve(16 << 30)
    be.synchronize()
    def token(cache, pos):
        # uploads staged on the side stream (sf_ct_stage), each joined before its stage
        for i, (slot, (w, _)) in enumerate(zip(layer.inputs[:4], host_in)):
            be.stage(slot, w, i)
        o = pos % t
        be.stage_wait(0)
        q, k, v = sf.vmm_interleaved_multi(be, x, [layer.wq, wk[o], wv[o]])
        qr = sf.rope_apply(be, q, cfg, pos)
        kr = sf.rope_apply(be, k, cfg, pos)
        cache = sf.v_append(be, cache, sf.make_v_pieces(be, cache, v, pos))
        cache = sf.k_append(be, cache, kr)
        maps = sf.qk_dot(be, qr, cache)
        att = sf.softmax_times_v(be, probs[:len(maps)], cache)
        be.stage_wait(1)
        sf.vmm_interleaved(be, h7, None, plan=layer.wo)
        be.stage_wait(2)
        sf.vmm_interleaved_multi(be, h3, [layer.wg, layer.wu])
        be.stage_wait(3)
        dn = sf.vmm_interleaved(be, h1, None, plan=layer.wd)
        # next token's RoPE plaintexts: encoded on the host while this token runs
        sf.rope_prepare(be, cfg, pos + 1, rope_level, 0)
        sf.rope_prepare(be, cfg, pos + 1, rope_level, (pos + 1) % t)
        return cache, maps, [att.data(), dn.data()]  # D2H: synchronises the token

    # two untimed warm-up tokens (positions 2047, 2048: the second opens a K-ct,
    # a V group and a score map) on the copy-on-write cache, which stays at n' = 2047
    c_w = cache
    for i in range(2):
        c_w, _, _ = token(c_w, layer.pos + i)
    del c_w
    sf.rope_prepare(be, cfg, layer.pos, rope_level, 0)
    sf.rope_prepare(be, cfg, layer.pos, rope_level, layer.pos % t)
    be.synchronize()
    per_token = []
    be.event_record(20)
    t0 = time.perf_counter()
    tok_log = os.environ.get("SF_STREAM_LOG")
    for i in range(T):
        if tok_log:
            print(f"[stream] token {i}", file=sys.stderr, flush=True)
        ti = time.perf_counter()
        cache, maps, res = token(cache, layer.pos + i)
        per_token.append((time.perf_counter() - ti) * 1e3)
    be.event_record(21)
    wall = (time.perf_counter() - t0) * 1e3 / T
    dev = be.event_elapsed_ms(20, 21) / T
    return {"value": round(wall, 3), "unit": "ms/token", "tokens": T, "n_prime": [NP - 1, NP - 1 + T],
            "device_ms_per_token": round(dev, 3), "first_token_ms": round(per_token[0], 3),
            "median_token_ms": round(float(np.median(per_token)), 3),
            "token_ms": [round(x, 1) for x in per_token],
            "h2d_bytes_per_token": int(sum(w.nbytes for w, _ in host_in)),
            "d2h_bytes_per_token": int(sum(r.nbytes for r in res)),
            "maps_at_end": len(maps), "k_cts_at_end": cache.n_prime // t + (1 if cache.n_prime % t else 0),
            "execution": "eager (host-issued); cache persists and grows; RoPE plaintexts encoded per position "
                         "(the next token's while the current one runs: sf_rope_prepare); value-piece masks of "
                         "every lane offset encoded at setup"}


def emulated_shards(be, sf, layer, steps, worlds=(2, 4, 8)):
    """Predicted strong scaling of ONE token over N GPUs, measured on this one:
    for every rank r of a world W, the rank's own work -- its partials (VMM giant
    groups, QK^T key-ct groups, Score*V giant groups; csrc/protocols.cpp *_partial),
    the W-way modular sum of the exchanged partials (sf_sum_partials over W
    ciphertexts: the same reads and adds as the peer-memory reduce kernel) and
    the replicated tail (reduce ladders, RoPE, appends, lane fold,
    relinearisation) -- is captured into a graph and timed with CUDA events.
    The prediction ignores the NVLink transfer itself (reported separately as
    bytes per exchange); a rank's step time is the max over ranks because every
    exchange waits for all of them."""
    from paper_2602_11470_b200 import shard
    x, h7, h3, h1, p0, p1 = layer.inputs
    wl = [layer.wq, layer.wk, layer.wv]

    def step_rank(r, W):
        be.set_value_shard(r, W)  # this rank's aligned companions only
        parts = shard.vmm_multi_partial(be, x, wl, r, W)
        q, k, v = shard.vmm_multi_finish(be, [shard.sum_partials(be, [p] * W) for p in parts], wl)
        qr = sf.rope_apply(be, q, layer.cfg, layer.pos)
        kr = sf.rope_apply(be, k, layer.cfg, layer.pos)
        cache = sf.v_append(be, layer.cache, sf.make_v_pieces(be, layer.cache, v, layer.pos))
        cache = sf.k_append(be, cache, kr)
        mp = shard.qk_dot_partial(be, qr, cache, r, W)
        maps = [shard.sum_partials(be, [m] * W) for m in mp]
        sv = shard.softmax_times_v_partial(be, [p0, p1], cache, r, W)
        att = shard.softmax_times_v_finish(be, [sv] * W, cache)
        po = shard.vmm_partial(be, h7, layer.wo, r, W)
        o = shard.vmm_finish(be, shard.sum_partials(be, [po] * W), layer.wo)
        gu = shard.vmm_multi_partial(be, h3, [layer.wg, layer.wu], r, W)
        g, u = shard.vmm_multi_finish(be, [shard.sum_partials(be, [p] * W) for p in gu], [layer.wg, layer.wu])
        pd = shard.vmm_partial(be, h1, layer.wd, r, W)
        dn = shard.vmm_finish(be, shard.sum_partials(be, [pd] * W), layer.wd)
        return [q, att, o, g, u, dn] + maps, [parts, mp, sv, gu, [po], [pd]]

    out = {}
    for W in worlds:
        per_rank, xbytes = [], 0
        for r in range(W):
            graph, (outs, partials) = be.capture(step_rank, r, W)
            if r == 0:  # bytes each rank publishes per token: every partial ciphertext of the step
                flat = [c for grp in partials for c in grp]
                xbytes = int(sum(2 * (c.level + 1) * 2 * SLOTS * 8 for c in flat if not c.is_zero))
            graph.launch()
            be.synchronize()
            be.event_record(0)
            for _ in range(steps):
                graph.launch()
            be.event_record(1)
            per_rank.append(round(be.event_elapsed_ms(0, 1) / steps, 3))
            del graph, outs, partials
        out[str(W)] = {"rank_ms": per_rank, "max_rank_ms": max(per_rank),
                       "exchange_bytes_published_per_rank": xbytes,
                       "nvlink_ms_at_900GBps": round(xbytes * (W - 1) / 900e9 * 1e3, 3)}
    be.set_value_shard(0, 1)
    return out


def hevmm_c1(sf, steps):
    """BASELINE.json configs[0] as a throughput number: independent 768x768 BSGS
    HE-VMMs (encrypted 1x768 activation x plaintext weight) at ring 2^15,
    level 4, 16 inputs per captured graph, outputs per second (SURVEY.md §8(d):
    one output ciphertext per VMM)."""
    slots, B = 1 << 14, int(os.environ.get("SF_HEVMM_BATCH", "16"))
    be = sf.Backend(slots, 4, alpha=2, seed=7)
    rng = np.random.default_rng(11)
    W = rng.normal(size=(768, 768)) / np.sqrt(768.0)
    ly = sf.make_interleaved(1024, slots, 0)
    plan = sf.VmmPlan(be, W, 768, 768, 4, 0, 0, True)
    xs = []
    for i in range(B):
        v = np.zeros(slots)
        v[np.arange(768) * ly.t] = rng.normal(size=768)
        xs.append(be.encrypt(v, 4, ly, seed=100 + i))
    run = lambda: sf.vmm_interleaved_many(be, xs, plan)  # noqa: E731  (one batched VMM over the 16 inputs)
    run()
    be.synchronize()
    graph, _ = be.capture(run)
    graph.launch()
    be.synchronize()
    be.event_record(0)
    for _ in range(steps):
        graph.launch()
    be.event_record(1)
    ms = be.event_elapsed_ms(0, 1) / steps
    be.synchronize()
    return {"value": round(B / (ms * 1e-3), 1), "unit": "ciphertexts/s", "ms_per_vmm": round(ms / B, 4),
            "config": f"768x768 BSGS HE-VMM (BASELINE configs[0]), ring 2^15, level 4, {B} independent inputs "
                      "batched through sf_vmm_interleaved_many per graph replay, device-resident, CUDA events"}


def c2_attention(sf, steps):
    """BASELINE.json configs[1]: GPT-2 attention, 12 heads x
    d_head 64 (run as H = 16 with 4 zero heads, d = 1024), ring 2^15 (2^14
    slots); the KV cache grows from n' = 128 to 1024 by per-token append. Each
    decode step = make_v_pieces + v_append + k_append of the new token, then
    qk_dot and softmax_times_v over the whole cache (kv_attention.cpp:131-241),
    issued eagerly through the public API (the cache grows, so every step has a
    new shape). Reported: the stream's mean ms per decode step (device time,
    CUDA events around the whole stream; and host wall), plus one captured step
    replayed at n' = 1024 (device-resident, graph)."""
    N, d, H = 16384, 1024, 16
    cfg = sf.AttentionConfig(N, d, H, 0, 1024)
    be = sf.Backend(N, 5, alpha=2, seed=3)
    t = cfg.t
    rng = np.random.default_rng(4)
    vs_in, ks_in = [], []
    for off in range(t):  # one fresh encryption per lane offset, reused by every token at that offset
        vs = np.full(N, 0.5)
        vs[np.arange(d) * t + off] = rng.normal(size=d)
        vs_in.append(be.encrypt(vs, 4, sf.make_interleaved(d, N, off, H).with_(deferred_mask=True), seed=100 + off))
        ks = np.zeros(N)
        ks[np.arange(d) * t + off] = rng.normal(size=d) * 0.15
        ks_in.append(be.encrypt(ks, 3, sf.make_interleaved(d, N, off, H), seed=200 + off))
    qs = np.zeros(N)
    qs[np.arange(d) * t] = rng.normal(size=d) * 0.15
    qc = be.encrypt(qs, 3, sf.make_interleaved(d, N, 0, H), seed=5)
    probs = [be.encrypt(np.full(N, 1.0 / 1024), 3, seed=6)]

    def append(cache, u):
        cache = sf.v_append(be, cache, sf.make_v_pieces(be, cache, vs_in[u % t], u))
        return sf.k_append(be, cache, ks_in[u % t])

    def step(cache, u):
        cache = append(cache, u)
        maps = sf.qk_dot(be, qc, cache)
        att = sf.softmax_times_v(be, probs[:len(maps)], cache)
        return cache, att

    cache = sf.KVCache(be, cfg)
    for u in range(128):  # the prompt stands in as appended tokens (off the timed region)
        cache = append(cache, u)
    step(cache, 128)  # warm: keys, masks, conversion tables
    be.synchronize()
    be.ledger.reset()
    be.event_record(0)
    t0 = time.perf_counter()
    for u in range(128, 1024):
        cache, att = step(cache, u)
    be.event_record(1)
    dev = be.event_elapsed_ms(0, 1)
    be.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    counts = be.ledger.totals().asdict()
    # one decode step at n' = 1023 -> 1024, captured and replayed (device-resident)
    n_before = cache  # noqa: F841 (kept alive)
    full = sf.KVCache(be, cfg)
    for u in range(1023):
        full = append(full, u)
    graph, _ = be.capture(step, full, 1023)
    graph.launch()
    be.synchronize()
    be.event_record(2)
    for _ in range(steps):
        graph.launch()
    be.event_record(3)
    g_ms = be.event_elapsed_ms(2, 3) / steps
    be.synchronize()
    return {"stream_ms_per_step": round(dev / 896, 3), "stream_wall_ms_per_step": round(wall / 896, 3),
            "graph_ms_per_step_at_1024": round(g_ms, 3), "steps": 896, "ledger_stream": counts,
            "config": "GPT-2 attention (12 heads x 64, as H=16, d=1024), ring 2^15, L=5, alpha=2: 896 decode "
                      "steps n'=128->1024, each append + QK^T + Score*V; device time (CUDA events) over the eager "
                      "stream, and one step at n'=1024 captured and replayed"}


def c3_linear(sf, steps):
    """BASELINE.json configs[2]: the GPT-2-small decoder-layer
    linear path per decode token at ring 2^16 (2^15 slots), level 4: Q/K/V
    (one multi-VMM of three 768x768 plans), the output projection 768x768, the
    FFN 768->3072 and 3072->768 BSGS HE-VMMs, captured into one graph.
    Reference bench weights (W = None plans), fresh encrypted inputs."""
    N, lvl = SLOTS, 4
    be = sf.Backend(N, lvl, alpha=2, seed=2)
    mk = lambda r, c: sf.VmmPlan(be, None, r, c, lvl, 0, 0, True)  # noqa: E731
    wq, wk, wv, wo, wu, wd = mk(768, 768), mk(768, 768), mk(768, 768), mk(768, 768), mk(768, 3072), mk(3072, 768)
    rng = np.random.default_rng(21)

    def fresh(d, seed):
        dp = 1 << (d - 1).bit_length()
        s = np.zeros(N)
        s[np.arange(d) * (N // dp)] = rng.normal(size=d)
        return be.encrypt(s, lvl, sf.make_interleaved(dp, N, 0), seed=seed)
    x, h, hu, hd = fresh(768, 1), fresh(768, 2), fresh(768, 3), fresh(3072, 4)

    def step():
        q, k, v = sf.vmm_interleaved_multi(be, x, [wq, wk, wv])
        o = sf.vmm_interleaved(be, h, None, plan=wo)
        u = sf.vmm_interleaved(be, hu, None, plan=wu)
        dn = sf.vmm_interleaved(be, hd, None, plan=wd)
        return [q, k, v, o, u, dn]

    step()
    be.synchronize()
    be.ledger.reset()
    graph, _ = be.capture(step)
    counts = be.ledger.totals().asdict()
    graph.launch()
    be.synchronize()
    be.event_record(0)
    for _ in range(steps):
        graph.launch()
    be.event_record(1)
    ms = be.event_elapsed_ms(0, 1) / steps
    be.synchronize()
    return {"ms_per_token": round(ms, 3), "vmm_ct_per_s": round(6 / (ms * 1e-3), 1), "ledger": counts,
            "config": "GPT-2-small layer linear path (QKV 3x768^2 multi-VMM, out 768^2, 768->3072, 3072->768), "
                      "ring 2^16, level 4, alpha=2, bench weights; one graph, CUDA events"}


def prefill_c4(sf, be, steps, n0=64):
    """SURVEY.md §8(f) rank 2 measured: the batched prefill of an n0-token
    prompt at the C4 layer shape (d 4096, 32 heads, ring 2^16) -- token-batched
    Q/K/V VMMs, batched RoPE, causal score maps, attention -- captured into one
    graph and replayed. The softmax between scores and attention is the
    reference's client hook; here it returns pre-made encrypted probability
    maps, as the decode bench does, so the timed region is homomorphic work."""
    cfg = sf.AttentionConfig(SLOTS, D, H, n0, NP)
    t = cfg.t
    P = (n0 + t - 1) // t
    lvl = 6
    r = np.arange(D, dtype=np.float64)[:, None]
    cidx = np.arange(D, dtype=np.float64)[None, :]
    Wm = np.sin(0.001 * (31.0 * r + cidx) + 0.25)  # the reference bench weight (slotforge_cli.cpp:88-92)
    plans = [sf.VmmBatchPlan(be, Wm, lvl) for _ in range(3)]
    rng = np.random.default_rng(13)
    xs = []
    for p in range(P):
        v = np.zeros(SLOTS)
        for tau in range(min(t, n0 - p * t)):
            v[np.arange(D) * t + tau] = rng.normal(size=D) / 8
        xs.append(be.encrypt(v, lvl, sf.make_interleaved(D, SLOTS, 0, H), seed=900 + p))
    made = {}

    def probs_fn(be_, maps, cfg_, n0_):
        if "p" not in made:  # first (eager) call: synthetic probabilities at each map's level
            made["p"] = [[[be_.encrypt(np.full(SLOTS, 1.0 / n0_), m.level, m.layout) for m in row] for row in mp]
                         for mp in maps]
        return made["p"]

    run = lambda: sf.prefill(be, xs, plans[0], plans[1], plans[2], cfg, probs_fn)  # noqa: E731
    run()
    be.synchronize()
    be.ledger.reset()
    graph, _ = be.capture(run)
    counts = be.ledger.totals().asdict()
    graph.launch()
    be.synchronize()
    be.event_record(0)
    for _ in range(steps):
        graph.launch()
    be.event_record(1)
    ms = be.event_elapsed_ms(0, 1) / steps
    be.synchronize()
    return {"ms_per_prompt": round(ms, 3), "ms_per_prompt_token": round(ms / n0, 3), "n0": n0,
            "config": f"prefill of {n0} tokens at the C4 layer shape (d {D}, {H} heads, ring 2^16, level {lvl}): "
                      "vmm_batch Q/K/V, rope_apply_batch, causal score maps, attention; one graph, CUDA events",
            "ledger": counts}


def nonlinear_c4(sf):
    """SURVEY.md §8(f) rank 3 measured at the C4 shape (ring 2^16): the
    homomorphic softmax over the two score maps of n' = 2048 (32 heads), the
    layer norm of a 4096-wide hidden vector and the SiLU of the 14336-wide gate
    projection, with the harness's desk-shallow schedules (nonlinear.py). Wall
    clock around synchronised calls: the client-side domain guard decrypts."""
    from paper_2602_11470_b200 import nonlinear as NL
    be = sf.Backend(SLOTS, 14, alpha=2, seed=17)
    rng = np.random.default_rng(19)
    gt = SLOTS // H
    maps = []
    for m in range(2):
        v = np.zeros(SLOTS)
        for h in range(H):
            v[h * gt:h * gt + gt] = rng.uniform(-8, -3, size=gt)  # normaliser inside the inverse domain
        maps.append(be.encrypt(v, 14, seed=40 + m))
    hid = np.zeros(SLOTS)
    lyh = sf.make_interleaved(D, SLOTS, 0, 1)
    hid[np.arange(D) * lyh.t] = rng.normal(size=D)
    xh = be.encrypt(hid, 14, lyh, seed=50)
    gate = be.encrypt(rng.uniform(-8, 8, size=SLOTS), 14, sf.make_interleaved(16384, SLOTS, 0, 1), seed=51)
    sm, nm, si = (NL.desk_spec("desk-shallow", f) for f in ("softmax", "norm", "silu"))
    nm.iterations, nm.depth_budget = 3, 0  # the harness's approx-mode norm (harness.cpp:353-374)
    for spec in (sm, nm, si):
        spec.strict_domain = False
    gamma, beta = 1 + 0.1 * rng.normal(size=D), 0.01 * rng.normal(size=D)
    ops = {"approx_softmax (2 maps, n'=2048, 32 heads)": lambda: NL.approx_softmax(be, maps, NP, H, sm),
           "approx_norm (d 4096)": lambda: NL.approx_norm(be, xh, gamma, beta, 1e-5, nm),
           "approx_silu (14336-wide gate, padded 16384)": lambda: NL.approx_silu(be, gate, si)}
    out = {}
    for name, fn in ops.items():
        be.ledger.reset()
        fn()
        be.synchronize()
        counts = be.ledger.totals().asdict()
        t0 = time.perf_counter()
        fn()
        be.synchronize()
        out[name] = {"ms": round((time.perf_counter() - t0) * 1e3, 2), "ledger": counts}
    return out


def cpu_twin_sample(be, sf, layer, alpha, gpu_phases):
    """SURVEY.md §8(d)(ii) + the bench's own word-parity check. The bit-exact CPU
    CKKS twin (oracle/ckks_oracle.cpp, OpenMP on every host core; test
    infrastructure, run here only as the checker / baseline, after the timed
    region) executes bounded samples of every stage of the step at the bench's
    parameters (ring 2^16, L = 7, this alpha, key seed 1, bench weights); the
    GPU runs the SAME samples on the same encryptions and every output word is
    compared. Per-stage CPU times are extrapolated to the full step with the
    stated factors:
      Q,K,V / out / up+gate / down: one full 4096x4096 VMM at level 4, scaled by
        (diagonals x limbs) of each projection relative to it;
      RoPE & Cache: measured in full (2 rope_apply, 128 V pieces, 2 appends);
      QK^T: 8 of the 256 K-cts (x 32);
      Score*V: one 40-token group (132 probability rotations + products) scaled
        by the step's 510 (group, variant) pairs."""
    out = {"kind": "port", "cores": os.cpu_count(), "stages": {}}
    try:
        sys.path.insert(0, ROOT)
        from oracle.ckks import CkksOracle, bench_weight as twin_bench_weight
        from oracle import protocols as P
        from oracle.layout import make_interleaved as oly
        o = CkksOracle(SLOTS, 7, alpha=alpha, seed=1)
        words, equal, checked = 0, True, []

        def cmp(name, g_ct, o_ct):
            nonlocal words, equal
            a, b = g_ct.data(), o_ct.data()
            same = a.shape == b.shape and bool(np.array_equal(a, b))
            equal = equal and same
            words += a.size
            checked.append(f"{name}: {'equal' if same else 'DIFFER'}")

        def enc(slots, lvl, lg, lo, seed):
            return be.encrypt(slots, lvl, lg, seed=seed), o.encrypt(slots, lvl, lo, seed=seed)

        rng = np.random.default_rng(77)
        t = SLOTS // D
        cfg_g, cfg_o = sf.AttentionConfig(SLOTS, D, H, 0, NP), P.AttentionConfig(SLOTS, D, H, 0, NP)
        # --- VMM unit: Q projection at level 4 with the bench's W = None plan
        xs = np.zeros(SLOTS)
        xs[np.arange(D) * t] = rng.normal(size=D)
        xg, xo = enc(xs, LEVELS["qkv"], sf.make_interleaved(D, SLOTS, 0), oly(D, SLOTS, 0), 501)
        W = twin_bench_weight(D, D)
        t0 = time.perf_counter()
        qo = P.vmm_interleaved(o, xo, W, bsgs=True)
        vmm_s = time.perf_counter() - t0
        cmp("vmm 4096^2 @ level 4 (bench plan)", sf.vmm_interleaved(be, xg, None, plan=layer.wq), qo)

        def diag_limbs(rows, cols, lvl):  # interleaved diagonals k = d_in d_out / N, times limbs
            p2 = lambda v: 1 << (v - 1).bit_length()  # noqa: E731
            return max(1, p2(rows) * p2(cols) // SLOTS) * (lvl + 1)
        unit = diag_limbs(D, D, LEVELS["qkv"])
        vmm_scale = {"Q, K, V": 3 * unit, "Output projection": diag_limbs(D, D, LEVELS["out"]),
                     "Up & Gate projection": 2 * diag_limbs(D, FF, LEVELS["up"]),
                     "Down projection": diag_limbs(FF, D, LEVELS["down"])}
        for ph, wgt in vmm_scale.items():
            out["stages"][ph] = {"sample": "one 4096^2 VMM at level 4", "sample_ms": round(vmm_s * 1e3, 1),
                                 "factor": round(wgt / unit, 3), "ms": round(vmm_s * 1e3 * wgt / unit, 1)}
        # --- RoPE & cache at position 2047 (cache of shared encryptions)
        pos = NP - 1
        off = pos % t
        dly_g = sf.make_interleaved(D, SLOTS, 0).with_(deferred_mask=True)
        dly_o = oly(D, SLOTS, 0).with_(deferred_mask=True)

        def rnd(o_=0):
            v = np.zeros(SLOTS)
            v[np.arange(D) * t + o_] = rng.normal(size=D)
            return v
        qg, qo2 = enc(rnd(), 3, dly_g, dly_o, 502)
        kg, ko = enc(rnd(off), 3, dly_g.with_(offset=off), dly_o.with_(offset=off), 503)
        vg, vo = enc(rnd(off), 3, dly_g.with_(offset=off), dly_o.with_(offset=off), 504)
        ka, kb = enc(rng.normal(size=SLOTS), 2, sf.make_interleaved(D, SLOTS, 0, H), oly(D, SLOTS, 0, H), 505)
        va, vb = enc(rng.normal(size=SLOTS), 2, None, None, 506)
        n_k = (pos + t - 1) // t
        cache_g = sf.kv_from_cts(be, cfg_g, pos, [ka] * n_k, [[va] * (2 * cfg_g.d_head - 1)] * 2)
        cache_o = P.KVCache(pos, [kb] * n_k, [[vb] * (2 * cfg_g.d_head - 1) for _ in range(2)])
        t0 = time.perf_counter()
        qr_o, kr_o = P.rope_apply(o, qo2, cfg_o, pos), P.rope_apply(o, ko, cfg_o, pos)
        c2_o = P.k_append(o, P.v_append(o, cache_o, P.make_v_pieces(o, vo, cfg_o, pos), cfg_o), kr_o, cfg_o)
        rope_s = time.perf_counter() - t0
        qr_g, kr_g = sf.rope_apply(be, qg, cfg_g, pos), sf.rope_apply(be, kg, cfg_g, pos)
        c2_g = sf.k_append(be, sf.v_append(be, cache_g, sf.make_v_pieces(be, cache_g, vg, pos)), kr_g)
        cmp("rope_apply(q) @ 2047", qr_g, qr_o)
        cmp("k_append (last K-ct)", c2_g.k_cts[-1], c2_o.k_cts[-1])
        cmp("v_append (group 1, variant 127)", c2_g.v_cts[1][127], c2_o.v_cts[1][127])
        out["stages"]["RoPE & Cache"] = {"sample": "full stage", "sample_ms": round(rope_s * 1e3, 1), "factor": 1.0,
                                         "ms": round(rope_s * 1e3, 1)}
        # --- QK^T over 8 distinct K-cts
        kk = [enc(rng.normal(size=SLOTS), 2, sf.make_interleaved(D, SLOTS, 0, H), oly(D, SLOTS, 0, H), 600 + j)
              for j in range(8)]
        qs = np.zeros(SLOTS)
        qs[np.arange(D) * t] = rng.normal(size=D)
        q2g, q2o = enc(qs, 2, sf.make_interleaved(D, SLOTS, 0, H), oly(D, SLOTS, 0, H), 610)
        kc_g = sf.kv_from_cts(be, cfg_g, 8 * t, [a for a, _ in kk], [[va] * (2 * cfg_g.d_head - 1)])
        kc_o = P.KVCache(8 * t, [b for _, b in kk], [[vb] * (2 * cfg_g.d_head - 1)])
        P.qk_dot(o, q2o, kc_o, cfg_o)  # rotation keys generated here, untimed
        t0 = time.perf_counter()
        mo = P.qk_dot(o, q2o, kc_o, cfg_o)
        qk_s = time.perf_counter() - t0
        cmp("qk_dot over 8 K-cts", sf.qk_dot(be, q2g, kc_g)[0], mo[0])
        out["stages"]["QK^T"] = {"sample": "8 of 256 K-cts (keys warm)", "sample_ms": round(qk_s * 1e3, 1),
                                 "factor": 32.0, "ms": round(qk_s * 32e3, 1)}
        # --- Score*V over one 40-token group
        ntok = 40
        pr = np.zeros(SLOTS)
        for h in range(H):
            pr[h * cfg_g.group_tokens:h * cfg_g.group_tokens + ntok] = 1.0 / ntok
        pg, po = enc(pr, 2, None, None, 620)
        sv_g = sf.kv_from_cts(be, cfg_g, ntok, [a for a, _ in kk[:5]], [[va] * (2 * cfg_g.d_head - 1)])
        sv_o = P.KVCache(ntok, [b for _, b in kk[:5]], [[vb] * (2 * cfg_g.d_head - 1)])
        lo, hi = P.touched_variants(cfg_o, ntok)
        t0 = time.perf_counter()
        ao = P.softmax_times_v(o, [po], sv_o, cfg_o)
        sv_s = time.perf_counter() - t0
        cmp("softmax_times_v (40 tokens)", sf.softmax_times_v(be, [pg], sv_g), ao)
        pairs_step = 2 * (2 * cfg_g.d_head - 1)
        out["stages"]["Score*V"] = {"sample": f"one {ntok}-token group ({hi - lo} pairs)",
                                    "sample_ms": round(sv_s * 1e3, 1), "factor": round(pairs_step / (hi - lo), 3),
                                    "ms": round(sv_s * 1e3 * pairs_step / (hi - lo), 1)}
        total = sum(v["ms"] for v in out["stages"].values())
        out.update({
            "sample": "bounded samples of every stage at the bench parameters on the bit-exact CPU CKKS twin "
                      "(OpenMP, all host cores); per-stage factors extrapolate to one decode token",
            "value": round((vmm_s + rope_s + qk_s + sv_s) * 1e3, 1), "unit": "ms of samples",
            "step_extrapolated_ms": round(total, 1),
            "gpu_step_ms": round(sum(gpu_phases.values()), 3) if gpu_phases else None,
            "gpu_speedup_extrapolated": round(total / sum(gpu_phases.values()), 1) if gpu_phases else None,
            "parity": {"bit_exact_twin": equal, "words_compared": int(words), "checked": checked}})
    except Exception as e:  # pragma: no cover
        out.update({"sample": f"failed: {e}"})
    return out


# ----------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nvtx-step", action="store_true", help="run one NVTX-ranged step after warm-up and exit")
    ap.add_argument("--alpha", type=int, default=2, help="special primes per key-switching digit")
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="split ONE token over the ranks (the default for --gpus > 1; with one GPU: a world of one)")
    ap.add_argument("--replicas", action="store_true",
                    help="with --gpus > 1: N independent replicas (throughput) instead of one sharded token")
    ap.add_argument("--shard-host", action="store_true",
                    help="with --shard: exchange on torch's stream (eager) instead of the library stream + graph")
    ap.add_argument("--shard-nccl", action="store_true",
                    help="with --shard: NCCL all-gather on the library stream instead of the peer-memory exchange")
    ap.add_argument("--no-extras", action="store_true",
                    help="only the headline step (skip C1/C2/C3/C5, prefill and nonlinearity lines)")
    ap.add_argument("--no-stream", action="store_true", help="skip the T-token decode stream (e2e_stream)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the reduced C5 NTT / key-switch sweep")
    ap.add_argument("--no-emulate", action="store_true",
                    help="skip the emulated per-rank timings of worlds 2/4/8 (N=1 only)")
    args = ap.parse_args()

    # NCCL announces its version on stdout at communicator creation unless told
    # otherwise; rank 0's stdout must carry exactly one JSON line
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `bench.py --gpus N` without a launcher: re-run under torch.distributed.run, one rank per GPU
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":  # host cores only: rank 0 runs, the other ranks exit without work
        run_reference(args, rank)
        return
    if world > 1 and not args.replicas:
        args.shard = True  # N > 1: one token split over the ranks (strong scaling, per-token latency)
    dist = None
    if world > 1 or args.shard:
        import torch
        import torch.distributed as dist
        ngpu = torch.cuda.device_count()
        local = local % max(ngpu, 1)  # more ranks than GPUs: ranks share devices (CUDA IPC still works)
        torch.cuda.set_device(local)
        backend = "nccl" if ngpu >= world else "gloo"  # NCCL refuses two ranks on one device
        if world > 1:
            dist.init_process_group(backend)
        else:  # --shard on one GPU: a world of one (exercises the exchange path)
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
        if backend == "gloo" and args.shard_nccl:
            raise SystemExit("--shard-nccl needs one GPU per rank")

    log = (lambda *a: None) if (args.quiet or rank != 0) else (lambda *a: print(*a, file=sys.stderr, flush=True))
    import paper_2602_11470_b200 as sf
    t0 = time.time()
    be = sf.Backend(SLOTS, 7, alpha=args.alpha, seed=1, device=local)
    layer = LlamaLayer(be, sf, log)
    log(f"[bench] setup {time.time() - t0:.1f}s")

    clk = Clocks(local).__enter__()  # sampling starts before the warm-up
    clk.wait_first()
    if args.shard:
        run_sharded(args, be, sf, layer, dist, rank, world, clk)
        dist.barrier()
        dist.destroy_process_group()
        return
    for _ in range(args.warmup):
        layer.step()
    be.synchronize()
    if args.nvtx_step:
        # profiling hook: one decode step inside an NVTX range, e.g.
        #   ncu --nvtx --nvtx-include "sf_step/" ... python bench.py --nvtx-step
        import torch
        torch.cuda.nvtx.range_push("sf_step")
        layer.step()
        be.synchronize()
        torch.cuda.nvtx.range_pop()
        clk.__exit__()
        return

    def barrier():
        if dist:
            import torch
            torch.cuda.synchronize()
            dist.barrier()

    # ---- eager reference timing (host-issued step, for the record)
    hprof = None
    if os.environ.get("SF_HOST_PROF"):
        import ctypes as C
        buf = C.create_string_buffer(1 << 16)
        sf._native.lib().sf_host_profile(buf, len(buf), 1)  # reset: count only the timed eager steps
    be.ledger.reset()
    barrier()
    be.synchronize()
    be.event_record(0)
    t_host = time.perf_counter()
    for _ in range(args.steps):
        outs = layer.step()
    t_host = (time.perf_counter() - t_host) * 1e3 / args.steps
    be.event_record(1)
    ms_eager = be.event_elapsed_ms(0, 1) / args.steps
    counts = be.ledger.totals()
    be.synchronize()
    # host issue cost per step from an empty launch queue (the loop above
    # blocks on the queue once it is a few hundred launches deep, so its wall
    # time is device time, not host work)
    t_idle = 0.0
    for _ in range(args.steps):
        be.synchronize()
        t0 = time.perf_counter()
        layer.step()
        t_idle += time.perf_counter() - t0
    be.synchronize()
    t_idle = t_idle * 1e3 / args.steps
    if os.environ.get("SF_HOST_PROF"):  # host time per internal scope over the eager steps (diagnostics)
        sf._native.lib().sf_host_profile(buf, len(buf), 1)
        rows = [l.rsplit(" ", 2) for l in buf.value.decode().splitlines() if l.strip()]
        hprof = {k: {"us_per_step": round(float(us) / args.steps, 1), "calls_per_step": int(n) // args.steps}
                 for k, us, n in sorted(rows, key=lambda r: -float(r[1]))[:25]}

    # ---- capture the decode step once into a CUDA graph (nothing runs during
    # the capture); every replay re-executes all of the step's kernels
    graph, gouts = be.capture(layer.step)
    graph.launch()
    be.synchronize()

    # ---- value: graph replays, device-resident inputs, CUDA events on the library stream
    barrier()
    be.synchronize()
    l0 = be.kernel_launches()
    clk.mark()
    be.event_record(0)
    for _ in range(args.steps):
        graph.launch()
    be.event_record(1)
    ms_total = be.event_elapsed_ms(0, 1)
    clk.__exit__()
    be.synchronize()
    barrier()
    launches = be.kernel_launches() - l0
    if dist:
        ms_total = reduce_ranks(dist, ms_total, dist.ReduceOp.MAX)
    ms_step = ms_total / args.steps
    value = ms_step / world  # whole-job: `world` independent tokens per step time


    # ---- roofline: live per-family kernel timing over the same steps
    import ctypes as C
    lib = sf._native.lib()
    _ = lib.sf_profile_begin(be.ctx, 0x3F)
    for _ in range(args.steps):
        layer.step()
    ms = (C.c_double * 6)()
    by = (C.c_double * 6)()
    nl = (C.c_longlong * 6)()
    lib.sf_profile_end(be.ctx, ms, by, nl)
    bf = (C.c_double * 6)()
    lib.sf_profile_butterflies(be.ctx, bf)
    # families: 0 row passes (plain / epilogue), 1 key-switch row stages (ks_row, ks_sum),
    # 2 MACs, 3 fused column stages (ModUp / ModDown / rescale conversions), 4 elementwise, 5 sampling
    fams = ["ntt_rows", "keyswitch_rows", "ctpt_mac", "fused_col", "elementwise", "sampling"]
    prof = {f: {"ms_per_step": ms[i] / args.steps, "launches_per_step": nl[i] / args.steps,
                # algorithmic-byte model (counts L2- and shared-memory-served re-reads: an
                # upper bound on DRAM traffic; measured DRAM bytes: profiles/r2_traffic_v7.json)
                "alg_GBps": (by[i] / (ms[i] * 1e-3) / 1e9) if ms[i] > 0 else None} for i, f in enumerate(fams)}
    dom = max(range(6), key=lambda i: ms[i])
    P = peaks()
    peak = P.get("hbm_gbs", 6650.0)
    achieved = by[dom] / (ms[dom] * 1e-3) / 1e9 if ms[dom] > 0 else 0.0
    traffic = None
    try:  # ncu DRAM bytes per launch of the same family (profiles/r2_traffic_v7.json, tools/traffic.py)
        traffic = json.load(open(os.path.join(ROOT, "profiles", "r2_traffic_v7.json")))["families"][fams[dom]][
            "dram_bytes_per_launch"]
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": fams[dom], "achieved": round(achieved, 1), "peak": peak,
                "unit": "GB/s", "frac": round(achieved / peak, 4),
                "traffic": traffic, "traffic_source": "profiles/r2_traffic_v7.json (ncu launch list, same family)",
                "peak_source": "measured" if not P.get("_fallback") else "fallback",
                "algorithmic_bytes_per_launch": by[dom] / max(nl[dom], 1),
                "avg_launch_us": ms[dom] * 1e3 / max(nl[dom], 1)}

    # INT roofline: the NTT-bearing kernels (row / column / key-switch row passes)
    # against the measured register-resident butterfly peak
    try:
        bpk = json.load(open(os.path.join(ROOT, "profiles", "r1_butterfly_peak.json")))["exact_shoup_G_butterflies_per_s"]
    except Exception:
        bpk = None
    nt_ms = ms[0] + ms[1] + ms[3]
    bf_tot = bf[0] + bf[1] + bf[3]
    int_roofline = {"bound": "int (FMA-heavy pipe: 64-bit IMAD of the Shoup butterflies)",
                    "kernels": "ntt_rows + keyswitch_rows + fused_col families",
                    "butterflies_per_step": bf_tot / args.steps,
                    "achieved": round(bf_tot / (nt_ms * 1e-3) / 1e9, 1) if nt_ms > 0 else None,
                    "peak": bpk, "unit": "G butterfly/s",
                    "frac": round(bf_tot / (nt_ms * 1e-3) / 1e9 / bpk, 4) if (nt_ms > 0 and bpk) else None,
                    "peak_source": "profiles/r1_butterfly_peak.json (tools/microbench/butterfly.cu on B200)"}
    try:  # the same kernels' FMA-heavy pipe utilisation from the committed ncu capture
        pu = json.load(open(os.path.join(ROOT, "profiles", "r2_pipe_util_v7.json")))
        int_roofline["fmaheavy_pipe_pct_share_weighted"] = pu["share_weighted_fmaheavy_pct"]
        int_roofline["fmaheavy_pipe_source"] = "profiles/r2_pipe_util_v7.json (ncu, top-6 kernels, %.1f%% of the step)" % \
            pu["covered_step_share_pct"]
    except Exception:
        pass

    # ---- e2e: public API with host buffers (import inputs from pinned host
    # memory, read the results back), host wall clock around whole steps
    host_in = [(c.data(), c.level, c.scale, c.layout) for c in layer.inputs]
    pinned_in = []
    try:
        import torch
        for w, lvl, sc, ly in host_in:
            t = torch.empty(w.shape, dtype=torch.uint64 if hasattr(torch, "uint64") else torch.int64, pin_memory=True)
            a = t.numpy().view(np.uint64)
            a[...] = w
            pinned_in.append((a, lvl, sc, ly, t))
        pinned = True
    except Exception:
        pinned_in = [(w, lvl, sc, ly, None) for w, lvl, sc, ly in host_in]
        pinned = False
    h2d = sum(w.nbytes for w, *_ in host_in)
    d2h = 0
    be.synchronize()
    barrier()

    def e2e_run(g, outs, refill, pinned_out=None):
        t_imp = t_iss = t_rd = 0.0
        t_e = time.perf_counter()
        for _ in range(args.steps):
            t1 = time.perf_counter()
            if refill:
                for slot, (w, *_r) in zip(layer.inputs, pinned_in):  # H2D into the step's input ciphertexts
                    be.refill(slot, w)
            t2 = time.perf_counter()
            g.launch()
            t3 = time.perf_counter()
            if pinned_out is not None:  # read back inside the step (sf_ct_stage_out)
                be.synchronize()
                res = pinned_out
            else:
                res = [outs[4].data(), outs[8].data()]  # attention output and the layer's down-projection output
            t4 = time.perf_counter()
            t_imp, t_iss, t_rd = t_imp + t2 - t1, t_iss + t3 - t2, t_rd + t4 - t3
        be.synchronize()
        barrier()
        ms = (time.perf_counter() - t_e) * 1e3 / args.steps
        parts = {"h2d_enqueue_ms": round(t_imp * 1e3 / args.steps, 3), "graph_launch_ms": round(t_iss * 1e3 / args.steps, 3),
                 "readback_wait_ms": round(t_rd * 1e3 / args.steps, 3), "pinned": pinned}
        return ms, parts, sum(r.nbytes for r in res)

    # serial: all six uploads, then the step (the round-1 form, kept for comparison)
    e2e_serial, serial_parts, d2h = e2e_run(graph, gouts, True)
    gouts_lv = [o.level for o in gouts]
    graph_kernels = graph.kernel_launches
    del graph, gouts  # the timed graph's memory is not the stream's to fight over
    be.synchronize()
    e2e_ms, e2e_parts = e2e_serial, dict(serial_parts, h2d="serial: six sf_ct_refill copies, then the step")
    if pinned:
        # staged: the uploads are part of the captured step (sf_ct_stage on a side stream,
        # memcpy nodes re-reading the pinned words on every replay); each input joins
        # right before its stage, so only x's upload precedes the first kernel
        pin_out = []
        for lvl in (gouts_lv[4], gouts_lv[8]):
            t_o = torch.empty((2, lvl + 1, be.n), dtype=torch.uint64 if hasattr(torch, "uint64") else torch.int64,
                              pin_memory=True)
            pin_out.append((t_o.numpy().view(np.uint64), t_o))
        g_e2e, outs_e2e = be.capture(layer.step, staged=[w for w, *_r in pinned_in],
                                     staged_out=[a for a, _t in pin_out])
        g_e2e.launch()
        be.synchronize()
        barrier()
        e2e_ms, e2e_parts, d2h = e2e_run(g_e2e, outs_e2e, False, [a for a, _t in pin_out])
        e2e_parts["h2d"] = "staged: in-graph uploads overlapping the earlier stages (sf_ct_stage)"
        e2e_parts["d2h"] = "staged: in-graph read-backs into pinned words (sf_ct_stage_out), the attention output's overlapping the projections"
        e2e_parts["serial_ms"] = round(e2e_serial / world, 3)
        del g_e2e, outs_e2e
        be.synchronize()
    if dist:
        e2e_ms = reduce_ranks(dist, e2e_ms, dist.ReduceOp.MAX)
    be.synchronize()
    phases = layer.phase_ms(args.steps)  # last: its graph's memory must not disturb the timed graph
    stream = None
    if not args.no_stream:
        try:
            stream = token_stream(be, sf, layer, max(16, args.steps))
        except Exception as e:  # pragma: no cover
            stream = {"error": str(e)}
    emu = None
    if world == 1 and not args.no_emulate:
        try:
            emu = emulated_shards(be, sf, layer, args.steps)
            for W, e in emu.items():
                e["predicted_speedup"] = round(ms_step / e["max_rank_ms"], 2)
        except Exception as e:  # pragma: no cover
            emu = {"error": str(e)}
    hevmm = prefill = c2 = c3 = c5 = nonlin = None
    if not args.no_extras:
        try:
            hevmm = hevmm_c1(sf, args.steps)
        except Exception as e:  # pragma: no cover
            hevmm = {"value": None, "error": str(e)}
        try:
            prefill = prefill_c4(sf, be, args.steps)
        except Exception as e:  # pragma: no cover
            prefill = {"ms_per_prompt": None, "error": str(e)}
        try:
            c2 = c2_attention(sf, args.steps)
        except Exception as e:  # pragma: no cover
            c2 = {"error": str(e)}
        try:
            c3 = c3_linear(sf, args.steps)
        except Exception as e:  # pragma: no cover
            c3 = {"error": str(e)}
        c5 = None
        if not args.no_sweep:
            try:
                sys.path.insert(0, os.path.join(ROOT, "tools"))
                from sweep import sweep
                c5 = sweep(levels=(8, 24, 40), logns=(15, 16), alpha=4, log=lambda m: None)
            except Exception as e:  # pragma: no cover
                c5 = {"error": str(e)}
        try:
            nonlin = nonlinear_c4(sf)
        except Exception as e:  # pragma: no cover
            nonlin = {"error": str(e)}
    cpu = None if (args.no_cpu_baseline or rank != 0) else cpu_baseline_sample()
    parity = {"decrypt_max_rel_err": decrypt_parity(be, layer, outs), "tolerance": 1e-3}
    parity["decrypt_ok"] = all(v <= parity["tolerance"] for v in parity["decrypt_max_rel_err"].values())
    twin = None if (args.no_cpu_baseline or rank != 0) else cpu_twin_sample(be, sf, layer, args.alpha, phases)
    if twin and "parity" in twin:
        parity["bit_exact_twin"] = twin["parity"]["bit_exact_twin"]
        parity["twin_words_compared"] = twin["parity"]["words_compared"]
    vmm_per_step = 7
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "ms/token", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic: reference bench weights sin(0.001(31r+c)+0.25), N(0,1) activations/cache, seeded",
        "config": bench_config(args.alpha, world, False),
        # the decode step's 7 VMMs over the WHOLE step time (attention included); the
        # HE-VMM throughput proper is hevmm_c1
        "step_vmms_per_s": round(vmm_per_step * world / (ms_step * 1e-3), 2),
        "hevmm_c1": hevmm,
        "attention_c2": c2,
        "linear_c3": c3,
        "sweep_c5": c5,
        "prefill_c4": prefill,
        "nonlinear_c4": nonlin,
        "roofline": roofline,
        "int_roofline": int_roofline,
        "cpu_baseline": cpu,
        "cpu_baseline_ckks_twin": twin,
        "parity": parity,
        "emulated_sharding": emu,
        "e2e": {"value": round(e2e_ms / world, 3), "unit": "ms/token", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "breakdown": e2e_parts},
        "e2e_stream": stream,
        "gpu_launches": int(launches),
        "keys": dict(zip(("count", "GiB", "GiB_untruncated"),
                         (lambda k: (k[0], round(k[1] / 2**30, 2), round(k[2] / 2**30, 2)))(be.key_stats()))),
        "host_issue_ms_per_step": round(t_idle, 3),
        "host_issue_ms_per_step_queued": round(t_host, 3),
        "host_profile": hprof,
        "eager_ms_per_step": round(ms_eager, 3),
        "execution": f"CUDA graph of the whole decode step ({graph_kernels} kernels), replayed per token",
        "clocks": clk.summary(),
        "ledger_per_step": {k: v // args.steps for k, v in counts.asdict().items()},
        "kernel_families": prof,
        "phase_ms": phases,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
