"""C5 microbench sweep (BASELINE.json configs[4]): batched NTT and key-switching
throughput vs RNS limb count at ring degree 2^15 / 2^16 on one B200.

  python tools/sweep.py [--out profiles/r1_sweep.json]

NTT: sf_bench_ntt (batched two-pass transforms, device time per limb NTT);
roofline = 16 n bytes per limb transform against the measured
HBM peak, and n/2 log2 n butterflies against the measured butterfly peak.
Key switching: sf_rotate_many of B ciphertexts at level L by one slot (one
batched hybrid key switch each); bytes per rotation = 8 n [2l + 2 beta (l + alpha) + 2l]
(SURVEY §8(d)), l = L + 1 limbs, beta = ceil(l / alpha).
"""
import argparse
import json
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def sweep(levels=(8, 16, 24, 32, 40), logns=(15, 16), alpha=4, log=print):
    """One row per (ring, L): batched NTT and batched key-switch timings."""
    import paper_2602_11470_b200 as sf
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    bpk = json.load(open(os.path.join(ROOT, "profiles", "r1_butterfly_peak.json")))["exact_shoup_G_butterflies_per_s"]
    rows = []
    for logn in logns:
        n = 1 << logn
        for L in levels:
            be = sf.Backend(n // 2, L, alpha=alpha, seed=7)
            limbs = L + 1
            count = max(1, 512 // limbs)
            be.bench_ntt(limbs, count, reps=2)  # warm-up (tables, scratch) before the timed call
            ms = be.bench_ntt(limbs, count, reps=10)
            ntt_gbs = 16.0 * n / (ms * 1e-3) / 1e9
            bfly = 0.5 * n * logn / (ms * 1e-3) / 1e9
            # key switching: B rotations by one slot at level L
            B = max(2, min(32, 256 // limbs))
            rng = np.random.default_rng(1)
            cts = [be.encrypt(rng.normal(size=n // 2), L, seed=100 + i) for i in range(B)]
            be.rotate_many(cts, 1)  # key generation + warm-up
            be.rotate_many(cts, 1)
            be.synchronize()
            reps = 3
            be.event_record(0)
            for _ in range(reps):
                outs = be.rotate_many(cts, 1)
            be.event_record(1)
            ks_ms = be.event_elapsed_ms(0, 1) / (reps * B)
            beta = math.ceil(limbs / alpha)
            ks_bytes = 8.0 * n * (2 * limbs + 2 * beta * (limbs + alpha) + 2 * limbs)
            ks_gbs = ks_bytes / (ks_ms * 1e-3) / 1e9
            err = float(np.max(np.abs(be.decrypt(outs[0]) - np.roll(be.decrypt(cts[0]), -1))))
            row = {"log_n": logn, "L": L, "limbs": limbs, "alpha": alpha, "beta": beta,
                   "ntt_us_per_limb": round(ms * 1e3, 3), "ntt_limb_per_s": round(1e3 / ms),
                   "ntt_hbm_frac": round(ntt_gbs / peaks["hbm_gbs"], 4),
                   "ntt_butterfly_frac": round(bfly / bpk, 4),
                   "ks_us_per_rotation": round(ks_ms * 1e3, 2), "ks_rotations_per_s": round(1e3 / ks_ms),
                   "ks_batch": B, "ks_alg_GBps": round(ks_gbs, 1), "ks_hbm_frac": round(ks_gbs / peaks["hbm_gbs"], 4),
                   "rotation_max_err": err}
            log(json.dumps(row))
            rows.append(row)
            del be, cts, outs
    return {"what": "C5 sweep: batched NTT / key-switch throughput vs limb count on one B200",
            "hbm_peak_gbs": peaks["hbm_gbs"], "butterfly_peak_G_per_s": bpk, "rows": rows}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--levels", default="8,16,24,32,40")
    ap.add_argument("--logn", default="15,16")
    ap.add_argument("--alpha", type=int, default=4)
    a = ap.parse_args()
    res = sweep([int(x) for x in a.levels.split(",")], [int(x) for x in a.logn.split(",")], a.alpha,
                log=lambda m: print(m, flush=True))
    if a.out:
        json.dump(res, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
