"""Pipe utilisation, conflicts and DRAM bytes of the ncu --set full captures of one
tools/gpu_profile.sh run, weighted by each kernel's share of the step (launch list):

  python tools/pipe_util.py gpurun_out/TAG > profiles/rNN_pipe_util.json
"""
import collections
import csv
import glob
import json
import os
import sys

d = sys.argv[1]
rows = [r for r in csv.reader(open(os.path.join(d, "launches.csv"))) if len(r) > 10]
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
tot, step = collections.Counter(), 0.0
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
    us = float(r[vi].replace(",", "")) / 1e3
    tot[name] += us
    step += us
out = {"source": f"ncu --set full --clock-control none of the largest launch of each top kernel ({d}); "
                 "launch list of one decode step for the shares",
       "metric": "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed (the FMA-heavy pipe that "
                 "executes the 64-bit IMAD.WIDE of the modular products)",
       "kernels": {}}
wsum = wf = 0.0


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3,
         "ms": 1e3, "us": 1.0, "ns": 1e-3, "s": 1e6, "second": 1e6}


def g(dd, k, units=None):
    """metric value; bytes / microseconds when the unit row names a scale"""
    try:
        v = float(dd[k].replace(",", ""))
    except (KeyError, ValueError, AttributeError):
        return None
    return v * SCALE.get((units or {}).get(k, ""), 1.0)


for f in sorted(glob.glob(os.path.join(d, "big_*.raw.csv"))):
    rr = list(csv.reader(open(f)))
    dd = dict(zip(rr[0], rr[2]))
    un = dict(zip(rr[0], rr[1]))
    name = os.path.basename(f)[4:].rsplit("_", 1)[0]
    share = 100.0 * tot.get(name, 0.0) / step if step else 0.0
    fma = g(dd, "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed")
    bc = g(dd, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
    wv = g(dd, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    out["kernels"][name] = {
        "step_share_pct": round(share, 1),
        "duration_us": round(g(dd, "gpu__time_duration.sum", un), 1),
        "fmaheavy_pct": fma,
        "alu_pct": g(dd, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": g(dd, "sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "warps_active_pct": g(dd, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "dram_pct": g(dd, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "dram_bytes": (g(dd, "dram__bytes_read.sum", un) or 0) + (g(dd, "dram__bytes_write.sum", un) or 0),
        "smem_conflict_share_pct": round(100.0 * bc / wv, 1) if bc is not None and wv else None,
    }
    if fma is not None:
        wsum += share * fma
        wf += share
out["share_weighted_fmaheavy_pct"] = round(wsum / wf, 1) if wf else None
out["covered_step_share_pct"] = round(wf, 1)
json.dump(out, sys.stdout, indent=1)
print()
