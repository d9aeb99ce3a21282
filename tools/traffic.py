"""Per-family DRAM traffic of one decode step from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum:
average DRAM bytes per launch for each kernel family of bench.py's profile.
  python tools/traffic.py launches.csv > profiles/r1_traffic.json"""
import collections
import csv
import json
import sys

FAMILY = {"ntt_row_pass": "ntt_rows", "ntt_row_epi": "ntt_rows", "ks_row_kernel": "keyswitch_rows",
          "ks_sum_kernel": "keyswitch_rows", "fused_col_kernel": "fused_col", "vmm_mac_kernel": "ctpt_mac",
          "tensor_sum_kernel": "ctpt_mac", "mulpt_batch_kernel": "ctpt_mac", "mac_kernel": "ctpt_mac"}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
        "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
per = collections.defaultdict(dict)
for r in rows[1:]:
    per[(r[ii], r[ki])][r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1)
fam = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "seconds": 0.0})
for (_, name), m in per.items():
    short = name.split("(")[0].split("::")[-1].split("<")[0]
    f = FAMILY.get(short, "elementwise")
    fam[f]["launches"] += 1
    fam[f]["dram_bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    fam[f]["seconds"] += m.get("gpu__time_duration.sum", 0)
out = {f: {"launches": v["launches"], "dram_bytes_per_launch": v["dram_bytes"] / max(v["launches"], 1),
           "dram_GBps_serialised": v["dram_bytes"] / max(v["seconds"], 1e-12) / 1e9} for f, v in fam.items()}
json.dump({"source": sys.argv[1], "note": "ncu launch list of one eager decode step (serialised, cold L2 per launch)",
           "families": out}, sys.stdout, indent=1)
