"""From an ncu launch list, print "kernel_regex:skip" for the largest launch of each of the top-K kernels."""
import collections
import csv
import sys

path, k = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 5
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, gi, vi = h.index("Kernel Name"), h.index("Grid Size"), h.index("Metric Value")
mi = h.index("Metric Name")
rows = [rows[0]] + [r for r in rows[1:] if r[mi] == "gpu__time_duration.sum"]
tot, idx, best = collections.Counter(), collections.Counter(), {}
for r in rows[1:]:
    name = r[ki].split("(")[0].split("::")[-1].split("<")[0]
    us = float(r[vi].replace(",", "")) / 1e3
    tot[name] += us
    if name not in best or us > best[name][1]:
        best[name] = (idx[name], us)
    idx[name] += 1
print(" ".join(f"{n}:{best[n][0]}" for n, _ in tot.most_common(k)))
