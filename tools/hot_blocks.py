"""Hot basic blocks of an ncu --set full report (SASS source page): instruction
share, stall share and opcode mix per straight-line block.
  python tools/hot_blocks.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = [r for r in rows[2:] if len(r) >= len(h)]
ia, isrc = h.index("Address"), h.index("Source")
iex, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
blocks, cur = [], None
for r in data:
    ex = float(r[iex] or 0)
    if cur and cur[0] == ex:
        cur[2] += 1
        cur[3].append(r[isrc])
        cur[4] += float(r[iss] or 0)
    else:
        cur = [ex, r[ia], 1, [r[isrc]], float(r[iss] or 0)]
        blocks.append(cur)
tot = sum(b[0] * b[2] for b in blocks)
ts = sum(b[4] for b in blocks) or 1
print(f"total warp instructions {tot / 1e6:.1f} M")
for b in sorted(blocks, key=lambda b: -b[0] * b[2])[:top]:
    ops = {}
    for x in b[3]:
        t = x.split()
        o = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")
        o = o.split(".")[0]
        ops[o] = ops.get(o, 0) + 1
    mix = ", ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:6])
    print(f"{b[1][-5:]} x{b[0]:.0f} len {b[2]} inst {100 * b[0] * b[2] / tot:.1f}% stall {100 * b[4] / ts:.1f}%  {mix}")
