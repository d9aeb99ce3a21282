"""Dynamic SASS profile of one ncu capture (the `--page source --csv
--print-source sass` export written by tools/gpu_profile.sh): executed warp
instructions per opcode (grouped by pipe family) and the hottest instructions
by warp-stall samples.

  python tools/sass_hot.py gpurun_out/TAG/big_ks_sum_kernel_8.sass.csv.gz [top]
"""
import collections
import csv
import gzip
import io
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = gzip.open(path, "rt").read() if path.endswith(".gz") else open(path).read()
lines = raw.splitlines()
start = next(i for i, ln in enumerate(lines) if ln.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))


def num(x):
    try:
        return float(x.replace(",", ""))
    except (ValueError, AttributeError):
        return 0.0


def family(op):
    if op.startswith("IMAD.WIDE"):
        return "IMAD.WIDE (fmaheavy, 64-bit result)"
    if op.startswith("IMAD"):
        return "IMAD* other (fmaheavy)"
    if op.startswith(("IADD3", "LOP3", "SHF", "SEL", "ISETP", "PRMT", "LEA", "IABS", "VIADD", "IMNMX", "FLO", "POPC")):
        return "ALU (int add / logic / select / compare)"
    if op.startswith(("LDG", "STG", "LDS", "STS", "LD", "ST", "ATOM", "RED", "LDC", "LDSM", "LDGSTS")):
        return "memory (LSU)"
    if op.startswith("SHFL"):
        return "SHFL"
    if op.startswith(("BRA", "BRX", "EXIT", "BAR", "WARPSYNC", "BSYNC", "BSSY", "CALL", "RET", "NOP", "DEPBAR")):
        return "control / barrier"
    if op.startswith(("MOV", "S2R", "S2UR", "CS2R", "R2UR", "UMOV", "ULDC", "UIADD", "ULOP", "USHF", "UIMAD", "ULEA",
                      "UISETP", "USEL", "UPRMT", "UFLO", "LDCU")):
        return "move / uniform"
    return "other"


inst = collections.Counter()
fam = collections.Counter()
samples = []
tot_inst = tot_samp = 0.0
for r in rows:
    src = r["Source"].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    n = num(r["Instructions Executed"])
    s = num(r["Warp Stall Sampling (All Samples)"])
    inst[op] += n
    fam[family(op)] += n
    tot_inst += n
    tot_samp += s
    samples.append((s, r["Address"][-5:], src[:70]))
print(f"{path}: {tot_inst:.3e} warp instructions executed, {tot_samp:.0f} stall samples")
print("by family:")
for k, v in fam.most_common():
    print(f"  {k:44s} {v:12.3e}  {100 * v / tot_inst:5.1f}%")
print("top opcodes:")
for k, v in inst.most_common(18):
    print(f"  {k:28s} {v:12.3e}  {100 * v / tot_inst:5.1f}%")
print(f"top {top} instructions by stall samples:")
for s, a, src in sorted(samples, reverse=True)[:top]:
    print(f"  {s:7.0f} {100 * s / max(tot_samp, 1):5.1f}%  {a}  {src}")
