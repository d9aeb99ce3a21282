"""Static SASS opcode mix of one kernel instantiation (cuobjdump -sass), with
the FMA-heavy-pipe opcodes (IMAD*, the 32-bit integer multiplies the 64-bit
modular products decompose into) grouped.
  python tools/sass_mix.py paper_2602_11470_b200/build/ntt.cu.o 'fused_col_kernelILi8ELi8ELi8ELi1ELb1E'"""
import collections
import re
import subprocess
import sys

obj, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
blocks = re.split(r"\n\s+Function : ", out)
for b in blocks[1:]:
    name = b.split("\n", 1)[0].strip()
    if pat not in name:
        continue
    ops = collections.Counter()
    for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", b):
        ops[m.group(1)] += 1
    tot = sum(ops.values())
    print(f"{name}: {tot} instructions")
    imad = {k: v for k, v in ops.items() if k.startswith("IMAD")}
    print(f"  IMAD* (FMA-heavy pipe): {sum(imad.values())} ({100 * sum(imad.values()) / tot:.1f}%)")
    for k, v in sorted(imad.items(), key=lambda kv: -kv[1]):
        print(f"    {k:24s} {v}")
    print("  top opcodes:")
    for k, v in ops.most_common(20):
        print(f"    {k:24s} {v}")
