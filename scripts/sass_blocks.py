"""Largest basic blocks of one kernel's SASS with their opcode mix.

    python scripts/sass_blocks.py LIB.so KERNEL_SUBSTRING [N]
"""
import collections
import re
import subprocess
import sys

lib, sub = sys.argv[1], sys.argv[2]
nshow = int(sys.argv[3]) if len(sys.argv) > 3 else 3
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", sass)
body = next(f for f in funcs[1:] if sub in f.split("\n")[0])
ins = []
for line in body.split("\n"):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for a, t in ins:
    m = re.search(r"BRA.*?(0x[0-9a-f]+)", t)
    if m:
        targets.add(int(m.group(1), 16))
blocks, cur = [], []
for a, t in ins:
    if a in targets and cur:
        blocks.append(cur)
        cur = []
    cur.append((a, t))
    if re.match(r"(@!?U?P\w+\s+)?(BRA|EXIT|RET|BAR)", t):
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
print(f"{len(ins)} instructions, {len(blocks)} blocks")
for b in sorted(blocks, key=len, reverse=True)[:nshow]:
    c = collections.Counter()
    for _, t in b:
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        c[op.split(".")[0]] += 1
    print(f"block 0x{b[0][0]:x}-0x{b[-1][0]:x}: {len(b)} instr: " + ", ".join(f"{k} {v}" for k, v in c.most_common()))
