"""Per-opcode warp-stall breakdown of an `ncu --page source --csv` SASS dump.

    python scripts/stall_by_op.py SOURCE.csv [--lines N]
"""
import collections
import csv
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]


def f(r, k):
    try:
        return float(r[ix[k]] or 0)
    except (ValueError, IndexError):
        return 0.0


tot = collections.Counter()
per_op = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    src = r[ix["Source"]].split()
    if not src:
        continue
    op = src[1] if src[0].startswith("@") else src[0]
    op = op.split(".")[0]
    for s in stalls:
        v = f(r, s)
        tot[s] += v
        per_op[op][s] += v
    per_op[op]["inst"] += f(r, "Instructions Executed")
all_s = sum(tot.values())
print("stall totals:")
for s, v in tot.most_common():
    if v:
        print(f"  {s:26s} {100 * v / all_s:5.1f}%")
print("by opcode (share of all samples; top stall reasons):")
ops = sorted(per_op.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "inst"))
for op, c in ops[:18]:
    n = sum(v for k, v in c.items() if k != "inst")
    top = ", ".join(f"{k[6:]} {100 * v / all_s:.1f}" for k, v in c.most_common(5) if k != "inst" and v)
    print(f"  {op:8s} {100 * n / all_s:5.1f}%  inst {c['inst'] / 1e9:7.2f}G  [{top}]")
