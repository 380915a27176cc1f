"""Instruction mix of one kernel from `ncu -i rep --page source --csv --print-source sass` output."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(h) and r[h.index("Instructions Executed")].isdigit()]
ie = h.index("Instructions Executed")
ws = h.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie] or 0) for r in data)
tws = sum(int(r[ws] or 0) for r in data)
print("sass lines", len(data), "warp instructions", tot)
c = collections.Counter()
s = collections.Counter()
for r in data:
    t = r[1].split()
    op = t[1] if t[0].startswith("@") else t[0]
    op = op.split(".")[0]
    c[op] += int(r[ie] or 0)
    s[op] += int(r[ws] or 0)
for op, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{op:10s} instr {v / tot * 100:5.1f}%  stall-samples {s[op] / max(tws, 1) * 100:5.1f}%")
