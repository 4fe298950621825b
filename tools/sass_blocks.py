"""Instruction counts of an ncu SASS source page (csv) by execution count: per-task
(loop) cost of the layer kernel. usage: python tools/sass_blocks.py src.csv [lo hi]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
ie = idx["Instructions Executed"]
cnt = [float(r[ie] or 0) for r in data]
tot = sum(cnt)
print(f"total warp instructions {tot:.0f} over {len(data)} SASS lines")
c = Counter()
for k in cnt:
    c[int(k)] += k
for k, v in sorted(c.items(), key=lambda x: -x[1])[:25]:
    print(f"  exec {k:7d}: {v:10.0f} ({100 * v / tot:4.1f}%)  {v / max(k, 1):6.0f} lines")
