#!/usr/bin/env python3
"""Per-point instruction histogram from an ncu source-page SASS csv
(`ncu -i rep --page source --csv --print-source sass`):
    python tools/sass_hist.py <sass.csv> <points per launch> [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
pts = int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
hdr, data = rows[1], rows[2:]
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
c = Counter()
for r in data:
    if not r[ie].isdigit():
        continue
    toks = r[src].split()
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    c[op] += int(r[ie])
tot = sum(c.values())
print(f"{rows[0][1][:110]}")
print(f"thread instructions per point: {tot * 32 / pts:.1f}")
print(", ".join(f"{k} {v * 32 / pts:.2f}" for k, v in c.most_common(top)))
