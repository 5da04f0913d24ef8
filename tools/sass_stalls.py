"""Per-region stall breakdown from an ncu source page (SASS) CSV:
    ncu -i rep --page source --csv --print-source sass > x.csv; python tools/sass_stalls.py x.csv"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
iSrc = hdr.index("Source")
tot = Counter()
by_op = defaultdict(Counter)
for r in data:
    src = r[iSrc].split()
    op = (src[1] if src and src[0].startswith("@") else (src[0] if src else "?")).split(".")[0]
    for k in reasons:
        v = r[hdr.index(k)]
        if v.isdigit() and int(v):
            tot[k] += int(v)
            by_op[op][k] += int(v)
s = sum(tot.values())
print("all:", ", ".join(f"{k[6:]} {100*v/s:.1f}%" for k, v in tot.most_common(8)))
for op, c in sorted(by_op.items(), key=lambda x: -sum(x[1].values()))[:12]:
    t = sum(c.values())
    print(f"{op:8s} {100*t/s:5.1f}%: " + ", ".join(f"{k[6:]} {100*v/s:.1f}" for k, v in c.most_common(4)))
