"""Stall samples by reason and the instructions they fall on, from an
``ncu --page source --csv --print-source sass`` export (read here, no GPU)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hh = rows[1]
i_src = hh.index("Source")
cols = [c for c in hh if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: hh.index(c) for c in cols}
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
for r in rows[2:]:
    try:
        vals = {c: float(r[idx[c]] or 0) for c in cols}
    except (ValueError, IndexError):
        continue
    op = r[i_src].split()
    if not op:
        continue
    o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
    for c, x in vals.items():
        tot[c] += x
        byop[c][o] += x
s = sum(tot.values()) or 1.0
print(rows[0][0][:120])
for c, x in tot.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 10):
    print(f"  {c:24s} {x / s:.3f}  " + ", ".join(f"{o} {v / s:.3f}" for o, v in byop[c].most_common(4)))
