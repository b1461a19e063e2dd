"""Per-phase stall samples of a kernel: SASS split at every BAR.SYNC (program order).

usage: ncu_phases.py <rep.ncu-rep> [min_pct]
Prints, per segment between barriers: executed warp instructions, share of all
stall samples, the top stall reasons and the segment's dominant opcodes.
"""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
min_pct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
iA, iS, iE, iN = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = {c: h.index(c) for c in reasons}
segs, cur = [], None


def new_seg(addr, label):
    return {"start": addr, "label": label, "inst": 0.0, "samples": 0.0, "stall": collections.Counter(),
            "ops": collections.Counter()}


cur = new_seg("start", "entry")
for r in rows[2:]:
    if not r or not r[iA].startswith("0x"):
        continue
    tok = r[iS].split()
    op = ""
    if tok:
        op = (tok[1] if tok[0].startswith("@") else tok[0])
    e = float(r[iE] or 0)
    s = float(r[iN] or 0)
    cur["inst"] += e
    cur["samples"] += s
    cur["ops"][op.split(".")[0]] += e
    for c in reasons:
        cur["stall"][c[6:]] += float(r[ri[c]] or 0)
    if op.startswith("BAR"):
        segs.append(cur)
        cur = new_seg(r[iA], op)
segs.append(cur)
tot_s = sum(x["samples"] for x in segs)
tot_i = sum(x["inst"] for x in segs)
for k, x in enumerate(segs):
    if x["samples"] / tot_s * 100 < min_pct:
        continue
    top = ", ".join(f"{n} {v / max(x['samples'], 1) * 100:.0f}%" for n, v in x["stall"].most_common(5))
    ops = ", ".join(f"{n} {v / max(x['inst'], 1) * 100:.0f}%" for n, v in x["ops"].most_common(5))
    print(f"seg {k:2d} after {x['label']:10s} @{x['start']}: samples {x['samples'] / tot_s * 100:5.1f}%  "
          f"inst {x['inst'] / tot_i * 100:5.1f}%\n      stalls: {top}\n      ops: {ops}")
