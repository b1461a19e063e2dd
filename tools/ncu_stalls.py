"""Per-source-line stall samples (by reason) for an .ncu-rep joined with nvdisasm line info."""
import collections, csv, io, re, subprocess, sys

rep, cubin = sys.argv[1], sys.argv[2]
reasons = sys.argv[3].split(",") if len(sys.argv) > 3 else ["stall_barrier", "stall_mio", "stall_short_sb", "stall_wait", "stall_long_sb", "stall_dispatch"]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
addr2line, cur = {}, None
for ln in dis.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*)", ln)
    if m:
        addr2line[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
iA = h.index("Address")
idx = {r: h.index(r) for r in reasons}
base = min(int(r[iA], 16) for r in rows[2:] if r and r[iA].startswith("0x"))
tot = collections.Counter()
per = {r: collections.Counter() for r in reasons}
for r in rows[2:]:
    if not r or not r[iA].startswith("0x"):
        continue
    line = addr2line.get(int(r[iA], 16) - base, "?")
    for rr in reasons:
        val = float(r[idx[rr]] or 0)
        per[rr][line] += val
        tot[rr] += val
for rr in reasons:
    print(f"== {rr} total {tot[rr]:.0f}")
    for line, c in per[rr].most_common(6):
        print(f"   {c / max(tot[rr], 1) * 100:5.1f}%  {line}")
