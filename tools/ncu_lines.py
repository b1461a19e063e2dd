"""Join ncu per-SASS execution counts with nvdisasm line info: instructions per source line.

usage: ncu_lines.py <rep.ncu-rep> <kernel.cubin> [top]
"""
import collections, csv, io, re, subprocess, sys

rep, cubin = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
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
iA, iS, iE = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
base_addr = None
for r in rows[2:]:
    try:
        a0 = int(r[iA], 16)
    except (ValueError, IndexError):
        continue
    base_addr = a0 if base_addr is None else min(base_addr, a0)
per_line = collections.Counter()
per_line_ops = collections.defaultdict(collections.Counter)
tot = 0.0
for r in rows[2:]:
    try:
        a = int(r[iA], 16) - base_addr; e = float(r[iE] or 0)
    except ValueError:
        continue
    tok = r[iS].split()
    op = (tok[1] if tok and tok[0].startswith("@") else (tok[0] if tok else "?")).split(".")[0]
    line = addr2line.get(a, "?")
    per_line[line] += e
    per_line_ops[line][op] += e
    tot += e
for line, c in per_line.most_common(top):
    ops = ", ".join(f"{o}:{n / c * 100:.0f}%" for o, n in per_line_ops[line].most_common(4))
    print(f"{c / tot * 100:5.1f}%  {line:32s} {ops}")
