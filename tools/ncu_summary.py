"""Summarise an .ncu-rep: key raw metrics, instruction mix and stall reasons (read here, no GPU)."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for k in keys:
    if k in d:
        print(f"{k:80s} {d[k]} {u[h.index(k)]}")
for k in h:
    m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active.ratio", k)
    if m and float(d[k] or 0) > 0.05:
        print(f"  stall {m.group(1):24s} {float(d[k]):.3f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hh = rows[1]
iS, iE = hh.index("Source"), hh.index("Instructions Executed")
tot = 0.0
ops = collections.Counter()
for r in rows[2:]:
    try:
        e = float(r[iE] or 0)
    except ValueError:
        continue
    tok = r[iS].split()
    if not tok:
        continue
    op = tok[1] if tok[0].startswith("@") else tok[0]
    ops[op.split(".")[0]] += e
    tot += e
print("instruction mix:", ", ".join(f"{o} {c / tot * 100:.1f}%" for o, c in ops.most_common(14)))
