"""Condense an ncu --set full capture and a launch list into profiles/<round>/ summaries.

usage: profile_summary.py <rep.ncu-rep> <launches.csv> <out_prefix> [samples_per_launch]
writes <out_prefix>_ncu.json (key metrics, stalls, instruction mix) and
<out_prefix>_launches.csv (kernel, duration ns) and prints the JSON.
"""
import collections, csv, io, json, re, subprocess, sys

rep, launches, prefix = sys.argv[1], sys.argv[2], sys.argv[3]
samples = float(sys.argv[4]) if len(sys.argv) > 4 else 512 * 2 ** 18
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
d = dict(zip(h, v))
units = dict(zip(h, u))


def num(k):
    try:
        return float(d[k])
    except (KeyError, ValueError):
        return None


def scaled(k, to):
    val, un = num(k), units.get(k, "")
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "s": 1}.get(un, 1.0)
    return None if val is None else val * f / to


out = {
    "kernel": d.get("Kernel Name"),
    "duration_ms": scaled("gpu__time_duration.sum", 1e-3),
    "dram_read_bytes": scaled("dram__bytes_read.sum", 1),
    "dram_write_bytes": scaled("dram__bytes_write.sum", 1),
    "samples_per_launch": samples,
    "warp_instructions": num("smsp__inst_executed.sum"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "fma_pipe_pct": num("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
    "alu_pipe_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "lsu_pipe_pct": num("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "l1_wavefronts_pct": num("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
    "smem_wavefronts_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "smem_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "registers_per_thread": num("launch__registers_per_thread"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "stalls_per_issue": {},
}
out["dram_traffic_bytes"] = (out["dram_read_bytes"] or 0) + (out["dram_write_bytes"] or 0)
out["dram_bytes_per_sample"] = out["dram_traffic_bytes"] / samples
out["thread_instructions_per_sample"] = (out["warp_instructions"] or 0) * 32 / samples
for k in h:
    m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active.ratio", k)
    if m and (num(k) or 0) > 0.03:
        out["stalls_per_issue"][m.group(1)] = round(num(k), 3)
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
sh = srows[1]
iS, iE = sh.index("Source"), sh.index("Instructions Executed")
ops, tot = collections.Counter(), 0.0
for r in srows[2:]:
    try:
        e = float(r[iE] or 0)
    except (ValueError, IndexError):
        continue
    tok = r[iS].split()
    if tok:
        op = (tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]
        ops[op] += e
        tot += e
out["instruction_mix_pct"] = {o: round(c / tot * 100, 2) for o, c in ops.most_common(16)}
json.dump(out, open(prefix + "_ncu.json", "w"), indent=1)
if launches == "-":   # no launch list
    print(json.dumps(out, indent=1))
    sys.exit(0)
with open(launches) as fh:
    lines = [ln for ln in fh if not ln.startswith("==")]
lr = list(csv.reader(lines))
hh = lr[0]
ki, vi, ui = hh.index("Kernel Name"), hh.index("Metric Value"), hh.index("Metric Unit")
with open(prefix + "_launches.csv", "w", newline="") as fh:
    w = csv.writer(fh)
    w.writerow(["kernel", "duration", "unit"])
    for r in lr[1:]:
        w.writerow([r[ki][:80], r[vi], r[ui]])
print(json.dumps(out, indent=1))
