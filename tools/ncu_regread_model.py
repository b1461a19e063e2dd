"""Dynamic register-operand model of a kernel from an ncu source-page export
(``ncu -i X.ncu-rep --page source --csv --print-source sass``; read here, no GPU).

For every SASS line: warp-level executions x (FP-pipe issue cycles, vector
register-file reads not served by the operand reuse cache).  The fp_rate
probes (profiles/r2/fp_rate_probe.txt) put the per-SMSP register-file read
rate at ~2 32-bit registers per lane per clock (FFMA2 with three pair
operands 0.33/clk x 6, FADD2 0.49/clk x 4, FFMA 0.63/clk x 3) and the packed
ops at 2 FMA-pipe cycles, scalar FFMA/FADD/FMUL at 1.  Usage:
  python tools/ncu_regread_model.py src.csv duration_ms clock_mhz [sms]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hh = rows[1]
i_src, i_ex = hh.index("Source"), hh.index("Instructions Executed")
dur_ms, mhz = float(sys.argv[2]), float(sys.argv[3])
sms = int(sys.argv[4]) if len(sys.argv) > 4 else 148
PACKED = {"FFMA2", "FADD2", "FMUL2"}
SCALAR = {"FFMA", "FADD", "FMUL"}
ex_by = collections.Counter()
reads_by = collections.Counter()
fp_cycles = 0.0
reads = 0.0
total_ex = 0.0
for r in rows[2:]:
    try:
        ex = float(r[i_ex] or 0)
    except (ValueError, IndexError):
        continue
    s = r[i_src].strip()
    if not s or ex == 0:
        continue
    if s.startswith("@"):
        s = s.split(None, 1)[1] if " " in s else s
    op_full, _, rest = s.partition(" ")
    op = op_full.split(".")[0]
    total_ex += ex
    args = [a.strip() for a in rest.rstrip(";").split(",")]
    srcs = args[1:] if op not in ("STS", "ST", "STG", "STL", "RED", "ATOMS") else args
    nr = 0
    for a in srcs:
        a2 = a.lstrip("-|!").strip()
        m = re.match(r"\[?(R\d+)", a2)
        if not m or a2.startswith("RZ") or ".reuse" in a2:
            continue
        if op in PACKED:
            nr += 2 if "F32x2" in a2 else 1
        elif op.startswith("STS") or op.startswith("LDS"):
            w = re.search(r"\.(64|128)", op_full)
            nr += (int(w.group(1)) // 32 if w and not a2.startswith("[") else 1)
        else:
            nr += 1
    reads += nr * ex
    reads_by[op] += nr * ex
    ex_by[op] += ex
    if op in PACKED:
        fp_cycles += 2 * ex
    elif op in SCALAR:
        fp_cycles += ex
cyc = dur_ms * 1e-3 * mhz * 1e6       # elapsed SM cycles
per_smsp = sms * 4
print(f"warp instructions executed {total_ex:.4g}; elapsed {cyc:.4g} cycles per SMSP")
print(f"FP pipe (packed 2 cycles, scalar 1): {fp_cycles / per_smsp:.4g} cycles per SMSP = {fp_cycles / per_smsp / cyc:.3f} of elapsed")
print(f"register-file reads (not reuse-served, all instructions): {reads / per_smsp:.4g} per SMSP "
      f"= {reads / per_smsp / 2 / cyc:.3f} of elapsed at 2 per clock")
for op, v in reads_by.most_common(10):
    print(f"  {op:8s} executions {ex_by[op] / per_smsp:10.4g}/SMSP  reads {v / per_smsp:10.4g}/SMSP  "
          f"avg {v / max(ex_by[op], 1):.2f}")
