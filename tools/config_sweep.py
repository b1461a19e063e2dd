#!/usr/bin/env python
"""Every BASELINE configuration point through bench.py (clock-sampled lines).

    python tools/config_sweep.py [--steps 20] [--waveforms 512] > profiles/r2/configs_r2.jsonl

configs[0] (2048/700, ESSFM N_s=1 N_c=17, symmetric and linear-first),
configs[1] (FFE, N in {1024, 2048, 4096}, M = 700), configs[2] (SSFM-20
linear-first at 2048/700 and 8192/1024), configs[3] (N_s in {1, 2, 4} x N_c
in {1, 9, 17, 33} x N in {1024, 2048, 4096, 8192}, M per tools/sweep.py).
One bench.py run per point (its JSON line: value, rooflines, clocks), on the
512 x 2^18 per-GPU batch; a `config_point` key names the point.
"""
import argparse
import json
import subprocess
import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
M3 = {1024: 768, 2048: 1400, 4096: 1400, 8192: 1400}


def points():
    yield "config0-sym", ["--nc", "17"]
    yield "config0-lf", ["--nc", "17", "--arrangement", "linear-first"]
    for n in (1024, 2048, 4096):
        yield f"config1-ffe-{n}", ["--algorithm", "ffe", "--block-len", str(n), "--overlap", "700"]
    for n, m in ((2048, 700), (8192, 1024)):
        yield f"config2-ssfm20-{n}", ["--algorithm", "ssfm", "--num-steps", "20", "--arrangement", "linear-first",
                                      "--nc", "0", "--block-len", str(n), "--overlap", str(m)]
    for n in (1024, 2048, 4096, 8192):
        for ns in (1, 2, 4):
            for nc in (1, 9, 17, 33):
                yield f"config3-{n}-ns{ns}-nc{nc}", ["--block-len", str(n), "--overlap", str(M3[n]),
                                                      "--num-steps", str(ns), "--nc", str(nc)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--waveforms", type=int, default=512)
    ap.add_argument("--only", default="", help="substring filter on the point names")
    a = ap.parse_args()
    for name, args in points():
        if a.only and a.only not in name:
            continue
        cmd = [sys.executable, str(REPO / "bench.py"), "--steps", str(a.steps), "--warmup", "3", "--no-e2e",
               "--no-cpu-baseline", "--waveforms", str(a.waveforms), *args]
        res = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
        try:
            line = json.loads(res.stdout.strip().splitlines()[-1])
        except (IndexError, json.JSONDecodeError):
            print(json.dumps({"config_point": name, "error": res.stderr[-400:]}), flush=True)
            continue
        line["config_point"] = name
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
