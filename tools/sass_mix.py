#!/usr/bin/env python
"""Static SASS instruction mix of one kernel in an object file.

    python tools/sass_mix.py build/obj/dbp_kernel_n11.o 'dbp_block_kernelILi11ELi0E'
"""
import collections
import re
import subprocess
import sys


def mix(obj: str, pattern: str) -> collections.Counter:
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    cnt = collections.Counter()
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            continue
        if cur is None or pattern not in cur:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            cnt[m.group(2)] += 1
    return cnt


if __name__ == "__main__":
    c = mix(sys.argv[1], sys.argv[2])
    tot = sum(c.values())
    print(f"total {tot}")
    for k, v in c.most_common(25):
        print(f"{k:10s} {v}")
