"""Attribute each SASS instruction of a cubin to its source line (code-size map)."""
import collections, re, subprocess, sys
cubin = sys.argv[1]
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
cur = None; cnt = collections.Counter(); func = None; per_func = collections.Counter()
for ln in out.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"; continue
    if re.search(r'\.text\.(\S+):', ln):
        func = re.search(r'\.text\.(\S+):', ln).group(1)
    if re.match(r'\s+/\*[0-9a-f]{4,5}\*/', ln):
        cnt[cur] += 1; per_func[func] += 1
for f, c in per_func.items(): print("function", f[:60], c)
for k, c in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30): print(f"{c:6d} {k}")
