"""Pinned-copy bandwidth with the process bound to each NUMA node's CPUs (e2e placement check)."""
import os
import subprocess
import sys
import time
from pathlib import Path


def gpu_local_cpus(dev=0):
    import torch
    bus = torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(torch.cuda.get_device_properties(dev), "pci_bus_id") else None
    out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                         capture_output=True, text=True).stdout.strip()
    bus = out.lower().replace("00000000:", "0000:")
    p = Path(f"/sys/bus/pci/devices/{bus}/local_cpulist")
    node = Path(f"/sys/bus/pci/devices/{bus}/numa_node")
    return bus, (p.read_text().strip() if p.exists() else None), (node.read_text().strip() if node.exists() else None)


def parse(cpulist):
    cpus = set()
    for part in cpulist.split(","):
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        elif part:
            cpus.add(int(part))
    return cpus


def measure():
    import torch
    n = 1 << 30
    h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h_in.fill_(1)
    h_out.fill_(2)
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        d_a.copy_(h_in, non_blocking=True)
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); d_a.copy_(h_in, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    h_out.copy_(d_b, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize(); t3 = time.perf_counter()
    return n / (t1 - t0) / 1e9, n / (t2 - t1) / 1e9, 2 * n / (t3 - t2) / 1e9


if __name__ == "__main__":
    if len(sys.argv) > 1:
        os.sched_setaffinity(0, parse(sys.argv[1]))
        print(sys.argv[1], "H2D %.1f D2H %.1f both %.1f GB/s" % measure())
    else:
        print("gpu", gpu_local_cpus(), "cpus", os.cpu_count(), "allowed", len(os.sched_getaffinity(0)))
        nodes = sorted(Path("/sys/devices/system/node").glob("node[0-9]*"))
        for nd in nodes:
            cl = (nd / "cpulist").read_text().strip()
            subprocess.run([sys.executable, __file__, cl])
        print("unbound", "H2D %.1f D2H %.1f both %.1f GB/s" % measure())
