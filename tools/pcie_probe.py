"""Pinned host<->device copy bandwidth on the box (one direction and both at once)."""
import time
import torch

n = 1 << 30  # bytes
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(2):
    d_a.copy_(h_in, non_blocking=True); h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize()
t0 = time.perf_counter(); d_a.copy_(h_in, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
h_out.copy_(d_b, non_blocking=True); torch.cuda.synchronize(); t2 = time.perf_counter()
with torch.cuda.stream(s1):
    d_a.copy_(h_in, non_blocking=True)
with torch.cuda.stream(s2):
    h_out.copy_(d_b, non_blocking=True)
torch.cuda.synchronize(); t3 = time.perf_counter()
print(f"H2D {n / (t1 - t0) / 1e9:.1f} GB/s  D2H {n / (t2 - t1) / 1e9:.1f} GB/s  both {2 * n / (t3 - t2) / 1e9:.1f} GB/s total")
