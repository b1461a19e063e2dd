"""FP32 peak probes: scalar FFMA, packed FFMA2 and the two interleaved (is there a second FMA pipe?)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1507_00921_b200._native as n
for _ in range(2):
    print("ffma", n.probe_fp32_peak(0, 4096)[0], "ffma2", n.probe_fp32x2_peak(0, 4096)[0])
    for s in (2, 4, 8, 16):
        print("mixed", s, n.probe_fp32_mixed_peak(0, 4096, s)[0])
