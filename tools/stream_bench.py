"""BASELINE configs[4]: one continuous 2^30-sample dual-pol stream, sharded by block range.

    python tools/stream_bench.py [--log2-samples 30] [--steps 5]
    torchrun --nproc-per-node G tools/stream_bench.py ...

The stream (28 GBd, 2 sps, 0 dBm complex Gaussian stand-in) is defined tile
by tile (2^20 samples, torch generator seeded with the tile index), so every
GPU count sees the identical stream.  Rank g owns blocks [b_g, b_{g+1}),
b_g = floor(g nb / G) (multiples of N - M), builds its halo'd span
[b_g step - M/2, b_{g+1} step - M/2 + M) on its own device (cyclic wrap at
the stream ends) and runs ``dbp_run_chunk`` -- no collective on the data
path.  Prints one JSON line (rank 0): whole-stream Gsamples/s (max over
ranks), per-chunk latency, and a per-rank output checksum that must be
identical to the 1-GPU run's for the same sample ranges
(``--digest-splits K`` on a 1-rank run prints the digests of the K-way shard
ranges of its output, for comparison with a K-rank run).

``--backend gloo`` runs the collectives (barrier, max-time reduction, digest
gather, optional final gather) on CPU tensors, so a K-rank run also works with
several ranks on ONE GPU (ranks map to ``LOCAL_RANK % device_count``) -- the
multi-rank correctness check on a single-GPU box; its timing is not a scaling
number.
"""

import argparse
import hashlib
import json
import math
import os
import sys
import time
import warnings
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

TILE = 1 << 20


def tile_values(torch, idx, dev, amp):
    g = torch.Generator(device=dev)
    g.manual_seed(10_000 + idx)
    return torch.randn((2, TILE, 2), generator=g, device=dev) * amp


def build_span(torch, lo, hi, n, dev, amp):
    """Samples [lo, hi) of the circular stream as a (2, hi-lo, 2) float32 tensor."""
    out = torch.empty((2, hi - lo, 2), device=dev)
    pos = lo
    while pos < hi:
        g = pos % n
        tile, off = divmod(g, TILE)
        take = min(hi - pos, TILE - off, n - g)
        out[:, pos - lo:pos - lo + take] = tile_values(torch, tile, dev, amp)[:, off:off + take]
        pos += take
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2-samples", type=int, default=30)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--backend", choices=("nccl", "gloo"), default="nccl")
    ap.add_argument("--digest-splits", type=int, default=0,
                    help="1-rank runs: also print the output digests of the K-way shard ranges")
    ap.add_argument("--gather", action="store_true",
                    help="after timing, assemble the whole output stream on rank 0 (NCCL point-to-point over "
                         "NVLink; not part of the timed path) and report its digest and the gather time")
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    import bench
    import paper_1507_00921_b200 as pb

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if a.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    dev = f"cuda:{local}"
    red_dev = dev if a.backend == "nccl" else "cpu"
    warnings.simplefilter("ignore")
    args = bench.parse_args([])
    cfg = bench.make_cfg(args)
    eng = pb.get_engine(cfg, bench.SAMPLE_RATE, local)
    n = 1 << a.log2_samples
    nb = eng.num_blocks(n)
    b0, b1 = pb.shard_blocks(nb, world)[rank]
    lo, hi = cfg.plan.input_span(b0, b1)
    olo, ohi = cfg.plan.output_span(b0, b1, n)
    amp = math.sqrt(1e-3 / 4.0)
    span = build_span(torch, lo, hi, n, dev, amp)
    out = torch.empty((2, ohi - olo, 2), device=dev)
    stream = torch.cuda.Stream()

    def step():
        eng.native.run_chunk(span.data_ptr(), out.data_ptr(), n, 1, b0, b1, hi - lo, ohi - olo, stream.cuda_stream)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    digest = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
    digests = [None] * world
    if world > 1:
        dist.all_gather_object(digests, (rank, olo, ohi, digest))
    else:
        digests = [(0, olo, ohi, digest)]
    split_digests = None
    if world == 1 and a.digest_splits > 1:
        split_digests = []
        host = out.cpu().numpy()
        for k, (s0, s1) in enumerate(pb.shard_blocks(nb, a.digest_splits)):
            klo, khi = cfg.plan.output_span(s0, s1, n)
            split_digests.append([k, klo, khi, hashlib.sha256(host[:, klo - olo:khi - olo].tobytes()).hexdigest()[:16]])
    gather = None
    if a.gather:
        # optional final gather: rank r's output span [olo, ohi) -> rank 0, no data-path collective
        spans = [None] * world
        if world > 1:
            dist.all_gather_object(spans, (olo, ohi))
        else:
            spans = [(olo, ohi)]
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        if rank == 0:
            full = torch.empty((2, n, 2), device=dev)
            full[:, olo:ohi] = out
            for r in range(1, world):
                rlo, rhi = spans[r]
                buf = torch.empty((2, rhi - rlo, 2), device=red_dev)
                dist.recv(buf, src=r)
                full[:, rlo:rhi] = buf.to(dev)
            torch.cuda.synchronize()
            gather = {"seconds": time.perf_counter() - g0,
                      "digest": hashlib.sha256(full.cpu().numpy().tobytes()).hexdigest()[:16]}
        else:
            dist.send(out.contiguous().to(red_dev), dst=0)
    if rank == 0:
        ms_max = float(t.item())
        print(json.dumps({
            "metric": "ESSFM 1-step DBP Gsamples/s (dual-pol), configs[4] stream", "unit": "Gsamples/s",
            "value": n / (ms_max * 1e-3) / 1e9, "n_gpus": world, "stream_samples": n, "blocks": nb,
            "chunk_latency_ms": ms_max, "halo_samples": [cfg.plan.lead, cfg.plan.overlap - cfg.plan.lead],
            "shards": [list(d) for d in digests], "split_digests": split_digests, "backend": a.backend,
            "device_resident": True,
            "gather": gather,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
