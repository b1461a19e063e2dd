"""Multi-process (gloo, world_size 2) cover of the N>1 path's host logic.

Each rank takes its contiguous block range b_g = floor(g nb / G) of one
stream, builds its halo'd input span exactly as the GPU chunk
mode expects it (``OverlapPlan.input_span`` + ``gather_span``), runs the
oracle's block operator on its blocks only, and the ranks all-gather their
output spans.  The assembled stream must be bitwise equal to the unsharded
oracle run -- the same property the GPU tests assert on the device.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import dbp_port
from paper_1507_00921_b200.framing import OverlapPlan, gather_span, shard_blocks


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    rng = np.random.default_rng(5)
    n = 20000
    x = 0.02 * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))
    cfg = dbp_port.PortConfig("essfm", 1024, 300, -21.68, 1.3, 0.2, 80.0, 10, num_steps=2,
                              coeffs=np.array([0.6, 0.15, 0.05]), arrangement="symmetric")
    return x, cfg


def _shard_output(rank, world, x, cfg):
    plan = OverlapPlan(cfg.block_len, cfg.overlap)
    n = x.shape[1]
    b0, b1 = shard_blocks(plan.num_blocks(n), world)[rank]
    lo, hi = plan.input_span(b0, b1)
    span = gather_span(x, lo, hi)                      # what rank `rank` copies to its GPU
    op = dbp_port.block_operator(cfg, 56e9)
    step, lead = plan.usable, plan.lead
    olo, ohi = plan.output_span(b0, b1, n)
    out = np.zeros((2, ohi - olo), dtype=np.complex128)
    for b in range(b0, b1):
        blk = span[:, (b - b0) * step:(b - b0) * step + cfg.block_len]
        res = op(blk)[:, lead:lead + step]
        s = b * step - olo
        e = min(s + step, ohi - olo)
        out[:, s:e] = res[:, :e - s]
    return olo, ohi, out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, cfg = _case()
        olo, ohi, out = _shard_output(rank, world, x, cfg)
        gathered = [None] * world
        dist.all_gather_object(gathered, (olo, ohi, out))
        if rank == 0:
            full = np.zeros_like(x)
            for lo, hi, part in gathered:
                full[:, lo:hi] = part
            q.put(full)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_block_range_sharding_bit_equal_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x, cfg = _case()
    want = dbp_port.backpropagate_arrays(x, 56e9, cfg)
    np.testing.assert_array_equal(full, want)


def test_shard_plan_covers_every_block_once():
    for nb in (1, 7, 98, 796545):
        for parts in (1, 2, 3, 8):
            ranges = shard_blocks(nb, parts)
            assert ranges[0][0] == 0 and ranges[-1][1] == nb
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    plan = OverlapPlan(2048, 700)
    assert plan.input_span(3, 5) == (3 * 1348 - 350, 5 * 1348 - 350 + 700)
    assert plan.output_span(97, 98, 1 << 17) == (97 * 1348, 1 << 17)
