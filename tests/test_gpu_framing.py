"""overlap_save_run with caller-written block processors (the reference's seam
accepts any callable, spectral.py:84-92): GPU framing (dbp_frame_blocks) and
keep-centre assembly (dbp_unframe_blocks) around a host numpy callable or a
device torch operator.  Pure data movement, so the bar is bit-exact against the
oracle's restatement of the reference framing (oracle/dbp_port.py cut_blocks /
join_blocks, spectral.py:122-145) applying the same callable."""

import numpy as np
import pytest

import paper_1507_00921_b200 as pb
from paper_1507_00921_b200 import _native
from oracle import dbp_port

pytestmark = pytest.mark.gpu


def _sig(n, seed, dtype=np.complex128):
    g = np.random.default_rng(seed)
    s = (g.normal(size=(2, n)) + 1j * g.normal(size=(2, n))).astype(dtype)
    return pb.DualPolSignal(s[0], s[1], 56e9)


def _nonlinear(blk):
    # position-dependent and nonlinear, so any misplaced sample shows
    w = np.arange(blk.shape[1])
    return blk * np.exp(1j * np.abs(blk) ** 2) + 0.25 * np.roll(blk, 3, axis=1) * (w % 7)


def _oracle(sig, plan, fn):
    stacked = sig.stack()
    blocks = dbp_port.cut_blocks(stacked, plan.block_len, plan.overlap)
    return dbp_port.join_blocks(np.stack([np.asarray(fn(b)) for b in blocks]), stacked.shape[1], plan.overlap)


def test_host_callable_identity_every_length():
    # test_spectral.py:119-125 with the reference's own ``lambda b: b``
    plan = pb.OverlapPlan(128, 32)
    for n_total in range(1, 301):
        sig = _sig(n_total, n_total)
        out = pb.overlap_save_run(sig, plan, lambda b: b)
        np.testing.assert_array_equal(out.stack(), sig.stack())
        assert out.x.dtype == np.complex128 and out.sample_rate == sig.sample_rate


@pytest.mark.parametrize("n_blk,m", [(16, 0), (64, 17), (2048, 700), (4096, 1400), (8192, 1024)])
@pytest.mark.parametrize("n_total", [1, 7, 1348, 1349, 20000, 131072])
def test_host_callable_matches_oracle_framing(n_blk, m, n_total):
    plan = pb.OverlapPlan(n_blk, m)
    sig = _sig(n_total, n_blk + n_total)
    got = pb.overlap_save_run(sig, plan, _nonlinear).stack()
    np.testing.assert_array_equal(got, _oracle(sig, plan, _nonlinear))


def test_host_callable_jobs_bit_identical_and_errors():
    plan = pb.OverlapPlan(2048, 700)
    sig = _sig(50000, 3)
    one = pb.overlap_save_run(sig, plan, _nonlinear).stack()
    four = pb.overlap_save_run(sig, plan, _nonlinear, jobs=4).stack()
    np.testing.assert_array_equal(one, four)
    with pytest.raises(ValueError, match="expected \\(2, 2048\\)"):   # spectral.py:141-142
        pb.overlap_save_run(sig, plan, lambda b: b[:, :100])
    with pytest.raises(ValueError):
        pb.overlap_save_run(sig, plan, lambda b: b, jobs=0)
    with pytest.raises(TypeError):
        pb.overlap_save_run(sig, plan, 3)


@pytest.mark.parametrize("dtype", ["complex64", "complex128"])
def test_device_block_processor_matches_oracle(dtype):
    import torch

    plan = pb.OverlapPlan(2048, 700)
    np_dt = np.complex64 if dtype == "complex64" else np.complex128
    sig = _sig(262144, 11, np_dt)
    calls = []

    def op(blocks):   # one call on the whole (nb, 2, N) device stack
        calls.append(tuple(blocks.shape))
        assert blocks.is_cuda and str(blocks.dtype) == f"torch.{dtype}"
        return blocks * torch.exp(1j * blocks.abs() ** 2) + 0.5 * torch.roll(blocks, 5, dims=-1)

    got = pb.overlap_save_run(sig, plan, pb.DeviceBlockProcessor(op, dtype=dtype)).stack()
    nb = dbp_port.count_blocks(262144, 2048, 700)
    assert calls == [(nb, 2, 2048)]

    def ref(b):   # the same operator on each block, on the device, for the oracle framing
        t = torch.from_numpy(np.ascontiguousarray(b.astype(np_dt))[None]).cuda()
        return op(t)[0].cpu().numpy()

    calls.clear()
    want = _oracle(pb.DualPolSignal(sig.x.astype(np_dt), sig.y.astype(np_dt), 56e9), plan, ref)
    # elementwise + roll along the block: the same values whichever batch shape ran them
    np.testing.assert_array_equal(got, want.astype(np.complex128))
    with pytest.raises(ValueError):
        pb.overlap_save_run(sig, plan, pb.DeviceBlockProcessor(lambda b: b[:, :, :10]))


def test_frame_unframe_block_ranges_and_batch():
    # the C-ABI directly: a block range of a batch, both element widths
    import torch

    n, n_blk, m = 10007, 512, 100
    step, nb = n_blk - m, dbp_port.count_blocks(n, n_blk, m)
    g = np.random.default_rng(5)
    x = (g.normal(size=(3, 2, n)) + 1j * g.normal(size=(3, 2, n)))
    for np_dt, elem in ((np.complex64, 8), (np.complex128, 16)):
        d = torch.from_numpy(x.astype(np_dt)).cuda()
        b0, b1 = 4, nb - 3
        blocks = torch.empty((3, b1 - b0, 2, n_blk), dtype=d.dtype, device="cuda")
        _native.frame_blocks(d.data_ptr(), blocks.data_ptr(), n, 3, n_blk, m, b0, b1, elem)
        out = torch.zeros_like(d)
        _native.unframe_blocks(blocks.data_ptr(), out.data_ptr(), n, 3, n_blk, m, b0, b1, elem)
        torch.cuda.synchronize()
        hb, ho = blocks.cpu().numpy(), out.cpu().numpy()
        for i in range(3):
            np.testing.assert_array_equal(hb[i], dbp_port.cut_blocks(x[i].astype(np_dt), n_blk, m)[b0:b1])
            lo, hi = b0 * step, min(n, b1 * step)
            np.testing.assert_array_equal(ho[i][:, lo:hi], x[i].astype(np_dt)[:, lo:hi])
            assert not ho[i][:, :lo].any() and not ho[i][:, hi:].any()
