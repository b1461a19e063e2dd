"""Concurrent callers on one device give the results of sequential calls.

The reference's functions are plain numpy and safe to call from several
threads; the GPU drop-ins share cached device objects per (device, size) --
DBP engines, the link simulator, the receiver -- so every call sequence on
one of them runs under that object's lock.  Each test runs the same work
from 6 threads at once and compares bitwise with the sequential results.
"""

from __future__ import annotations

import math
import warnings
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_1507_00921_b200 as pb
from oracle import waveforms

from .helpers import quiet_link

pytestmark = pytest.mark.gpu

THREADS = 6
SPAN = pb.FiberParams(beta2=-21.7, gamma=1.3, alpha_db_per_km=0.2, length=80.0)


def _parallel(fn, items):
    with ThreadPoolExecutor(max_workers=THREADS) as pool:
        return list(pool.map(fn, items))


def _waves(n, count, seed):
    rng = np.random.default_rng(seed)
    amp = math.sqrt(10 ** ((0.0 - 30) / 10) / 4.0)
    return [(amp * (rng.normal(size=(2, n)) + 1j * rng.normal(size=(2, n)))).astype(np.complex64)
            for _ in range(count)]


def test_concurrent_backpropagate_equals_sequential():
    cfg = pb.DbpConfig("essfm", pb.OverlapPlan(2048, 700), quiet_link(4, SPAN),
                       coeffs=pb.EssfmCoefficients(waveforms.gaussian_coeffs(17)))
    xs = _waves(30000, 12, 1)

    def run(x):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            return pb.backpropagate(pb.DualPolSignal(x[0], x[1], 56e9), cfg).stack()

    seq = [run(x) for x in xs]
    for got, want in zip(_parallel(run, xs), seq):
        np.testing.assert_array_equal(got, want)


def test_concurrent_link_simulation_equals_sequential():
    xs = _waves(1 << 14, 12, 2)
    link = pb.LinkConfig(span=SPAN, num_spans=2, amp_noise_figure_db=5.0, pol_rotation=True)

    def run(args):
        i, x = args
        return pb.propagate_link(pb.DualPolSignal(x[0], x[1], 56e9), link, pb.SsfmStepConfig(8), rng=100 + i).stack()

    items = list(enumerate(xs))
    seq = [run(a) for a in items]
    for got, want in zip(_parallel(run, items), seq):
        np.testing.assert_array_equal(got, want)


def test_concurrent_receivers_equal_sequential():
    # (dispersion-free) QPSK through the receiver chain from several threads,
    # batches of different sizes so the cached receiver is also regrown meanwhile
    tx, sym = waveforms.qpsk_rrc(1 << 12, seed=3)
    rng = np.random.default_rng(4)
    batches = []
    for k in range(8):
        b = 1 + k % 3
        noise = 0.05 * (rng.normal(size=(b, 2, tx.shape[1])) + 1j * rng.normal(size=(b, 2, tx.shape[1])))
        batches.append((tx[None] / np.sqrt(np.mean(np.abs(tx) ** 2)) + noise).astype(np.complex64))

    def run(x):
        return [(m.ber, m.evm_percent) for m in pb.receive_batch(x, 28e9, sym)]

    seq = [run(x) for x in batches]
    assert _parallel(run, batches) == seq
