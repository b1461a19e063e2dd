"""CPU proofs of the fused kernel's index algebra (no GPU needed)."""

import numpy as np
import pytest

from .layout_model import TILE_LEN, TILE_PITCH, fir_phys


def test_fir_padding_conflict_free():
    # float4 window loads at 16 t (stride 20 physical floats) hit 8 distinct 16-byte groups
    for m in range(0, 40, 4):
        groups = [(fir_phys(16 * t + m) // 4) % 8 for t in range(8)]
        assert len(set(groups)) == 8


# ---- v2 (default) kernel: one polarisation per thread, radix R0 first ----

from .layout_model import Geo2, conv_model2, pair_layout, side2, twiddles2, xchg2  # noqa: E402


@pytest.mark.parametrize("logn", list(range(4, 14)))
def test_v2_conv_model_equals_fft_filter(logn):
    n = 1 << logn
    if n > 4096:
        pytest.skip("pure-python model too slow above 4096")
    rng = np.random.default_rng(100 + logn)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    h = np.exp(1j * rng.uniform(-np.pi, np.pi, n))
    got = conv_model2(x, h / n, logn)
    want = np.fft.ifft(np.fft.fft(x) * h)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-11 * np.max(np.abs(want)))


@pytest.mark.parametrize("logn", list(range(5, 14)))
def test_v2_exchanges_bijective_and_conflict_free(logn):
    # 8-byte accesses: the 16 lanes of one polarisation share a shared-memory phase
    g = Geo2(logn)
    n, T = g.N, g.T
    cta_boundaries = [p for p in range(g.NP - 1) if not (g.NP >= 3 and p == g.NP - 2)
                      and not (g.NP == 3 and g.R0 == 8 and p == 0)]   # paired: own test
    for p in cta_boundaries:
        idx = [xchg2(g, p, i) for i in range(n)]
        assert len(set(idx)) == n and max(idx) < n + n // 8
        if T < 16:
            continue
        ls1 = g.log_s(p + 1)
        for h0 in range(0, T, 16):
            lanes = range(h0, h0 + 16)
            for m in range(16):
                assert len({side2(g, p, t, m) % 16 for t in lanes}) == 16
                assert side2(g, p, h0, m) == xchg2(g, p, h0 + T * m)
            for e in range(16):
                banks = {xchg2(g, p, ((t >> ls1) << (ls1 + 4)) + (t & ((1 << ls1) - 1)) + (e << ls1)) % 16
                         for t in lanes}
                assert len(banks) == 16, (p, e)
    if g.NP >= 3:
        # the gathers of the exchange into pass NP-2 stay inside each half-warp's tile
        p, ls1 = g.NP - 3, 4
        for h in range(T // 16):
            reads = {xchg2(g, p, ((t >> ls1) << (ls1 + 4)) + (t & 15) + (e << ls1))
                     for t in range(16 * h, 16 * h + 16) for e in range(16)}
            assert min(reads) >= TILE_LEN * h and max(reads) < TILE_LEN * h + 256
        # tile accesses: 8-byte column side l + 18 k (fixed k): 16 consecutive elements;
        # 16-byte row side 18 l + e (e even, 16-byte aligned): 8 lanes per phase hit
        # 8 distinct 16-byte bank groups
        for k in range(16):
            assert len({(l + TILE_PITCH * k) % 16 for l in range(16)}) == 16
        for e in range(0, 16, 2):
            assert all((TILE_PITCH * l + e) % 2 == 0 for l in range(16))
            for l0 in (0, 8):
                assert len({((TILE_PITCH * l + e) // 2) % 8 for l in range(l0, l0 + 8)}) == 8
        assert TILE_PITCH * 15 + 15 < TILE_LEN


def test_v2_side_index_linear_forms():
    # the kernel's closed forms equal the padded index of t + T m
    for logn in range(5, 14):
        g = Geo2(logn)
        for p in range(g.NP - 1):
            for t in range(g.T):
                for m in range(16):
                    i = t + g.T * m
                    if g.NP >= 3 and p + 1 == g.NP - 2:
                        closed = (t + g.T * m + (((g.T * m) >> 8) << 5)) if g.T <= 256 else \
                                 (t + ((t >> 8) << 5)) + m * (g.T + g.T // 8)
                        assert closed == i + ((i >> 8) << 5)


def test_v2_twiddle_table_size():
    for logn in range(4, 14):
        g = Geo2(logn)
        if g.NP > 1:
            assert twiddles2(g).size == g.tw_offset(g.NP - 1)


def test_x01_paired_closed_forms_and_banks():
    # N = 2048: the kernel's 16-byte accesses st/ld_pair(2t + TILE_LEN (m/2)) and
    # ld/st_pair(TILE_LEN (t >> 4) + 2 (t & 15) + 32 e) address pair_layout exactly
    g = Geo2(11)
    T = g.T
    for t in range(T):
        for m in range(0, 16, 2):
            assert pair_layout(t + T * m) == 2 * t + TILE_LEN * (m // 2)
            assert pair_layout(t + T * (m + 1)) == 2 * t + TILE_LEN * (m // 2) + 1
        k0, ns = t >> 4, t & 15
        for e in range(8):
            i = 256 * k0 + 16 * e + ns
            assert pair_layout(i) == TILE_LEN * k0 + 32 * e + 2 * ns
            assert pair_layout(i + 128) == pair_layout(i) + 1
    # 16-byte accesses: 8 lanes per shared-memory phase hit 8 distinct 16-byte groups
    for t0 in range(0, T, 8):
        for m in range(0, 16, 2):
            assert len({((2 * t + TILE_LEN * (m // 2)) // 2) % 8 for t in range(t0, t0 + 8)}) == 8
        for e in range(8):
            assert len({((TILE_LEN * (t >> 4) + 2 * (t & 15) + 32 * e) // 2) % 8 for t in range(t0, t0 + 8)}) == 8


# ---- v9: decimation-in-time forward with fused input twiddles ----

from .layout_model import conv_model_dit, dit_fwd_base_exp, dit_inv_base_exp  # noqa: E402


@pytest.mark.parametrize("logn", list(range(4, 14)))
def test_dit_conv_model_equals_fft_filter(logn):
    # the v9 forward (input twiddles W_{R0 16^p}^{K_p} as powers of one base per
    # thread and pass) and the inverse walk give ifft(fft(x) * h) with the
    # unchanged digit-reversed table order (last_pass_bin)
    n = 1 << logn
    if n > 4096:
        pytest.skip("pure-python model too slow above 4096")
    rng = np.random.default_rng(300 + logn)
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    h = np.exp(1j * rng.uniform(-np.pi, np.pi, n))
    got = conv_model_dit(x, h / n, logn)
    want = np.fft.ifft(np.fft.fft(x) * h)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-11 * np.max(np.abs(want)))


def dit_table_sizes(g):
    """Entries of the kernel's DIT base tables (Geo::dit_fwd_size / dit_inv_size)."""
    fwd = [g.R0 * 16 ** (p - 1) for p in range(1, g.NP)]
    inv = [g.N // g.R0 if p == 0 else (1 << g.log_s(p)) for p in range(g.NP - 1)]
    return fwd, inv


@pytest.mark.parametrize("logn", list(range(5, 14)))
def test_dit_base_indices_fit_their_tables(logn):
    # every thread's base index lies inside its pass's table (forward: by
    # sub-problem K, the last pass by thread t; inverse: by g = t + T q or ns)
    g = Geo2(logn)
    fwd, inv = dit_table_sizes(g)
    for p in range(1, g.NP):
        for t in range(g.T):
            k, period = dit_fwd_base_exp(g, p, t)
            idx = t if p == g.NP - 1 else t >> g.log_s(p)
            assert idx < fwd[p - 1] and k < period and period == g.R0 * 16 ** p
            if p < g.NP - 1:
                assert k == idx
    for p in range(g.NP - 1):
        for t in range(g.T):
            for q in range(g.G0 if p == 0 else 1):
                k, period = dit_inv_base_exp(g, p, t, q)
                assert (t + g.T * q if p == 0 else t & ((1 << g.log_s(p)) - 1)) < inv[p]
