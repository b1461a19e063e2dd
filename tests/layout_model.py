"""Executable numpy model of the fused kernel's FFT data movement.

A line-by-line restatement of ``fft_fwd`` / ``fft_inv`` / ``side_index`` /
``xchg_index`` in paper_1507_00921_b200/csrc/dbp_block_kernel.cuh (thread
registers, shared-memory exchange addresses, the twiddle table layout of
``make_twiddles``), evaluated in complex128.  The CPU tests use it to prove
the index algebra (pass decomposition, digit-reversed spectrum order, swizzle
bijectivity and bank-conflict freedom) before any GPU run.
"""

from __future__ import annotations

import numpy as np


def fir_phys(u: int) -> int:
    return u + ((u >> 4) << 2)


# ---------------------------------------------------------------------------
# v2 kernel (one polarisation per thread, radix R0 first), dbp_block_kernel.cuh
# ---------------------------------------------------------------------------

class Geo2:
    def __init__(self, logn: int):
        self.logn = logn
        self.N = 1 << logn
        self.T = self.N // 16
        self.NP = (logn + 3) // 4
        self.LOGR0 = logn - 4 * (self.NP - 1)
        self.R0 = 1 << self.LOGR0
        self.G0 = 16 // self.R0

    def log_s(self, p):
        return self.logn - self.LOGR0 - 4 * p

    def tw_offset(self, p):
        off = 0
        for q in range(p):
            off += (self.R0 - 1) * (self.N // self.R0) if q == 0 else 15 * (1 << self.log_s(q))
        return off


def twiddles2(g: Geo2) -> np.ndarray:
    n, r0 = g.N, g.R0
    out = []
    if g.NP > 1:
        for k in range(1, r0):
            for gg in range(n // r0):
                out.append(np.exp(-2j * np.pi * ((gg * k) % n) / n))
        for p in range(1, g.NP - 1):
            s = n >> (g.LOGR0 + 4 * p)
            for k in range(1, 16):
                for ns in range(s):
                    out.append(np.exp(-2j * np.pi * ((ns * k) % (16 * s)) / (16 * s)))
    return np.asarray(out if out else [1.0 + 0j])


TILE_PITCH = 18                 # kernel kTilePitch
TILE_LEN = 16 * TILE_PITCH      # kernel kTileLen


def pair_layout(i: int) -> int:
    """X01_PAIRED layout (N = 2048): i and i + 128 adjacent, then pad256."""
    j = 256 * (i >> 8) + 2 * (i & 127) + ((i >> 7) & 1)
    return j + ((j >> 8) << 5)


def xchg2(g: Geo2, p: int, i: int) -> int:
    """Gather-side plane index of exchange p (kernel xchg_index)."""
    if g.NP == 3 and g.R0 == 8 and p == 0:
        return pair_layout(i)
    if g.NP == 2 and p == 0:
        return i + (i >> 4)                      # pad16
    if g.NP >= 3 and p + 1 == g.NP - 2:
        return i + ((i >> 8) << 5)               # pad256 (32 per 256)
    return i


def side2(g: Geo2, p: int, t: int, m: int) -> int:
    """Strided-side plane index of exchange p (kernel side_index)."""
    return xchg2(g, p, t + g.T * m)


def last_pass_bin(g: Geo2, t: int, e: int) -> int:
    if g.NP >= 3:
        return (t >> 4) + (g.N // 256) * (t & 15) + (g.N // 16) * e
    return t + g.T * e


def conv_model2(block: np.ndarray, table: np.ndarray, logn: int, trace=None) -> np.ndarray:
    """Emulate the kernel's conv_block<LOGN> on one polarisation (table: natural order, 1/N folded)."""
    g = Geo2(logn)
    N, T = g.N, g.T
    tw = twiddles2(g)
    tab = np.array([table[last_pass_bin(g, t, e)] for e in range(16) for t in range(T)])  # [t + T e]
    regs = np.zeros((T, 16), dtype=np.complex128)
    for t in range(T):
        for m in range(16):
            regs[t, m] = block[t + T * m]
    plane = np.full(N + N // 8, np.nan + 0j)

    def dft(v, inv):
        return np.fft.ifft(v) * v.size if inv else np.fft.fft(v)

    def read_base(t, ls1):
        return ((t >> ls1) << (ls1 + 4)) + (t & ((1 << ls1) - 1))

    def cta_exchange_fwd(p):
        ls1 = g.log_s(p + 1)
        plane[:] = np.nan
        for t in range(T):
            for m in range(16):
                plane[side2(g, p, t, m)] = regs[t, m]
        for t in range(T):
            for e in range(16):
                regs[t, e] = plane[xchg2(g, p, read_base(t, ls1) + (e << ls1))]

    def cta_exchange_inv(p):
        ls1 = g.log_s(p + 1)
        plane[:] = np.nan
        for t in range(T):
            for e in range(16):
                plane[xchg2(g, p, read_base(t, ls1) + (e << ls1))] = regs[t, e]
        for t in range(T):
            for m in range(16):
                regs[t, m] = plane[side2(g, p, t, m)]

    def last(t):
        u = dft(regs[t], False)
        for e in range(16):
            u[e] *= tab[t + T * e]
        regs[t] = dft(u, True)

    def rec(p):
        if g.NP == 1:
            for t in range(T):
                regs[t] = dft(regs[t], False) * tab[:16]
                regs[t] = dft(regs[t], True)
            return
        if p == 0:
            for t in range(T):
                for q in range(g.G0):
                    idx = [q + g.G0 * e for e in range(g.R0)]
                    u = dft(regs[t, idx], False)
                    for k in range(1, g.R0):
                        u[k] *= tw[(k - 1) * (N // g.R0) + t + T * q]
                    regs[t, idx] = u
            cta_exchange_fwd(0)
            if g.NP == 2:
                for t in range(T):
                    last(t)
            else:
                rec(1)
            cta_exchange_inv(0)
            for t in range(T):
                for q in range(g.G0):
                    idx = [q + g.G0 * e for e in range(g.R0)]
                    u = regs[t, idx].copy()
                    for k in range(1, g.R0):
                        u[k] *= np.conj(tw[(k - 1) * (N // g.R0) + t + T * q])
                    regs[t, idx] = dft(u, True)
            return
        s = 1 << g.log_s(p)
        for t in range(T):
            regs[t] = dft(regs[t], False)
            for k in range(1, 16):
                regs[t, k] *= tw[g.tw_offset(p) + (t & (s - 1)) + (k - 1) * s]
        if p == g.NP - 2:
            # half-warp-local transpose through the 288-element tile (pitch 18)
            for h in range(T // 16):
                tile = np.full(TILE_LEN, np.nan + 0j)
                base = TILE_LEN * h
                for l in range(16):
                    for k in range(16):
                        tile[l + TILE_PITCH * k] = regs[16 * h + l, k]
                        if trace is not None:
                            trace.append(("tile", h, base + l + TILE_PITCH * k))
                for l in range(16):
                    for e in range(16):
                        regs[16 * h + l, e] = tile[TILE_PITCH * l + e]
            for t in range(T):
                last(t)
            for h in range(T // 16):
                tile = np.full(TILE_LEN, np.nan + 0j)
                for l in range(16):
                    for e in range(16):
                        tile[TILE_PITCH * l + e] = regs[16 * h + l, e]
                for l in range(16):
                    for k in range(16):
                        regs[16 * h + l, k] = tile[l + TILE_PITCH * k]
        else:
            cta_exchange_fwd(p)
            rec(p + 1)
            cta_exchange_inv(p)
        for t in range(T):
            for k in range(1, 16):
                regs[t, k] *= np.conj(tw[g.tw_offset(p) + (t & (s - 1)) + (k - 1) * s])
            regs[t] = dft(regs[t], True)

    rec(0)
    out = np.zeros(N, dtype=np.complex128)
    for t in range(T):
        for m in range(16):
            out[t + T * m] = regs[t, m]
    return out


# ---------------------------------------------------------------------------
# v9 forward FFT: decimation in time (input twiddles, fused into the DFT)
# ---------------------------------------------------------------------------

def dit_fwd_base_exp(g: Geo2, p: int, t: int) -> tuple[int, int]:
    """(K, period) of the forward pass-p input twiddle base W_period^K for thread t.

    Pass p >= 1 multiplies its input register e by base^e, base =
    W_{R0 16^p}^{K_p}, K_p the thread's accumulated sub-problem index: the
    reader's sub-problem t >> log_s(p) after a CTA exchange, and
    (t >> 4) + (N / 256) (t & 15) after the half-warp tile transpose into the
    last pass (NP >= 3)."""
    period = g.R0 * 16 ** p
    if g.NP >= 3 and p == g.NP - 1:
        k = (t >> 4) + (g.N // 256) * (t & 15)
    else:
        k = t >> g.log_s(p)
    return k % period, period


def dit_inv_base_exp(g: Geo2, p: int, t: int, q: int = 0) -> tuple[int, int]:
    """(K, period) of the inverse pass-p input twiddle base W_period^{-K}:
    pass 0 group q: W_N^{-(t + T q)}; middle pass p: W_{16 S_p}^{-(t mod S_p)}."""
    if p == 0:
        return (t + g.T * q) % g.N, g.N
    s = 1 << g.log_s(p)
    return t & (s - 1), 16 * s


def conv_model_dit(block: np.ndarray, table: np.ndarray, logn: int) -> np.ndarray:
    """conv_block with the v9 forward (DIT, input twiddles as powers of one base
    per thread and pass) and the unchanged inverse walk (input twiddles)."""
    g = Geo2(logn)
    N, T = g.N, g.T
    tab = np.array([table[last_pass_bin(g, t, e)] for e in range(16) for t in range(T)])
    regs = np.zeros((T, 16), dtype=np.complex128)
    for t in range(T):
        for m in range(16):
            regs[t, m] = block[t + T * m]
    plane = np.full(N + N // 8, np.nan + 0j)
    pw = np.arange(16)

    def dft(v, inv):
        return np.fft.ifft(v) * v.size if inv else np.fft.fft(v)

    def w(k, period, sign=-1):
        return np.exp(sign * 2j * np.pi * k / period)

    def read_base(t, ls1):
        return ((t >> ls1) << (ls1 + 4)) + (t & ((1 << ls1) - 1))

    def xfwd(p):
        ls1 = g.log_s(p + 1)
        plane[:] = np.nan
        for t in range(T):
            for m in range(16):
                plane[side2(g, p, t, m)] = regs[t, m]
        for t in range(T):
            for e in range(16):
                regs[t, e] = plane[xchg2(g, p, read_base(t, ls1) + (e << ls1))]

    def xinv(p):
        ls1 = g.log_s(p + 1)
        plane[:] = np.nan
        for t in range(T):
            for e in range(16):
                plane[xchg2(g, p, read_base(t, ls1) + (e << ls1))] = regs[t, e]
        for t in range(T):
            for m in range(16):
                regs[t, m] = plane[side2(g, p, t, m)]

    def tile(forward):
        for h in range(T // 16):
            blk = regs[16 * h:16 * h + 16].copy()
            regs[16 * h:16 * h + 16] = blk.T

    def fwd_dit(p):
        for t in range(T):
            k, period = dit_fwd_base_exp(g, p, t)
            regs[t] = dft(regs[t] * w(k, period) ** pw, False)

    def inv_dit(p):
        for t in range(T):
            k, period = dit_inv_base_exp(g, p, t)
            regs[t] = dft(regs[t] * w(k, period, +1) ** pw, True)

    if g.NP == 1:
        for t in range(T):
            regs[t] = dft(dft(regs[t], False) * tab[:16], True)
    else:
        for t in range(T):
            for q in range(g.G0):
                idx = [q + g.G0 * e for e in range(g.R0)]
                regs[t, idx] = dft(regs[t, idx], False)
        for p in range(1, g.NP):
            if g.NP >= 3 and p == g.NP - 1:
                tile(True)
            else:
                xfwd(p - 1)
            fwd_dit(p)
        for t in range(T):
            regs[t] = dft(regs[t] * tab[t + T * pw], True)    # x table, last inverse pass (no twiddle)
        for p in range(g.NP - 2, 0, -1):
            if g.NP >= 3 and p == g.NP - 2:
                tile(False)
            else:
                xinv(p)
            inv_dit(p)
        xinv(0) if not (g.NP >= 3 and g.NP - 2 == 0) else None
        for t in range(T):
            for q in range(g.G0):
                idx = [q + g.G0 * e for e in range(g.R0)]
                k, period = dit_inv_base_exp(g, 0, t, q)
                regs[t, idx] = dft(regs[t, idx] * w(k, period, +1) ** np.arange(g.R0), True)
    out = np.zeros(N, dtype=np.complex128)
    for t in range(T):
        for m in range(16):
            out[t + T * m] = regs[t, m]
    return out
