"""Executable numpy model of the fused kernel's FFT data movement.

A line-by-line restatement of ``conv_pass`` / ``side_index`` /
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


def xchg2(g: Geo2, p: int, i: int) -> int:
    if p + 1 == g.NP - 1:
        return i + (i >> 4)          # pad16: one pad element per 16
    return i


def conv_model2(block: np.ndarray, table: np.ndarray, logn: int, trace=None) -> np.ndarray:
    """Emulate the v2 conv_pass<LOGN,0> on one polarisation."""
    g = Geo2(logn)
    N, T = g.N, g.T
    tw = twiddles2(g)
    regs = np.zeros((T, 16), dtype=np.complex128)
    for t in range(T):
        for m in range(16):
            regs[t, m] = block[t + T * m]
    plane = np.full(N + N // 16, np.nan + 0j)

    def dft(v, inv):
        return np.fft.ifft(v) * v.size if inv else np.fft.fft(v)

    def read_base(t, ls1):
        return ((t >> ls1) << (ls1 + 4)) + (t & ((1 << ls1) - 1))

    def rec(p):
        if g.NP == 1:
            for t in range(T):
                regs[t] = dft(regs[t], False) * table[:16]
                regs[t] = dft(regs[t], True)
            return
        if p < g.NP - 1:
            ls1 = g.log_s(p + 1)
            for t in range(T):
                if p == 0:
                    for q in range(g.G0):
                        idx = [q + g.G0 * e for e in range(g.R0)]
                        u = dft(regs[t, idx], False)
                        for k in range(1, g.R0):
                            u[k] *= tw[(k - 1) * (N // g.R0) + t + T * q]
                        regs[t, idx] = u
                else:
                    s = 1 << g.log_s(p)
                    regs[t] = dft(regs[t], False)
                    for k in range(1, 16):
                        regs[t, k] *= tw[g.tw_offset(p) + (t & (s - 1)) + (k - 1) * s]
            plane[:] = np.nan
            for t in range(T):
                for m in range(16):
                    a = xchg2(g, p, t + T * m)
                    if trace is not None:
                        trace.append(("w", p, t, a))
                    plane[a] = regs[t, m]
            for t in range(T):
                for e in range(16):
                    a = xchg2(g, p, read_base(t, ls1) + (e << ls1))
                    if trace is not None:
                        trace.append(("r", p, t, a))
                    regs[t, e] = plane[a]
            rec(p + 1)
            plane[:] = np.nan
            for t in range(T):
                for e in range(16):
                    plane[xchg2(g, p, read_base(t, ls1) + (e << ls1))] = regs[t, e]
            for t in range(T):
                for m in range(16):
                    regs[t, m] = plane[xchg2(g, p, t + T * m)]
            for t in range(T):
                if p == 0:
                    for q in range(g.G0):
                        idx = [q + g.G0 * e for e in range(g.R0)]
                        u = regs[t, idx].copy()
                        for k in range(1, g.R0):
                            u[k] *= np.conj(tw[(k - 1) * (N // g.R0) + t + T * q])
                        regs[t, idx] = dft(u, True)
                else:
                    s = 1 << g.log_s(p)
                    for k in range(1, 16):
                        regs[t, k] *= np.conj(tw[g.tw_offset(p) + (t & (s - 1)) + (k - 1) * s])
                    regs[t] = dft(regs[t], True)
        else:
            for t in range(T):
                u = dft(regs[t], False)
                for e in range(16):
                    u[e] *= table[t + T * e]
                regs[t] = dft(u, True)

    rec(0)
    out = np.zeros(N, dtype=np.complex128)
    for t in range(T):
        for m in range(16):
            out[t + T * m] = regs[t, m]
    return out
