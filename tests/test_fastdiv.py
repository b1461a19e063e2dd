"""The block -> (item, block) split by multiply-high (dbp_capi.cu launch(),
dbp_block_kernel.cuh process_group): for 32-bit operands,
umulhi64(~0 / d + 1, n) == n // d (Lemire et al.'s fastdiv).  The launcher only
takes this path when blocks_per_item and total_blocks fit 32 bits."""

import numpy as np


def _magic(d: int) -> int:
    return (2 ** 64 - 1) // d + 1


def test_fastdiv_exact_for_32_bit_operands():
    rng = np.random.default_rng(5)
    ds = [2, 3, 7, 97, 98, 195, 196, 1000, 65535, 65536, 2 ** 31 - 1, 2 ** 31, 2 ** 32 - 1]
    ds += [int(v) for v in rng.integers(2, 2 ** 32, size=200)]
    for d in ds:
        m = _magic(d)
        ns = [0, 1, d - 1, d, d + 1, 2 * d - 1, 2 * d, 2 ** 32 - 1, 2 ** 32 - 2]
        ns += [int(v) for v in rng.integers(0, 2 ** 32, size=200)]
        for n in ns:
            if n >= 2 ** 32:
                continue
            assert (m * n) >> 64 == n // d, (n, d)
