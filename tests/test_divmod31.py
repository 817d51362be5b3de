"""The generic stage kernel's 31-bit index division (lsg_device.cuh
divmod31, multipliers from slab_params in lsg_host.cu): q = umulhi(x, m) >> (l-1)
with m = ceil(2^(31+l) / d), l = ceil(log2 d), must equal x // d for every
0 <= x < 2^31 and 2 <= d < 2^31.  Checked here with the same integer
arithmetic at the edges of every quotient step plus random dividends."""
import numpy as np


def magic(d):
    l = 0
    while (1 << l) < d:
        l += 1
    m = ((1 << (31 + l)) + d - 1) // d
    assert m < (1 << 32)
    return m, l - 1


def divmod31(x, d, m, sh):
    q = ((x * m) >> 32) >> sh
    return q, x - q * d


def test_divmod31_exact():
    rng = np.random.default_rng(7)
    divisors = list(range(2, 300)) + [2 ** k + e for k in range(2, 31) for e in (-1, 0, 1) if 2 <= 2 ** k + e < 2 ** 31]
    divisors += [int(v) for v in rng.integers(2, 2 ** 31, 200)]
    for d in divisors:
        m, sh = magic(d)
        xs = {0, 1, d - 1, d, d + 1, 2 ** 31 - 1, 2 ** 31 - 2, (2 ** 31 - 1) // d * d, (2 ** 31 - 1) // d * d - 1}
        xs |= {int(v) for v in rng.integers(0, 2 ** 31, 200)}
        xs |= {int(k) * d + o for k in rng.integers(0, (2 ** 31 - 1) // d + 1, 50) for o in (-1, 0, 1)}
        for x in xs:
            if 0 <= x < 2 ** 31:
                assert divmod31(x, d, m, sh) == divmod(x, d), (x, d)
