"""Host-side check of the multiply-shift division the cast kernel uses to
decode its tile index (cast.cu `fast_div`, constants from `launch_model`):
for n < 2^31 and l = ceil(log2 d), m = floor(2^(31+l) / d) + 1 gives
floor(n / d) = (n * m) >> (31 + l) exactly.  The identity is checked here
against Python's integer division (a library primitive, not the formula),
at the divisors the configs use, at every power of two and its neighbours,
and at random divisors; n covers multiples of d and their neighbours up to
2^31 - 1."""
import numpy as np


def magic(d):
    l = 0
    while (1 << l) < d:
        l += 1
    return (1 << (31 + l)) // d + 1, 31 + l


def check(d, ns):
    m, s = magic(d)
    assert m < (1 << 32), d  # fits the unsigned 32-bit constant
    for n in ns:
        assert (n * m) >> s == n // d, (n, d)


def test_fast_div_exact():
    rng = np.random.default_rng(0)
    # tiles per image (4x8 tiles) / tiles per row / sensors of the configs
    divisors = {1, 2, 3, 4, 60 * 34, 60, 120 * 34, 120, 128 * 16, 128, 7, 1000003}
    for k in range(1, 31):
        divisors |= {(1 << k) - 1, 1 << k, (1 << k) + 1}
    divisors |= set(int(x) for x in rng.integers(1, 1 << 31, 200))
    top = (1 << 31) - 1
    for d in sorted(divisors):
        ns = {0, 1, d - 1, d, d + 1, top, top - 1}
        q = top // d
        for j in (1, 2, 3, q // 2, q - 1, q):
            if j >= 0:
                ns |= {max(j * d - 1, 0), j * d, min(j * d + 1, top)}
        ns |= set(int(x) for x in rng.integers(0, top, 64))
        check(d, [n for n in ns if 0 <= n <= top])
