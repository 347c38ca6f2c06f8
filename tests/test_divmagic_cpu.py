"""The frame source's multiply-shift divisions (ash_map.cu `divmagic`:
position -> pixel, pixel -> image row): floor(n / d) == (n * m) >> k for
every n < 2^31 with k = 31 + ceil(log2 d), m = ceil(2^k / d)
(Granlund-Montgomery, Thm 4.2).  The same derivation restated in Python and
checked at the divisors the kernel meets (samples per pixel 1-4096, 27;
image widths up to 2^30 - 1) on the n where an error would first show: the
multiples of d and their neighbours at the top of the range, plus random n;
and the product stays inside 64 bits."""
import numpy as np


def divmagic(d: int):
    l = 0
    while (1 << l) < d:
        l += 1
    k = 31 + l
    return ((1 << k) + d - 1) // d, k


def _check(d: int, ns) -> None:
    m, k = divmagic(d)
    assert m <= 2 ** 32
    # the theorem's condition, then the identity itself
    assert 2 ** k <= m * d < 2 ** k + 2 ** (k - 31)
    for n in ns:
        assert n * m < 2 ** 64
        assert (n * m) >> k == n // d, (n, d)


def test_samples_per_pixel_divisors():
    rng = np.random.default_rng(0)
    top = 2 ** 31 - 1
    for d in list(range(1, 4097)) + [27]:
        q = top // d
        ns = {0, 1, d - 1, d, d + 1, top, top - 1, q * d, q * d - 1, (q - 1) * d + d - 1}
        ns |= set(int(x) for x in rng.integers(0, 2 ** 31, size=16))
        _check(d, sorted(n for n in ns if 0 <= n <= top))


def test_image_width_divisors():
    rng = np.random.default_rng(1)
    top = 2 ** 31 - 1
    ds = [320, 640, 1280, 1920, 4096, 37, 61, 5, 2 ** 20 - 1, 2 ** 20 + 1, 2 ** 29 + 7, 2 ** 30 - 1]
    ds += [int(x) for x in rng.integers(2, 2 ** 30, size=200)]
    for d in ds:
        q = top // d
        ns = {0, d - 1, d, top, q * d, q * d - 1} | set(int(x) for x in rng.integers(0, 2 ** 31, size=32))
        _check(d, sorted(n for n in ns if 0 <= n <= top))
