"""The cloud claim's reciprocal quantize (ash_map.cu `quantize_try`), restated
in numpy: q = RN(x * RN(1 / cell)), tol = RN(|q| * 2^-50 + 2^-1000),
lo = RN(q - tol), hi = RN(q + tol); when floor(lo) == floor(hi) and
|q| < 2^30 the fast result floor(lo) must equal numpy's floor(x / cell)
(the reference's quantize, geometry.py:53), and otherwise the kernel divides
exactly.  Checked at the adversarial points: exact multiples of the cell and
1-4 ulps around them, across cells and magnitudes, plus zeros and
subnormals.  (The kernel forms tol with one FMA; the two roundings here give
a tol that is no smaller, so the same bracket argument applies.)"""
import numpy as np
import pytest


def fast_quantize(x: np.ndarray, cell: float):
    rc = 1.0 / cell
    q = x * rc
    tol = np.abs(q) * 2.0 ** -50 + 2.0 ** -1000
    lo, hi = np.floor(q - tol), np.floor(q + tol)
    ok = (np.abs(q) < 2.0 ** 30) & (lo == hi)
    return lo, ok


@pytest.mark.parametrize("cell", [0.005, 0.1, 1.0 / 3.0, 7.3e-4, 0.0058 * 8, 1e-7, 12345.678, 0.3, 2.5e-3])
def test_fast_path_agrees_with_numpy_where_taken(cell):
    rng = np.random.default_rng(int(cell * 1e7) % 9973)
    k = np.concatenate([np.arange(-3000, 3000), rng.integers(-2 ** 30, 2 ** 30, size=20000)]).astype(np.float64)
    base = k * cell
    pts = [base]
    for steps in (1, 2, 3, 4):
        up, dn = base.copy(), base.copy()
        for _ in range(steps):
            up, dn = np.nextafter(up, np.inf), np.nextafter(dn, -np.inf)
        pts += [up, dn]
    pts.append(rng.uniform(-2e6, 2e6, size=50000) * cell)
    pts.append(np.array([0.0, -0.0, 5e-324, -5e-324, 1e-310, -1e-310, 2.0 ** -1020]))
    x = np.concatenate(pts)
    with np.errstate(all="ignore"):
        want = np.floor(x / cell)
    fast, ok = fast_quantize(x, cell)
    assert np.array_equal(fast[ok], want[ok])
    # the slow path is rare away from the cell boundaries
    free = pts[-2]
    assert fast_quantize(free, cell)[1].mean() > 0.99
