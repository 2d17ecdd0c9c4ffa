"""The sweep's hoisted-reciprocal division equals IEEE x/d bitwise."""

import ctypes as C

import numpy as np
import pytest

from paper_2510_22221_b200 import _native

pytestmark = pytest.mark.gpu

SPACINGS = [10e-6, 8e-6, 6e-6, 5e-6, 4e-6, 3e-6, 2e-6, 1e-6, 19e-6, 4e-6 / 3,
            1.0, 3.0, 0.1, 7.123456789e-5, 2.0**-20, 0.5, 2.0, 8.0]   # powers of two: exact ties
# LLG divisors (llg.py:93-95,134): Ms values, 1 + |a|^2 just above 1 and
# large, |M| near Ms -- ddiv with y = recip_of(d) replaces x / d there too
LLG_DIVISORS = [9.7e5, 1.3926e5, 1.3926e5 * (1 + 2.0**-40), 1.0 + 2.0**-52, 1.0 + 1e-9,
                1.0000123, 1.5, 2.0 - 2.0**-52, 37.25, 1e12, 1e150, 2.0**-500]


def _samples(seed, n):
    rng = np.random.default_rng(seed)
    # random bit patterns over the whole double range plus field-like values
    bits = rng.integers(0, 2**63, size=n, dtype=np.uint64)
    bits |= rng.integers(0, 2, size=n, dtype=np.uint64) << np.uint64(63)
    x = bits.view(np.float64)
    y = rng.normal(size=n) * 10.0 ** rng.uniform(-320, 300, size=n)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324,
                        2.2250738585072014e-308, 1.7976931348623157e308,
                        1e-300, 1e-310, 2.0**-969, 2.0**-970, 2.0**-1000])
    return np.concatenate([x, y, special])


def _near_subnormal_midpoints(d, seed, n=20000):
    """x = RN(m d) for m a midpoint (2j+1) 2^-1075 of the subnormal grid (and
    its neighbours): quotients on and next to the ties that the scaled
    subnormal path of ddiv must round like IEEE x / d."""
    from fractions import Fraction
    rng = np.random.default_rng(seed)
    js = np.concatenate([rng.integers(0, 2**20, n // 2), rng.integers(0, 2**52, n // 2)])
    fd = Fraction(d)
    out = []
    for j in js.tolist():
        m = Fraction(2 * int(j) + 1, 2**1075)
        x = float(m * fd)
        out += [x, -x, np.nextafter(x, np.inf), np.nextafter(x, -np.inf)]
    return np.array(out)


@pytest.mark.parametrize("d", SPACINGS + LLG_DIVISORS)
def test_ddiv_matches_ieee_division(d):
    lib = _native.load_library()
    x = np.ascontiguousarray(np.concatenate([_samples(hash(d) & 0xffff, 4_000_000),
                                             _near_subnormal_midpoints(d, 7)]))
    mism = C.c_int64()
    bad = C.c_double()
    _native.check(lib.mpb_selftest_division(0, d, x.ctypes.data_as(C.POINTER(C.c_double)),
                                            x.size, C.byref(mism), C.byref(bad)))
    assert mism.value == 0, f"first mismatch at x={bad.value!r}"
