"""The controller's pow (csrc/bode_pow.cuh), host build: correctly rounded
against 50-digit decimal arithmetic, and therefore equal to glibc's pow
(what the reference's NumPy calls) wherever glibc is correctly rounded."""
import ctypes as C
import math
import os
import random
from decimal import Decimal, getcontext

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2210_12375_b200", "_build", "libbode_hostpow.so")


@pytest.fixture(scope="module")
def crpow():
    if not os.path.exists(LIB):
        pytest.skip("host pow library not built")
    lib = C.CDLL(LIB)
    lib.bode_cr_pow_host.restype = C.c_double
    lib.bode_cr_pow_host.argtypes = [C.c_double, C.c_double]
    return lib.bode_cr_pow_host


@pytest.mark.parametrize("e", [-0.2, -0.12, 0.04, 1 / 6, -1 / 30, -1 / 90, 2.5, -3.7])
def test_correctly_rounded(crpow, e):
    getcontext().prec = 50
    rng = random.Random(hash(e) & 0xFFFF)
    bad = glibc_bad = 0
    n = 4000
    for _ in range(n):
        x = 10 ** rng.uniform(-10, 3) if abs(e) < 1 else rng.uniform(1e-3, 1e3)
        ref = float((Decimal(e) * Decimal(x).ln()).exp())
        bad += crpow(x, e) != ref
        glibc_bad += math.pow(x, e) != ref
    assert bad == 0
    assert glibc_bad <= n * 0.005  # glibc itself: ~0.1% not correctly rounded


def test_special_values(crpow):
    assert crpow(1.0, -0.2) == 1.0
    assert crpow(4.0, 0.5) == 2.0
    assert crpow(0.0, -0.2) == math.inf
    assert crpow(math.inf, -0.2) == 0.0
    assert crpow(math.inf, 0.3) == math.inf
    assert math.isnan(crpow(-1.0, 0.5))
    assert math.isnan(crpow(math.nan, 0.5))
    assert crpow(2.0 ** -1060, 0.5) == math.pow(2.0 ** -1060, 0.5)   # subnormal input
    assert crpow(1e300, 0.9) == math.pow(1e300, 0.9)
    assert crpow(1e-300, 2.5) == math.pow(1e-300, 2.5)  # underflow edge -> libm


@pytest.mark.parametrize("e", [-0.2, -0.12, 0.04, 1 / 6, -1 / 30, -1 / 90])
def test_fast_mode_pow_within_1_ulp(e):
    """BODE_MODE_FAST's controller pow (plain-double log/exp on the same
    tables): within 1 ulp of the exact value over the controller's range."""
    if not os.path.exists(LIB):
        pytest.skip("host pow library not built")
    lib = C.CDLL(LIB)
    lib.bode_fast_pow_host.restype = C.c_double
    lib.bode_fast_pow_host.argtypes = [C.c_double, C.c_double]
    getcontext().prec = 50
    rng = random.Random(7 + (hash(e) & 0xFF))
    worst = 0
    for _ in range(4000):
        x = 10 ** rng.uniform(-10, 3)
        ref = float((Decimal(e) * Decimal(x).ln()).exp())
        got = lib.bode_fast_pow_host(x, e)
        worst = max(worst, abs(got - ref) / math.ulp(ref))
    assert worst <= 1, worst
    assert lib.bode_fast_pow_host(1.0, e) == 1.0
