"""DMMA (mma.sync m8n8k4 f64 = SASS DMMA.8x8x4) known answers on the device.

The tile engine's contract (reference tiles.py:153-166, test_tiles.py:117-122) is
D = A(8x4) B(4x8) + C(8x8).  Exactly representable operands pin the fragment
layout bit-for-bit; random and cancelling operands pin the accumulation error the
guard band of the DMMA kernels relies on (within 4 ulp of the
absolute sum |A||B| + |C|), so the band's soundness is measured on every box the
suite runs on."""

import ctypes
from fractions import Fraction

import numpy as np
import pytest

from paper_2209_11287_b200 import _native

pytestmark = pytest.mark.gpu
P = ctypes.POINTER(ctypes.c_double)


def dmma(a, b, c):
    lib = _native.load_library()
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    c = np.ascontiguousarray(c, np.float64)
    d = np.zeros((8, 8))
    assert lib.tj_dmma_known_answer(a.ctypes.data, b.ctypes.data, c.ctypes.data,
                                    d.ctypes.data) == 0
    return d


def test_fragment_layout_exact():
    a = np.arange(32, dtype=np.float64).reshape(8, 4)
    b = np.arange(32, dtype=np.float64).reshape(4, 8) * 0.5
    c = np.arange(64, dtype=np.float64).reshape(8, 8)
    assert np.array_equal(dmma(a, b, c), a @ b + c)
    # orthonormal rows (test_kernels.py:138-141 shape): -2 e_i . e_j + 1 + 1 = 2(1 - I)
    e = np.eye(4)
    a = np.vstack([e, e])
    b = -2.0 * np.hstack([e, e])
    c = np.full((8, 8), 2.0)
    want = np.tile(2.0 * (1.0 - np.eye(4)), (2, 2))
    assert np.array_equal(dmma(a, b, c), want)


def test_accumulation_error_within_guard_assumption():
    rng = np.random.default_rng(0)
    worst = 0.0
    for t in range(300):
        a = rng.normal(size=(8, 4)) * (10.0 ** rng.integers(-3, 4))
        b = rng.normal(size=(4, 8))
        c = rng.normal(size=(8, 8)) * (10.0 ** rng.integers(-3, 4))
        if t % 2:  # near-total cancellation, the hard case for the expanded form
            c = -(a @ b) * (1 + 1e-15)
        d = dmma(a, b, c)
        exact = np.array([[float(sum(Fraction(a[r, k]) * Fraction(b[k, j]) for k in range(4))
                                 + Fraction(c[r, j])) for j in range(8)] for r in range(8)])
        scale = np.abs(a) @ np.abs(b) + np.abs(c)
        worst = max(worst, float((np.abs(d - exact) / (scale * 2.0 ** -53)).max()))
    assert worst <= 4.0, worst
