"""Pins for the oracle's step 4 (PAPER.md:135 spherical reference at (0, 30, -400) mm, :137
binary-amplitude conversion; R-A14, R-A15).  References: closed-form inputs u = +-R, u = iR
 and a crafted sign pattern that fixes the bit order (MSB first)."""
import math

import numpy as np


def _P(orc):
    return orc.Params(633e-9, 1e-6, 256, 1, 3, 0.1e-3, 0.1e-3, 0.1)


def _ref_wave(P, ref, x0, y0, w, h):
    Y, X = np.mgrid[y0:y0 + h, x0:x0 + w]
    x = (X - P.n_h // 2) * P.pitch
    y = (Y - P.n_h // 2) * P.pitch
    r = np.sqrt((x - ref[0]) ** 2 + (y - ref[1]) ** 2 + ref[2] ** 2)
    return np.exp(1j * 2 * math.pi / P.wavelength * r)


REF = (0.0, 0.030, -0.400)


def test_u_equal_reference_is_all_ones_and_minus_all_zero(orc):
    P = _P(orc)
    R = _ref_wave(P, REF, 64, 32, 128, 16)
    bits, I = orc.quantize(P, REF, R, 64, 32)
    assert np.all(bits == 0xFF)
    np.testing.assert_allclose(I, 1.0, atol=1e-6)
    bits, I = orc.quantize(P, REF, -R, 64, 32)
    assert np.all(bits == 0)


def test_u_quadrature_is_threshold_band(orc):
    """u = iR gives I = Re(iR conj(R)) = 0: the whole window sits in the A16 threshold band."""
    P = _P(orc)
    R = _ref_wave(P, REF, 0, 0, 64, 8)
    _, I = orc.quantize(P, REF, 1j * R, 0, 0)
    assert np.max(np.abs(I)) < 1e-6


def test_bit_order_msb_first(orc):
    """Pixel X -> byte X >> 3, bit 7 - (X & 7), 1 = I >= 0."""
    P = _P(orc)
    R = _ref_wave(P, REF, 0, 0, 64, 2)
    rng = np.random.default_rng(0)
    s = rng.choice([-1.0, 1.0], size=(2, 64))
    bits, _ = orc.quantize(P, REF, s * R, 0, 0)
    exp = np.packbits((s > 0).astype(np.uint8), axis=1, bitorder="big")
    assert np.array_equal(bits, exp)
