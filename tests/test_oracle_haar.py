"""Pins for the oracle's Haar FWT (PAPER.md:91, :94 steps 1 and 3; reading R-A1/R-A6).

Independent references: a textbook separable orthonormal Haar filter bank written here with
numpy matrices in the Mallat layout, closed forms (constant, impulse), Parseval/perfect
reconstruction (north_star validation 1), and exact shift commutation.
"""
import numpy as np
import pytest


def _rand_field(rng, h, w):
    return rng.standard_normal((h, w)) + 1j * rng.standard_normal((h, w))


def _haar_matrix(n):
    """1-D orthonormal Haar analysis, one level: rows 0..n/2-1 lowpass, n/2.. highpass."""
    W = np.zeros((n, n))
    s = 1 / np.sqrt(2)
    for i in range(n // 2):
        W[i, 2 * i] = s; W[i, 2 * i + 1] = s
        W[n // 2 + i, 2 * i] = s; W[n // 2 + i, 2 * i + 1] = -s
    return W


def _mallat(f, L):
    """Textbook 2-D separable Haar (x then y), Mallat layout: returns dict level -> (HL, LH, HH), LL."""
    out = {}
    cur = f.copy()
    for l in range(1, L + 1):
        h, w = cur.shape
        Wx, Wy = _haar_matrix(w), _haar_matrix(h)
        t = Wy @ cur @ Wx.T
        LL = t[: h // 2, : w // 2]
        HL = t[: h // 2, w // 2:]     # x-high, y-low
        LH = t[h // 2:, : w // 2]     # x-low, y-high
        HH = t[h // 2:, w // 2:]
        out[l] = (HL, LH, HH)
        cur = LL
    return out, cur


@pytest.mark.parametrize("L", [1, 2, 3, 4, 5, 6, 7])
@pytest.mark.parametrize("mult", [1, 3, 8])
def test_v1_perfect_reconstruction_and_parseval(orc, L, mult):
    rng = np.random.default_rng(100 + L * 10 + mult)
    n = (1 << L) * mult
    if n > 512:
        n = 1 << L
    f = _rand_field(rng, n, n)
    W = orc.haar_fwd(f, L)
    back = orc.haar_inv(W, L)
    assert np.max(np.abs(back - f)) <= 1e-13 * np.max(np.abs(f))
    e0, e1 = np.sum(np.abs(f) ** 2), np.sum(np.abs(W) ** 2)
    assert abs(e1 - e0) <= 1e-13 * e0


@pytest.mark.parametrize("L", [1, 3, 4])
def test_matches_textbook_mallat_filter_bank(orc, L):
    """Interleaved in-place layout (R-A6) equals the textbook separable Haar re-indexed:
    level-l block (m, n) sits at X0 = m 2^l, Y0 = n 2^l; HL at (X0+s, Y0), LH at (X0, Y0+s),
    HH at (X0+s, Y0+s), LL_L at (X0, Y0)."""
    rng = np.random.default_rng(7 + L)
    n = 8 << L
    f = _rand_field(rng, n, n // 2 if n >= 16 else n)
    h, w = f.shape
    W = orc.haar_fwd(f, L)
    det, LL = _mallat(f, L)
    for l in range(1, L + 1):
        s = 1 << (l - 1)
        HL, LH, HH = det[l]
        np.testing.assert_allclose(W[0::2 * s, s::2 * s], HL, atol=1e-12)
        np.testing.assert_allclose(W[s::2 * s, 0::2 * s], LH, atol=1e-12)
        np.testing.assert_allclose(W[s::2 * s, s::2 * s], HH, atol=1e-12)
    np.testing.assert_allclose(W[0::1 << L, 0::1 << L], LL, atol=1e-12)


@pytest.mark.parametrize("L", [1, 3, 6])
def test_constant_field(orc, L):
    """constant c -> every detail 0, scaling coefficients 2^L c."""
    n = 2 << L
    f = np.full((n, n), 0.7 - 0.2j)
    W = orc.haar_fwd(f, L)
    B = 1 << L
    mask = np.zeros((n, n), bool)
    mask[0::B, 0::B] = True
    np.testing.assert_allclose(W[mask], (2 ** L) * (0.7 - 0.2j), rtol=0, atol=1e-14)
    assert np.max(np.abs(W[~mask])) <= 1e-14


@pytest.mark.parametrize("L", [1, 2, 4, 6])
def test_unit_impulse(orc, L):
    """Unit impulse at (0,0): every level-l detail of block (0,0) = 2^-l, LL_L = 2^-L, rest 0."""
    n = 1 << L
    f = np.zeros((n, n), complex)
    f[0, 0] = 1.0
    W = orc.haar_fwd(f, L)
    exp = np.zeros((n, n))
    exp[0, 0] = 2.0 ** -L
    for l in range(1, L + 1):
        s = 1 << (l - 1)
        exp[0, s] = exp[s, 0] = exp[s, s] = 2.0 ** -l
    np.testing.assert_allclose(W, exp, atol=1e-15)


@pytest.mark.parametrize("L", [2, 4])
def test_shift_by_multiple_of_2L_commutes_exactly(orc, L):
    """SPEC.md:142 keystone: a shift by a multiple of 2^L shifts every coefficient identically
    (bitwise: same operations on the same values)."""
    rng = np.random.default_rng(3)
    B = 1 << L
    f = _rand_field(rng, 4 * B, 4 * B)
    g = np.roll(np.roll(f, B, axis=1), 2 * B, axis=0)
    Wf = orc.haar_fwd(f, L)
    Wg = orc.haar_fwd(g, L)
    assert np.array_equal(np.roll(np.roll(Wf, B, axis=1), 2 * B, axis=0), Wg)


def test_non_multiple_shift_does_not_commute(orc):
    """Sanity: a 1-pixel shift is NOT a coefficient shift (why Eq.(2) needs the alpha rule)."""
    rng = np.random.default_rng(4)
    f = _rand_field(rng, 16, 16)
    W1 = orc.haar_fwd(np.roll(f, 1, axis=1), 2)
    assert not np.allclose(np.roll(orc.haar_fwd(f, 2), 1, axis=1), W1)
