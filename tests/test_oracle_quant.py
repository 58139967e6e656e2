"""Pins for the fp8 K/V quantiser oracle (oracle/quant.py; gt_opts.kv_fp8, reading Z25):

Q1 e4m3 itself: every one of the 256 codes decodes to the value its bits define (sign, 4-bit exponent
   with bias 7, 3-bit mantissa, subnormals, 0x7f / 0xff NaN - OCP FP8 E4M3); rne_e4m3 maps every finite
   code to itself, every midpoint between neighbours to the even one, and points just off a midpoint
   to the nearer neighbour;
Q2 the exponent rule as a closed form: e is minimal with max|x| <= 448 2^e (boundary values 448 2^k
   and their float successors), the vectorised form equals the scalar one;
Q3 quantisation invariants: the row's max maps to a code of magnitude in [224, 448], x^ = x when x is
   already e4m3 times a power of two, |x^ - x| <= half a code spacing, scaling invariance
   (quantize(2^s x) = 2^s quantize(x)).
"""
import math

import numpy as np

from oracle import quant


def e4m3_decode(code: int) -> float:
    s = -1.0 if code & 0x80 else 1.0
    ex = (code >> 3) & 0xF
    m = code & 0x7
    if ex == 0xF and m == 0x7:
        return math.nan
    if ex == 0:
        return s * m / 8.0 * 2.0 ** -6
    return s * (1.0 + m / 8.0) * 2.0 ** (ex - 7)


def finite_codes():
    vals = sorted({e4m3_decode(c) for c in range(256) if not math.isnan(e4m3_decode(c))})
    return np.array(vals)


def test_q1_codes_and_rne():
    vals = finite_codes()
    assert vals.max() == 448.0 and vals.min() == -448.0 and len(vals) == 253   # +-0 collapse: 254 - 1
    np.testing.assert_array_equal(quant.rne_e4m3(vals.astype(np.float32)), vals)
    pos = vals[vals >= 0]
    for a, b in zip(pos[:-1], pos[1:]):
        mid = (a + b) / 2.0
        # even neighbour: the one whose mantissa bit 0 is 0
        ca = int(np.round(a / (2.0 ** math.floor(math.log2(a))) * 8)) if a > 0 else 0
        even = a if (a == 0 or ca % 2 == 0) else b
        if a >= 2.0 ** -6:
            assert quant.rne_e4m3(np.array([mid], np.float32))[0] == even, (a, b)
        eps = (b - a) * 2.0 ** -6
        assert quant.rne_e4m3(np.array([mid - eps], np.float32))[0] == a
        assert quant.rne_e4m3(np.array([mid + eps], np.float32))[0] == b


def test_q2_exponent_rule():
    for k in range(-20, 21):
        b = 448.0 * 2.0 ** k
        assert quant.exponent(b) == k
        assert quant.exponent(float(np.nextafter(np.float32(b), np.float32(np.inf)))) == k + 1
        assert quant.exponent(b / 2.0) == k - 1
        assert quant.exponent(b * 0.75) == k
    assert quant.exponent(0.0) == -126
    rng = np.random.default_rng(1)
    a = np.abs(rng.standard_normal(5000) * np.exp2(rng.integers(-30, 30, 5000))).astype(np.float32)
    a[:10] = 0.0
    want = np.array([quant.exponent(float(x)) for x in a])
    np.testing.assert_array_equal(quant.exponents(a), want)
    for x, e in zip(a[10:200], want[10:200]):
        assert x <= 448.0 * 2.0 ** e and x > 448.0 * 2.0 ** (e - 1)


def test_q3_invariants():
    rng = np.random.default_rng(2)
    x = (rng.standard_normal((50, 4, 16)) * np.exp2(rng.integers(-8, 8, (50, 4, 1)))).astype(np.float32)
    xh, e = quant.quantize(x)
    amax = np.abs(x).max(axis=2)
    top = np.abs(xh).max(axis=2) / np.exp2(e)
    assert np.all(top >= 224.0) and np.all(top <= 448.0)   # (224, 448] before rounding
    # half a code spacing: e4m3 has 3 mantissa bits -> relative spacing <= 2^-3 (normal range)
    spacing = np.exp2(np.floor(np.log2(np.maximum(np.abs(x), 1e-30))) - 3)
    normal = np.abs(x) / np.exp2(e)[:, :, None] >= 2.0 ** -6
    assert np.all(np.abs(xh - x)[normal] <= spacing[normal] / 2 + 1e-30)
    assert np.all(np.abs(xh - x)[~normal] <= (2.0 ** -10 * np.exp2(e)[:, :, None] * np.ones_like(x))[~normal])
    # e4m3 values times a power of two are reproduced
    vals = finite_codes()
    sh = np.exp2(rng.integers(-5, 5, (20, 2, 1)))
    y = rng.choice(vals, size=(20, 2, 16)) * sh
    y[:, :, :1] = 448.0 * sh   # the row's max pins its scale to sh
    yh, _ = quant.quantize(y.astype(np.float32))
    np.testing.assert_array_equal(yh, y)
    # scaling by powers of two commutes with quantisation
    x2h, e2 = quant.quantize((x * 2.0 ** 5).astype(np.float32))
    np.testing.assert_array_equal(x2h, xh * 2.0 ** 5)
    np.testing.assert_array_equal(e2, e + 5)
    # bf16 bit patterns are read as their float values
    b = (x.view(np.uint32) >> 16).astype(np.uint16)
    bh, _ = quant.quantize(b)
    xb = (b.astype(np.uint32) << 16).view(np.float32)
    np.testing.assert_array_equal(bh, quant.quantize(xb)[0])
