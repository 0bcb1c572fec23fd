"""FP8 E4M3 codec, written out from the format definition.

Paper: "FP8 MMA takes FP8_E4M3 inputs and accumulates in FP32"; E4M3
"can exactly represent consecutive integers in the range of -16 to 16";
diag(mu')A is "cast to the FP8_E4M3 matrices ... in round-up mode".

Format (sign 1 / exponent 4, bias 7 / mantissa 3): exponent field 0 is subnormal
(value m * 2^-9); exponent field 15 with mantissa 7 is NaN; there is no infinity;
the largest finite magnitude is 448 (code 0x7E).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from bisect import bisect_left
from fractions import Fraction

NAN_CODES = (0x7F, 0xFF)


def decode(code: int):
    """Exact value of an E4M3 code as a Fraction; None for NaN."""
    code &= 0xFF
    sign = code >> 7
    e = (code >> 3) & 0xF
    m = code & 0x7
    if e == 0xF and m == 0x7:
        return None
    if e == 0:
        v = Fraction(m, 2 ** 9)                       # subnormal: m * 2^-9
    else:
        v = Fraction(8 + m, 8) * Fraction(2) ** (e - 7)  # (1 + m/8) * 2^(e-7)
    return -v if sign else v


# The 127 non-negative finite codes 0x00..0x7E, in increasing value order
# (the encoding is monotone in the magnitude bits).
_POS_CODES = list(range(0x00, 0x7F))
_POS_VALUES = [decode(c) for c in _POS_CODES]
assert all(_POS_VALUES[i] < _POS_VALUES[i + 1] for i in range(len(_POS_VALUES) - 1))
MAX_FINITE = _POS_VALUES[-1]  # 448


def encode_ru_nonneg(x) -> int:
    """Code of the smallest E4M3 value >= x, for 0 <= x <= 448 (round-up).

    Exact comparison against every non-negative E4M3 value.
    """
    x = Fraction(x)
    if x < 0 or x > MAX_FINITE:
        raise ValueError("encode_ru_nonneg: x out of [0, 448]")
    i = bisect_left(_POS_VALUES, x)
    return _POS_CODES[i]


def encode_rne(x) -> int:
    """Round-to-nearest-even encode (used only to pin the codec)."""
    x = Fraction(x)
    sign = 0x80 if x < 0 else 0
    a = -x if x < 0 else x
    if a >= MAX_FINITE:
        return sign | 0x7E
    i = bisect_left(_POS_VALUES, a)
    if _POS_VALUES[i] == a:
        return sign | _POS_CODES[i]
    lo, hi = _POS_VALUES[i - 1], _POS_VALUES[i]
    if a - lo < hi - a:
        c = _POS_CODES[i - 1]
    elif a - lo > hi - a:
        c = _POS_CODES[i]
    else:
        c = _POS_CODES[i - 1] if (_POS_CODES[i - 1] & 1) == 0 else _POS_CODES[i]
    return sign | c


def encode_int(v: int) -> int:
    """Exact code of an integer |v| <= 16."""
    if not -16 <= v <= 16:
        raise ValueError("encode_int: |v| > 16 is not exactly representable")
    c = encode_ru_nonneg(abs(v))
    assert decode(c) == abs(v)
    return (0x80 | c) if v < 0 else c
