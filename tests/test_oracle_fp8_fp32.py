"""Pins for oracle.fp8 (E4M3 codec) and oracle.fp32 (directed binary32 rounding).

Pinned against: the E4M3 format definition enumerated independently here with
numpy's float16 (every E4M3 value is exactly representable in binary16), the
paper's facts and IEEE neighbours from numpy.nextafter.
"""
import struct
from fractions import Fraction

import numpy as np
import pytest

from oracle import fp8, fp32


def _e4m3_via_f16(code):
    """Independent decode: build the binary16 bit pattern of the same value.
    E4M3 exponent e (bias 7) -> binary16 exponent e - 7 + 15; subnormals m*2^-9."""
    s = (code >> 7) & 1
    e = (code >> 3) & 0xF
    m = code & 7
    if e == 15 and m == 7:
        return None
    if e == 0:
        v = np.float16(m) * np.float16(2.0 ** -9)
    else:
        bits = (s << 15) | ((e - 7 + 15) << 10) | (m << 7)
        return float(np.frombuffer(struct.pack("<H", bits), dtype=np.float16)[0])
    return -float(v) if s else float(v)


def test_decode_matches_independent_enumeration():
    for c in range(256):
        a = fp8.decode(c)
        b = _e4m3_via_f16(c)
        if b is None:
            assert a is None and c in fp8.NAN_CODES
        else:
            assert a == Fraction(b), hex(c)


def test_format_facts(facts, spec):
    vals = {fp8.decode(c) for c in range(256)} - {None}
    assert len(vals) == 253                     # 254 finite codes, +0 and -0 coincide
    assert max(vals) == 448 == spec["fp8_codec"]["max_finite"]
    # consecutive integers -16..16 exactly representable, 17 not
    n = facts["fp8_facts"]["consecutive_int_max"]
    for v in range(-n, n + 1):
        assert Fraction(v) in vals
        assert fp8.decode(fp8.encode_int(v)) == v
    assert Fraction(17) not in vals
    for c, v in spec["fp8_codec"]["decode"]:
        assert fp8.decode(c) == Fraction(v)
    assert fp8.decode(spec["fp8_codec"]["nan_code"]) is None
    assert fp8.decode(fp8.encode_rne(17)) == spec["fp8_codec"]["rne_17"]
    assert fp8.decode(fp8.encode_ru_nonneg(Fraction("255.9"))) == spec["fp8_codec"]["ru_255_9"]


def test_round_up_is_minimal_upper_bound():
    rng = np.random.default_rng(1)
    xs = list(rng.random(2000) * 256.0) + [0.0, 2.0 ** -10, 2.0 ** -9, 255.999, 256.0]
    pos = sorted({fp8.decode(c) for c in range(0x7F)})
    for x in xs:
        c = fp8.encode_ru_nonneg(Fraction(x))
        v = fp8.decode(c)
        assert v >= Fraction(x)
        below = [p for p in pos if p < v]
        assert not below or below[-1] < Fraction(x)


def _f32(x):
    return Fraction(float(np.float32(x)))


def test_fp32_directed_vs_nextafter():
    rng = np.random.default_rng(2)
    for _ in range(3000):
        q = Fraction(int(rng.integers(1, 2 ** 60)), int(rng.integers(1, 2 ** 40)))
        if rng.random() < 0.3:
            q = -q
        d = fp32.round_down(q)
        u = fp32.round_up(q)
        assert d <= q <= u
        if d != u:
            # neighbours: nothing representable strictly between
            nd = np.nextafter(np.float32(float(d)), np.float32(np.inf))
            assert Fraction(float(nd)) == u
        n = fp32.round_nearest(q)
        assert n in (d, u)
        assert abs(n - q) <= abs((u if n == d else d) - q)


def test_fp32_subnormals_and_exact():
    tiny = Fraction(1, 2 ** 149)
    assert fp32.round_up(tiny / 3) == tiny
    assert fp32.round_down(tiny / 3) == 0
    for v in [1.0, 0.5, 3.25, 2.0 ** -130, 1e30]:
        x = _f32(v)
        assert fp32.round_down(x) == x == fp32.round_up(x) == fp32.round_nearest(x)
    # ties to even
    one = Fraction(1)
    assert fp32.round_nearest(one + Fraction(1, 2 ** 24)) == one
    assert fp32.round_nearest(one + Fraction(3, 2 ** 24)) == one + Fraction(4, 2 ** 24)


def test_delta_bit_pattern(facts):
    from oracle import moduli
    d = moduli.delta()
    assert fp32.f32_bits(d) == int(facts["delta"]["bits_hex"], 16)
    assert d == -(Fraction(1, 2) + Fraction(3, 2 ** 24))
