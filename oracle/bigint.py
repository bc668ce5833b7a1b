"""TEST INFRASTRUCTURE ONLY — arbitrary-precision oracle for small inputs.

A pure-Python restatement of the reference's verification oracle
(/root/reference/proj/src/oracle.cpp, which needs Boost.Multiprecision and
cannot be compiled here): every finite double is an integer multiple of
2^-1074, so exact sums are Python ints.  It also restates the accumulators'
special-value state machine (small_accumulator.cpp:230-242), which the oracle
deliberately does not model (it returns a canonical NaN, oracle.cpp:107-108),
and the canonical chunk form of a value (small_accumulator.cpp:244-303).

Pinned against the compiled reference (oracle/_ref) and the SPEC.md golden
vectors in tests/test_oracle.py.  Only tests/ may import this module.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass

MANT_BITS = 52
EXP_BIAS = 1023
SCALE = -(EXP_BIAS + MANT_BITS - 1)  # value = numerator * 2^SCALE  (2^-1074)
CANONICAL_QNAN = 0x7FF8000000000000
POS_INF = 0x7FF0000000000000
NEG_INF = 0xFFF0000000000000
NCHUNKS = 67


def to_bits(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def from_bits(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b & ((1 << 64) - 1)))[0]


@dataclass
class ExactValue:
    """oracle.hpp:29-33: numerator * 2^-1074, inf sign (-1/0/+1), nan flag."""

    numerator: int = 0
    inf_sign: int = 0
    nan: bool = False


def add(ev: ExactValue, v) -> None:
    """oracle.cpp:66-96.  Accepts a float or a raw 64-bit pattern (int)."""
    b = v if isinstance(v, int) else to_bits(v)
    sign = b >> 63
    e = (b >> 52) & 0x7FF
    m = b & ((1 << 52) - 1)
    if e == 0x7FF:
        if m:
            ev.nan = True
        else:
            s = -1 if sign else 1
            if ev.inf_sign == 0:
                ev.inf_sign = s
            elif ev.inf_sign != s:
                ev.nan = True
        return
    if e == 0:
        units = m  # zero or denormal: m units of 2^-1074
    else:
        units = ((1 << 52) | m) << (e - 1)
    ev.numerator += -units if sign else units


def exact(values) -> ExactValue:
    """oracle.cpp:98-104."""
    ev = ExactValue()
    for v in values:
        add(ev, int(v) if not isinstance(v, float) else v)
    return ev


def _round_magnitude(mag: int, scale_pow2: int, extra_sticky: bool) -> float:
    """oracle.cpp:36-58: keep 53 bits with nearest-even, scale with ldexp."""
    bits = mag.bit_length()
    if bits <= MANT_BITS + 1:
        return math.ldexp(float(mag), scale_pow2)
    shift = bits - (MANT_BITS + 1)
    keep = mag >> shift
    round_bit = (mag >> (shift - 1)) & 1
    sticky = extra_sticky or (mag & ((1 << (shift - 1)) - 1)) != 0
    if round_bit and (sticky or (keep & 1)):
        keep += 1
    try:
        return math.ldexp(float(keep), scale_pow2 + shift)
    except OverflowError:
        return math.inf


def round_bits(ev: ExactValue) -> int:
    """oracle.cpp:106-122 as a bit pattern: canonical NaN, +-Inf, +0.0 for zero."""
    if ev.nan:
        return CANONICAL_QNAN
    if ev.inf_sign:
        return POS_INF if ev.inf_sign > 0 else NEG_INF
    if ev.numerator == 0:
        return 0
    neg = ev.numerator < 0
    r = _round_magnitude(abs(ev.numerator), SCALE, False)
    return to_bits(-r if neg else r)


def mean_bits(ev: ExactValue, n: int) -> int:
    """oracle.cpp:124-165."""
    if n <= 0:
        raise ValueError("oracle::mean: divisor must be positive")
    if ev.nan:
        return CANONICAL_QNAN
    if ev.inf_sign:
        return POS_INF if ev.inf_sign > 0 else NEG_INF
    if ev.numerator == 0:
        return 0
    neg = ev.numerator < 0
    a = abs(ev.numerator)
    if a < (n << (MANT_BITS + 1)):
        q, r = divmod(a, n)
        twice_r = r << 1
        if twice_r > n or (twice_r == n and (q & 1)):
            q += 1
        mag = math.ldexp(float(q), SCALE)
    else:
        extra = 4
        q, r = divmod(a << extra, n)
        mag = _round_magnitude(q, SCALE - extra, r != 0)
    return to_bits(-mag if neg else mag)


def accumulator_specials(values) -> tuple[int, int]:
    """(inf_bits, nan_bits) of the serial add order (small_accumulator.cpp:230-242)."""
    inf_bits = nan_bits = 0
    for v in values:
        b = v if isinstance(v, int) else to_bits(v)
        if (b >> 52) & 0x7FF != 0x7FF:
            continue
        if b & ((1 << 52) - 1) == 0:
            if inf_bits == 0:
                inf_bits = b
            elif inf_bits != b and nan_bits == 0:
                nan_bits = CANONICAL_QNAN
        elif nan_bits == 0:
            nan_bits = b
    return inf_bits, nan_bits


def exact_sum_bits(values) -> int:
    """Result bits of exact_sum (either method) including the NaN payload rule:
    NaN state first, then Inf, then the oracle's rounding (small_accumulator.cpp:330-348)."""
    vals = list(values)
    inf_bits, nan_bits = accumulator_specials(vals)
    if nan_bits:
        return nan_bits
    if inf_bits:
        return inf_bits
    return round_bits(exact(vals))


def canonical_chunks(numerator: int) -> tuple[list[int], int]:
    """Unique post-carry_propagate chunk vector of value numerator * 2^-1074.

    Chunk i weighs 2^(32 i - 1075) (small_accumulator.hpp:27-35): the value in
    chunk units is 2 * numerator.  Digits below the top are in [0, 2^32); the top
    chunk is in [-2^32, 2^32) and is -1 only at index 0 (small_accumulator.cpp:244-303).
    Returns (chunks, top) with top = -1 for zero.
    """
    v = 2 * numerator
    if v == 0:
        return [0] * NCHUNKS, -1
    ch = [0] * NCHUNKS
    if v > 0:
        i = 0
        while v:
            ch[i] = v & 0xFFFFFFFF
            v >>= 32
            i += 1
        return ch, i - 1
    # negative: smallest top with floor(v / 2^(32 top)) in [-2^32, -2] (or top = 0)
    top = 0
    while True:
        d = v >> (32 * top)
        if d >= -(1 << 32) and (d != -1 or top == 0):
            break
        top += 1
    for i in range(top):
        ch[i] = (v >> (32 * i)) & 0xFFFFFFFF
    ch[top] = v >> (32 * top)
    return ch, top
