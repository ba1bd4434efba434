"""ORACLE twin (O2) - test infrastructure only; pure Python ints, small n.

Same definition as ``oracle/xsum_oracle.c`` (the exact
fixed-point sum) in independent code: the exact sum is a Python ``int`` A with
sum(x) = A * 2^-1074, and the rounding is the standard library's correctly
rounded int/int true division (``float(Fraction)``), not a re-typing of O1's
bit-level rounding. Used to pin O1 on inputs up to ~2^20 elements.
"""
from __future__ import annotations

import math
import struct
from fractions import Fraction

F_NAN, F_PINF, F_NINF, F_OVERFLOW, F_INEXACT = 1, 2, 4, 8, 16
F_OVERFLOW32, F_INEXACT32 = 64, 128
NLIMB = 34


def decode(x: float) -> tuple[int, int, int]:
    """(sign, biased exponent, fraction) of a binary64 (IEEE 754; R1)."""
    (b,) = struct.unpack("<Q", struct.pack("<d", x))
    return b >> 63, (b >> 52) & 0x7FF, b & ((1 << 52) - 1)


def exact_int(xs) -> tuple[int, int]:
    """(A, flags): A = sum of the finite x_i times 2^1074, exactly; specials only flagged."""
    A = 0
    flags = 0
    for x in xs:
        s, e, m = decode(float(x))
        if e == 0x7FF:
            flags |= F_NAN if m else (F_NINF if s else F_PINF)
            continue
        if e == 0:
            v = m                       # subnormal (or zero): m * 2^-1074
        else:
            v = (m | (1 << 52)) << (e - 1)   # (2^52 + m) * 2^(e-1075) = ... * 2^-1074
        A += -v if s else v
    return A, flags


def round_int(A: int, flags: int = 0) -> tuple[float, int, int]:
    """(value, direction, flags) for the exact integer A (units of 2^-1074)."""
    flags &= F_NAN | F_PINF | F_NINF
    direction = 0
    exact = Fraction(A, 1 << 1074)
    try:
        value = float(exact)            # correctly rounded (RN-even), raises on overflow
    except OverflowError:
        value = math.inf if A > 0 else -math.inf
        flags |= F_OVERFLOW
    if math.isinf(value) and not (flags & F_OVERFLOW):
        flags |= F_OVERFLOW             # defensive: some Python builds return inf
    if math.isinf(value):
        direction = 1 if A > 0 else -1
    else:
        fv = Fraction(value)
        direction = (fv > exact) - (fv < exact)
    if direction:
        flags |= F_INEXACT
    _, f32flags = round_int_f32(A, 0)           # the binary32 rounding's flags (independent)
    flags |= f32flags & (F_OVERFLOW32 | F_INEXACT32)
    if value == 0.0:
        value = 0.0                     # exact zero -> +0.0 (R9)
    if (flags & F_NAN) or ((flags & F_PINF) and (flags & F_NINF)):
        value, direction = struct.unpack("<d", struct.pack("<Q", 0x7FF8000000000000))[0], 0
    elif flags & F_PINF:
        value, direction = math.inf, 0
    elif flags & F_NINF:
        value, direction = -math.inf, 0
    return value, direction, flags


def bits_of(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def exact_sum(xs) -> tuple[float, int, int, int]:
    """(value, direction, flags, A)."""
    A, flags = exact_int(xs)
    value, direction, flags = round_int(A, flags)
    return value, direction, flags, A


def limbs(A: int) -> list[int]:
    """34 little-endian u64 limbs of A in two's complement."""
    v = A & ((1 << (64 * NLIMB)) - 1)
    return [(v >> (64 * L)) & 0xFFFFFFFFFFFFFFFF for L in range(NLIMB)]


def decode32(bits: int) -> tuple[int, int, int]:
    """(sign, biased exponent, fraction) of a binary32 bit pattern."""
    return bits >> 31, (bits >> 23) & 0xFF, bits & 0x7FFFFF


def exact_int_f32(bit_patterns) -> tuple[int, int]:
    """(A, flags) for binary32 inputs given as uint32 bit patterns: A = sum * 2^1074."""
    A = 0
    flags = 0
    for b in bit_patterns:
        s, e, m = decode32(int(b))
        if e == 0xFF:
            flags |= F_NAN if m else (F_NINF if s else F_PINF)
            continue
        v = (m << 925) if e == 0 else ((m | (1 << 23)) << (e - 1 + 925))
        A += -v if s else v
    return A, flags


def _f32_value(bits: int) -> Fraction:
    s, e, m = decode32(bits)
    v = Fraction(m, 1 << 149) if e == 0 else Fraction(m | (1 << 23), 1) * Fraction(2) ** (e - 150)
    return -v if s else v


def round_int_f32(A: int, flags: int = 0) -> tuple[int, int]:
    """(binary32 bits, flags) of the RN-even binary32 rounding of A * 2^-1074, by search:
    the two binary32 neighbours of the exact value are found from a float64 guess and
    compared exactly as rationals (independent of the oracle's bit-level rounding)."""
    flags &= F_NAN | F_PINF | F_NINF
    if (flags & F_NAN) or ((flags & F_PINF) and (flags & F_NINF)):
        return 0x7FC00000, flags
    if flags & F_PINF:
        return 0x7F800000, flags
    if flags & F_NINF:
        return 0xFF800000, flags
    if A == 0:
        return 0, flags
    S = Fraction(A, 1 << 1074)
    sign = 0x80000000 if A < 0 else 0
    mag = abs(S)
    top = Fraction((1 << 24) - 1) * Fraction(2) ** 104            # FLT_MAX
    if mag >= top + Fraction(2) ** 103:                           # >= FLT_MAX + half ulp: tie -> even = inf
        return sign | 0x7F800000, flags | F_OVERFLOW32 | F_INEXACT32
    # candidate neighbours: magnitudes are monotone in the bit pattern
    guess = struct.unpack("<I", struct.pack("<f", min(float(mag), 3.4028234663852886e38)))[0]
    best = None
    for b in range(max(0, guess - 2), min(0x7F7FFFFF, guess + 2) + 1):
        d = abs(_f32_value(b) - mag)
        key = (d, b & 1)                                           # nearest, then even
        if best is None or key < best[0]:
            best = (key, b)
    b = best[1]
    if _f32_value(b) != mag:
        flags |= F_INEXACT32
    return sign | b, flags


# 16-bit formats (binary16: t = 10, l = 5; bfloat16: t = 7, l = 8), the paper's t-bit fraction /
# l-bit exponent format with the IEEE bias (R1). Python ints, one element at
# a time: x = (-1)^s M 2^(max(e,1) - bias - t), A = x 2^1074.
H16 = {"f16": (10, 5), "bf16": (7, 8)}


def exact_int_h16(bit_patterns, fmt: str) -> tuple[int, int]:
    """(A, flags) for 16-bit inputs given as uint16 bit patterns: A = sum * 2^1074."""
    t, l = H16[fmt]
    bias = (1 << (l - 1)) - 1
    A = 0
    flags = 0
    for b in bit_patterns:
        b = int(b)
        s, e, m = b >> 15, (b >> t) & ((1 << l) - 1), b & ((1 << t) - 1)
        if e == (1 << l) - 1:
            flags |= F_NAN if m else (F_NINF if s else F_PINF)
            continue
        M = m if e == 0 else m + (1 << t)
        v = M << (max(e, 1) - bias - t + 1074)
        A += -v if s else v
    return A, flags
