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
