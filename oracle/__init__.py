"""ORACLE - test infrastructure only.

Plain CPU exact summation of binary64 / binary32 / binary16 / bfloat16 (the oracle of DESIGN.md §3). Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package. It shares no code with the
CUDA path (``paper_1605_05436_b200``) and never imports it.

Two independent implementations of one definition (§2
fixed-point view: the exact sum is an integer multiple of 2^-1074):
  * O1  ``xsum_oracle.c``  big-integer limbs, threaded, any n   (this module)
  * O2  ``oracle.pytwin``  Python ints / fractions, small n     (pins O1)
and, for the condition-number-sensitive algorithm of PAPER.md:851-965 (r-truncated sparse
superaccumulators, r <- r^2, stopping conditions; a faithful, not a unique, result):
  * O3  ``oracle.condsens`` Python ints / fractions, step by step in the paper's order,
        pinned by tests/test_condsens_pins.py
Rounding: round-to-nearest ties-to-even of the exact sum (PAPER.md:172-179
faithful; §5 PAPER.md:1066-1069 "correctly rounded").

Every function here is pinned by ``tests/test_oracle_pins.py``; DESIGN.md lists
the readings of the paper it follows (R1-R12).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

NLIMB = 34                    # 2176-bit two's complement image, little-endian u64 limbs
F_NAN, F_PINF, F_NINF, F_OVERFLOW, F_INEXACT = 1, 2, 4, 8, 16
F_OVERFLOW32, F_INEXACT32 = 64, 128          # the binary32 rounding (value_f32)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "xsum_oracle.c")


class _CResult(ctypes.Structure):
    _fields_ = [("value", ctypes.c_double), ("direction", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("msb_exp", ctypes.c_int32), ("sign", ctypes.c_int32), ("count", ctypes.c_uint64),
                ("sig53", ctypes.c_uint64), ("exp2", ctypes.c_int32), ("value_f32", ctypes.c_uint32)]


@dataclass(frozen=True)
class Result:
    value: float
    bits: int            # uint64 bit pattern of value
    direction: int       # sign(value - exact) of the finite part; 0 if a special is returned
    flags: int
    msb_exp: int | None  # floor(log2|exact|), None for an exact zero
    sign: int
    count: int
    sig53: int           # unbounded-exponent rounding: |exact| ~= sig53 * 2^exp2
    exp2: int
    bits_f32: int        # uint32 bit pattern of the RN-even binary32 rounding


def build() -> None:
    if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-pthread", _SRC, "-o", _SO])


_lib = None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        p, u64, i32, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint32
        lib.oracle_sum.argtypes = [p, p, p, u64, i32]
        lib.oracle_sum.restype = None
        lib.oracle_sum_f32.argtypes = [p, p, p, u64, i32]
        lib.oracle_sum_f32.restype = None
        lib.oracle_sum_h16.argtypes = [p, p, p, u64, i32, i32]
        lib.oracle_sum_h16.restype = None
        lib.oracle_round.argtypes = [p, u32, u64, ctypes.POINTER(_CResult)]
        lib.oracle_round.restype = None
        lib.oracle_limbs_add.argtypes = [p, p]
        lib.oracle_limbs_add.restype = None
        lib.oracle_sum_segments.argtypes = [p, i32, p, u64, p, p, p, p, i32]
        lib.oracle_sum_segments.restype = None
        _lib = lib
    return _lib


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class Accumulator:
    """Streaming exact sum: ``add`` chunks in any order, then ``result``."""

    def __init__(self, nthreads: int | None = None):
        self.limbs = np.zeros(NLIMB, dtype=np.uint64)
        self._flags = ctypes.c_uint32(0)
        self.count = 0
        self.nthreads = nthreads or host_threads()

    @property
    def flags(self) -> int:
        return int(self._flags.value)

    def add(self, x: np.ndarray, fmt: str | None = None) -> "Accumulator":
        """Add float64 values (float32 arrays are summed exactly as binary32, float16 arrays as
        binary16). 16-bit bit patterns (uint16 arrays) need fmt = "f16" or "bf16"."""
        x = np.asarray(x)
        if x.dtype == np.float16 or fmt is not None:
            if fmt is None:
                fmt = "f16"
            if fmt not in ("f16", "bf16"):
                raise ValueError("fmt must be 'f16' or 'bf16'")
            x = np.ascontiguousarray(x).view(np.uint16)
            if x.size:
                _L().oracle_sum_h16(self.limbs.ctypes.data, ctypes.addressof(self._flags), x.ctypes.data, x.size,
                                    self.nthreads, 1 if fmt == "bf16" else 0)
            self.count += int(x.size)
            return self
        f32 = x.dtype == np.float32
        x = np.ascontiguousarray(x, dtype=np.float32 if f32 else np.float64)
        if x.size:
            fn = _L().oracle_sum_f32 if f32 else _L().oracle_sum
            fn(self.limbs.ctypes.data, ctypes.addressof(self._flags), x.ctypes.data, x.size, self.nthreads)
        self.count += int(x.size)
        return self

    def merge(self, other: "Accumulator") -> "Accumulator":
        _L().oracle_limbs_add(self.limbs.ctypes.data, other.limbs.ctypes.data)
        self._flags.value |= other._flags.value
        self.count += other.count
        return self

    def result(self) -> Result:
        return round_limbs(self.limbs, self.flags, self.count)


def round_limbs(limbs: np.ndarray, flags: int, count: int = 0) -> Result:
    limbs = np.ascontiguousarray(limbs, dtype=np.uint64)
    assert limbs.size == NLIMB
    r = _CResult()
    _L().oracle_round(limbs.ctypes.data, flags, count, ctypes.byref(r))
    bits = int(np.array([r.value], dtype=np.float64).view(np.uint64)[0])
    return Result(value=r.value, bits=bits, direction=r.direction, flags=r.flags,
                  msb_exp=None if r.msb_exp == -(2 ** 31) else r.msb_exp, sign=r.sign,
                  count=r.count, sig53=r.sig53, exp2=r.exp2, bits_f32=r.value_f32)


def exact_sum(x, nthreads: int | None = None, fmt: str | None = None) -> tuple[Result, np.ndarray]:
    """(rounded result, 34-limb two's complement image of sum(x)*2^1074); float32 arrays are
    summed as binary32 values, float16 arrays as binary16, uint16 bit patterns per fmt
    ("f16" / "bf16"), anything else as float64."""
    x = np.asarray(x)
    if fmt is not None or x.dtype == np.float16:
        acc = Accumulator(nthreads).add(x, fmt=fmt)
        return acc.result(), acc.limbs.copy()
    acc = Accumulator(nthreads).add(x if x.dtype == np.float32 else np.asarray(x, dtype=np.float64))
    return acc.result(), acc.limbs.copy()


def limbs_to_int(limbs: np.ndarray) -> int:
    """Signed Python int of a 34-limb two's complement image."""
    v = 0
    for L in reversed(range(NLIMB)):
        v = (v << 64) | int(limbs[L])
    if v >> (64 * NLIMB - 1):
        v -= 1 << (64 * NLIMB)
    return v


def int_to_limbs(v: int) -> np.ndarray:
    v &= (1 << (64 * NLIMB)) - 1
    return np.array([(v >> (64 * L)) & 0xFFFFFFFFFFFFFFFF for L in range(NLIMB)], dtype=np.uint64)


_FMT = {None: 0, "f64": 0, "f32": 1, "f16": 2, "bf16": 3}


def sum_segments(x, offsets=None, seg_len: int | None = None, fmt: str | None = None, canon: bool = False,
                 nthreads: int | None = None):
    """Per-segment exact sums, each rounded like exact_sum (segment s = x[offsets[s]:offsets[s+1]], or
    equal segments of seg_len): returns (binary64 bits uint64[nseg], binary32 bits uint32[nseg],
    flags uint32[nseg], canonical images uint64[nseg, 34] or None). float32 arrays are binary32;
    uint16 bit patterns need fmt "f16" / "bf16"."""
    x = np.ascontiguousarray(x)
    if fmt is None and x.dtype == np.float32:
        fmt = "f32"
    if fmt is None and x.dtype == np.float16:
        fmt, x = "f16", x.view(np.uint16)
    if offsets is None:
        if not seg_len or x.size % seg_len:
            raise ValueError("x.size must be a multiple of seg_len")
        offsets = np.arange(0, x.size + 1, seg_len, dtype=np.uint64)
    off = np.ascontiguousarray(offsets, dtype=np.uint64)
    nseg = off.size - 1
    b64 = np.zeros(nseg, dtype=np.uint64)
    b32 = np.zeros(nseg, dtype=np.uint32)
    fl = np.zeros(nseg, dtype=np.uint32)
    cn = np.zeros((nseg, NLIMB), dtype=np.uint64) if canon else None
    if nseg:
        _L().oracle_sum_segments(x.ctypes.data if x.size else None, _FMT[fmt], off.ctypes.data, nseg,
                                 b64.ctypes.data, b32.ctypes.data, fl.ctypes.data,
                                 cn.ctypes.data if cn is not None else None, nthreads or host_threads())
    return b64, b32, fl, cn
