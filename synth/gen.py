"""Seeded synthetic inputs for the five BASELINE.json configs (numpy implementation).

This module holds NONE of the method's arithmetic: it only assembles IEEE-754
binary64 bit patterns from a counter-based generator. It is the one module that
both sides (the CPU oracle in ``oracle/`` and the CUDA path in
``paper_1605_05436_b200/``) may consume. ``synth/gen.c`` (host, threaded) and
``synth/csrc/gen.cu`` (device) are independent implementations of the same
definition; tests check that all three agree bit for bit.

Definition (all arithmetic mod 2^64):

    mix64(z)      = splitmix64 finaliser
    key(seed, st) = mix64(seed + G*(st+1)),            G = 0x9E3779B97F4A7C15
    U(seed, st, j)= mix64(key(seed, st) + G*(j+1))
    draw(seed, st, i, lo, hi):
        u = U(seed, st, 2i); v = U(seed, st, 2i+1)
        frac = u & (2^52-1); sign = u >> 63
        E = lo + (((v >> 32) * (hi-lo+1)) >> 32)        # unbiased exponent in [lo, hi]
        bits = sign<<63 | (E+1023)<<52 | frac           # always a normal double

The workloads stand in for the paper's four dataset families (PAPER.md:1216-1230,
§6.3) - see DESIGN.md "Input recipe".
"""
from __future__ import annotations

import numpy as np

G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK52 = np.uint64((1 << 52) - 1)

# name -> generator parameters (BASELINE.json "configs")
CONFIGS = {
    "c1": dict(kind="uniform", n=1 << 20, seed=1, st=0, lo=-10, hi=10),
    "c2": dict(kind="uniform", n=1 << 28, seed=2, st=0, lo=-1000, hi=1000),
    "c3": dict(kind="cancel", n=(1 << 28) + (1 << 20), seed=3, npairs=1 << 27,
               pair_lo=0, pair_hi=600, ntiny=1 << 20, tiny_lo=-900, tiny_hi=-800),
    "c4": dict(kind="uniform", n=1 << 33, seed=4, st=0, lo=-1022, hi=1023),
    "c5": dict(kind="segments", n=1 << 28, seed=5, st=0, lo=-200, hi=200,
               nseg=1 << 16, seg_len=1 << 12),
}

# Measurement workloads of the NEXT rows, not BASELINE.json configs:
#  * c5csr: 2^16 variable-length segments, len_s = 1 + (U(seed, 1, s) >> 51) in [1, 8192]
#    (mean ~4096), elements drawn like c5 (f1, CSR segments);
#  * c2f32 / c2f16 / c2bf16: 2^28 elements of another format (f2), element j = the low 32 / 16
#    bits of U(seed, 0, j), an all-ones exponent field (NaN/Inf) moved down by one exponent:
#    uniform over the finite bit patterns (every exponent incl. subnormals, both signs, zeros).
FORMAT_BITS = {"f32": (32, 0x7F800000, 1 << 23), "f16": (16, 0x7C00, 1 << 10), "bf16": (16, 0x7F80, 1 << 7)}
CONFIGS.update({
    "c5csr": dict(kind="csr", nseg=1 << 16, seed=9, st=0, lo=-200, hi=200, maxlen=1 << 13),
    "c2f32": dict(kind="bits", fmt="f32", n=1 << 28, seed=6, st=0),
    "c2f16": dict(kind="bits", fmt="f16", n=1 << 28, seed=7, st=0),
    "c2bf16": dict(kind="bits", fmt="bf16", n=1 << 28, seed=8, st=0),
    # f1 measurement workloads: c2's elements as a [4096, 65536] matrix reduced over dim 0 (K10,
    # strided), and 2^24 segments of 16 doubles drawn like c5 with seed 10 (K11, one lane each)
    "c2dim0": dict(kind="uniform", n=1 << 28, seed=2, st=0, lo=-1000, hi=1000, op="dim0", shape=(4096, 65536)),
    "c5s16": dict(kind="segments", n=1 << 28, seed=10, st=0, lo=-200, hi=200, nseg=1 << 24, seg_len=16),
    # f4 measurement workloads: the condition-number-sensitive sum (K12) over c2 (well conditioned)
    # and c3 (ill conditioned, C(X) ~ 2^1413) - the same elements as those configs
    "c2cs": dict(kind="uniform", n=1 << 28, seed=2, st=0, lo=-1000, hi=1000, op="condsens"),
    "c3cs": dict(kind="cancel", n=(1 << 28) + (1 << 20), seed=3, npairs=1 << 27,
                 pair_lo=0, pair_hi=600, ntiny=1 << 20, tiny_lo=-900, tiny_hi=-800, op="condsens"),
})


def mix64(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * _M1
        z = z ^ (z >> np.uint64(27))
        z = z * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def key(seed: int, st: int) -> np.uint64:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + G * np.uint64(st + 1)
    return mix64(np.array([z], dtype=np.uint64))[0]


def U(seed: int, st: int, j: np.ndarray) -> np.ndarray:
    k = key(seed, st)
    j = np.asarray(j, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(k + G * (j + np.uint64(1)))


def draw_bits(seed: int, st: int, i: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """uint64 bit patterns of draw(seed, st, i, lo, hi) for an index array ``i``."""
    i = np.asarray(i, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = U(seed, st, np.uint64(2) * i)
        v = U(seed, st, np.uint64(2) * i + np.uint64(1))
    frac = u & _MASK52
    sign = u >> np.uint64(63)
    span = np.uint64(hi - lo + 1)
    e = ((v >> np.uint64(32)) * span) >> np.uint64(32)          # in [0, span)
    biased = (e.astype(np.int64) + (lo + 1023)).astype(np.uint64)
    return (sign << np.uint64(63)) | (biased << np.uint64(52)) | frac


def draw(seed: int, st: int, i: np.ndarray, lo: int, hi: int) -> np.ndarray:
    return draw_bits(seed, st, i, lo, hi).view(np.float64)


def uniform(seed: int, lo: int, hi: int, start: int, count: int, st: int = 0) -> np.ndarray:
    """Elements [start, start+count) of the uniform-exponent family (c1, c2, c4, c5)."""
    idx = np.arange(start, start + count, dtype=np.uint64)
    return draw(seed, st, idx, lo, hi)


def cancel_unpermuted(cfg: dict, start: int, count: int) -> np.ndarray:
    """Elements [start, start+count) of c3 BEFORE the permutation:
    [a_0, -a_0, a_1, -a_1, ..., t_0, ..., t_{ntiny-1}].
    a_j = draw(seed, 0, j, pair_lo, pair_hi); t_m = draw(seed, 1, m, tiny_lo, tiny_hi)."""
    seed = cfg["seed"]
    npair2 = 2 * cfg["npairs"]
    pos = np.arange(start, start + count, dtype=np.int64)
    out = np.empty(count, dtype=np.uint64)
    pm = pos < npair2
    if pm.any():
        p = pos[pm]
        a = draw_bits(seed, 0, (p // 2).astype(np.uint64), cfg["pair_lo"], cfg["pair_hi"])
        a = a ^ ((p & 1).astype(np.uint64) << np.uint64(63))      # odd positions: negation
        out[pm] = a
    tm = ~pm
    if tm.any():
        m = (pos[tm] - npair2).astype(np.uint64)
        out[tm] = draw_bits(seed, 1, m, cfg["tiny_lo"], cfg["tiny_hi"])
    return out.view(np.float64)


def cancel_perm_keys(cfg: dict, start: int, count: int) -> np.ndarray:
    """Permutation keys U(seed, 2, idx) for c3 pre-permutation positions idx."""
    return U(cfg["seed"], 2, np.arange(start, start + count, dtype=np.uint64))


def cancel_permuted(cfg: dict) -> np.ndarray:
    """Full c3 in its permuted order (stable sort of positions by key). Large: n doubles."""
    n = cfg["n"]
    keys = cancel_perm_keys(cfg, 0, n)
    perm = np.argsort(keys, kind="stable")
    return cancel_unpermuted(cfg, 0, n)[perm]


def csr_offsets(cfg: dict) -> np.ndarray:
    """int64 offsets [0, len_0, len_0+len_1, ...] of a "csr" config (nseg + 1 entries)."""
    u = U(cfg["seed"], 1, np.arange(cfg["nseg"], dtype=np.uint64))
    lens = (u >> np.uint64(64 - int(np.log2(cfg["maxlen"])))).astype(np.int64) + 1
    return np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)


CONFIGS["c5csr"]["n"] = int(csr_offsets(CONFIGS["c5csr"])[-1])


def bits_fix(u: np.ndarray, fmt: str) -> np.ndarray:
    """Finite bit patterns of format ``fmt`` from raw 64-bit draws (see FORMAT_BITS)."""
    width, em, low = FORMAT_BITS[fmt]
    b = (u & np.uint64((1 << width) - 1)).astype(np.uint32 if width == 32 else np.uint16)
    spec = (b & b.dtype.type(em)) == b.dtype.type(em)
    b[spec] ^= b.dtype.type(low)
    return b


def bits(name: str, start: int = 0, count: int | None = None) -> np.ndarray:
    """Elements [start, start+count) of a "bits" config as bit patterns (uint32 / uint16)."""
    cfg = CONFIGS[name]
    if count is None:
        count = cfg["n"] - start
    return bits_fix(U(cfg["seed"], cfg["st"], np.arange(start, start + count, dtype=np.uint64)), cfg["fmt"])


def generate(name: str, start: int = 0, count: int | None = None, permute: bool = True) -> np.ndarray:
    """Elements [start, start+count) of config ``name`` as float64 (host memory).

    For c3 the permuted order needs the whole array; ``permute=False`` returns the
    pre-permutation order (the exact sum is order-independent)."""
    cfg = CONFIGS[name]
    n = cfg["n"]
    if count is None:
        count = n - start
    if start < 0 or start + count > n:
        raise ValueError("range outside config")
    if cfg["kind"] in ("uniform", "segments", "csr"):
        return uniform(cfg["seed"], cfg["lo"], cfg["hi"], start, count, cfg["st"])
    if cfg["kind"] == "bits":
        raise ValueError("use gen.bits() for the other formats")
    if permute:
        if start != 0 or count != n:
            raise ValueError("permuted c3 is only available whole; use permute=False")
        return cancel_permuted(cfg)
    return cancel_unpermuted(cfg, start, count)
