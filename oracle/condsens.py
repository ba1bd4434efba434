"""ORACLE (O3) - test infrastructure only; pure Python ints and fractions, small n.

The paper's condition-number-sensitive algorithm (§4 "Our
Condition-Number Sensitive PRAM Algorithm"), step by step in the paper's order and
notation, for binary64 inputs. Only ``tests/`` may import this module; it shares no
code with the CUDA path and does not import it (nor ``oracle.xsum_oracle``).

Objects:
  * a superaccumulator Y = (y_k, ..., y_0) has value sum_i y_i R^i in units of
    2^-1074 (PAPER.md:527-531 fixed point), radix R = 2^52 (R5), and is
    (alpha, beta)-regularized with alpha = beta = R-1: |y_i| <= R-1;
  * a sparse superaccumulator keeps only its active entries, here a
    dict {index i: y_i} with y_i != 0 (reading C1: an entry that became zero is
    inactive; the paper's "has ever been non-zero" is bookkeeping);
  * the gamma-truncated sparse superaccumulator keeps the gamma most significant
    entries.

The algorithm:
  1. a summation tree T of depth O(log n) with x_i at leaf i (reading C2: the complete
     binary tree over the index order - node (L, j) covers [j 2^L, (j+1) 2^L), a node
     whose right child is empty takes its left child unchanged);
  2. every leaf is converted to a sparse regularized superaccumulator (PAPER.md:744-750
     step 2: two components at digit i = floor(k/52));
  3. bottom-up, every internal node is the r-truncated sum of its children's r-truncated
     sparse superaccumulators, the sum by the carry rule of Lemma 1 on
     the merged active indices (Lemma 2);
  4. y = the floating-point value of the root (rounded to nearest even);
  5. stop if a stopping condition holds or nothing was truncated
     anywhere; else r <- r^2 and repeat from 3, starting at r = 2.

Reading C3: the paper takes eps_min = eps * 2^{E_{i_r}} from the root's least
significant retained component and argues that every truncated amount is below it
(PAPER.md:946-962). With cancellation between subtrees that is false (the root may keep
components far below a subtree's truncation point; tests/test_condsens_pins.py builds
such an input on which the literal rule stops with a non-faithful y). We keep the
paper's principle - "a bound whose magnitude is larger than any value we truncated"
 - and take eps_min = R^{E_cut} 2^-1074 with E_cut the largest index
of the r-th (least significant retained) entry over every node that dropped entries:
each node drops regularized digits below that index, of total magnitude <= R^{E_cut} - 1,
and there are < n nodes, so |S - T| < n eps_min as the paper's argument needs.

Reading C4: stopping condition (1) "y = y (+) n eps_min = y (+) -n eps_min" with (+) the
round-to-nearest-even addition, evaluated exactly (no overflow of n eps_min); y must be
finite and non-zero. Condition (2), "the exponent of the least significant bit of y is at
least ceil(log n) greater than E_{i_r}", is NOT sufficient as stated
(the rounding half-gap and the smaller gap below a power of two cost two more bits); we
use ulp(y) >= 2^(ceil(log2 n) + 2) eps_min.

Specials (NaN / +-Inf, R10) enter the tree as empty leaves and set flags.
"""
from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from fractions import Fraction

W = 52
R = 1 << W                 # radix (R5)
ND = 42                    # digit indices 0..41 (R7)
F_NAN, F_PINF, F_NINF = 1, 2, 4
UNIT = Fraction(1, 1 << 1074)


def leaf(x: float) -> tuple[dict, int]:
    """Step 2: x -> sparse regularized superaccumulator {i: y_i}, flags.
    |x| = M 2^(k-1074) (R1/R2); M 2^(k mod 52) = hi R + lo with 0 <= lo, hi < R;
    the components are +-lo at index floor(k/52) and +-hi at the next index."""
    (b,) = struct.unpack("<Q", struct.pack("<d", x))
    s, e, m = b >> 63, (b >> 52) & 0x7FF, b & (R - 1)
    if e == 0x7FF:
        return {}, (F_NAN if m else (F_NINF if s else F_PINF))
    M = m + (R if e else 0)
    k = max(e, 1) - 1
    i, o = divmod(k, W)
    v = M << o
    lo, hi = v % R, v // R
    sign = -1 if s else 1
    Y = {}
    if lo:
        Y[i] = sign * lo
    if hi:
        Y[i + 1] = sign * hi
    return Y, 0


def lemma1_sum(Y: dict, Z: dict) -> dict:
    """Sum of two regularized sparse superaccumulators (Lemma 1 :578-628,
    sparse form :703-711): on the merged active indices P_i = Y_i + Z_i; the signed carry out
    of position i is C_{i+1} = 1 if P_i >= R-1, -1 if P_i <= -(R-1), else 0; W_i = P_i - C_{i+1} R;
    S_i = W_i + C_i. An index is active in the sum if it was active in Y or Z or becomes
    non-zero through a carry; entries that end up zero are dropped (reading C1)."""
    active = sorted(set(Y) | set(Z))
    P = {i: Y.get(i, 0) + Z.get(i, 0) for i in active}
    C = {}                                      # C[i+1] = carry out of position i
    for i in active:
        if P[i] >= R - 1:
            C[i + 1] = 1
        elif P[i] <= -(R - 1):
            C[i + 1] = -1
        else:
            C[i + 1] = 0
    S = {}
    for i in sorted(set(active) | {j for j, c in C.items() if c}):
        Wi = P.get(i, 0) - C.get(i + 1, 0) * R
        Si = Wi + C.get(i, 0)
        if Si:
            S[i] = Si
    return S


def truncate(Y: dict, r: int) -> tuple[dict, int | None]:
    """The r-truncated sparse superaccumulator: the r most significant
    entries. Returns (Y'', cut) with cut the index of the least significant kept entry if any
    entry was dropped (every dropped index is below it), else None."""
    keys = sorted(Y, reverse=True)
    if len(keys) <= r:
        return dict(Y), None
    kept = keys[:r]
    return {i: Y[i] for i in kept}, kept[-1]


@dataclass
class TreeResult:
    root: dict            # the root's r-truncated sparse superaccumulator
    e_cut: int | None     # largest truncation index over all nodes (None: nothing dropped)
    ntrunc: int           # nodes that dropped entries
    flags: int


def tree_sum(leaves: list, r: int) -> TreeResult:
    """Steps 1 and 3: bottom-up over the complete binary tree of
    the index order (reading C2), every internal node = truncate_r(Lemma-1 sum of its
    children); a node without a right child is its left child."""
    level = [Y for Y in leaves]
    e_cut, ntrunc = None, 0
    while len(level) > 1:
        nxt = []
        for j in range(0, len(level), 2):
            if j + 1 == len(level):
                nxt.append(level[j])
                continue
            Y, cut = truncate(lemma1_sum(level[j], level[j + 1]), r)
            if cut is not None:
                ntrunc += 1
                e_cut = cut if e_cut is None else max(e_cut, cut)
            nxt.append(Y)
        level = nxt
    return TreeResult(root=level[0] if level else {}, e_cut=e_cut, ntrunc=ntrunc, flags=0)


def value(Y: dict) -> Fraction:
    """Exact value of a sparse superaccumulator."""
    return sum((Fraction(y * R ** i) for i, y in Y.items()), Fraction(0)) * UNIT


def rn(q: Fraction) -> float:
    """Round to nearest, ties to even (the standard library's correctly rounded division);
    +-inf beyond the binary64 range (R11)."""
    try:
        return float(q)
    except OverflowError:
        return math.inf if q > 0 else -math.inf


def stop_rule_1(y: float, n: int, e_cut: int) -> bool:
    """Stopping condition (1) (reading C4): y = y (+) n eps_min = y (+) -n eps_min,
    eps_min = R^{E_cut} 2^-1074, (+) round-to-nearest-even, evaluated exactly."""
    if math.isinf(y) or math.isnan(y) or y == 0:
        return False
    d = n * Fraction(R ** e_cut) * UNIT
    return rn(Fraction(y) + d) == y and rn(Fraction(y) - d) == y


def ulp_exp(y: float) -> int:
    """Exponent of the least significant bit of a finite non-zero binary64."""
    (b,) = struct.unpack("<Q", struct.pack("<d", abs(y)))
    e = (b >> 52) & 0x7FF
    return max(e, 1) - 1075


def stop_rule_2(y: float, n: int, e_cut: int) -> bool:
    """Stopping condition (2) (reading C4): the least significant bit of y at
    least ceil(log2 n) + 2 binary orders above eps_min = 2^(52 E_cut - 1074)."""
    if math.isinf(y) or math.isnan(y) or y == 0:
        return False
    return ulp_exp(y) >= (W * e_cut - 1074) + (n - 1).bit_length() + 2


@dataclass
class CondSensResult:
    value: float
    r: int                # the truncation parameter of the last iteration
    iterations: int
    exact: bool           # the last iteration truncated nothing (value = RN of the exact sum)
    e_cut: int | None
    root: dict
    flags: int


def condsens_sum(xs, rule: int = 1) -> CondSensResult:
    """The iteration of PAPER.md:895-918: r = 2, then r <- r^2 until a stopping condition holds
    or nothing was truncated. Returns the last iteration's y (a faithful rounding of the exact
    sum; the RN-even rounding when the iteration was exact)."""
    xs = [float(v) for v in xs]
    n = len(xs)
    leaves, flags = [], 0
    for v in xs:
        Y, f = leaf(v)
        leaves.append(Y)
        flags |= f
    stop = stop_rule_1 if rule == 1 else stop_rule_2
    r, it = 2, 0
    while True:
        it += 1
        t = tree_sum(leaves, r)
        y = rn(value(t.root))
        if t.e_cut is None or stop(y, n, t.e_cut):
            break
        r = r * r
    if flags & F_NAN or (flags & F_PINF and flags & F_NINF):
        y = math.nan
    elif flags & F_PINF:
        y = math.inf
    elif flags & F_NINF:
        y = -math.inf
    if y == 0:
        y = 0.0                # +0.0 for an exact zero (R9)
    return CondSensResult(value=y, r=r, iterations=it, exact=t.e_cut is None, e_cut=t.e_cut, root=t.root,
                          flags=flags)
