"""Independent brute-force referees used to pin the oracle and to check the
CUDA path where several results are correct. Plain Python; shares no code
with oracle/ or the CUDA package.

- ``tree_results``: every evaluation tree of a commutative, associative-in-
  exact-arithmetic combiner over n <= 8 terms, evaluated in the given float
  precision (associativity/commutativity allow any order;
  P:50 fn 2: in floating point different orders give different results).
- ``exact_sum`` / ``exact_prod``: rational arithmetic (fractions.Fraction) as
  the exact referee ("exact-rational oracle" idea).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

WIDTH = {"int32": 32, "uint32": 32, "int64": 64}


def _f32(v):
    return np.float32(v)


def _combine_float(op, a, b, prec):
    if prec == "float32":
        a, b = np.float32(a), np.float32(b)
        with np.errstate(all="ignore"):
            r = a + b if op == "sum" else a * b
        return float(r)
    return a + b if op == "sum" else a * b


def tree_results(values, op, prec):
    """Set of results (as float bit patterns -> float) over all binary trees.

    Bitmask DP over subsets: R(S) = { a (x) b : S = A u B disjoint, a in R(A), b in R(B) }.
    Returns a set of python floats (NaN-free inputs assumed)."""
    n = len(values)
    assert 1 <= n <= 8
    R = {}
    for i, v in enumerate(values):
        R[1 << i] = {float(_f32(v)) if prec == "float32" else float(v)}
    for mask in range(1, 1 << n):
        if mask in R:
            continue
        low = mask & -mask
        out = set()
        sub = (mask - 1) & mask
        while sub:
            if sub & low:
                other = mask ^ sub
                if other:
                    for a in R[sub]:
                        for b in R[other]:
                            out.add(_combine_float(op, a, b, prec))
            sub = (sub - 1) & mask
        R[mask] = out
    return R[(1 << n) - 1]


def mixed_tree_results(values, prec):
    """Set of float sums over all binary trees whose every node is rounded EITHER to the
    element precision OR kept in the library's wide accumulator (fp64 for float32 data;
    double-double, exact at n <= 8 up to ~2^-100 relative, for float64 data), the root then
    rounded once to the element precision -- the results the default float sum can give
    (include/b200reduce.h: input-precision block trees added into a wide accumulator).
    n <= 8; NaN-free finite inputs."""
    n = len(values)
    assert 1 <= n <= 8

    def narrow(v):
        if prec == "float32":
            return Fraction(float(np.float32(float(v))))
        return Fraction(float(v))            # Fraction -> nearest double (correctly rounded)

    def wide(v):
        return Fraction(float(v)) if prec == "float32" else v   # fp64 rounding / exact

    R = {1 << i: {Fraction(float(v))} for i, v in enumerate(values)}
    for mask in range(1, 1 << n):
        if mask in R:
            continue
        low = mask & -mask
        out = set()
        sub = (mask - 1) & mask
        while sub:
            if sub & low and mask ^ sub:
                for a in R[sub]:
                    for b in R[mask ^ sub]:
                        out.add(narrow(a + b))
                        out.add(wide(a + b))
            sub = (sub - 1) & mask
        R[mask] = out
    return {float(narrow(v)) for v in R[(1 << n) - 1]}


def int_exact(values, op, dtype):
    """Exact integer reduction with Python big ints, reduced mod 2^w (two's complement)."""
    w = WIDTH[dtype]
    mask = (1 << w) - 1
    signed = dtype != "uint32"

    def to_py(v):
        v = int(v) & mask
        if signed and v >> (w - 1):
            v -= 1 << w
        return v

    vals = [to_py(v) for v in values]
    if op == "sum":
        r = sum(vals)
    elif op == "prod":
        r = 1
        for v in vals:
            r *= v
    elif op == "min":
        r = min(vals)
    elif op == "max":
        r = max(vals)
    elif op == "and":
        r = -1
        for v in vals:
            r &= v
    elif op == "or":
        r = 0
        for v in vals:
            r |= v
    elif op == "xor":
        r = 0
        for v in vals:
            r ^= v
    else:
        raise ValueError(op)
    return to_py(r)


def exact_sum(values) -> Fraction:
    return sum((Fraction(float(v)) for v in values), Fraction(0))


def exact_prod(values) -> Fraction:
    r = Fraction(1)
    for v in values:
        r *= Fraction(float(v))
    return r


def ulp(x: float, dtype: str) -> float:
    if dtype == "float32":
        x32 = np.float32(abs(x))
        return float(np.spacing(x32))
    return math.ulp(abs(x))


def total_order_min(values):
    """IEEE 754-2019 minimum over a list: NaN if any NaN, else smallest with -0 < +0."""
    if any(math.isnan(v) for v in values):
        return math.nan
    return min(values, key=lambda v: (v, 0 if math.copysign(1.0, v) < 0 else 1))


def total_order_max(values):
    if any(math.isnan(v) for v in values):
        return math.nan
    return max(values, key=lambda v: (v, 0 if math.copysign(1.0, v) < 0 else 1))
