"""Pins of the oracle's exact sum (reading R17): the real
sum of the float values, computed exactly, rounded once to nearest-even.

The references here are independent of oracle.c's multi-limb arithmetic:
Python's exact rationals (fractions.Fraction) for the sum, ``float(Fraction)``
(CPython rounds int/int true division correctly) for fp64, a nearest-float32
search by exact comparison for fp32, hand-derived values from
``tests/golden/exact_sum.txt`` (ties, sticky bits, overflow threshold,
subnormals, signed zeros, specials), and invariants (any order, any split into
blocks gives the same bits). CPU only.
"""
from __future__ import annotations

import math
import os
from fractions import Fraction

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
F32_MAX = Fraction(np.finfo(np.float32).max.item())


def _bits(v, dtype):
    return np.array([v], dtype=dtype).view(np.uint32 if dtype == "float32" else np.uint64)[0]


def _rn64(s: Fraction) -> float:
    """Fraction -> nearest double, ties to even (CPython's correctly rounded int/int division);
    beyond the range -> +-inf (the IEEE 754 overflow threshold is 2^1024 - 2^970)."""
    try:
        return float(s)
    except OverflowError:
        return math.inf if s > 0 else -math.inf


def _rn32(s: Fraction) -> np.float32:
    """Fraction -> nearest float32, ties to even, by comparing the exact distances to the
    neighbouring float32 values (no bit manipulation)."""
    thresh = F32_MAX + (Fraction(2) ** 104) / 2        # 2^128 - 2^103: the overflow threshold
    if s >= thresh:
        return np.float32(np.inf)
    if s <= -thresh:
        return np.float32(-np.inf)
    guess = np.float32(float(s)) if abs(s) <= F32_MAX else np.float32(math.copysign(float(F32_MAX), float(s)))
    with np.errstate(over="ignore"):
        cands = {guess, np.nextafter(guess, np.float32(np.inf)), np.nextafter(guess, np.float32(-np.inf))}
    cands = [c for c in cands if np.isfinite(c)]
    best = min(cands, key=lambda c: (abs(Fraction(c.item()) - s),
                                     int(np.array([c]).view(np.uint32)[0]) & 1))   # tie -> even mantissa
    return np.float32(best)


def _expected(x: np.ndarray) -> np.floating:
    """R17 from the definition: specials first, then the exact rational sum rounded once."""
    dt = x.dtype.name
    if np.isnan(x).any() or (np.isposinf(x).any() and np.isneginf(x).any()):
        return x.dtype.type(np.nan)
    if np.isposinf(x).any():
        return x.dtype.type(np.inf)
    if np.isneginf(x).any():
        return x.dtype.type(-np.inf)
    s = sum((Fraction(v.item()) for v in x), Fraction(0))
    if s == 0:
        all_neg = x.size > 0 and all(v == 0 and np.signbit(v) for v in x)
        return x.dtype.type(-0.0 if all_neg else 0.0)
    return np.float32(_rn32(s)) if dt == "float32" else np.float64(_rn64(s))


def _same(a, b, dtype):
    if np.isnan(a) or np.isnan(b):
        return bool(np.isnan(a) and np.isnan(b))
    return _bits(a, dtype) == _bits(b, dtype)


def _term(t: str, dtype: str):
    t = t.strip()
    if t.startswith(("2^", "-2^")) or "*2^" in t:
        sign = -1 if t.startswith("-") else 1
        t = t.lstrip("-")
        mult = 1
        if "*" in t:
            m, t = t.split("*")
            mult = int(m)
        return np.dtype(dtype).type(sign * mult * math.ldexp(1.0, int(t[2:])))
    return np.dtype(dtype).type(float(t))


def _golden():
    rows = []
    with open(os.path.join(GOLDEN, "exact_sum.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            dt, terms, exp, why = [c.strip() for c in line.split("|")]
            rows.append((dt, [_term(t, dt) for t in terms.split(",")], np.dtype(dt).type(float(exp)), why))
    return rows


@pytest.mark.parametrize("dtype,terms,expected,why", _golden(), ids=lambda v: None)
def test_exact_golden(dtype, terms, expected, why):
    x = np.array(terms, dtype=dtype)
    got = oracle.reduce(x, "sum_exact").value
    assert _same(got, expected, dtype), (terms, got, expected, why)
    # the golden values agree with the independent rational reference too
    assert _same(_expected(x), expected, dtype), why
    # and with every order of the terms (P:50 fn 2: the exact sum does not depend on it)
    for k in range(6):
        perm = np.random.default_rng(k).permutation(x.size)
        assert _same(oracle.reduce(x[perm], "sum_exact").value, expected, dtype)


def _wide_floats(rng, n, dtype, lo_exp, hi_exp):
    """floats with random signs, mantissas and exponents over [lo_exp, hi_exp] (incl. subnormals)"""
    m = rng.random(n) + 0.5
    e = rng.integers(lo_exp, hi_exp + 1, n)
    s = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    return (s * np.ldexp(m, e)).astype(dtype)


@pytest.mark.parametrize("seed", range(12))
@pytest.mark.parametrize("dtype,lo,hi", [("float32", -160, 127), ("float32", -20, 20),
                                         ("float64", -1080, 1023), ("float64", -60, 60)])
def test_exact_vs_rationals(seed, dtype, lo, hi):
    """Random terms over the whole exponent range (incl. subnormals and overflowing partial sums)
    vs the exact rational sum rounded once."""
    rng = np.random.default_rng(1000 * seed + abs(lo))
    x = _wide_floats(rng, int(rng.integers(1, 300)), dtype, lo, hi)
    x = x[np.isfinite(x)]
    got = oracle.reduce(x, "sum_exact").value
    assert _same(got, _expected(x), dtype)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_exact_near_ties(dtype):
    """Sums constructed to land on, just above and just below rounding midpoints."""
    rng = np.random.default_rng(7)
    p = 24 if dtype == "float32" else 53
    for _ in range(200):
        e = int(rng.integers(-20, 20))
        base = np.dtype(dtype).type(math.ldexp(1.0 + float(rng.integers(0, 1 << 20)) * 2.0 ** -20, e))
        half_ulp = math.ldexp(1.0, e - p)                      # half an ulp of base
        for tweak in (0.0, math.ldexp(1.0, e - p - 30), -math.ldexp(1.0, e - p - 30)):
            terms = [base, np.dtype(dtype).type(half_ulp)]
            if tweak:
                terms.append(np.dtype(dtype).type(tweak))
            x = np.array(terms, dtype=dtype)
            assert _same(oracle.reduce(x, "sum_exact").value, _expected(x), dtype)


@settings(max_examples=300, deadline=None)
@given(st.lists(st.floats(width=64, allow_nan=True, allow_infinity=True), min_size=0, max_size=40))
def test_exact_fp64_hypothesis(vals):
    x = np.array(vals, dtype=np.float64)
    got = oracle.reduce(x, "sum_exact").value
    if x.size == 0:
        assert _bits(got, "float64") == 0          # empty -> +0.0 (R1)
        return
    assert _same(got, _expected(x), "float64")


@settings(max_examples=300, deadline=None)
@given(st.lists(st.floats(width=32, allow_nan=True, allow_infinity=True), min_size=1, max_size=40))
def test_exact_fp32_hypothesis(vals):
    x = np.array(vals, dtype=np.float32)
    assert _same(oracle.reduce(x, "sum_exact").value, _expected(x), "float32")


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_exact_order_and_block_invariance(dtype):
    """Any order and any split into consecutive blocks merged in order give the same bits."""
    rng = np.random.default_rng(3)
    x = _wide_floats(rng, 5000, dtype, -40, 40)
    ref = oracle.reduce(x, "sum_exact").value
    for k in range(5):
        perm = rng.permutation(x.size)
        assert _same(oracle.reduce(x[perm], "sum_exact").value, ref, dtype)
        cuts = sorted(rng.choice(np.arange(1, x.size), size=k + 1, replace=False))
        blocks = np.split(x, cuts)
        f = oracle.Fold(dtype, "sum_exact").fold(blocks[0])
        for b in blocks[1:]:
            f.merge(oracle.Fold(dtype, "sum_exact").fold(b))
        assert _same(f.result().value, ref, dtype)


def test_exact_u01_matches_fsum():
    """u01 float32 terms are multiples of 2^-24 below 1: with n = 2^20 the exact sum has < 45
    significant bits, so math.fsum (a correctly rounded library sum) returns it exactly, and one
    numpy float32 conversion rounds it once."""
    import inputs
    x = inputs.generate(1 << 20, "float32", "u01", seed=1)
    s = math.fsum(x.astype(np.float64))
    assert Fraction(s) == sum((Fraction(int(v * 2 ** 24)) for v in x), Fraction(0)) / 2 ** 24
    assert _same(oracle.reduce(x, "sum_exact").value, np.float32(s), "float32")


def test_exact_integers_are_the_sum():
    rng = np.random.default_rng(5)
    for dt in ("int32", "uint32", "int64"):
        x = rng.integers(0, 1 << 30, 1000).astype(dt)
        assert oracle.reduce(x, "sum_exact").value == oracle.reduce(x, "sum").value
    assert oracle.identity("float32", "sum_exact") == 0 and not np.signbit(oracle.identity("float32", "sum_exact"))
