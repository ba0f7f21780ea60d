"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics
fix -- closed forms, the paper's worked absorption example, brute force over
all evaluation orders, exact rational referees, identity laws and invariants.
None of these re-types the oracle's formula: each would fail on a plausible
mistake in it (dropped term, wrong sign/index, wrong identity, lost
compensation, wrong width or signedness). CPU only.
"""
from __future__ import annotations

import itertools
import math
import os
import random
import struct

import numpy as np
import pytest

import inputs
import oracle
from tests import _brute

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
INT_DTYPES = ["int32", "uint32", "int64"]
FLOAT_DTYPES = ["float32", "float64"]
INT_OPS = ["sum", "prod", "min", "max", "and", "or", "xor"]
FLOAT_OPS = ["sum", "prod", "min", "max"]
W = {"int32": 32, "uint32": 32, "int64": 64}


def _as_int(v, dtype):
    """numpy scalar -> python int with the dtype's signedness"""
    return int(v)


def _wrap(v, dtype):
    w = W[dtype]
    v &= (1 << w) - 1
    if dtype != "uint32" and v >> (w - 1):
        v -= 1 << w
    return v


def _bits(x: float, dtype: str) -> int:
    if dtype == "float32":
        return struct.unpack("<I", struct.pack("<f", x))[0]
    return struct.unpack("<Q", struct.pack("<d", x))[0]


# ---------------------------------------------------------------- closed forms
def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            rows.append([c.strip() for c in line.split("|")])
    return rows


@pytest.mark.parametrize("row", _golden_rows("closed_forms.txt"), ids=lambda r: "-".join(r[:3]))
def test_golden_closed_forms(row):
    """tests/golden/closed_forms.txt: BASELINE configs[0] (iota int32 sum n=2^20 = -524288)."""
    dtype, op, n, expected = row[0], row[1], int(row[2]), int(row[3])
    x = inputs.generate(n, dtype, "iota")
    assert _as_int(oracle.reduce(x, op).value, dtype) == expected


@pytest.mark.parametrize("dtype", INT_DTYPES)
@pytest.mark.parametrize("n", [1, 2, 7, 8, 9, 1023, 1024, 1025, 65535, 65537, 1 << 20])
def test_iota_closed_forms(dtype, n):
    """sum = n(n-1)/2 mod 2^w; xor(0..m) = [m,1,m+1,0][m mod 4]; min 0; max n-1."""
    x = inputs.generate(n, dtype, "iota")
    assert int(oracle.reduce(x, "sum").value) == _wrap(n * (n - 1) // 2, dtype)
    m = n - 1
    assert int(oracle.reduce(x, "xor").value) == [m, 1, m + 1, 0][m % 4]
    assert int(oracle.reduce(x, "min").value) == 0
    assert int(oracle.reduce(x, "max").value) == n - 1
    # or of 0..m = 2^bitlen(m) - 1; and of 0..m = 0 for n >= 2
    assert int(oracle.reduce(x, "or").value) == (1 << m.bit_length()) - 1
    if n >= 2:
        assert int(oracle.reduce(x, "and").value) == 0


@pytest.mark.parametrize("dtype", INT_DTYPES)
def test_iota_product_closed_form(dtype):
    """prod of 1..k (iota shifted by one element) = k! mod 2^w."""
    for k in [1, 5, 12, 13, 20, 21, 33, 40]:
        x = inputs.generate(k + 1, dtype, "iota")[1:]
        assert int(oracle.reduce(x, "prod").value) == _wrap(math.factorial(k), dtype)


@pytest.mark.parametrize("dtype", INT_DTYPES + FLOAT_DTYPES)
@pytest.mark.parametrize("n", [2, 3, 1000, 1 << 16])
def test_planted_extremes(dtype, n):
    """planted workload: min / max are the planted values at their hashed positions."""
    x = inputs.generate(n, dtype, "planted", seed=3)
    pmax, pmin = inputs.planted_positions(3, n)
    assert pmax != pmin
    if dtype.startswith("float"):
        assert float(oracle.reduce(x, "max").value) == 2.0 ** 20
        assert float(oracle.reduce(x, "min").value) == -(2.0 ** 20)
    else:
        assert int(oracle.reduce(x, "max").value) == 1 << 30
        assert int(oracle.reduce(x, "min").value) == 3
    assert x[pmax] == x.max() and x[pmin] == x.min()


# ------------------------------------------------------ the paper's worked example
def test_absorption_golden():
    """PAPER.md P:50 fn 2 (tests/golden/absorption.txt): 1.5 + 4^50 - 4^50 -> 0 or 1.5."""
    big = 4.0 ** 50
    # the paper's claim, pinned with the independent brute-force enumerator
    for prec in FLOAT_DTYPES:
        assert _brute.tree_results([1.5, big, -big], "sum", prec) == {0.0, 1.5}
    # the golden left fold in each precision (the plain fold the footnote describes)
    for order, want in [([1.5, big, -big], 0.0), ([big, -big, 1.5], 1.5)]:
        for prec in FLOAT_DTYPES:
            acc = np.array([order[0]], dtype=prec)[0]
            for t in order[1:]:
                acc = acc + np.array([t], dtype=prec)[0]
            assert float(acc) == want
    # the oracle: its double-double accumulator (fp32 and fp64 data) keeps 1.5 in every
    # order -- the exact sum the footnote calls "always the same"
    for prec in FLOAT_DTYPES:
        for order in ([1.5, big, -big], [big, -big, 1.5], [big, 1.5, -big]):
            r = oracle.reduce(np.array(order, dtype=prec), "sum")
            assert float(r.value) == 1.5
            assert r.sum_abs == 2 * big + 1.5


def test_compensation_golden():
    """tests/golden/kahan.txt: [1, 1e100, 1, -1e100] -> exact 2.0; naive fp64 fold 0.0."""
    terms = [1.0, 1e100, 1.0, -1e100]
    naive = 0.0
    for t in terms:
        naive += t
    assert naive == 0.0  # the case discriminates a plain fold
    assert float(oracle.reduce(np.array(terms), "sum").value) == 2.0
    assert float(_brute.exact_sum(terms)) == 2.0


# ------------------------------------------------------ brute force, n <= 8
@pytest.mark.parametrize("dtype", INT_DTYPES)
@pytest.mark.parametrize("op", INT_OPS)
def test_int_brute_force_all_orders(dtype, op):
    """Integers: every permutation x parenthesisation gives one value = the oracle."""
    rng = random.Random(hash((dtype, op)) & 0xFFFF)
    for n in range(1, 7):
        for _ in range(6):
            if op == "prod":
                vals = [rng.randrange(1 << 20) | 1 for _ in range(n)]
            elif op in ("and", "or"):
                vals = [rng.randrange(1 << W[dtype]) for _ in range(n)]
            else:
                vals = [rng.randrange(-(1 << (W[dtype] - 1)), 1 << (W[dtype] - 1)) for _ in range(n)]
            x = np.array([v & ((1 << W[dtype]) - 1) for v in vals], dtype=np.uint64).astype(
                inputs.NP_DTYPES[dtype])
            got = int(oracle.reduce(x, op).value)
            want = _brute.int_exact(list(x), op, dtype)
            assert got == want, (n, vals)
            # any permutation of the input gives the same oracle value
            for perm in itertools.islice(itertools.permutations(range(n)), 24):
                assert int(oracle.reduce(x[list(perm)], op).value) == got


@pytest.mark.parametrize("prec", FLOAT_DTYPES)
def test_float_sum_brute_force_contains_exact(prec):
    """Floats, n <= 7: the exactly-rounded sum is always one of the tree results in
    small-exponent-range cases; the oracle (wider accumulator) returns it."""
    rng = np.random.default_rng(5)
    for n in range(1, 8):
        for _ in range(5):
            v = rng.integers(-1000, 1000, n) / 64.0   # exact in fp32: no rounding anywhere
            x = v.astype(prec)
            trees = _brute.tree_results(list(x), "sum", prec)
            assert len(trees) == 1  # exact inputs: all orders agree
            assert float(oracle.reduce(x, "sum").value) in trees


# ------------------------------------------------------ exact rational referee
@pytest.mark.parametrize("prec", FLOAT_DTYPES)
@pytest.mark.parametrize("wl", ["u01", "normalish"])
def test_float_sum_exact_referee(prec, wl):
    """|oracle - exact| within the oracle's own rounding (double-double, fp32 and fp64
    data: 4n*2^-104*sum|x|) + 1/2 ulp of the final rounding (+ the fp64 step of fp32 data)."""
    for n in [1, 2, 3, 17, 1000, 4099]:
        x = inputs.generate(n, prec, wl, seed=n)
        r = oracle.reduce(x, "sum")
        ex = _brute.exact_sum(x)
        sabs = float(sum(abs(_brute.Fraction(float(t))) for t in x))
        acc_err = 4 * n * 2.0 ** -104 * sabs
        got = _brute.Fraction(r.hi) + _brute.Fraction(r.lo)     # the unrounded double-double
        assert abs(got - ex) <= _brute.Fraction(acc_err)
        step = 2.0 ** -53 * abs(float(ex)) if prec == "float32" else 0.0   # hi + lo -> fp64 -> fp32
        assert abs(float(r.value) - float(ex)) <= 0.5 * _brute.ulp(float(r.value), prec) + acc_err + step
        assert math.isclose(r.sum_abs, sabs, rel_tol=1e-15)


@pytest.mark.parametrize("prec", FLOAT_DTYPES)
def test_float_prod_exact_referee(prec):
    for n in [1, 2, 5, 64, 300]:
        x = inputs.generate(n, prec, "near_one", seed=n + 11)
        r = oracle.reduce(x, "prod")
        ex = float(_brute.exact_prod(x))
        acc_err = 4 * n * 2.0 ** -104 * abs(ex)
        got = _brute.Fraction(r.hi) + _brute.Fraction(r.lo)
        assert abs(got - _brute.exact_prod(x)) <= _brute.Fraction(acc_err * 1.0000001)
        step = 2.0 ** -53 * abs(ex) if prec == "float32" else 0.0
        assert abs(float(r.value) - ex) <= 0.5 * _brute.ulp(float(r.value), prec) + acc_err * 1.0000001 + step


def test_plain_fp64_fold_is_not_enough():
    """Why the fp64 oracle uses double-double: a plain fp64 fold
    misses the exact sum by many ulps; the oracle does not."""
    n = 1 << 14
    x = inputs.generate(n, "float64", "u01", seed=9)
    ex = _brute.exact_sum(x)
    plain = 0.0
    for t in x.tolist():
        plain += t
    err_plain = abs(_brute.Fraction(plain) - ex)
    err_oracle = abs(_brute.Fraction(float(oracle.reduce(x, "sum").value)) - ex)
    assert err_oracle <= _brute.Fraction(math.ulp(float(ex))) / 2
    assert err_plain > 4 * err_oracle


def test_fp32_data_plain_fp64_fold_is_not_enough():
    """Why fp32 data also take the double-double accumulator (a plain fp64 fold
    of fp32 data can err by (n-1) 2^-53 sum|x| = 16 eps32 sum|x| at n = 2^34, above the 4 eps32
    tolerance it referees): 2^30 followed by 2^-30 terms -- each is absorbed by a plain fp64
    running sum (2^30 + 2^-30 needs 61 bits), the double-double keeps every one exactly."""
    k = 3000
    x = np.array([2.0 ** 30] + [2.0 ** -30] * k, dtype=np.float32)
    ex = _brute.exact_sum(x)
    plain = 0.0
    for t in x.tolist():
        plain += t
    assert plain == 2.0 ** 30 and _brute.Fraction(plain) != ex
    r = oracle.reduce(x, "sum")
    assert _brute.Fraction(r.hi) + _brute.Fraction(r.lo) == ex
    r = oracle.reduce(x[::-1].copy(), "sum")            # small terms first: exact either way
    assert _brute.Fraction(r.hi) + _brute.Fraction(r.lo) == ex


@pytest.mark.parametrize("prec", FLOAT_DTYPES)
@pytest.mark.parametrize("op,wl", [("sum", "u01"), ("sum", "normalish"), ("sum", "wide"), ("prod", "near_one")])
def test_merge_float_branch_vs_fraction(prec, op, wl):
    """or_merge's float + / x branch (the rank-order combine of the host-logic tests) against
    exact rationals on split arrays, at the double-double bound 4n 2^-104 sum|x| (+) /
    8n 2^-104 |prod| (x): a dropped lo word (the merge adding only hi) misses it by ~2^-53."""
    n = 3001
    x = inputs.generate(n, prec, wl, seed=21)
    if op == "sum":
        ex = _brute.exact_sum(x)
        bound = _brute.Fraction(4 * n * 2.0 ** -104) * sum(abs(_brute.Fraction(float(t))) for t in x)
    else:
        ex = _brute.exact_prod(x)
        bound = _brute.Fraction(8 * n * 2.0 ** -104) * abs(ex)
    for cuts in ([1], [1500], [2999], [7, 700, 2000, 3000]):
        parts = np.split(x, cuts)
        acc = oracle.Fold(prec, op)
        for p in parts:
            acc.merge(oracle.Fold(prec, op).fold(p))
        r = acc.result()
        assert r.count == n
        got = _brute.Fraction(r.hi) + _brute.Fraction(r.lo)
        assert abs(got - ex) <= bound, (cuts, float(got - ex))
        # and the merged fold is the one-shot fold's value
        one = oracle.reduce(x, op)
        assert abs(float(r.value) - float(one.value)) <= _brute.ulp(float(one.value), prec)


# ------------------------------------------------------ exact-representable workloads
@pytest.mark.parametrize("n", [1, 1000, 1 << 16, (1 << 18) + 3])
def test_exact_float_workloads(n):
    """fp64 + of |x| <= 2^16 integers and fp32 + of sparse +-1 are exact in ANY order;
    x of sparse powers of two is the closed form 2^(#2 - #0.5)."""
    xi = inputs.generate(n, "int64", "int_small", seed=4)
    xd = inputs.generate(n, "float64", "int_small", seed=4)
    assert np.array_equal(xi.astype(np.float64), xd)
    assert float(oracle.reduce(xd, "sum").value) == float(int(xi.sum()))
    xs = inputs.generate(n, "float32", "sparse_pm1", seed=4)
    assert float(oracle.reduce(xs, "sum").value) == float(int(xs.astype(np.int64).sum()))
    for prec in FLOAT_DTYPES:
        xp = inputs.generate(n, prec, "pow2_sparse", seed=4)
        e = int((xp == 2.0).sum()) - int((xp == 0.5).sum())
        assert int((xp != 1.0).sum()) == int((xp == 2.0).sum() + (xp == 0.5).sum())
        assert float(oracle.reduce(xp, "prod").value) == 2.0 ** e


# ------------------------------------------------------ identities and special values
SPECIALS32 = [0.0, -0.0, 1.0, -1.0, 1.5, float("inf"), float("-inf"), 1e-45, -1e-45, 1e-40,
              3.4028234663852886e38, -3.4028234663852886e38, 2.0 ** -126]


@pytest.mark.parametrize("dtype", INT_DTYPES + FLOAT_DTYPES)
@pytest.mark.parametrize("op", INT_OPS)
def test_identity_table_and_law(dtype, op):
    """n=0 -> Algorithm 1's initial accumulator (INFINITY for min);
    identity (x) x == x."""
    if dtype.startswith("float") and op in ("and", "or", "xor"):
        with pytest.raises(oracle.OracleError):
            oracle.identity(dtype, op)
        return
    ident = oracle.identity(dtype, op)
    empty = oracle.reduce(np.zeros(0, dtype=inputs.NP_DTYPES[dtype]), op).value
    if dtype.startswith("float"):
        want = {"sum": 0.0, "prod": 1.0, "min": math.inf, "max": -math.inf}[op]
        assert float(ident) == want and _bits(float(empty), dtype) == _bits(want, dtype)
        pad = -0.0 if op == "sum" else want     # -0.0 is the true additive identity
        for v in SPECIALS32:
            x = np.array([pad, v], dtype=dtype)
            r = float(oracle.reduce(x, op).value)
            assert _bits(r, dtype) == _bits(float(np.array(v, dtype=dtype)), dtype), (op, v)
    else:
        w = W[dtype]
        want = {"sum": 0, "prod": 1, "and": -1, "or": 0, "xor": 0,
                "min": (1 << (w - 1)) - 1 if dtype != "uint32" else (1 << w) - 1,
                "max": -(1 << (w - 1)) if dtype != "uint32" else 0}[op]
        assert int(ident) == _wrap(want, dtype) and int(empty) == int(ident)
        rng = random.Random(1)
        for _ in range(50):
            v = rng.randrange(1 << w)
            x = np.array([int(ident) & ((1 << w) - 1), v], dtype=np.uint64).astype(dtype)
            assert int(oracle.reduce(x, op).value) == int(x[1])


@pytest.mark.parametrize("dtype", FLOAT_DTYPES)
def test_minmax_ieee_brute_force(dtype):
    """Reading R4 (IEEE minimum/maximum: NaN propagates, -0 < +0) over all pairs and
    triples of a special-value domain, against an independent total-order definition."""
    dom = [0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, 1e-45, -2.5]
    for k in (1, 2, 3):
        for combo in itertools.product(dom, repeat=k):
            x = np.array(combo, dtype=dtype)
            xs = [float(t) for t in x]
            for op, ref in (("min", _brute.total_order_min), ("max", _brute.total_order_max)):
                got, want = float(oracle.reduce(x, op).value), ref(xs)
                if math.isnan(want):
                    assert math.isnan(got)
                else:
                    assert _bits(got, dtype) == _bits(want, dtype), (op, combo)


@pytest.mark.parametrize("dtype", FLOAT_DTYPES)
def test_signed_zero_sum(dtype):
    """Reading R2: the fold starts at x_0, so [-0,-0] -> -0.0; any +0 or cancellation -> +0."""
    z = lambda v: _bits(float(oracle.reduce(np.array(v, dtype=dtype), "sum").value), dtype)
    assert z([-0.0]) == _bits(-0.0, dtype)
    assert z([-0.0, -0.0, -0.0]) == _bits(-0.0, dtype)
    assert z([-0.0, 0.0]) == _bits(0.0, dtype)
    assert z([1.0, -1.0]) == _bits(0.0, dtype)
    assert z([]) == _bits(0.0, dtype)


@pytest.mark.parametrize("dtype", FLOAT_DTYPES)
def test_inf_nan_sum(dtype):
    r = lambda v, op="sum": float(oracle.reduce(np.array(v, dtype=dtype), op).value)
    assert r([1.0, math.inf, 2.0]) == math.inf
    assert math.isnan(r([math.inf, 1.0, -math.inf]))
    assert math.isnan(r([1.0, math.nan]))
    assert r([2.0, math.inf], "prod") == math.inf
    assert math.isnan(r([0.0, math.inf], "prod"))


# ------------------------------------------------------ invariants
@pytest.mark.parametrize("dtype", INT_DTYPES)
@pytest.mark.parametrize("op", INT_OPS)
def test_int_shuffle_invariance(dtype, op):
    """>= 100 random shuffles of an n <= 2^12 integer array give identical results."""
    wl = inputs.default_workload(dtype, op)
    x = inputs.generate(4096, dtype, wl, seed=2)
    want = int(oracle.reduce(x, op).value)
    rng = np.random.default_rng(0)
    for _ in range(100):
        assert int(oracle.reduce(rng.permutation(x), op).value) == want


@pytest.mark.parametrize("dtype,op", [(d, o) for d in INT_DTYPES for o in INT_OPS] +
                         [(d, o) for d in FLOAT_DTYPES for o in FLOAT_OPS])
def test_streaming_fold_equals_one_shot(dtype, op):
    """Algorithm 1 is one left fold: folding chunk by chunk gives identical bits."""
    wl = inputs.default_workload(dtype, op)
    x = inputs.generate(10007, dtype, wl, seed=6)
    one = oracle.reduce(x, op)
    f = oracle.Fold(dtype, op)
    for a, b in [(0, 1), (1, 1000), (1000, 1001), (1001, 10007)]:
        f.fold(x[a:b])
    two = f.result()
    assert one.value.tobytes() == two.value.tobytes()
    assert one.hi == two.hi and one.lo == two.lo


@pytest.mark.parametrize("dtype", INT_DTYPES)
@pytest.mark.parametrize("op", INT_OPS)
def test_block_merge_exact_for_ints(dtype, op):
    """fold(A) (x) fold(B) == fold(A ++ B) bit-exactly for integers, any split."""
    wl = inputs.default_workload(dtype, op)
    x = inputs.generate(5000, dtype, wl, seed=8)
    want = oracle.reduce(x, op).value
    for cut in [0, 1, 2500, 4999, 5000]:
        a = oracle.Fold(dtype, op).fold(x[:cut])
        b = oracle.Fold(dtype, op).fold(x[cut:])
        assert a.merge(b).result().value == want


def test_paper_n_int32_sum_matches_numpy_wrap():
    """n = 5,533,214 (the paper's only workload): int32 sum == numpy's exact
    int64 sum reduced mod 2^32 (an independent library routine)."""
    n = 5533214
    x = inputs.generate(n, "int32", "uniform_bits", seed=1)
    want = _wrap(int(x.astype(np.int64).sum()), "int32")
    assert int(oracle.reduce(x, "sum").value) == want
    assert int(oracle.reduce(x, "xor").value) == int(np.bitwise_xor.reduce(x))
    assert int(oracle.reduce(x, "min").value) == int(x.min())
    assert int(oracle.reduce(x, "max").value) == int(x.max())
    assert int(oracle.reduce(x, "and").value) == int(np.bitwise_and.reduce(x))
    assert int(oracle.reduce(x, "or").value) == int(np.bitwise_or.reduce(x))


def test_bitwise_on_float_rejected():
    for op in ("and", "or", "xor"):
        with pytest.raises(oracle.OracleError):
            oracle.reduce(np.ones(3, np.float32), op)


# ------------------------------------------------------ argmin / argmax (f4, reading R6)
def _ref_arg(values, op):
    """Independent definition: smallest index attaining the min/max under the
    total order NaN-first, then value, then -0 < +0."""
    def key(i):
        v = float(values[i])
        if math.isnan(v):
            return (0, 0.0, 0, i)
        neg0 = 1 if (v == 0.0 and math.copysign(1.0, v) < 0) else 0
        if op == "argmin":
            return (1, v, 0 if neg0 else 1, i)
        return (1, -v, 1 if neg0 else 0, i)
    return min(range(len(values)), key=key)


@pytest.mark.parametrize("dtype", INT_DTYPES + FLOAT_DTYPES)
@pytest.mark.parametrize("op", ["argmin", "argmax"])
def test_arg_ops_against_definition_and_numpy(dtype, op):
    rng = np.random.default_rng(7)
    for n in (1, 2, 5, 100, 4097):
        for _ in range(5):
            if dtype.startswith("float"):
                x = rng.integers(-20, 20, n).astype(dtype) / 4   # many ties
            else:
                x = rng.integers(0, 50, n).astype(dtype)
            r = oracle.reduce(x, op)
            assert r.index == _ref_arg(list(x), op)
            np_idx = int(np.argmin(x) if op == "argmin" else np.argmax(x))  # first occurrence
            if not (dtype.startswith("float") and np.any(x == 0)):
                assert r.index == np_idx
            assert x[r.index] == r.value


@pytest.mark.parametrize("dtype", FLOAT_DTYPES)
def test_arg_ops_special_values(dtype):
    dom = [0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, 2.5]
    for k in (1, 2, 3):
        for combo in itertools.product(dom, repeat=k):
            x = np.array(combo, dtype=dtype)
            for op in ("argmin", "argmax"):
                r = oracle.reduce(x, op)
                want = _ref_arg(list(x), op)
                assert r.index == want, (op, combo)
                if math.isnan(combo[want]):
                    assert math.isnan(float(r.value))
                else:
                    assert _bits(float(r.value), dtype) == _bits(float(x[want]), dtype)


@pytest.mark.parametrize("dtype", INT_DTYPES + FLOAT_DTYPES)
def test_arg_ops_planted_and_empty(dtype):
    n = 100000
    x = inputs.generate(n, dtype, "planted", seed=5)
    pmax, pmin = inputs.planted_positions(5, n)
    assert oracle.reduce(x, "argmax").index == pmax
    assert oracle.reduce(x, "argmin").index == pmin
    e = oracle.reduce(x[:0], "argmin")
    assert e.index == -1 and e.value == oracle.identity(dtype, "min")


@pytest.mark.parametrize("dtype", ["int32", "uint32", "float32", "float64"])
def test_arg_ops_block_merge(dtype):
    """fold(A) merged with fold(B) == fold(A ++ B): indices of B shift by |A|; ties keep A."""
    rng = np.random.default_rng(3)
    x = (rng.integers(0, 7, 3000)).astype(dtype)
    for op in ("argmin", "argmax"):
        want = oracle.reduce(x, op)
        for cut in (0, 1, 1500, 2999, 3000):
            a = oracle.Fold(dtype, op).fold(x[:cut])
            b = oracle.Fold(dtype, op).fold(x[cut:])
            got = a.merge(b).result()
            assert got.index == want.index and got.value == want.value


def test_overflowing_double_double_sum_is_inf_not_nan():
    """A finite fp64 sum whose running value overflows gives +inf (IEEE 754 overflow of a sum of
    positive terms), in the value and in sum|x|; TwoSum's error term of an overflowed sum is NaN and
    must not leak into the double-double accumulators."""
    big = np.finfo(np.float64).max
    r = oracle.reduce(np.array([big, big, 1.0], np.float64), "sum")
    assert r.value == np.inf and r.sum_abs == np.inf
    r = oracle.reduce(np.array([-big, -big], np.float64), "sum")
    assert r.value == -np.inf and r.sum_abs == np.inf
