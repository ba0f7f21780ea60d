"""Property-based checks (hypothesis): the oracle on arbitrary inputs (CPU), and
the CUDA path against the oracle on arbitrary inputs incl. special values (GPU)."""
import math

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st
from hypothesis.extra import numpy as hnp

import oracle
from tests import _brute

INT_DT = ["int32", "uint32", "int64"]
INT_OPS = ["sum", "prod", "min", "max", "and", "or", "xor", "argmin", "argmax"]


@settings(max_examples=200, deadline=None)
@given(st.sampled_from(INT_DT), st.sampled_from(INT_OPS), st.data())
def test_oracle_int_order_invariance(dtype, op, data):
    """Integers: any permutation gives the same value; arg ops give the
    same value and the index moves with the element."""
    x = data.draw(hnp.arrays(np.dtype(dtype), st.integers(1, 64)))
    perm = np.array(data.draw(st.permutations(range(x.size))), dtype=np.int64)
    a, b = oracle.reduce(x, op), oracle.reduce(x[perm], op)
    assert a.value == b.value
    if op in ("argmin", "argmax"):
        assert x[a.index] == a.value and x[perm][b.index] == b.value
    elif op not in ("prod",):
        assert int(a.value) == _brute.int_exact(list(x), op, dtype)


@settings(max_examples=200, deadline=None)
@given(hnp.arrays(np.float64, st.integers(1, 40), elements=st.floats(-1e6, 1e6, allow_nan=False)))
def test_oracle_fp64_sum_is_nearly_exact(x):
    """double-double accumulation: within 1/2 ulp + 4 n 2^-104 sum|x| of the exact sum."""
    from fractions import Fraction
    r = oracle.reduce(x, "sum")
    ex = _brute.exact_sum(x)                      # exact rational
    sabs = float(np.sum(np.abs(x)))
    err = abs(Fraction(float(r.value)) - ex)      # no rounding of the referee
    assert err <= Fraction(0.5 * math.ulp(float(ex))) + Fraction(4 * x.size * 2.0 ** -104 * sabs) \
        + Fraction(2.0 ** -1074)


torch = pytest.importorskip("torch")

_specials = st.sampled_from([0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, 3.5e38, 1e-45])


@pytest.mark.gpu
@settings(max_examples=150, deadline=None, suppress_health_check=list(HealthCheck))
@given(st.sampled_from(["float32", "float64"]), st.sampled_from(["min", "max", "argmin", "argmax"]),
       st.data())
def test_gpu_float_minmax_arbitrary(dtype, op, data):
    from tests._parity import check
    from tests.test_gpu_parity import to_dev, val
    import paper_1710_07358_b200 as rd
    n = data.draw(st.integers(1, 3000))
    base = data.draw(hnp.arrays(np.dtype(dtype), n, elements=st.floats(-1e3, 1e3, width=32)))
    k = data.draw(st.integers(0, 4))
    for _ in range(k):
        base[data.draw(st.integers(0, n - 1))] = data.draw(_specials)
    off = data.draw(st.integers(0, 7))
    variant = data.draw(st.sampled_from(["vector", "bulk"]))
    check(val(rd.reduce_ex(to_dev(base, off), op, variant=variant)[0]), base, op)


@pytest.mark.gpu
@settings(max_examples=150, deadline=None, suppress_health_check=list(HealthCheck))
@given(st.sampled_from(INT_DT), st.sampled_from(INT_OPS + ["sum_compensated"]), st.data())
def test_gpu_int_arbitrary(dtype, op, data):
    from tests._parity import check
    from tests.test_gpu_parity import to_dev, val
    import paper_1710_07358_b200 as rd
    x = data.draw(hnp.arrays(np.dtype(dtype), st.integers(0, 5000)))
    off = data.draw(st.integers(0, 7))
    grid = data.draw(st.sampled_from([0, 1, 3, 200]))
    variant = data.draw(st.sampled_from(["vector", "bulk"]))
    check(val(rd.reduce_ex(to_dev(x, off), op, variant=variant, grid=grid)[0]), x, op)


@pytest.mark.gpu
@settings(max_examples=200, deadline=None, suppress_health_check=list(HealthCheck))
@given(st.sampled_from(["float32", "float64"]), st.data())
def test_gpu_exact_sum_arbitrary(dtype, data):
    """The exact sum (reading R17) on arbitrary floats -- any exponent, subnormals, signed
    zeros, inf/NaN, values that overflow any running sum -- is bit-exact against the oracle
    through both variants, any grid and any base offset."""
    from tests._parity import check
    from tests.test_gpu_parity import to_dev, val
    import paper_1710_07358_b200 as rd
    width = 32 if dtype == "float32" else 64
    x = data.draw(hnp.arrays(np.dtype(dtype), st.integers(0, 4000),
                             elements=st.floats(width=width, allow_nan=True, allow_infinity=True)))
    off = data.draw(st.integers(0, 7))
    grid = data.draw(st.sampled_from([0, 1, 5, 300]))
    variant = data.draw(st.sampled_from(["vector", "bulk"]))
    check(val(rd.reduce_ex(to_dev(x, off), "sum_exact", variant=variant, grid=grid)[0]), x, "sum_exact")


@pytest.mark.gpu
@settings(max_examples=120, deadline=None, suppress_health_check=list(HealthCheck))
@given(st.sampled_from([("int32", "sum"), ("uint32", "max"), ("int64", "xor"), ("float32", "sum"),
                        ("float64", "min"), ("float32", "argmax"), ("int64", "argmin"), ("float64", "sum_exact"),
                        ("float32", "sum_exact")]), st.data())
def test_gpu_random_block_splits(case, data):
    """Any split of an array into consecutive blocks (not only rd_shard_range's), each reduced
    to a record (exact records for the exact sum) and the records folded in block order, gives
    the oracle's result on the whole array (the partials of consecutive blocks combine
    in block order)."""
    from tests._parity import check
    from tests.test_gpu_parity import to_dev, val
    import paper_1710_07358_b200 as rd
    dtype, op = case
    n = data.draw(st.integers(0, 20000))
    if dtype.startswith("float"):
        x = data.draw(hnp.arrays(np.dtype(dtype), n, elements=st.floats(-1e6, 1e6, width=32)))
    else:
        x = data.draw(hnp.arrays(np.dtype(dtype), n))
    cuts = sorted(data.draw(st.lists(st.integers(0, n), max_size=6)))
    bounds = list(zip([0] + cuts, cuts + [n]))
    xd = to_dev(x, data.draw(st.integers(0, 7)))
    exact = op == "sum_exact" and dtype.startswith("float")
    RB = rd.EXACT_RECORD_BYTES if exact else rd.RECORD_BYTES
    recs = torch.empty(len(bounds) * RB, dtype=torch.uint8, device="cuda")
    for k, (b, e) in enumerate(bounds):
        if exact:
            rd.reduce_exact_partial(xd[b:e], rec=recs[k * RB:(k + 1) * RB])
        else:
            rd.reduce_partial(xd[b:e], op, rec=recs[k * RB:(k + 1) * RB])
    got = rd.combine_exact_records(recs, dtype) if exact else rd.combine_records(recs, dtype, op)
    check(val(got), x, op)
