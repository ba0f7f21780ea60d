"""Comparison of a CUDA-path result with the oracle.

- integers, all ops: bit-exact;
- float min/max: bit-exact (NaN compared as "is NaN");
- float sum_exact: bit-exact (the exact sum rounded once is unique; reading R17);
- float sum: |gpu - exact| <= 4 * eps(dtype) * sum|x_i|  (BASELINE.json north_star),
  where exact = oracle's unrounded hi + lo; a zero sum of zeros compares the sign bit;
- float prod: |gpu - exact| <= 4 * eps(dtype) * |exact| (the analogous bound);
- non-finite oracle results: the GPU result must be the same class and sign.
"""
from __future__ import annotations

import math

import numpy as np

import oracle

EPS = {"float32": 2.0 ** -23, "float64": 2.0 ** -52}
# unit roundoff of the compensated-sum accumulators (fp64 for fp32 data, double-double for fp64)
U_ACC = {"float32": 2.0 ** -53, "float64": 2.0 ** -106}


def to_bits(v, dtype):
    return np.array([v], dtype=np.dtype(dtype)).tobytes()


def check(got, x: np.ndarray, op: str, ref=None, factor: float = 4.0):
    """Assert parity of `got` (numpy scalar / python number; (value, index) for
    argmin / argmax) with the oracle on x."""
    dtype = x.dtype.name          # with ref given, x only supplies the dtype
    r = ref if ref is not None else oracle.reduce(x, op)
    if op in ("argmin", "argmax"):
        gv, gi = got
        assert int(gi) == r.index, f"{dtype} {op} n={x.size}: index {int(gi)} want {r.index}"
        g = np.array([gv], dtype=x.dtype)[0]
        if dtype.startswith("float") and math.isnan(float(r.value)):
            assert math.isnan(float(g))
        else:
            assert to_bits(g, dtype) == to_bits(r.value, dtype), f"{op}: value {g!r} want {r.value!r}"
        return r
    g = np.array([got], dtype=x.dtype)[0]
    if not dtype.startswith("float") or op in ("min", "max", "sum_exact"):
        if dtype.startswith("float") and math.isnan(float(r.value)):
            assert math.isnan(float(g)), f"{op}: want NaN, got {g}"
            return r
        assert to_bits(g, dtype) == to_bits(r.value, dtype), \
            f"{dtype} {op} n={r.count}: got {g!r} want {r.value!r}"
        return r
    want = float(r.value)
    gv = float(g)
    if not math.isfinite(want) or not math.isfinite(r.exact):
        if math.isnan(want):
            assert math.isnan(gv), f"want NaN got {gv}"
        else:
            assert gv == want, f"want {want} got {gv}"
        return r
    if op in ("sum", "sum_compensated"):
        if r.sum_abs == 0.0:
            assert to_bits(g, dtype) == to_bits(r.value, dtype), f"signed zero: got {gv!r} want {want!r}"
            return r
        tol = factor * EPS[dtype] * r.sum_abs
        if op == "sum_compensated":   # include/b200reduce.h: 1/2 ulp + 4 u_acc sum|x|
            tol = 0.5 * float(np.spacing(np.abs(g))) + factor * U_ACC[dtype] * r.sum_abs
    else:
        tol = factor * EPS[dtype] * abs(r.exact)
    err = abs(gv - r.exact)
    assert err <= tol, f"{dtype} {op} n={r.count}: |{gv!r} - {r.exact!r}| = {err:.3e} > {tol:.3e}"
    return r


def rel_error(got, x, op, ref):
    """error in units of the tolerance scale (for reports)"""
    dtype = x.dtype.name
    if not dtype.startswith("float") or op in ("min", "max"):
        return 0.0
    scale = ref.sum_abs if op == "sum" else abs(ref.exact)
    if scale == 0 or not math.isfinite(scale):
        return 0.0
    return abs(float(got) - ref.exact) / (EPS[dtype] * scale)
