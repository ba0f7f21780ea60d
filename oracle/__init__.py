"""oracle -- TEST INFRASTRUCTURE ONLY.

ctypes binding for ``oracle/oracle.c``: the plain sequential CPU oracle of the
reduction x_0 (x) x_1 (x) ... (x) x_{n-1} (§1.1), evaluated as
Algorithm 1 "Summation(A)" generalised to the combiner.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package. The
product path (``paper_1710_07358_b200``) never imports it.

Readings R1-R5 are listed in oracle.c and DESIGN.md. Every function is pinned
by ``tests/test_oracle_pins.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# restated codes (not imported from the CUDA package)
DTYPES = {"int32": 0, "uint32": 1, "int64": 2, "float32": 3, "float64": 4}
OPS = {"sum": 0, "prod": 1, "min": 2, "max": 3, "and": 4, "or": 5, "xor": 6, "argmin": 7, "argmax": 8,
       "sum_compensated": 9, "sum_exact": 10}
NP_DTYPES = {"int32": np.int32, "uint32": np.uint32, "int64": np.int64,
             "float32": np.float32, "float64": np.float64}


class OracleState(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("op", ctypes.c_int32),
                ("count", ctypes.c_uint64), ("ibits", ctypes.c_uint64),
                ("hi", ctypes.c_double), ("lo", ctypes.c_double),
                ("abs_hi", ctypes.c_double), ("abs_lo", ctypes.c_double),
                ("all_negzero", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("best_idx", ctypes.c_uint64),
                ("big", ctypes.c_uint32 * 72),
                ("nan_seen", ctypes.c_int32), ("pinf_seen", ctypes.c_int32),
                ("ninf_seen", ctypes.c_int32), ("pad2", ctypes.c_int32)]


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc -O2 (no -ffast-math: IEEE semantics kept)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        dp = ctypes.POINTER(ctypes.c_double)
        sp = ctypes.POINTER(OracleState)
        L.or_init.argtypes = [sp, i32, i32]
        L.or_fold.argtypes = [sp, vp, u64]
        L.or_result.argtypes = [sp, vp, dp, dp, dp]
        L.or_reduce.argtypes = [vp, u64, i32, i32, vp, dp, dp, dp]
        L.or_identity.argtypes = [i32, i32, vp]
        L.or_merge.argtypes = [sp, sp]
        L.or_state_size.restype = u64
        L.or_result_index.argtypes = [sp]
        L.or_result_index.restype = ctypes.c_int64
        for f in (L.or_init, L.or_fold, L.or_result, L.or_reduce, L.or_identity, L.or_merge):
            f.restype = i32
        assert L.or_state_size() == ctypes.sizeof(OracleState)
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


@dataclass
class OracleResult:
    value: object        # numpy scalar of the dtype (narrowed with one rounding)
    hi: float            # unrounded float accumulator (hi + lo), floats only
    lo: float
    sum_abs: float       # sum |x_i| (floats only), for the tolerance 4*eps*sum|x|
    count: int
    index: int = -1      # argmin / argmax only: smallest index of the best element

    @property
    def exact(self) -> float:
        return self.hi + self.lo


def _check(rc: int):
    if rc == 1:
        raise OracleError("invalid argument")
    if rc == 2:
        raise OracleError("unsupported (bitwise op on a float dtype)")


def _result(st: OracleState, dtype: str) -> OracleResult:
    out = np.zeros(1, dtype=NP_DTYPES[dtype])
    hi, lo, sa = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _check(lib().or_result(ctypes.byref(st), out.ctypes.data, ctypes.byref(hi),
                           ctypes.byref(lo), ctypes.byref(sa)))
    return OracleResult(out[0], hi.value, lo.value, sa.value, int(st.count),
                        int(lib().or_result_index(ctypes.byref(st))))


def reduce(x: np.ndarray, op: str) -> OracleResult:
    """Algorithm 1 over the whole array, generalised to ``op``."""
    x = np.ascontiguousarray(x)
    dtype = x.dtype.name
    st = OracleState()
    _check(lib().or_init(ctypes.byref(st), DTYPES[dtype], OPS[op]))
    _check(lib().or_fold(ctypes.byref(st), x.ctypes.data if x.size else None, x.size))
    return _result(st, dtype)


class Fold:
    """Streaming form of the same left fold: fold(A); fold(B) == fold(A ++ B)."""

    def __init__(self, dtype: str, op: str):
        self.dtype = dtype
        self.st = OracleState()
        _check(lib().or_init(ctypes.byref(self.st), DTYPES[dtype], OPS[op]))

    def fold(self, x: np.ndarray) -> "Fold":
        x = np.ascontiguousarray(x)
        assert x.dtype.name == self.dtype
        _check(lib().or_fold(ctypes.byref(self.st), x.ctypes.data if x.size else None, x.size))
        return self

    def merge(self, other: "Fold") -> "Fold":
        """self := fold(self's block) (x) fold(other's block) -- block order."""
        _check(lib().or_merge(ctypes.byref(self.st), ctypes.byref(other.st)))
        return self

    def result(self) -> OracleResult:
        return _result(self.st, self.dtype)


def identity(dtype: str, op: str):
    """Result of the empty fold: Algorithm 1's initial accumulator (R1)."""
    out = np.zeros(1, dtype=NP_DTYPES[dtype])
    _check(lib().or_identity(DTYPES[dtype], OPS[op], out.ctypes.data))
    return out[0]
