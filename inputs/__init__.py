"""inputs -- seeded synthetic input generators shared by the oracle side and
the CUDA side of every parity check.

Holds none of the reduction's arithmetic: ``gen.h`` maps (seed, workload,
global index) to x_i, compiled twice (gcc host twin, nvcc device twin) so both
produce identical bits. Recipe: DESIGN.md "Input recipe" / SURVEY.md §8(d).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SRC = os.path.join(_HERE, "gen_host.c")
_DEV_SRC = os.path.join(_HERE, "gen_device.cu")
_HDR = os.path.join(_HERE, "gen.h")
HOST_LIB = os.path.join(_HERE, "libinputs_host.so")
DEV_LIB = os.path.join(_HERE, "libinputs_device.so")

DTYPES = {"int32": 0, "uint32": 1, "int64": 2, "float32": 3, "float64": 4}
NP_DTYPES = {"int32": np.int32, "uint32": np.uint32, "int64": np.int64,
             "float32": np.float32, "float64": np.float64}
WORKLOADS = {"iota": 0, "uniform_bits": 1, "odd": 2, "sparse_clear": 3, "sparse_set": 4,
             "u01": 5, "normalish": 6, "near_one": 7, "pow2_sparse": 8, "planted": 9,
             "int_small": 10, "sparse_pm1": 11, "wide": 12, "wide_full": 13}

# Workload used for each op on each dtype class: non-degenerate
# for products (odd / near-one) and for and/or (sparse bit patterns).
DEFAULT_WORKLOAD = {
    ("int", "sum"): "uniform_bits", ("int", "prod"): "odd", ("int", "min"): "uniform_bits",
    ("int", "max"): "uniform_bits", ("int", "and"): "sparse_clear", ("int", "or"): "sparse_set",
    ("int", "xor"): "uniform_bits",
    ("float", "sum"): "u01", ("float", "prod"): "near_one", ("float", "min"): "planted",
    ("float", "max"): "planted",
    # argmin / argmax: small value ranges so the extreme value is tied (lowest index wins)
    ("int", "argmin"): "int_small", ("int", "argmax"): "int_small",
    ("float", "argmin"): "u01", ("float", "argmax"): "u01",
    ("int", "sum_compensated"): "uniform_bits", ("float", "sum_compensated"): "normalish",
    # exact sum: terms spanning 2^-40..2^40 (most additions inexact: the slow path works)
    ("int", "sum_exact"): "uniform_bits", ("float", "sum_exact"): "wide",
}


def default_workload(dtype: str, op: str) -> str:
    return DEFAULT_WORKLOAD[("float" if dtype.startswith("float") else "int", op)]


def _newer(out, *srcs):
    return os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(s) for s in srcs)


def build_host(force=False):
    if force or not _newer(HOST_LIB, _HOST_SRC, _HDR):
        tmp = HOST_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off",
                               "-o", tmp, _HOST_SRC])
        os.replace(tmp, HOST_LIB)
    return HOST_LIB


def build_device(force=False):
    if force or not _newer(DEV_LIB, _DEV_SRC, _HDR):
        tmp = DEV_LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                               "-o", tmp, _DEV_SRC])
        os.replace(tmp, DEV_LIB)
    return DEV_LIB


_host = None
_dev = None


def _host_lib():
    global _host
    if _host is None:
        build_host()
        L = ctypes.CDLL(HOST_LIB)
        u64 = ctypes.c_uint64
        L.in_fill_host.argtypes = [ctypes.c_void_p, u64, ctypes.c_int, ctypes.c_int, u64, u64, u64]
        L.in_fill_host.restype = ctypes.c_int
        L.in_planted_positions.argtypes = [u64, u64, ctypes.POINTER(u64), ctypes.POINTER(u64)]
        _host = L
    return _host


def _dev_lib():
    global _dev
    if _dev is None:
        if not os.path.exists(DEV_LIB):
            build_device()
        L = ctypes.CDLL(DEV_LIB)
        u64 = ctypes.c_uint64
        L.in_fill_device.argtypes = [ctypes.c_void_p, u64, ctypes.c_int, ctypes.c_int, u64, u64,
                                     u64, ctypes.c_void_p]
        L.in_fill_device.restype = ctypes.c_int
        _dev = L
    return _dev


def generate(n: int, dtype: str, workload: str, seed: int = 1, offset: int = 0,
             n_total: int | None = None) -> np.ndarray:
    """Host twin: elements offset..offset+n-1 of the logical array of length n_total."""
    out = np.empty(n, dtype=NP_DTYPES[dtype])
    nt = n_total if n_total is not None else offset + n
    rc = _host_lib().in_fill_host(out.ctypes.data if n else None, n, DTYPES[dtype],
                                  WORKLOADS[workload], seed, offset, nt)
    if rc != 0:
        raise ValueError(f"workload {workload!r} undefined for {dtype}")
    return out


def fill_device(t, workload: str, seed: int = 1, offset: int = 0, n_total: int | None = None,
                stream=None):
    """Device twin: fill the contiguous CUDA tensor ``t`` (1-D) in place."""
    import torch
    dtype = str(t.dtype).replace("torch.", "")
    n = t.numel()
    nt = n_total if n_total is not None else offset + n
    st = stream if stream is not None else torch.cuda.current_stream(t.device).cuda_stream
    rc = _dev_lib().in_fill_device(t.data_ptr() if n else None, n, DTYPES[dtype],
                                   WORKLOADS[workload], seed, offset, nt, st)
    if rc != 0:
        raise ValueError(f"device generator failed rc={rc} ({workload!r}, {dtype})")
    return t


def planted_positions(seed: int, n_total: int):
    a, b = ctypes.c_uint64(), ctypes.c_uint64()
    _host_lib().in_planted_positions(seed, n_total, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value
