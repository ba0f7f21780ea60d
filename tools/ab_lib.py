#!/usr/bin/env python
"""A/B of library builds on the same box: back-to-back GB/s of `reduce` for a
few (dtype, op) at n = 2^28, through ctypes on each .so given (measurement
only).   python tools/ab_lib.py build/ab/lib_a.so build/ab/lib_b.so ..."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402

DT = {"int32": 0, "uint32": 1, "int64": 2, "float32": 3, "float64": 4}
OPS = {"sum": 0, "max": 3, "argmin": 7, "argmax": 8, "sum_compensated": 9, "sum_exact": 10}
PAIRS = [("float32", "argmin"), ("float32", "argmax"), ("int32", "argmax"), ("float64", "argmin"),
         ("float32", "sum"), ("int32", "sum"), ("float64", "max"), ("int64", "argmin"), ("uint32", "argmax")]
if os.environ.get("AB_PAIRS"):            # e.g. AB_PAIRS=uint32:argmax,float32:argmin
    PAIRS = [tuple(p.split(":")) for p in os.environ["AB_PAIRS"].split(",")]
# AB_WORKLOAD: the float workload (default u01; e.g. normalish, wide)
# AB_SOAK=S: S seconds of back-to-back calls before each timing (the sustained,
# power-capped regime bench.py measures); AB_REPS: calls per timing
SOAK = float(os.environ.get("AB_SOAK", "0"))
REPS = int(os.environ.get("AB_REPS", "20"))
if os.environ.get("AB_EXACT"):
    PAIRS.append(("float32", "sum_exact"))


def run(path, x_by_dtype):
    L = ctypes.CDLL(path)
    L.reduce.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    L.reduce.restype = ctypes.c_int
    out = torch.empty(2, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    res = {}
    for dtype, op in PAIRS:
        x = x_by_dtype[dtype]
        f = lambda: L.reduce(x.data_ptr(), x.numel(), DT[dtype], OPS[op], out.data_ptr(), st.cuda_stream)
        for _ in range(5):
            assert f() == 0
        import time
        t_end = time.perf_counter() + SOAK
        while time.perf_counter() < t_end:
            for _ in range(20):
                f()
            torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for _ in range(REPS):
                f()
            b.record(st)
            b.synchronize()
            ts.append(a.elapsed_time(b) / REPS * 1e-3)
        ts.sort()
        res[f"{dtype}-{op}"] = round(x.numel() * x.element_size() / ts[2] / 1e9, 1)
    return res


def run_small(path):
    """graph-captured us per launch at small n (float32 sum), 100 launches per replay"""
    L = ctypes.CDLL(path)
    L.reduce.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    out = torch.empty(2, dtype=torch.int64, device="cuda")
    res = {}
    for log2n in (10, 12, 13, 14, 16, 18):
        x = torch.rand(1 << log2n, device="cuda")
        gs = torch.cuda.Stream()
        with torch.cuda.stream(gs):
            L.reduce(x.data_ptr(), x.numel(), 3, 0, out.data_ptr(), gs.cuda_stream)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for _ in range(100):
                L.reduce(x.data_ptr(), x.numel(), 3, 0, out.data_ptr(), gs.cuda_stream)
        ts = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 10.0)
        ts.sort()
        res[f"2^{log2n}"] = round(ts[3], 3)
    return res


if __name__ == "__main__":
    if "--small" in sys.argv:
        for p in [a for a in sys.argv[1:] if a != "--small"]:
            print(json.dumps({"lib": os.path.basename(p), **run_small(p)}), flush=True)
        sys.exit(0)
    n = 1 << 28
    xs = {}
    for dtype in ("float32", "int32", "float64", "int64", "uint32"):
        xs[dtype] = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
        inputs.fill_device(xs[dtype], os.environ.get("AB_WORKLOAD", "u01") if dtype.startswith("float") else "int_small", seed=1)
    libs = sys.argv[1:]
    rounds = int(os.environ.get("AB_ROUNDS", "2"))
    for rnd in range(rounds):                 # ABBA...: clock / power drift cancels in the mean
        for p in (libs if rnd % 2 == 0 else libs[::-1]):
            print(json.dumps({"lib": os.path.relpath(p, ROOT), "round": rnd, **run(p, xs)}), flush=True)
