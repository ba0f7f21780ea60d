#!/usr/bin/env python
"""Bitwise comparison of two library builds (measurement / refactoring check):
the same (dtype, op, workload, n, base offset, variant, grid) through `reduce`
and `rd_reduce_ex` of each .so, every result compared bit for bit. For changes
that must not change results (e.g. a cheaper instruction sequence that computes
the same values).

    python tools/ab_bits.py LIB_A LIB_B [--dtype float64] [--op sum_compensated]
"""
import argparse
import ctypes
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402

DT = {"int32": 0, "uint32": 1, "int64": 2, "float32": 3, "float64": 4}
OPS = {"sum": 0, "prod": 1, "min": 2, "max": 3, "and": 4, "or": 5, "xor": 6, "argmin": 7, "argmax": 8,
       "sum_compensated": 9, "sum_exact": 10}
VARIANTS = {"auto": 0, "vector": 1, "bulk": 3, "cluster": 4}


class Cfg(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int32), ("vec_bytes", ctypes.c_int32), ("unroll", ctypes.c_int32),
                ("block", ctypes.c_int32), ("grid", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]


def load(path):
    L = ctypes.CDLL(path)
    L.rd_reduce_ex.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("lib_a")
    ap.add_argument("lib_b")
    ap.add_argument("--dtype", default="float64")
    ap.add_argument("--op", default="sum_compensated")
    ap.add_argument("--workloads", default="u01,normalish,wide,wide_full,near_one")
    args = ap.parse_args()
    A, B = load(args.lib_a), load(args.lib_b)
    st = torch.cuda.current_stream().cuda_stream
    tdt = getattr(torch, args.dtype)
    out = torch.zeros(4, dtype=torch.int64, device="cuda")
    sizes = [1, 7, 100, 4099, (1 << 16) + 3, (1 << 20) + 5, 5533214, (1 << 24) + 1, (1 << 25) + 7]
    cases = diffs = 0
    for wl, n in itertools.product(args.workloads.split(","), sizes):
        buf = torch.empty(n + 3, dtype=tdt, device="cuda")
        inputs.fill_device(buf, wl, seed=3)
        for off, (vname, grid) in itertools.product((0, 1), (("auto", 0), ("vector", 0), ("vector", 7),
                                                            ("bulk", 0), ("bulk", 5), ("cluster", 0))):
            x = buf[off:off + n]
            res = []
            for L in (A, B):
                out.zero_()
                cfg = Cfg(VARIANTS[vname], 0, 0, 0, grid)
                rc = L.rd_reduce_ex(x.data_ptr(), n, DT[args.dtype], OPS[args.op], out.data_ptr(), st,
                                    ctypes.byref(cfg), None)
                torch.cuda.synchronize()
                res.append((rc, tuple(out.tolist())))
            cases += 1
            if res[0] != res[1]:
                diffs += 1
                print(json.dumps({"diff": True, "workload": wl, "n": n, "off": off, "variant": vname, "grid": grid,
                                  "a": res[0], "b": res[1]}), flush=True)
        del buf
    print(json.dumps({"dtype": args.dtype, "op": args.op, "cases": cases, "bitwise_differences": diffs}))
    sys.exit(1 if diffs else 0)


if __name__ == "__main__":
    main()
