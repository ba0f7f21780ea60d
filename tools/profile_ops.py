#!/usr/bin/env python
"""One reduce per selected (dtype, op) at n = 2^28, for an ncu capture:

    ncu --set full -k regex:rd_ -o prof python tools/profile_ops.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402

PAIRS = [("int32", "sum"), ("float64", "sum"), ("float64", "prod"), ("float32", "max"),
         ("float32", "argmin"), ("float64", "sum_compensated"), ("float32", "argmax"), ("float64", "argmin"),
         ("float64", "max"), ("int64", "xor"), ("float32", "prod")]
# `python tools/profile_ops.py exact`: the exact sum on its two data classes
EXACT = [("float32", "sum_exact"), ("float64", "sum_exact")]

if __name__ == "__main__":
    n = 1 << 28
    wl_exact = sys.argv[2] if len(sys.argv) > 2 else "u01"    # u01: the fast path
    for dtype, op in (EXACT if sys.argv[1:2] == ["exact"] else PAIRS):
        x = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
        wl = wl_exact if op == "sum_exact" else inputs.default_workload(dtype, op)
        inputs.fill_device(x, wl, seed=1)
        rd.reduce(x, op)
        torch.cuda.synchronize()
        del x
    print("ok")
