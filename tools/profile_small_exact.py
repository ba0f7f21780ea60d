#!/usr/bin/env python
"""A few exact-sum launches at a small n (default 2^18), for an ncu capture of
the fixed per-launch cost:  ncu --set full -k regex:rd_exact python tools/profile_small_exact.py 18 [float64]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402

if __name__ == "__main__":
    n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 18)
    dt = getattr(torch, sys.argv[2] if len(sys.argv) > 2 else "float32")
    x = torch.empty(n, dtype=dt, device="cuda")
    inputs.fill_device(x, "u01", seed=1)
    for _ in range(3):
        rd.reduce(x, "sum_exact")
        rd.reduce(x, "sum")
    torch.cuda.synchronize()
    print("ok")
