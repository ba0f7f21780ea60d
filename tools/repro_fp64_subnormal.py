#!/usr/bin/env python
"""The fp64 exact-sum case a high-word-only exponent test gets wrong (measurement /
regression evidence): 2^-900 + 2^-1060 + (2^-900 + 2^-952) in one group of one thread.
2^-1060 is a subnormal with a zero high word; taken for a zero, the group's error tree
(2^-952 + 2^-1060) rounds and the correctly rounded total changes in its last bit.
The expected value is computed with Python fractions (exact, rounded once by float()).

    python tools/repro_fp64_subnormal.py LIB.so [LIB2.so ...]
"""
import ctypes
import json
import os
import sys
from fractions import Fraction

import numpy as np
import torch

DT_F64, SUM_EXACT = 4, 10


def main():
    a, t, b = 2.0 ** -900, 2.0 ** -1060, 2.0 ** -900 + 2.0 ** -952
    want = float(Fraction(a) + Fraction(t) + Fraction(b))
    for path in sys.argv[1:]:
        L = ctypes.CDLL(path)
        L.reduce.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                             ctypes.c_void_p]
        res = {}
        for pos in ([0, 1, 2], [0, 1, 1024]):
            for n in (4096, (1 << 20) + 8):
                x = np.zeros(n, np.float64)
                x[pos] = (a, t, b)
                xd = torch.from_numpy(x).cuda()
                out = torch.zeros(1, dtype=torch.float64, device="cuda")
                assert L.reduce(xd.data_ptr(), n, DT_F64, SUM_EXACT, out.data_ptr(),
                                torch.cuda.current_stream().cuda_stream) == 0
                got = out.item()
                res[f"pos{pos}-n{n}"] = "ok" if got == want else f"WRONG got {got.hex()} want {want.hex()}"
        print(json.dumps({"lib": os.path.relpath(path), **res}))


if __name__ == "__main__":
    main()
