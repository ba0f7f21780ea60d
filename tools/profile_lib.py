#!/usr/bin/env python
"""One exact sum per (dtype, workload) at n = 2^28 through a GIVEN library build
(ctypes), for ncu A/B captures of two builds (measurement only):

    ncu --set full -k regex:rd_exact -o prof python tools/profile_lib.py <lib.so> float64:u01 ...
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402

DT = {"float32": 3, "float64": 4}
SUM_EXACT = 10

if __name__ == "__main__":
    L = ctypes.CDLL(sys.argv[1])
    L.reduce.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    out = torch.empty(2, dtype=torch.int64, device="cuda")
    n = 1 << 28
    for spec in sys.argv[2:]:
        dtype, wl = spec.split(":")
        x = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
        inputs.fill_device(x, wl, seed=1)
        assert L.reduce(x.data_ptr(), n, DT[dtype], SUM_EXACT, out.data_ptr(), torch.cuda.current_stream().cuda_stream) == 0
        torch.cuda.synchronize()
        del x
    print("ok")
