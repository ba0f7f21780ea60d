#!/usr/bin/env python
"""One float32-sum launch per kernel variant at n = 2^28, for an ncu capture
(evidence for the variant choice and for Table 2 on B200):

    ncu --set full -k regex:rd_ -o prof python tools/profile_variants.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402

if __name__ == "__main__":
    x = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    inputs.fill_device(x, "u01", seed=1)
    for variant, u, vb in (("paper", 1, 0), ("paper", 8, 0), ("vector", 1, 4), ("vector", 4, 32), ("bulk", 0, 0)):
        rd.reduce_ex(x, "sum", variant=variant, unroll=u, vec_bytes=vb)
        torch.cuda.synchronize()
    print("ok")
