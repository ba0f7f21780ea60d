#!/usr/bin/env python
"""Small reductions of every kind, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck) runs on one GPU:

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Covers the kernel variants (vector, bulk, cluster), the paper-listing variant, every
(dtype, op) pair, misaligned bases, forced multi-CTA grids (ticket path), arg
ops, records + rd_combine_records, exact records, and reduce_host. Exits non-zero if a result
disagrees with the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402
from tests import _parity  # noqa: E402

INT_OPS = ["sum", "prod", "min", "max", "and", "or", "xor", "argmin", "argmax", "sum_compensated", "sum_exact"]
FLT_OPS = ["sum", "prod", "min", "max", "argmin", "argmax", "sum_compensated", "sum_exact"]


def dev(x, off=0):
    carrier = {4: np.int32, 8: np.int64}[x.itemsize]
    buf = torch.zeros(x.size + off + 1, dtype=getattr(torch, np.dtype(carrier).name), device="cuda")
    if x.size:
        buf[off:off + x.size].copy_(torch.from_numpy(x.view(carrier)))
    return buf.view(getattr(torch, x.dtype.name))[off:off + x.size]


def val(t):
    if isinstance(t, tuple):
        return val(t[0]), int(t[1].item())
    carrier = {4: torch.int32, 8: torch.int64}[t.element_size()]
    npdt = np.dtype(str(t.dtype).replace("torch.", ""))
    return np.array([t.view(carrier).item()], dtype=np.dtype(str(carrier).replace("torch.", ""))).view(npdt)[0]


def main():
    only = sys.argv[sys.argv.index("--only-op") + 1] if "--only-op" in sys.argv else None
    count = 0
    for dtype in ("int32", "uint32", "int64", "float32", "float64"):
        ops = FLT_OPS if dtype.startswith("float") else INT_OPS
        for op in ops:
            if only and op != only:
                continue
            wl = inputs.default_workload(dtype, op)
            for n, off in ((0, 0), (5, 1), (1000, 3), (70001, 2)):
                x = inputs.generate(n, dtype, wl, seed=3)
                xd = dev(x, off)
                for variant, grid in (("vector", 0), ("vector", 7), ("bulk", 0), ("bulk", 3), ("cluster", 0),
                                      ("cluster", 5)):
                    out, _ = rd.reduce_ex(xd, op, variant=variant, grid=grid)
                    _parity.check(val(out), x, op)
                    count += 1
    if only:
        torch.cuda.synchronize()
        print(f"sanitize cases ok: {count} launches checked ({only})")
        return
    x = inputs.generate(100003, "float32", "u01", seed=1)
    xd = dev(x, 1)
    for f in (1, 8, 16):
        _parity.check(val(rd.reduce_ex(xd, "sum", variant="paper", unroll=f)[0]), x, "sum")
    recs = torch.zeros(4 * 32, dtype=torch.uint8, device="cuda")
    for op in ("sum", "argmax"):
        for r in range(4):
            b, c = rd.shard_range(x.size, 4, r)
            rd.reduce_partial(xd[b:b + c], op, rec=recs[r * 32:(r + 1) * 32])
        _parity.check(val(rd.combine_records(recs, "float32", op)), x, op)
    RB = rd.EXACT_RECORD_BYTES
    xrecs = torch.zeros(4 * RB, dtype=torch.uint8, device="cuda")
    for r in range(4):
        b, c = rd.shard_range(x.size, 4, r)
        rd.reduce_exact_partial(xd[b:b + c], rec=xrecs[r * RB:(r + 1) * RB])
    _parity.check(val(rd.combine_exact_records(xrecs, "float32")), x, "sum_exact")
    w = inputs.generate(50001, "float64", "wide_full", seed=4)
    _parity.check(val(rd.reduce(dev(w, 1), "sum_exact")), w, "sum_exact")
    big = inputs.generate((1 << 23) + 5, "float64", "u01", seed=2)
    _parity.check(rd.reduce_host(big, "sum"), big, "sum")
    torch.cuda.synchronize()
    print(f"sanitize cases ok: {count} launches checked")


if __name__ == "__main__":
    main()
