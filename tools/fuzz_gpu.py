#!/usr/bin/env python
"""Randomised parity fuzzing of the CUDA path against the oracle, for a time
budget (measurement / robustness tooling, like the sanitizer cases):

    python tools/fuzz_gpu.py --seconds 300 --seed 1 > gpurun_out/fuzz.log

Every case draws a (dtype, op), a size (log-uniform up to 2^22, biased to the
vector/cluster/bulk boundaries), a base offset, a kernel variant and grid
(or AUTO), and an input (a synthetic workload, or random bits / special
values); the result must pass tests/_parity.check. Prints one JSON line per
failure and a summary; exits 1 on any failure.
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402
from tests import _parity  # noqa: E402
from tools.sanitize_cases import dev, val  # noqa: E402

INT = ["int32", "uint32", "int64"]
FLT = ["float32", "float64"]
INT_OPS = ["sum", "prod", "min", "max", "and", "or", "xor", "argmin", "argmax", "sum_compensated", "sum_exact"]
FLT_OPS = ["sum", "prod", "min", "max", "argmin", "argmax", "sum_compensated", "sum_exact"]
SPECIALS = [0.0, -0.0, math.inf, -math.inf, math.nan, 1e-45, 5e-324, 3.4e38, 1.7e308]


def draw_input(rng, dtype, op, n):
    kind = rng.integers(0, 3)
    if kind == 0 or op in ("prod", "sum_compensated"):
        wl = inputs.default_workload(dtype, op)
        return inputs.generate(n, dtype, wl, seed=int(rng.integers(1, 1 << 30))), wl
    if dtype in INT:
        if dtype == "int64":
            return rng.integers(-(1 << 63), (1 << 63) - 1, n, dtype=np.int64), "bits"
        return rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32).view(dtype), "bits"
    if op == "sum":                          # the float-sum contract is for inputs without overflow
        x = (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4)).astype(dtype)
        return x, "normal"
    if op == "sum_exact" and rng.integers(0, 2):
        # exponents over (a random window of) the whole format: every bin of the exact
        # sum's binned extraction, re-anchoring, and the per-element levels for fp64
        lo, hi = (-149, 127) if dtype == "float32" else (-1074, 1023)
        a = int(rng.integers(lo, hi))
        b = int(rng.integers(a, hi + 1))
        e = rng.integers(a, b + 1, n)
        with np.errstate(over="ignore", under="ignore"):
            x = (rng.choice([-1.0, 1.0], n) * np.ldexp(rng.random(n) + 0.5, e)).astype(dtype)
        x[~np.isfinite(x)] = 0
        return x, "full-range"
    x = (rng.standard_normal(n) * 2.0 ** rng.integers(-60, 60, n)).astype(dtype)
    if n and op != "prod":
        for _ in range(int(rng.integers(0, 4))):
            with np.errstate(over="ignore"):
                x[int(rng.integers(0, n))] = np.array(SPECIALS[int(rng.integers(0, len(SPECIALS)))]).astype(dtype)
    return x, "wide+specials"


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--seconds", type=float, default=120.0)
    p.add_argument("--seed", type=int, default=1)
    args = p.parse_args()
    rng = np.random.default_rng(args.seed)
    t_end = time.time() + args.seconds
    cases = fails = 0
    boundaries = [2 ** 13, 2 ** 15, 2 ** 18, 2 ** 20, 3 * 2 ** 20]
    while time.time() < t_end:
        dtype = [*INT, *FLT][int(rng.integers(0, 5))]
        ops = INT_OPS if dtype in INT else FLT_OPS
        op = ops[int(rng.integers(0, len(ops)))]
        if rng.random() < 0.3:
            b = boundaries[int(rng.integers(0, len(boundaries)))] // np.dtype(dtype).itemsize
            n = int(max(0, b + rng.integers(-40, 40)))
        else:
            n = int(2 ** rng.uniform(0, 22))
        x, wl = draw_input(rng, dtype, op, n)
        off = int(rng.integers(0, 8))
        variant = ["auto", "vector", "bulk", "cluster"][int(rng.integers(0, 4))]
        grid = 0 if rng.random() < 0.5 else int(rng.integers(1, 17 if variant == "cluster" else 600))
        try:
            out, info = rd.reduce_ex(dev(x, off), op, variant=variant, grid=grid)
            _parity.check(val(out), x, op)
        except AssertionError as e:
            fails += 1
            print(json.dumps({"fail": str(e)[:300], "dtype": dtype, "op": op, "n": n, "workload": wl,
                              "offset": off, "variant": variant, "grid": grid}), flush=True)
        cases += 1
    torch.cuda.synchronize()
    print(json.dumps({"cases": cases, "failures": fails, "seconds": args.seconds, "seed": args.seed}))
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
