#!/usr/bin/env python
"""BASELINE configs[2] (C3): every (dtype, op) x n = 2^10 .. 2^30, timed and
verified -- a report row is never written without its parity check
(SPEC S:385-393's idea: no unvalidated speedup).

    python tools/c3_report.py --out gpurun_out/c3   # -> c3.csv + c3.json

Per row: GB/s from back-to-back launches between CUDA events (the bench's
convention; for inputs < 4x L2 the numbers are L2-warm), the cold single-launch
time after an L2 read-flush, the kernel variant the planner chose, and the
parity verdict against the CPU oracle with |err| / tolerance for floats
(verified for n <= 2^28; at 2^30 only the closed forms of iota integer sums).
"""
from __future__ import annotations

import argparse
import csv
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
import oracle  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402
from tests import _parity  # noqa: E402

SIZE = {"int32": 4, "uint32": 4, "int64": 8, "float32": 4, "float64": 8}
INT_OPS = ["sum", "prod", "min", "max", "and", "or", "xor", "argmin", "argmax", "sum_compensated", "sum_exact"]
FLT_OPS = ["sum", "prod", "min", "max", "argmin", "argmax", "sum_compensated", "sum_exact"]
L2 = 126 * 2 ** 20


def val(t):
    if isinstance(t, tuple):
        return val(t[0]), int(t[1].item())
    carrier = {4: torch.int32, 8: torch.int64}[t.element_size()]
    npdt = np.dtype(str(t.dtype).replace("torch.", ""))
    return np.array([t.view(carrier).item()], dtype=np.dtype(str(carrier).replace("torch.", ""))).view(npdt)[0]


def read_probe_gbs(nbytes=1 << 30):
    """The same-run HBM read ceiling (tools/probe.cu; bench.py's roofline.read_probe)."""
    import ctypes
    lib = os.path.join(ROOT, "tools", "libprobe.so")
    if not os.path.exists(lib):
        return None
    pl = ctypes.CDLL(lib)
    pl.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    pl.probe_occupancy.argtypes = [ctypes.c_int, ctypes.c_int]
    x = torch.ones(nbytes // 4, dtype=torch.float32, device="cuda")
    sink = torch.zeros(1024, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    best = 0.0
    for thr, unr in ((256, 2), (1024, 2), (512, 1)):
        blocks = 148 * max(1, pl.probe_occupancy(unr, thr)) * 4
        for _ in range(3):
            pl.probe_read(x.data_ptr(), nbytes, unr, blocks, thr, sink.data_ptr(), s.cuda_stream, 0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(20):
            pl.probe_read(x.data_ptr(), nbytes, unr, blocks, thr, sink.data_ptr(), s.cuda_stream, 0)
        b.record(s)
        b.synchronize()
        best = max(best, nbytes * 20 / (a.elapsed_time(b) * 1e-3) / 1e9)
    return best


def copy_peak_gbs():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return None


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", required=True)
    p.add_argument("--log2n", type=int, nargs="+", default=[10, 14, 18, 22, 24, 26, 28, 30])
    p.add_argument("--verify-max-log2n", type=int, default=28)
    args = p.parse_args()
    flush = torch.ones(128 * 2 ** 20, dtype=torch.int32, device="cuda")
    probe, copy_peak = read_probe_gbs(), copy_peak_gbs()
    print(json.dumps({"read_probe_gbs": probe, "copy_peak_gbs": copy_peak}), flush=True)
    rows = []
    s = torch.cuda.current_stream()
    for dtype in ("int32", "uint32", "int64", "float32", "float64"):
        ops = FLT_OPS if dtype.startswith("float") else INT_OPS
        for log2n in args.log2n:
            n = 1 << log2n
            if n * SIZE[dtype] > 16 * 2 ** 30:
                continue
            # the exact sum twice: its default (adversarial, slow-path) workload and u01
            cases = [(op, inputs.default_workload(dtype, op)) for op in ops]
            if dtype.startswith("float"):
                cases.append(("sum_exact", "u01"))
            for op, wl in cases:
                x = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
                inputs.fill_device(x, wl, seed=1)
                res, info = rd.reduce_ex(x, op)
                got = val(res)
                verdict, err_ratio = "unverified", None
                if log2n <= args.verify_max_log2n:
                    xh = x.cpu().numpy()
                    try:
                        ref = _parity.check(got, xh, op)
                        verdict = "ok"
                        if dtype.startswith("float") and op in ("sum", "prod", "sum_compensated") \
                                and math.isfinite(ref.exact):
                            scale = ref.sum_abs if op != "prod" else abs(ref.exact)
                            eps = _parity.EPS[dtype]
                            err_ratio = abs(float(got) - ref.exact) / (4 * eps * scale) if scale else 0.0
                    except AssertionError as e:
                        verdict = f"FAIL: {e}"
                    del xh
                # timing: cold single launch (after an L2 read-flush) and back to back
                cold = []
                for _ in range(5):
                    flush.max()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s)
                    rd.reduce(x, op)
                    b.record(s)
                    b.synchronize()
                    cold.append(a.elapsed_time(b) * 1e3)
                reps = 50 if n <= 2 ** 26 else 20
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                for _ in range(reps):
                    rd.reduce(x, op)
                b.record(s)
                b.synchronize()
                us = a.elapsed_time(b) * 1e3 / reps
                nbytes = n * SIZE[dtype]
                row = {"dtype": dtype, "op": op, "n": n, "log2n": log2n, "workload": wl,
                       "variant": info["variant"], "grid": info["grid"], "block": info["block"],
                       "us_back_to_back": round(us, 3), "gbps_back_to_back": round(nbytes / us / 1e3, 1),
                       "elem_per_s_back_to_back": round(n / us * 1e6, 1),
                       "pct_read_probe": round(100 * nbytes / us / 1e3 / probe, 2) if probe else None,
                       "pct_copy_peak": round(100 * nbytes / us / 1e3 / copy_peak, 2) if copy_peak else None,
                       "us_cold_mean5": round(sum(cold) / 5, 3),
                       "gbps_cold": round(nbytes / (sum(cold) / 5) / 1e3, 1),
                       "l2_resident": nbytes < 4 * L2, "result_ok": verdict, "err_over_tol": err_ratio}
                rows.append(row)
                print(json.dumps(row), flush=True)
                del x
    with open(args.out + ".json", "w") as f:
        json.dump({"device": torch.cuda.get_device_name(), "when": time.strftime("%Y-%m-%dT%H:%M:%S"),
                   "read_probe_gbs": probe, "copy_peak_gbs": copy_peak, "rows": rows}, f, indent=1)
    with open(args.out + ".csv", "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(rows[0]))
        w.writeheader()
        w.writerows(rows)
    bad = [r for r in rows if r["result_ok"] not in ("ok", "unverified")]
    print(f"{len(rows)} rows, {len(bad)} failures")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
