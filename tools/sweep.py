#!/usr/bin/env python
"""Measurement sweeps on one B200 (run under gpurun); writes JSON to --out.

    python tools/sweep.py probe      --out gpurun_out/probe.json     # HBM read-bandwidth probe
    python tools/sweep.py ablation   --out gpurun_out/ablation.json  # U x VB and paper F (Table 2 on B200)
    python tools/sweep.py ops        --out gpurun_out/ops.json       # all 29 (dtype, op) pairs
    python tools/sweep.py sizes      --out gpurun_out/sizes.json     # n = 2^10 .. 2^30

Timing: CUDA events on the launching stream around each launch, after
warm-up; when the input is smaller than 4x L2 the L2 is flushed (a 512 MiB
memset) before every timed launch. GB/s = n * sizeof(dtype) / t (decimal,
PAPER.md Table 2's convention).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import inputs  # noqa: E402
import paper_1710_07358_b200 as rd  # noqa: E402

L2_BYTES = 126 * 2 ** 20
SIZE = {"int32": 4, "uint32": 4, "int64": 8, "float32": 4, "float64": 8}
_flush = None


def flush_l2():
    """Evict the input from L2 by READING a 512 MiB buffer (a write-based flush
    would leave ~126 MB of dirty lines whose write-back the timed kernel pays)."""
    global _flush
    if _flush is None:
        _flush = torch.ones(128 * 2 ** 20, dtype=torch.int32, device="cuda")
    _flush.max()


def time_launch(fn, nbytes, reps=30, warm=5):
    """Single launches after a synchronize (L2 read-flushed first when the input
    is < 4x L2): median / min / mean-of-5 (the paper's Table 2 convention is a
    mean of 5). For inputs >= 4x L2 also the steady state: `reps`
    back-to-back launches between two events (what bench.py measures)."""
    s = torch.cuda.current_stream()
    need_flush = nbytes < 4 * L2_BYTES
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if need_flush:
            flush_l2()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    med = statistics.median(ts)
    r = {"t_med_us": med * 1e6, "t_min_us": min(ts) * 1e6, "t_mean5_us": statistics.mean(ts[:5]) * 1e6,
         "gbps_med": nbytes / med / 1e9, "gbps_best": nbytes / min(ts) / 1e9, "l2_flushed": need_flush}
    if not need_flush:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        b.synchronize()
        t = a.elapsed_time(b) * 1e-3 / reps
        r.update({"t_stream_us": t * 1e6, "gbps_stream": nbytes / t / 1e9})
    return r


def make(n, dtype, wl, seed=1):
    x = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
    inputs.fill_device(x, wl, seed=seed)
    return x


def do_probe(args):
    lib = ctypes.CDLL(os.path.join(ROOT, "tools", "libprobe.so"))
    lib.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    nbytes = 1 << 30
    x = make(nbytes // 4, "float32", "u01")
    sink = torch.zeros(1024, dtype=torch.int32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    rows = []
    for threads in (256, 512, 1024):
        for u in (1, 2, 4, 8):
            occ = lib.probe_occupancy(u, threads)
            for waves in (1, 2, 4):
                for mode in (0, 1):
                    blocks = 148 * occ * waves
                    fn = lambda: lib.probe_read(x.data_ptr(), nbytes, u, blocks, threads, sink.data_ptr(), st, mode)
                    r = time_launch(fn, nbytes)
                    r.update({"threads": threads, "unroll": u, "ctas_per_sm": occ, "waves": waves,
                              "mode": ["grid-stride", "cta-contiguous"][mode], "grid": blocks})
                    rows.append(r)
                    print(json.dumps(r), flush=True)
    best = max(rows, key=lambda r: r["gbps_med"])
    # torch copy (the MEASURED_PEAKS method) for comparison, read+write bytes
    y = torch.empty_like(x)
    cp = time_launch(lambda: y.copy_(x), 2 * nbytes)
    return {"rows": rows, "best": best, "torch_copy_rw": cp}


def do_ablation(args):
    out = {}
    for dtype in ("float32", "int32"):
        wl = "u01" if dtype == "float32" else "uniform_bits"
        for n in (1 << 28, 5533214):
            x = make(n, dtype, wl)
            o = torch.empty((), dtype=x.dtype, device="cuda")
            rows = []
            cfgs = [("vector", u, vb) for vb in (4, 8, 16, 32) for u in (1, 2, 3, 4, 5, 6, 7, 8, 16)]
            cfgs += [("paper", u, 0) for u in (1, 2, 3, 4, 5, 6, 7, 8, 16)]
            cfgs += [("bulk", st, sb) for st, sb in ((4, 32768), (6, 32768), (3, 65536), (12, 16384),
                                                     (8, 16384), (6, 16384), (24, 8192), (3, 32768),
                                                     (5, 32768), (2, 65536), (4, 49152))]
            if args.only:
                cfgs = [c for c in cfgs if c[0] in args.only]
            for variant, u, vb in cfgs:
                _, info = rd.reduce_ex(x, "sum", variant=variant, unroll=u, vec_bytes=vb, out=o)
                fn = lambda: rd.reduce_ex(x, "sum", variant=variant, unroll=u, vec_bytes=vb, out=o)
                r = time_launch(fn, n * 4)
                r.update({"variant": variant, "unroll": u, "vec_bytes": info["vec_bytes"],
                          "grid": info["grid"], "regs": info["regs_per_thread"],
                          "ctas_per_sm": info["ctas_per_sm"]})
                rows.append(r)
                print(dtype, n, json.dumps(r), flush=True)
            out[f"{dtype}-{n}"] = rows
            del x
    return out


def do_ops(args):
    rows = []
    pairs = [(d, o) for d in ("int32", "uint32", "int64") for o in rd.OPS] + \
            [(d, o) for d in ("float32", "float64")
             for o in ("sum", "prod", "min", "max", "argmin", "argmax", "sum_compensated", "sum_exact")]
    for log2n in args.log2n:
        n = 1 << log2n
        for dtype, op in pairs:
            x = make(n, dtype, inputs.default_workload(dtype, op))
            o = torch.empty(2, dtype=torch.int64, device="cuda") if op in rd.ARG_OPS else \
                torch.empty((), dtype=x.dtype, device="cuda")
            _, info = rd.reduce_ex(x, op, out=o)
            r = time_launch(lambda: rd.reduce(x, op, out=o), n * SIZE[dtype])
            r.update({"dtype": dtype, "op": op, "n": n, "grid": info["grid"], "regs": info["regs_per_thread"],
                      "ctas_per_sm": info["ctas_per_sm"]})
            rows.append(r)
            print(json.dumps(r), flush=True)
            del x
    return rows


def do_exact(args):
    """RD_SUM_EXACT next to the plain and compensated sums, per workload:
    the exact kernel's fast path (one TwoSum per element) vs its slow path."""
    rows = []
    for log2n in args.log2n:
        n = 1 << log2n
        for dtype in ("float32", "float64"):
            for wl in ("u01", "normalish", "wide", "wide_full"):
                x = make(n, dtype, wl)
                o = torch.empty((), dtype=x.dtype, device="cuda")
                for op, var in (("sum", "auto"), ("sum_compensated", "auto"), ("sum_exact", "vector"),
                                ("sum_exact", "bulk")):
                    _, info = rd.reduce_ex(x, op, variant=var, out=o)
                    r = time_launch(lambda: rd.reduce_ex(x, op, variant=var, out=o), n * SIZE[dtype])
                    r.update({"dtype": dtype, "workload": wl, "op": op, "n": n, "grid": info["grid"],
                              "regs": info["regs_per_thread"], "ctas_per_sm": info["ctas_per_sm"],
                              "variant": info["variant"]})
                    rows.append(r)
                    print(json.dumps(r), flush=True)
                del x
    return rows


def do_sizes(args):
    rows = []
    for dtype in ("float32", "int32"):
        for log2n in range(10, 31):
            n = 1 << log2n
            x = make(n, dtype, "u01" if dtype == "float32" else "uniform_bits")
            o = torch.empty((), dtype=x.dtype, device="cuda")
            r = time_launch(lambda: rd.reduce(x, "sum", out=o), n * 4, reps=50)
            # launch-bound regime: also time 100 back-to-back launches (no flush)
            s = torch.cuda.current_stream()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(100):
                rd.reduce(x, "sum", out=o)
            b.record(s)
            b.synchronize()
            # ... and as a CUDA graph of 100 launches (no host launch overhead)
            gs = torch.cuda.Stream()
            with torch.cuda.stream(gs):
                rd.reduce(x, "sum", out=o)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                for _ in range(100):
                    rd.reduce(x, "sum", out=o)
            g.replay()
            torch.cuda.synchronize()
            c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c.record(s)
            g.replay()
            d.record(s)
            d.synchronize()
            r.update({"dtype": dtype, "n": n, "batched100_us_per_launch": a.elapsed_time(b) * 10.0,
                      "graph100_us_per_launch": c.elapsed_time(d) * 10.0})
            rows.append(r)
            print(json.dumps(r), flush=True)
            del x
    return rows


def graph_us(fn, reps=100):
    """per-launch time of `reps` launches captured in one CUDA graph (no host overhead)"""
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=gs):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(7):                       # median of 7 replays (clock / power noise)
        c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c.record(s)
        g.replay()
        d.record(s)
        d.synchronize()
        ts.append(c.elapsed_time(d) * 1e3 / reps)
    return statistics.median(ts)


def do_midgrids(args):
    """Mid sizes (2^16..2^27): grid and variant vs cold single-launch and graph-captured time."""
    rows = []
    for log2n in range(16, 28):
        n = 1 << log2n
        x = make(n, "float32", "u01")
        o = torch.empty((), dtype=x.dtype, device="cuda")
        _, info = rd.reduce_ex(x, "sum", out=o)
        for variant in ("vector", "bulk"):
            for g in (0, 37, 74, 148, 296, 444, 592, 888):
                try:
                    _, inf2 = rd.reduce_ex(x, "sum", variant=variant, grid=g, out=o)
                except rd.ReduceError:
                    continue
                fn = lambda: rd.reduce_ex(x, "sum", variant=variant, grid=g, out=o)
                cold = time_launch(fn, n * 4, reps=20)
                r = {"n": n, "log2n": log2n, "variant": variant, "grid": inf2["grid"], "auto_grid": info["grid"],
                     "auto_variant": info["variant"], "cold_us": cold["t_med_us"], "graph_us": graph_us(fn)}
                rows.append(r)
                print(json.dumps(r), flush=True)
        del x
    return rows


def do_midops(args):
    """Mid sizes, the AUTO plan for several (dtype, op): graph-captured us per launch
    (A/B the planner with RD_TUNE_VEC_CTAS_PER_SM: 1000 = uncapped)."""
    rows = []
    for dtype, op in (("float32", "sum"), ("int32", "sum"), ("float64", "sum"), ("float32", "argmin"),
                      ("float64", "prod"), ("float32", "sum_exact"), ("int64", "xor")):
        for log2n in range(18, 26):
            n = 1 << log2n
            x = make(n, dtype, inputs.default_workload(dtype, op) if op != "sum_exact" else "u01")
            o = torch.empty(2, dtype=torch.int64, device="cuda") if op in rd.ARG_OPS else \
                torch.empty((), dtype=x.dtype, device="cuda")
            _, info = rd.reduce_ex(x, op, out=o)
            r = {"dtype": dtype, "op": op, "log2n": log2n, "variant": info["variant"], "grid": info["grid"],
                 "graph_us": graph_us(lambda: rd.reduce(x, op, out=o)),
                 "cap": os.environ.get("RD_TUNE_VEC_CTAS_PER_SM", "default")}
            rows.append(r)
            print(json.dumps(r), flush=True)
            del x
    return rows


def do_exactvariants(args):
    """The exact sum's variants at mid sizes (2^18..2^27), per dtype and workload:
    vector vs bulk (and the one-cluster form where it applies), cold single launch
    (L2 flushed) and graph-captured back to back -- the basis of the exact sum's
    AUTO threshold."""
    rows = []
    for dtype in ("float32", "float64"):
        for wl in ("u01", "wide"):
            for log2n in range(18, 28):
                n = 1 << log2n
                x = make(n, dtype, wl)
                o = torch.empty((), dtype=x.dtype, device="cuda")
                _, info = rd.reduce_ex(x, "sum_exact", out=o)
                for variant in ("vector", "bulk", "cluster"):
                    if variant == "cluster" and n * x.element_size() > (1 << 20):
                        continue
                    fn = lambda: rd.reduce_ex(x, "sum_exact", variant=variant, out=o)
                    cold = time_launch(fn, n * x.element_size(), reps=20)
                    r = {"dtype": dtype, "workload": wl, "n": n, "log2n": log2n, "variant": variant,
                         "auto_variant": info["variant"], "cold_us": round(cold["t_med_us"], 2),
                         "graph_us": graph_us(fn)}
                    rows.append(r)
                    print(json.dumps(r), flush=True)
                del x
    return rows


def do_variants(args):
    """Plain ops at mid sizes (2^20..2^27): vector vs bulk, cold single launch (L2
    flushed) and graph-captured, for the 8-byte dtypes and a few 4-byte ones -- does
    the plain planner's 128 MiB bulk threshold (measured on float32 sum) hold?"""
    rows = []
    pairs = (("float64", "sum"), ("float64", "max"), ("int64", "sum"), ("float64", "argmax"),
             ("float32", "argmax"), ("float64", "sum_compensated"))
    if os.environ.get("SWEEP_PAIRS"):           # e.g. SWEEP_PAIRS=float64:sum,float32:prod
        pairs = [tuple(p.split(":")) for p in os.environ["SWEEP_PAIRS"].split(",")]
    for dtype, op in pairs:
        for log2n in (args.log2n if os.environ.get("SWEEP_PAIRS") else range(20, 28)):
            n = 1 << log2n
            x = make(n, dtype, inputs.default_workload(dtype, op))
            o = torch.empty(2, dtype=torch.int64, device="cuda") if op in rd.ARG_OPS else \
                torch.empty((), dtype=x.dtype, device="cuda")
            _, info = rd.reduce_ex(x, op, out=o)
            for variant in ("vector", "bulk"):
                fn = lambda: rd.reduce_ex(x, op, variant=variant, out=o)
                cold = time_launch(fn, n * x.element_size(), reps=20)
                r = {"dtype": dtype, "op": op, "n": n, "log2n": log2n, "variant": variant,
                     "auto_variant": info["variant"], "cold_us": round(cold["t_med_us"], 2),
                     "graph_us": graph_us(fn)}
                rows.append(r)
                print(json.dumps(r), flush=True)
            del x
    return rows


def do_grids(args):
    """Grid multiplier (waves of resident CTAs) for the default kernels at n = 2^28."""
    rows = []
    for dtype, op in (("float32", "sum"), ("int32", "sum"), ("float64", "sum"), ("float32", "max")):
        n = 1 << 28
        x = make(n, dtype, inputs.default_workload(dtype, op))
        o = torch.empty((), dtype=x.dtype, device="cuda")
        _, info = rd.reduce_ex(x, op, out=o)
        g0 = info["grid"]
        for mult in (0.5, 1, 2, 3, 4, 8):
            g = max(1, int(g0 * mult))
            _, info = rd.reduce_ex(x, op, grid=g, out=o)
            r = time_launch(lambda: rd.reduce_ex(x, op, grid=g, out=o), n * SIZE[dtype])
            r.update({"dtype": dtype, "op": op, "grid": g, "mult": mult})
            rows.append(r)
            print(json.dumps(r), flush=True)
        del x
    return rows


def do_crossover(args):
    """vector vs bulk variant around the AUTO threshold: L2-cold single launches
    (read-flush before each) and back-to-back launches in a CUDA graph."""
    rows = []
    for dtype in ("float32", "float64"):
        for log2n in range(18, 29):
            n = 1 << log2n
            x = make(n, dtype, "u01")
            o = torch.empty((), dtype=x.dtype, device="cuda")
            for variant in ("vector", "bulk"):
                fn = lambda: rd.reduce_ex(x, "sum", variant=variant, out=o)
                r = time_launch(fn, n * SIZE[dtype], reps=30)
                gs = torch.cuda.Stream()
                with torch.cuda.stream(gs):
                    fn()
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=gs):
                    for _ in range(20):
                        fn()
                g.replay()
                torch.cuda.synchronize()
                s = torch.cuda.current_stream()
                c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                c.record(s)
                g.replay()
                d.record(s)
                d.synchronize()
                r.update({"dtype": dtype, "n": n, "variant": variant, "graph_us_per_launch": c.elapsed_time(d) * 50.0})
                rows.append(r)
                print(json.dumps(r), flush=True)
            del x
    return rows


def do_multi(args):
    """Step latency of the exchange paths at one rank (what a 1-GPU box can
    measure): plain reduce vs reduce_multi (NCCL all-gather + combine kernel)
    vs reduce_fused (exchange inside the kernel), K back-to-back calls."""
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29544")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    comm = rd.Comm.from_process_group()
    fused = rd.FusedComm.from_process_group()
    rows = []
    for log2n in (10, 16, 20, 24, 28):
        n = 1 << log2n
        x = make(n, "float32", "u01")
        paths = {"reduce": lambda: rd.reduce(x, "sum"),
                 "reduce_multi_nccl": lambda: comm.reduce(x, "sum"),
                 "reduce_fused": lambda: fused.reduce(x, "sum")}
        for name, fn in paths.items():
            for _ in range(10):
                fn()
            torch.cuda.synchronize()
            s = torch.cuda.current_stream()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            K = 200
            a.record(s)
            for _ in range(K):
                fn()
            b.record(s)
            b.synchronize()
            us = a.elapsed_time(b) * 1e3 / K
            # graph-captured (GPU-side latency without host launch overhead)
            gs = torch.cuda.Stream()
            with torch.cuda.stream(gs):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                for _ in range(20):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c.record(s)
            g.replay()
            d.record(s)
            d.synchronize()
            r = {"n": n, "path": name, "us_per_step": us, "graph_us_per_step": c.elapsed_time(d) * 1e3 / 20}
            rows.append(r)
            print(json.dumps(r), flush=True)
        fused.check()
        comm.check()
    return rows


def do_overhead(args):
    """Host cost per call of the Python binding vs the C ABI (tiny n, back to back)."""
    rows = []
    x = make(1024, "float32", "u01")
    o = torch.empty((), dtype=torch.float32, device="cuda")
    import time as _t
    for name, fn in (("python reduce(x, op)", lambda: rd.reduce(x, "sum")),
                     ("python reduce(x, op, out=o)", lambda: rd.reduce(x, "sum", out=o))):
        for _ in range(100):
            fn()
        torch.cuda.synchronize()
        t0 = _t.perf_counter()
        for _ in range(2000):
            fn()
        torch.cuda.synchronize()
        r = {"path": name, "us_per_call": (_t.perf_counter() - t0) / 2000 * 1e6}
        rows.append(r)
        print(json.dumps(r), flush=True)
    return rows


def do_context(args):
    """SURVEY §8(d) context rows on the same box, across sizes: this library vs CUB
    DeviceReduce::Reduce (tools/libcubref.so) vs torch.sum / torch.amax vs the read
    probe, float32 / int32 sum and max. Per launch: graph-captured back to back (100
    launches in one CUDA graph; L2-warm below ~L2 size) and cold (L2 read-flushed,
    a device spin, %globaltimer stamp kernels around the launch; kernel boundaries
    land on ~2.05 us steps, so medians move in those steps)."""
    cub = ctypes.CDLL(os.path.join(ROOT, "tools", "libcubref.so"))
    cub.cub_ref_reduce.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p]
    pl = ctypes.CDLL(os.path.join(ROOT, "tools", "libprobe.so"))
    pl.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    pl.probe_stamp.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    sink = torch.zeros(1 << 20, dtype=torch.int32, device="cuda")
    stamps = torch.zeros(4, dtype=torch.int64, device="cuda")
    cur = lambda: torch.cuda.current_stream().cuda_stream
    rows = []
    sizes = args.log2n if args.log2n != [28] else list(range(16, 31, 2))
    for dtype in ("float32", "int32"):
        for op in ("sum", "max"):
            for log2n in sizes:
                n = 1 << log2n
                x = make(n, dtype, "u01" if dtype == "float32" else "uniform_bits")
                nbytes = 4 * n
                o = torch.empty((), dtype=x.dtype, device="cuda")
                ot = torch.empty((), dtype=torch.int64 if (dtype == "int32" and op == "sum") else x.dtype,
                                 device="cuda")
                co = torch.empty(2, dtype=torch.int64, device="cuda")
                code_dt, code_op = (3 if dtype == "float32" else 0), (0 if op == "sum" else 3)
                nb = ctypes.c_size_t(0)
                assert cub.cub_ref_reduce(x.data_ptr(), n, code_dt, code_op, co.data_ptr(), None, ctypes.byref(nb),
                                          cur()) == 0
                tmp = torch.empty(max(1, nb.value), dtype=torch.uint8, device="cuda")
                blocks = 148 * max(1, pl.probe_occupancy(2, 256)) * 4
                impls = {
                    "b200reduce": lambda: rd.reduce(x, op, out=o),
                    "cub": lambda: cub.cub_ref_reduce(x.data_ptr(), n, code_dt, code_op, co.data_ptr(),
                                                      tmp.data_ptr(), ctypes.byref(nb), cur()),
                    "torch": ((lambda: torch.sum(x, dim=0, dtype=ot.dtype, out=ot)) if op == "sum"
                              else (lambda: torch.amax(x, dim=0, out=ot))),
                    "read_probe": lambda: pl.probe_read(x.data_ptr(), nbytes, 2, blocks, 256, sink.data_ptr(),
                                                        cur(), 0),
                }
                for name, fn in impls.items():
                    g = graph_us(fn)
                    cold = []
                    for _ in range(7):
                        flush_l2()
                        torch.cuda._sleep(100_000)
                        pl.probe_stamp(stamps.data_ptr(), 0, cur())
                        fn()
                        pl.probe_stamp(stamps.data_ptr(), 1, cur())
                        torch.cuda.synchronize()
                        cold.append((int(stamps[1]) - int(stamps[0])) * 1e-3)
                    c = statistics.median(cold)
                    r = {"dtype": dtype, "op": op, "log2n": log2n, "impl": name, "graph_us": round(g, 3),
                         "graph_gbps": round(nbytes / g / 1e3, 1), "cold_us": round(c, 2),
                         "cold_gbps": round(nbytes / c / 1e3, 1)}
                    rows.append(r)
                    print(json.dumps(r), flush=True)
                del x, tmp
    return rows


def main():
    p = argparse.ArgumentParser()
    p.add_argument("what", choices=["probe", "ablation", "ops", "sizes", "grids", "crossover", "multi", "overhead",
                                    "exact", "midgrids", "midops", "context", "exactvariants", "variants"])
    p.add_argument("--out", required=True)
    p.add_argument("--log2n", type=int, nargs="+", default=[28])
    p.add_argument("--only", nargs="*", default=None, help="ablation: variants to run")
    args = p.parse_args()
    res = {"probe": do_probe, "ablation": do_ablation, "ops": do_ops, "sizes": do_sizes,
           "grids": do_grids, "crossover": do_crossover, "multi": do_multi,
           "overhead": do_overhead, "exact": do_exact, "exactvariants": do_exactvariants, "variants": do_variants,
           "midgrids": do_midgrids, "midops": do_midops, "context": do_context}[args.what](args)
    meta = {"device": torch.cuda.get_device_name(), "what": args.what}
    with open(args.out, "w") as f:
        json.dump({"meta": meta, "result": res}, f, indent=1)

if __name__ == "__main__":
    main()
