#!/usr/bin/env python
"""Where a single cold bulk-kernel launch spends its time (measurement only).

Loads an RD_TIMELINE build of the library (python -m paper_1710_07358_b200.build
--define RD_TIMELINE --out build/ab/timeline/libb200reduce.so), whose bulk
kernel stamps %globaltimer per CTA: 0 entry, 1 first full stage, 2 stream end
(consumers), 3 producer out of chunks, 4 ticket drawn, and for the last CTA
5 slots folded, 6 block reduce done, 7 output written.

Each rep: L2 read-flushed, a ~60 us device spin (torch.cuda._sleep) so the
host has enqueued the launch before the GPU reaches it (the event pair then
holds only device time: launch latency + kernel), event, reduce, event. The
read probe (tools/libprobe.so) is timed the same way on the same tensor.

    python tools/timeline.py [--lib PATH] [--log2n 25 26 28] [--reps 10]
    python tools/timeline.py --exp gaps      # launch gaps: stamp kernels around
        the launch, with and without a preceding 192 KB-shared-memory kernel
        (the SM's L1/shared carveout already switched), bulk vs vector vs probe
"""
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

DT = {"int32": 0, "uint32": 1, "int64": 2, "float32": 3, "float64": 4}
OPS = {"sum": 0, "prod": 1, "min": 2, "max": 3, "and": 4, "or": 5, "xor": 6, "argmin": 7, "argmax": 8,
       "sum_compensated": 9, "sum_exact": 10}
TORCH_DT = {"int32": torch.int32, "uint32": torch.uint32, "float32": torch.float32, "float64": torch.float64,
            "int64": torch.int64}

_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.ones(128 * 2 ** 20, dtype=torch.int32, device="cuda")
    _flush.max()


def cold(fn, reps, warm=False):
    """device time of single launches, host enqueue hidden behind a spin
    (warm: no L2 flush -- the previous launch left the input in L2)"""
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
        if warm:
            fn()
        else:
            flush_l2()
        torch.cuda._sleep(120_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return ts


def b2b(fn, reps=20):
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def gaps(L, P, args):
    """stamp0 (end of the preceding work) -> first CTA entry -> output -> stamp1"""
    st = torch.cuda.current_stream()
    out = torch.empty(4, dtype=torch.int64, device="cuda")
    stamps = torch.zeros(8, dtype=torch.int64, device="cuda")
    hog_sink = torch.zeros(4, dtype=torch.int32, device="cuda")
    sink = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
    cfg_t = type("cfg", (ctypes.Structure,), {"_fields_": [("variant", ctypes.c_int32), ("vec_bytes", ctypes.c_int32),
                                                             ("unroll", ctypes.c_int32), ("block", ctypes.c_int32),
                                                             ("grid", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]})
    L.rd_reduce_ex.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    P.probe_stamp.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    P.probe_smem_hog.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    for log2n in args.log2n:
        n = 1 << log2n
        x = torch.empty(n, dtype=torch.float32, device="cuda")
        inputs.fill_device(x, "u01")
        nbytes = 4 * n
        vec = cfg_t(1, 0, 0, 0, 0)
        impls = {
            "auto": lambda: L.reduce(x.data_ptr(), n, 3, 0, out.data_ptr(), st.cuda_stream),
            "vector": lambda: L.rd_reduce_ex(x.data_ptr(), n, 3, 0, out.data_ptr(), st.cuda_stream,
                                             ctypes.byref(vec), None),
            "probe": lambda: P.probe_read(x.data_ptr(), nbytes, 2, 148 * max(1, P.probe_occupancy(2, 256)) * 4, 256,
                                          sink.data_ptr(), st.cuda_stream, 0),
        }
        for name, fn in impls.items():
            for hog in (0, 1):
                for _ in range(3):
                    fn()
                evs, pre, post, tot = [], [], [], []
                for _ in range(args.reps):
                    flush_l2()
                    torch.cuda._sleep(120_000)
                    if hog:
                        P.probe_smem_hog(200 * 1024, 148, hog_sink.data_ptr(), st.cuda_stream)
                    if name == "auto":
                        L.rd_timeline_clear()
                    P.probe_stamp(stamps.data_ptr(), 0, st.cuda_stream)
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(st)
                    fn()
                    b.record(st)
                    P.probe_stamp(stamps.data_ptr(), 1, st.cuda_stream)
                    torch.cuda.synchronize()
                    evs.append(a.elapsed_time(b) * 1e3)
                    s0, s1 = int(stamps[0]), int(stamps[1])
                    tot.append((s1 - s0) * 1e-3)
                    if name == "auto":
                        tl = (ctypes.c_uint64 * (4096 * 8))()
                        L.rd_timeline_read(tl, 4096)
                        ent = [tl[i * 8] for i in range(4096) if tl[i * 8]]
                        outs = [tl[i * 8 + 7] for i in range(4096) if tl[i * 8 + 7]]
                        if ent and outs:      # AUTO took the bulk kernel (the instrumented one)
                            pre.append((min(ent) - s0) * 1e-3)
                            post.append((s1 - max(outs)) * 1e-3)
                med = lambda v: round(statistics.median(v), 2) if v else None
                r = {"exp": "gaps", "log2n": log2n, "impl": name, "after_smem_kernel": bool(hog),
                     "event_us": med(evs), "stamp_to_stamp_us": med(tot), "stamp0_to_first_entry_us": med(pre),
                     "output_to_stamp1_us": med(post), "event_gbps": round(nbytes / med(evs) / 1e3, 1)}
                print(json.dumps(r), flush=True)
        del x


def grids(L, P, args):
    """mid sizes: the vector kernel's (unroll, grid) -- cold (L2 read-flushed, stamp kernels
    around the launch: %globaltimer, finer than the events' 2.048 us steps) and L2-warm
    (100 launches in one CUDA graph) -- next to the bulk kernel and the read probe"""
    st = torch.cuda.current_stream()
    out = torch.empty(4, dtype=torch.int64, device="cuda")
    stamps = torch.zeros(8, dtype=torch.int64, device="cuda")
    sink = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
    cfg_t = type("cfg", (ctypes.Structure,), {"_fields_": [("variant", ctypes.c_int32), ("vec_bytes", ctypes.c_int32),
                                                             ("unroll", ctypes.c_int32), ("block", ctypes.c_int32),
                                                             ("grid", ctypes.c_int32), ("reserved", ctypes.c_int32 * 3)]})
    L.rd_reduce_ex.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    P.probe_stamp.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    for log2n, pair in [(a, b) for a in args.log2n for b in args.pairs.split(",")]:
        dtype, op = pair.split(":")
        dt, opc = DT[dtype], OPS[op]
        n = 1 << log2n
        x = torch.empty(n, dtype=TORCH_DT[dtype], device="cuda")
        inputs.fill_device(x, "u01" if dtype.startswith("float") else "uniform_bits")
        nbytes = x.element_size() * n
        cases = {"auto": None, "bulk": cfg_t(3, 0, 0, 0, 0)}
        for u in args.us:
            for g in args.gs:
                cases[f"vector_u{u}_g{g}"] = cfg_t(1, 32, u, 0, g)
        for g in (148, 296, 444, 592):      # the default vector kernel (any dtype / op)
            cases[f"vector_g{g}"] = cfg_t(1, 0, 0, 0, g)
        for name, cfg in list(cases.items()) + [("probe", "probe")]:
            cur = lambda: torch.cuda.current_stream().cuda_stream   # the capture stream inside the graph
            if cfg == "probe":
                fn = lambda: P.probe_read(x.data_ptr(), nbytes, 2, 148 * max(1, P.probe_occupancy(2, 256)) * 4, 256,
                                          sink.data_ptr(), cur(), 0)
            elif cfg is None:
                fn = lambda: L.reduce(x.data_ptr(), n, dt, opc, out.data_ptr(), cur())
            else:
                fn = (lambda c: lambda: L.rd_reduce_ex(x.data_ptr(), n, dt, opc, out.data_ptr(), cur(),
                                                       ctypes.byref(c), None))(cfg)
            if fn() != 0 and cfg != "probe":
                continue
            if args.cases and name not in args.cases:
                continue
            for _ in range(3):
                fn()
            tot = []
            for _ in range(args.reps):
                flush_l2()
                torch.cuda._sleep(120_000)
                P.probe_stamp(stamps.data_ptr(), 0, st.cuda_stream)
                fn()
                P.probe_stamp(stamps.data_ptr(), 1, st.cuda_stream)
                torch.cuda.synchronize()
                tot.append((int(stamps[1]) - int(stamps[0])) * 1e-3)
            # L2-warm: 100 launches captured in one graph
            gs = torch.cuda.Stream()
            gs.wait_stream(st)
            with torch.cuda.stream(gs):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=gs):
                for _ in range(100):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            ws = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                g.replay()
                b.record(st)
                b.synchronize()
                ws.append(a.elapsed_time(b) * 10.0)
            r = {"exp": "grids", "dtype": dtype, "op": op, "log2n": log2n, "case": name, "cold_stamp_us": round(statistics.median(tot), 2),
                 "cold_stamp_min_us": round(min(tot), 2), "warm_graph_us": round(statistics.median(ws), 2)}
            print(json.dumps(r), flush=True)
            del g
        del x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "build", "ab", "timeline", "libb200reduce.so"))
    ap.add_argument("--log2n", type=int, nargs="*", default=[25, 26, 27, 28])
    ap.add_argument("--pairs", default="float32:sum,int32:sum,float32:argmin")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--exp", default="timeline", choices=["timeline", "gaps", "grids"])
    ap.add_argument("--warm", action="store_true", help="timeline: no L2 flush (L2-resident inputs)")
    ap.add_argument("--cases", nargs="*", default=None, help="grids: only these cases")
    ap.add_argument("--us", type=int, nargs="*", default=[4, 8], help="grids: vector unrolls (ablation kernels)")
    ap.add_argument("--gs", type=int, nargs="*", default=[148, 296, 592, 1184], help="grids: vector grids")
    args = ap.parse_args()
    L = ctypes.CDLL(args.lib)
    L.reduce.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                         ctypes.c_void_p]
    if hasattr(L, "rd_timeline_read"):      # RD_TIMELINE builds only
        L.rd_timeline_read.argtypes = [ctypes.c_void_p, ctypes.c_int]
    P = ctypes.CDLL(os.path.join(ROOT, "tools", "libprobe.so"))
    P.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                             ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    P.probe_occupancy.argtypes = [ctypes.c_int, ctypes.c_int]
    sink = torch.zeros(1 << 20, dtype=torch.int64, device="cuda")
    out = torch.empty(4, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream()
    info = {"device": torch.cuda.get_device_name(), "lib": os.path.relpath(args.lib, ROOT), "reps": args.reps}
    print(json.dumps({"meta": info}), flush=True)
    if args.exp == "gaps":
        return gaps(L, P, args)
    if args.exp == "grids":
        return grids(L, P, args)
    for log2n in args.log2n:
        n = 1 << log2n
        for pair in args.pairs.split(","):
            dtype, op = pair.split(":")
            x = torch.empty(n, dtype=TORCH_DT[dtype], device="cuda")
            inputs.fill_device(x, "u01" if dtype.startswith("float") else "uniform_bits")
            nbytes = n * x.element_size()
            f = lambda: L.reduce(x.data_ptr(), n, DT[dtype], OPS[op], out.data_ptr(), st.cuda_stream)
            for _ in range(5):
                assert f() == 0
            torch.cuda.synchronize()
            assert L.rd_timeline_clear() == 0
            ev = cold(f, args.reps, args.warm)
            # the timeline of the last rep
            tl = (ctypes.c_uint64 * (4096 * 8))()
            assert L.rd_timeline_read(tl, 4096) == 0
            rows = [[tl[i * 8 + k] for k in range(8)] for i in range(4096)]
            rows = [r for r in rows if r[0] != 0]
            t0 = min(r[0] for r in rows)
            rel = lambda v: (v - t0) * 1e-3
            last = max(rows, key=lambda r: r[7])
            ent = [rel(r[0]) for r in rows]
            first = [(r[1] - r[0]) * 1e-3 for r in rows if r[1]]
            send = sorted(rel(r[2]) for r in rows if r[2])
            pend = sorted(rel(r[3]) for r in rows if r[3])
            tick = sorted(rel(r[4]) for r in rows if r[4])
            # the probe, cold and back to back (one of bench.py's configs: 256 thr, unroll 2)
            pf = lambda: P.probe_read(x.data_ptr(), nbytes, 2, 148 * max(1, P.probe_occupancy(2, 256)) * 4, 256,
                                      sink.data_ptr(), st.cuda_stream, 0)
            for _ in range(3):
                pf()
            pev = cold(pf, args.reps, args.warm)
            r = {"dtype": dtype, "op": op, "log2n": log2n, "grid": len(rows),
                 "cold_event_us": round(statistics.median(ev), 2), "cold_event_min_us": round(min(ev), 2),
                 "probe_cold_event_us": round(statistics.median(pev), 2),
                 "b2b_us": round(b2b(f), 2), "probe_b2b_us": round(b2b(pf), 2),
                 "span_us": round(rel(last[7]), 2),
                 "entry_spread_us": round(max(ent), 2), "entry_med_us": round(statistics.median(ent), 2),
                 "first_data_us_med": round(statistics.median(first), 2) if first else None,
                 "producer_done_us": [round(pend[0], 2), round(pend[len(pend) // 2], 2), round(pend[-1], 2)] if pend else None,
                 "stream_end_us": [round(send[0], 2), round(send[len(send) // 2], 2), round(send[-1], 2)],
                 "ticket_us": [round(tick[0], 2), round(tick[-1], 2)],
                 "last_fold_us": round((last[5] - last[4]) * 1e-3, 2),
                 "last_block_reduce_us": round((last[6] - last[5]) * 1e-3, 2),
                 "last_output_us": round((last[7] - last[6]) * 1e-3, 2)}
            r["cold_gbps"] = round(nbytes / r["cold_event_us"] / 1e3, 1)
            r["probe_cold_gbps"] = round(nbytes / r["probe_cold_event_us"] / 1e3, 1)
            r["b2b_gbps"] = round(nbytes / r["b2b_us"] / 1e3, 1)
            r["probe_b2b_gbps"] = round(nbytes / r["probe_b2b_us"] / 1e3, 1)
            print(json.dumps(r), flush=True)
            del x


if __name__ == "__main__":
    main()
