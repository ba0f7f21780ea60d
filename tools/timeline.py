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
OPS = {"sum": 0, "max": 3, "argmin": 7, "argmax": 8, "sum_exact": 10}
TORCH_DT = {"int32": torch.int32, "float32": torch.float32, "float64": torch.float64, "int64": torch.int64}

_flush = None


def flush_l2():
    global _flush
    if _flush is None:
        _flush = torch.ones(128 * 2 ** 20, dtype=torch.int32, device="cuda")
    _flush.max()


def cold(fn, reps):
    """device time of single launches, host enqueue hidden behind a spin"""
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps):
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
            "bulk": lambda: L.reduce(x.data_ptr(), n, 3, 0, out.data_ptr(), st.cuda_stream),
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
                    if name == "bulk":
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
                    if name == "bulk":
                        tl = (ctypes.c_uint64 * (4096 * 8))()
                        L.rd_timeline_read(tl, 4096)
                        ent = [tl[i * 8] for i in range(4096) if tl[i * 8]]
                        outs = [tl[i * 8 + 7] for i in range(4096) if tl[i * 8 + 7]]
                        pre.append((min(ent) - s0) * 1e-3)
                        post.append((s1 - max(outs)) * 1e-3)
                med = lambda v: round(statistics.median(v), 2) if v else None
                r = {"exp": "gaps", "log2n": log2n, "impl": name, "after_smem_kernel": bool(hog),
                     "event_us": med(evs), "stamp_to_stamp_us": med(tot), "stamp0_to_first_entry_us": med(pre),
                     "output_to_stamp1_us": med(post), "event_gbps": round(nbytes / med(evs) / 1e3, 1)}
                print(json.dumps(r), flush=True)
        del x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=os.path.join(ROOT, "build", "ab", "timeline", "libb200reduce.so"))
    ap.add_argument("--log2n", type=int, nargs="*", default=[25, 26, 27, 28])
    ap.add_argument("--pairs", default="float32:sum,int32:sum,float32:argmin")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--exp", default="timeline", choices=["timeline", "gaps"])
    args = ap.parse_args()
    L = ctypes.CDLL(args.lib)
    L.reduce.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                         ctypes.c_void_p]
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
            ev = cold(f, args.reps)
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
            pev = cold(pf, args.reps)
            r = {"dtype": dtype, "op": op, "log2n": log2n, "grid": len(rows),
                 "cold_event_us": round(statistics.median(ev), 2), "cold_event_min_us": round(min(ev), 2),
                 "probe_cold_event_us": round(statistics.median(pev), 2),
                 "b2b_us": round(b2b(f), 2), "probe_b2b_us": round(b2b(pf), 2),
                 "span_us": round(rel(last[7]), 2),
                 "entry_spread_us": round(max(ent), 2),
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
