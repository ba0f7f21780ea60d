#!/usr/bin/env python
"""Benchmark of the reduction hot path; prints ONE JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl {b200,reference}]
                    [--dtype float32] [--op sum] [--log2n 28]

A "step" is one pass of the whole hot path (plus a8
when N > 1) over the synthetic input resident in HBM: one `reduce` call (one
kernel launch) at N = 1; one `reduce_fused` call (the exchange inside the
reduce kernel; `--exchange nccl`: `reduce_multi`, reduce kernel + NCCL
all-gather of 32-byte records + rank-order combine kernel) at N > 1.

Beside the value (rank 0, `context`): the timed result checked against the
oracle on the same data; torch.sum, CUB DeviceReduce::Reduce and this
library's compensated / exact sums of the same tensor; int32 sum at the same
n (bit-exact check); and C5 (BASELINE configs[4]): float32 sum and max over
n_total = 2^34 strong-scaled over the N ranks, through reduce_multi and
reduce_fused.

Workload (BASELINE.json configs[1], the metric's config that fits one GPU):
float32 sum, n = 2^28 elements (1 GiB) per GPU, u01 data (inputs/, seed 1);
at N > 1 rank r holds global indices [r*2^28, (r+1)*2^28) of one 2^28*N array
(weak scaling). The input is 8x the 126 MB L2, so there is no L2 flush: each
pass streams from HBM.

`--impl reference` times the CPU oracle (oracle/, Algorithm 1 of PAPER.md
P:27-40) as it stands on the host, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# stdout carries exactly one JSON line. Everything else written to fd 1 --
# library banners such as NCCL's "NCCL version ..." -- is sent to stderr:
# fd 1 is re-pointed at stderr and the JSON line goes to a dup of the real one.
_JSON_OUT = os.fdopen(os.dup(1), "w")
os.dup2(2, 1)


def emit(line: dict) -> None:
    print(json.dumps(line), file=_JSON_OUT, flush=True)

METRIC = "reduce GB/s and % of HBM peak (fp32/int32, n=2^28..2^34) at 1/2/4/8 B200"
NP_BYTES = {"int32": 4, "uint32": 4, "int64": 8, "float32": 4, "float64": 8}
DTYPE_TAG = {"int32": "i32", "uint32": "u32", "int64": "i64", "float32": "f32", "float64": "f64"}


def gbps(nbytes: float, seconds: float) -> float:
    """Decimal GB/s, the paper's convention (Table 2: n*4 bytes / time)."""
    return nbytes / seconds / 1e9


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write bytes)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic(workload_key: str):
    """Per-launch dram bytes of the reduce kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get(workload_key)
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        loaded = [r for r in self.rows if r[2].isdigit() and int(r[2]) > 0] or self.rows
        sm = [float(r[0]) for r in loaded if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({names[i] for r in loaded for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "samples_under_load": len(loaded)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ====================================================================== reference arm
def run_reference(args):
    """The oracle as it stands, on the host cores, on a bounded sample per step."""
    import inputs
    import oracle
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    dt, op = args.dtype, args.op
    s = NP_BYTES[dt]
    n_full = 1 << args.log2n
    # size the per-step sample so the whole run stays within ~2 minutes
    probe = inputs.generate(1 << 20, dt, "u01" if dt.startswith("float") else inputs.default_workload(dt, op))
    t0 = time.perf_counter()
    oracle.reduce(probe, op)
    rate = (1 << 20) / (time.perf_counter() - t0)      # elements / s
    budget = 120.0 / max(1, args.steps + args.warmup)
    m = int(min(n_full, max(1 << 16, rate * budget)))
    wl = "u01" if dt.startswith("float") else inputs.default_workload(dt, op)
    x = inputs.generate(m, dt, wl, seed=1, offset=0, n_total=n_full)
    for _ in range(args.warmup):
        oracle.reduce(x, op)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.reduce(x, op)
    dt_s = time.perf_counter() - t0
    v = gbps(m * s * args.steps, dt_s)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": "GB/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt_s / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE_TAG[dt], "data": "synthetic",
        "config": {"workload": f"{dt} {op}, n=2^{args.log2n} per GPU (u01, seed 1); "
                               f"each reference step folds the first {m} elements (bounded sample)",
                   "n_per_gpu": n_full, "op": op, "sample_elements": m},
        "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"first {m} of {n_full} elements per step, {args.steps} steps"},
        "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def cpu_model() -> str:
    """The host CPU's model name (the report records it beside the core count)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


# ====================================================================== B200 arm
def time_b2b(fn, reps, stream, warm=3):
    """ms per call of `fn`, `reps` calls back to back between two CUDA events on
    `stream` (after `warm` untimed calls; synchronised on both sides)."""
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    b.synchronize()
    return a.elapsed_time(b) / reps


def to_np(t):
    """0-d CUDA tensor -> numpy scalar of its dtype (bit-preserving)."""
    import numpy as np
    import torch
    carrier = {4: torch.int32, 8: torch.int64}[t.element_size()]
    npdt = np.dtype(str(t.dtype).replace("torch.", ""))
    return np.array([t.view(carrier).item()], dtype=str(carrier).replace("torch.", "")).view(npdt)[0]


def check_against_oracle(got, ref, dtype: str, op: str) -> dict:
    """The timed result vs the oracle's fold of the same data (Algorithm 1):
    integers and min/max bit-exact, float + within the north-star bound 4 eps sum|x|."""
    import math
    import numpy as np
    if op in ("argmin", "argmax"):
        return {"ok": None, "note": "arg ops: index checked by the GPU tests"}
    want = ref.value
    if not dtype.startswith("float") or op in ("min", "max", "sum_exact"):
        ok = np.array([got]).tobytes() == np.array([want]).tobytes()
        return {"ok": bool(ok), "got": repr(got), "oracle": repr(want), "rule": "bit-exact"}
    eps = float(np.finfo(dtype).eps)
    scale = ref.sum_abs if op.startswith("sum") else abs(ref.exact)
    bound = 4 * eps * scale
    err = abs(float(got) - ref.exact)
    return {"ok": bool(err <= bound), "got": repr(float(got)), "oracle_exact": ref.exact,
            "err": err, "bound": bound, "err_over_bound": round(err / bound, 6) if bound else None,
            "rule": "|got - exact| <= 4 eps(dtype) sum|x_i| (BASELINE north_star)"}


def run_b200(args):
    import numpy as np
    import torch
    import inputs
    import paper_1710_07358_b200 as rd

    ws, rank, local = dist_env()
    if ws != args.gpus:
        if args.gpus > 1:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch with torchrun")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    use_comm = ws > 1 or args.force_comm
    c5_on = not args.profile and not args.no_c5
    dist = None
    if use_comm or c5_on or ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=dev)
    dt, op = args.dtype, args.op
    s = NP_BYTES[dt]
    n = 1 << args.log2n                              # per GPU (weak scaling)
    wl = "u01" if dt.startswith("float") else inputs.default_workload(dt, op)
    x = torch.empty(n, dtype=getattr(torch, dt), device=dev)
    inputs.fill_device(x, wl, seed=1, offset=rank * n, n_total=n * ws)
    # one element, or a 16-byte rd_arg_result for argmin / argmax
    out = torch.empty(2, dtype=torch.int64, device=dev) if op in rd.ARG_OPS else \
        torch.empty((), dtype=x.dtype, device=dev)
    comm = rd.Comm.from_process_group() if use_comm else None   # NCCL all-gather exchange
    exchange = "nccl"
    if use_comm and args.exchange == "fused":
        # the exchange fused into the reduce kernel, verified against
        # the NCCL path on this data before it is timed: both fold the same W
        # records in rank order, so the bits must agree on every rank. Every
        # step below is collective-safe: a failure on one rank makes all ranks
        # fall back to NCCL together (a stuck peer surfaces as RD_ERR_TIMEOUT).
        fused, a_f = None, None
        ok = torch.ones(1, device=dev)
        try:
            fused = rd.FusedComm.from_process_group()       # raises on all ranks or none
            a_f = fused.reduce(x, op)
            fused.check()
        except Exception as e:
            print(f"[bench] fused exchange unavailable on rank {rank}: {e}", file=sys.stderr)
            ok.fill_(0.0)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 1.0:
            a_n = comm.reduce(x, op)
            comm.check()
            pairs = zip(a_f, a_n) if op in rd.ARG_OPS else [(a_f, a_n)]
            same = all(bool((u.reshape(1).view(torch.uint8) == v.reshape(1).view(torch.uint8)).all().item())
                       for u, v in pairs)
            ok.fill_(1.0 if same else 0.0)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if ok.item() == 1.0:
            comm.destroy()
            comm, exchange = fused, "fused"
        elif fused is not None:
            torch.cuda.synchronize(dev)
            fused.destroy()
    stream = torch.cuda.current_stream(dev)

    def step():
        if comm is None:
            rd.reduce(x, op, out=out)
        else:
            comm.reduce(x, op, out=out)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v: float) -> float:
        if dist is None or ws == 1:
            return v
        tt = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    # warm-up (also creates the per-stream workspace)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(local).start()
    # clock soak: ~1 s of the same work so the clock record sees a loaded GPU
    t_end = time.perf_counter() + (0.0 if args.profile else 1.0)
    while time.perf_counter() < t_end:
        for _ in range(20):
            step()
        torch.cuda.synchronize(dev)

    # ---------------- timed region: exactly K steps
    # (no per-step events: an event between two launches would serialise them
    # and hide the programmatic-dependent-launch overlap of consecutive steps)
    K = args.steps
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    t0.record(stream)
    for i in range(K):
        step()
    t1.record(stream)
    barrier()
    clocks = sampler.stop()
    local_ms = t0.elapsed_time(t1)
    total_ms = max_over_ranks(local_ms)
    value = gbps(n * s * ws * K, total_ms / 1e3)
    timed_result = (to_np(out.view(torch.int64)[1]) if op in rd.ARG_OPS else to_np(out))

    # ---------------- dominant kernel (the reduce kernel) alone, for the roofline
    if comm is None:
        kern_ms = local_ms / K                      # one launch per step
        kern_src = "CUDA events around the K back-to-back steps of the timed region / K (1 launch per step)"
    else:
        rec = torch.empty(32, dtype=torch.uint8, device=dev)
        kern_ms = time_b2b(lambda: rd.reduce_partial(x, op, rec=rec), K, stream, warm=0)
        kern_src = "CUDA events around K back-to-back launches of the same reduce kernel (reduce_partial) / K"
    peak, peak_src = load_peaks()
    achieved = gbps(n * s, kern_ms / 1e3)

    # ---------------- host copy of the input (e2e source; the oracle check reads it)
    need_host = not args.profile
    host = torch.empty(n if need_host else 0, dtype=x.dtype, pin_memory=True)
    if need_host:
        host.copy_(x)
    torch.cuda.synchronize(dev)

    # ---------------- e2e: host (pinned) -> device -> result -> host, through the public API
    ke = 0 if args.profile else max(3, min(K, 10))
    if ke == 0:
        te, e2e_timer = float("nan"), "skipped (--profile)"
    elif comm is None:
        rd.reduce_host(host, op)                         # warm the pipeline
        te = time.perf_counter()
        for _ in range(ke):
            rd.reduce_host(host, op)
        te = time.perf_counter() - te
        e2e_timer = "host perf_counter around synchronous reduce_host calls (chunked H2D overlapped with reduce)"
    else:
        barrier()
        te = time.perf_counter()
        for _ in range(ke):
            x.copy_(host, non_blocking=True)
            comm.reduce(x, op, out=out)
            out.cpu()
        te = max_over_ranks(time.perf_counter() - te)
        e2e_timer = "host perf_counter, max over ranks: pinned H2D copy + reduce_multi + .item() per step"
    e2e = {"value": round(gbps(n * s * ws * ke, te), 3) if ke else None, "unit": "GB/s",
           "h2d_bytes_per_step": n * s * ws, "d2h_bytes_per_step": out.numel() * out.element_size() * ws,
           "steps": ke, "timer": e2e_timer}

    # ---------------- the timed result against the oracle on the same data (every rank
    # folds its own shard; rank 0 merges the folds in rank order, Algorithm 1's order)
    check, cpu, oracle_ref = None, None, None
    if not args.profile:
        import oracle
        xh = host.numpy()
        if ws == 1 and not args.no_cpu:
            # cpu_baseline: the oracle as it stands, single thread, full passes over the
            # same host array for ~cpu_seconds (its last pass is the check's reference)
            passes, tc = 0, time.perf_counter()
            while True:
                oracle_ref = oracle.reduce(xh, op)
                passes += 1
                el = time.perf_counter() - tc
                if el > args.cpu_seconds or passes >= 50:
                    break
            cpu = {"value": round(gbps(n * s * passes, el), 4), "unit": "GB/s", "cores": 1,
                   "kind": "oracle", "cpu_model": cpu_model(),
                   "sample": f"{passes} full pass(es) over the same {n}-element host array "
                             f"({el:.1f} s, single thread, gcc -O2)"}
            # all host cores: the same plain fold on contiguous chunks (ctypes drops
            # the GIL), partials merged in chunk order (oracle.Fold.merge)
            import concurrent.futures as cf
            cores = os.cpu_count() or 1
            bounds = [(n * i // cores, n * (i + 1) // cores) for i in range(cores)]
            tc = time.perf_counter()
            with cf.ThreadPoolExecutor(max_workers=cores) as ex:
                folds = list(ex.map(lambda be: oracle.Fold(dt, op).fold(xh[be[0]:be[1]]), bounds))
            acc = folds[0]
            for f in folds[1:]:
                acc.merge(f)
            el_all = time.perf_counter() - tc
            cpu["all_core"] = {"value": round(gbps(n * s, el_all), 4), "unit": "GB/s", "cores": cores,
                               "kind": "oracle per contiguous chunk, chunk partials merged in order",
                               "sample": f"one pass over the {n}-element host array"}
        else:
            import ctypes
            f = oracle.Fold(dt, op).fold(xh)
            if ws > 1:
                blob = bytes(ctypes.string_at(ctypes.addressof(f.st), ctypes.sizeof(f.st)))
                blobs = [None] * ws
                dist.all_gather_object(blobs, blob)
                f = oracle.Fold(dt, op)
                for bl in blobs:                         # rank order
                    g = oracle.Fold(dt, op)
                    ctypes.memmove(ctypes.addressof(g.st), bl, len(bl))
                    f.merge(g)
            oracle_ref = f.result()
        if rank == 0:
            check = check_against_oracle(timed_result, oracle_ref, dt, op)
            check["what"] = (f"the last timed step's result vs the oracle over the same {n * ws} elements "
                             + ("(one pass on rank 0)" if ws == 1 else "(per-rank folds merged in rank order)"))

    # ---------------- context rows, rank 0, on its own tensor (not the bench value)
    ctx = {}
    probe = None
    if rank == 0 and not args.profile:
        R = 20
        ctx["torch_sum_gbs"] = round(gbps(n * s, time_b2b(lambda: torch.sum(x), R, stream) / 1e3), 2) \
            if op == "sum" else None
        if op == "sum" and x.is_floating_point():
            # this library's other float sums of the same tensor
            for vop in ("sum_compensated", "sum_exact"):
                ctx[vop + "_gbs"] = round(gbps(n * s, time_b2b(lambda: rd.reduce(x, vop, out=out), R,
                                                               stream) / 1e3), 2)
        # CUB DeviceReduce::Reduce on the same tensor (library context)
        cub_lib = os.path.join(ROOT, "tools", "libcubref.so")
        cub = None
        if os.path.exists(cub_lib) and dt in ("float32", "int32") and op in ("sum", "max"):
            import ctypes
            cub = ctypes.CDLL(cub_lib)
            cub.cub_ref_reduce.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t),
                                           ctypes.c_void_p]

            def cub_gbs(t, code_dt, code_op):
                o = torch.empty(2, dtype=torch.int64, device=dev)
                nb = ctypes.c_size_t(0)
                assert cub.cub_ref_reduce(t.data_ptr(), t.numel(), code_dt, code_op, o.data_ptr(), None,
                                          ctypes.byref(nb), stream.cuda_stream) == 0
                tmp = torch.empty(max(1, nb.value), dtype=torch.uint8, device=dev)
                fn = lambda: cub.cub_ref_reduce(t.data_ptr(), t.numel(), code_dt, code_op, o.data_ptr(),
                                                tmp.data_ptr(), ctypes.byref(nb), stream.cuda_stream)
                return round(gbps(t.numel() * t.element_size(), time_b2b(fn, R, stream) / 1e3), 2)

            ctx["cub_device_reduce_gbs"] = cub_gbs(x, 3 if dt == "float32" else 0, 0 if op == "sum" else 3)
        # the metric's other dtype ("one of integers and one of single precision
        # floating points"): int32 sum at the same n, checked bit-exact against the oracle
        if dt == "float32" and op == "sum":
            import oracle
            xi = torch.empty(n, dtype=torch.int32, device=dev)
            inputs.fill_device(xi, "uniform_bits", seed=1)
            oi = torch.empty((), dtype=torch.int32, device=dev)
            ms = time_b2b(lambda: rd.reduce(xi, "sum", out=oi), R, stream)
            got = to_np(oi)
            want = oracle.reduce(xi.cpu().numpy(), "sum").value
            ctx["int32_sum"] = {"gbs": round(gbps(n * 4, ms / 1e3), 2), "n": n,
                                "workload": "uniform_bits, seed 1", "check_bit_exact": bool(got == want),
                                "cub_device_reduce_gbs": cub_gbs(xi, 0, 0) if cub is not None else None}
            del xi
            # the exact sum on its adversarial workload (exponents over 2^+-40: nearly
            # every group takes the binned-extraction fallback), same n,
            # checked bit-exact against the oracle's exact sum
            import numpy as np
            xw = torch.empty(n, dtype=torch.float32, device=dev)
            inputs.fill_device(xw, "wide", seed=1)
            ow = torch.empty((), dtype=torch.float32, device=dev)
            ms = time_b2b(lambda: rd.reduce(xw, "sum_exact", out=ow), R, stream)
            got = to_np(ow)
            want = oracle.reduce(xw.cpu().numpy(), "sum_exact").value
            ctx["sum_exact_wide"] = {"gbs": round(gbps(n * 4, ms / 1e3), 2), "n": n, "workload": "wide, seed 1",
                                     "check_bit_exact": bool(np.asarray(got).tobytes() == np.asarray(want).tobytes())}
            del xw

        # the same-run HBM read ceiling (SURVEY §8(d) peak 3): the read probe
        # (tools/probe.cu: 256-bit loads xor-folded, no reduction semantics) over
        # the same tensor, in its best configurations of profiles/r01_read_probe.json,
        # back to back like the timed steps; the north star's ">= 90% of measured HBM
        # read bandwidth" is achieved / this
        probe_lib = os.path.join(ROOT, "tools", "libprobe.so")
        if os.path.exists(probe_lib):
            import ctypes
            pl = ctypes.CDLL(probe_lib)
            pl.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            pl.probe_occupancy.argtypes = [ctypes.c_int, ctypes.c_int]
            sink = torch.zeros(1024, dtype=torch.int32, device=dev)
            best = 0.0
            for thr, unr in ((256, 2), (1024, 2), (512, 1)):
                blocks = 148 * max(1, pl.probe_occupancy(unr, thr)) * 4
                fn = lambda: pl.probe_read(x.data_ptr(), n * s, unr, blocks, thr, sink.data_ptr(),
                                           stream.cuda_stream, 0)
                best = max(best, gbps(n * s, time_b2b(fn, R, stream) / 1e3))
            probe = {"value": round(best, 2), "unit": "GB/s", "frac": round(achieved / best, 4),
                     "how": "tools/probe.cu read probe on the same tensor, best of 3 configs, 20 back-to-back "
                            "launches each (CUDA events)"}

    # ---------------- C5 (BASELINE configs[4]): sharded float32 sum and max over
    # n_total = 2^34 (64 GiB), STRONG-scaled: rank r holds rd.shard_range(2^34, W, r);
    # timed through reduce_multi (NCCL all-gather + rank-order fold) and reduce_fused
    # (the exchange inside the reduce kernel), max over ranks, every rank's result
    # checked: both paths bitwise equal, max == the planted 2^20, sum within
    # 4 eps sum|x| of the exact sum (RD_SUM_EXACT, bit-exact vs the oracle in the tests)
    c5 = None
    if c5_on:
        del host
        nt = 1 << args.c5_log2n
        b0, cnt = rd.shard_range(nt, ws, rank)
        xc = torch.empty(cnt, dtype=torch.float32, device=dev)
        inputs.fill_device(xc, "u01", seed=1, offset=b0, n_total=nt)
        p_max = nt - 12345                               # planted maximum (global index)
        if b0 <= p_max < b0 + cnt:
            xc[p_max - b0] = 2.0 ** 20
        torch.cuda.synchronize(dev)
        nccl_c = comm if (comm is not None and exchange == "nccl") else rd.Comm.from_process_group()
        fused_c = comm if (comm is not None and exchange == "fused") else None
        c5 = {"workload": f"float32, n_total=2^{args.c5_log2n} ({nt * 4 / 2**30:.0f} GiB) u01 seed 1, max planted "
                          f"2^20 at index {p_max}; rank r holds rd.shard_range(n_total, {ws}, r) (strong scaling)",
              "n_total": nt, "n_local": cnt, "ranks": ws}
        try:
            if fused_c is None:
                try:
                    fused_c = rd.FusedComm.from_process_group()
                except Exception as e:                    # collective: all ranks or none
                    c5["fused_error"] = str(e)
            Kc = max(3, min(K, 20))
            res = {}
            for cop in ("sum", "max"):
                oc = torch.empty((), dtype=torch.float32, device=dev)
                for path, cm in (("nccl", nccl_c), ("fused", fused_c)):
                    if cm is None:
                        continue
                    barrier()
                    ms = max_over_ranks(time_b2b(lambda: cm.reduce(xc, cop, out=oc), Kc, stream, warm=2))
                    cm.check()
                    res[(cop, path)] = to_np(oc)
                    c5[f"{cop}_{path}_gbs"] = round(gbps(nt * 4, ms / 1e3), 2)
                    c5[f"{cop}_{path}_ms"] = round(ms, 4)
            xs = nccl_c.reduce(xc, "sum_exact")
            exact = float(to_np(xs))
            chk = {"max_is_planted": all(float(v) == 2.0 ** 20 for (o, _), v in res.items() if o == "max"),
                   "fused_equals_nccl": all(res[(o, "nccl")].tobytes() == res[(o, "fused")].tobytes()
                                            for o in ("sum", "max") if (o, "fused") in res)}
            # u01 terms are >= 0, so sum|x_i| is the exact sum itself (to its rounding)
            err = abs(float(res[("sum", "nccl")]) - exact)
            chk["sum_err_over_bound"] = round(err / (4 * 2.0 ** -23 * exact), 6)
            chk["sum_within_bound"] = bool(err <= 4 * 2.0 ** -23 * exact * (1 + 2.0 ** -23))
            chk["sum"], chk["sum_exact"] = float(res[("sum", "nccl")]), exact
            c5["check"] = chk
            c5["steps"] = Kc
            c5["timer"] = ("CUDA events around Kc back-to-back calls per path and op, max over ranks; "
                           "GB/s = n_total * 4 B / time")
        finally:
            torch.cuda.synchronize(dev)
            if fused_c is not None and fused_c is not comm:
                fused_c.destroy()
            if nccl_c is not comm:
                nccl_c.destroy()
            del xc

    line = None
    if rank == 0:
        hbm_nominal = 8000.0
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws, "steps": K,
            "warmup": max(3, args.warmup), "ms_per_step": round(total_ms / K, 5), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": DTYPE_TAG[dt], "data": "synthetic",
            "config": {"workload": f"{dt} {op}, n=2^{args.log2n} per GPU ({wl}, seed 1), BASELINE configs[1]",
                       "n_per_gpu": n, "n_total": n * ws, "op": op,
                       "l2": "input (%.2f GB/GPU) > 126 MB L2: no flush" % (n * s / 1e9),
                       "parallelism": f"shard{ws}" if ws > 1 else "single",
                       "exchange": ("fused in-kernel over NVLink (reduce_fused)" if exchange == "fused"
                                    else "NCCL all-gather + rank-order fold (reduce_multi)") if use_comm else None},
            "pct_hbm_peak": round(100 * value / (hbm_nominal * ws), 2),
            "hbm_peak_basis": "nominal 8 TB/s per GPU (B200 datasheet, DGX; 7.7 HGX): read bandwidth",
            "pct_read_probe": round(100 * achieved / probe["value"], 2) if probe else None,
            "elements_per_s": round(value * 1e9 / s, 1),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "frac_of_read_probe": probe["frac"] if probe else None,
                         "traffic": load_traffic(f"{dt}-{op}-2^{args.log2n}"),
                         "traffic_source": "committed ncu --set full capture of this kernel at this size "
                                           "(profiles/traffic.json; dram__bytes_read.sum + dram__bytes_write.sum "
                                           "per launch), not measured in this run",
                         "kernel_ms": round(kern_ms, 5), "peak_source": peak_src + " -- a read+write copy, "
                         "so a read-only kernel can exceed 1.0; frac_of_read_probe is the same-run read ceiling",
                         "achieved_source": kern_src,
                         "algorithmic_bytes_per_launch": n * s,
                         "read_probe": probe},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": K * (1 if (comm is None or exchange == "fused") else 2),
            "clocks": clocks,
            "context": {"check": check, "result": repr(timed_result), **ctx, "c5": c5},
        }
        emit(line)
    if dist is not None:
        dist.barrier()
        if comm is not None:
            comm.destroy()
        dist.destroy_process_group()
    return 0


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=10)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--dtype", default="float32", choices=list(NP_BYTES))
    p.add_argument("--op", default="sum")
    p.add_argument("--log2n", type=int, default=28)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--exchange", choices=["fused", "nccl"], default="fused",
                   help="N>1: exchange partials inside the reduce kernel over NVLink (reduce_fused, verified "
                        "against NCCL first, falls back to it) or with an NCCL all-gather (reduce_multi)")
    p.add_argument("--force-comm", action="store_true",
                   help="use the reduce_multi (NCCL) step even at one rank (tests the N>1 path on one GPU)")
    p.add_argument("--profile", action="store_true",
                   help="for ncu: no clock soak, e2e, cpu baseline or context rows (not a bench value)")
    p.add_argument("--no-c5", action="store_true",
                   help="skip the C5 context (strong-scaled float32 sum/max over n_total = 2^34)")
    p.add_argument("--c5-log2n", type=int, default=34)
    args = p.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
