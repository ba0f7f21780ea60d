"""Command line front end of the library ("CLI exit codes follow
S:407 -- 0 ok, 1 verification failure, 2 usage, 3 runtime").

    python -m paper_1710_07358_b200 --op sum --dtype float32 --n 268435456 [--workload u01] [--seed 1]
    python -m paper_1710_07358_b200 --op max --input x.npy          # a .npy array, copied to the GPU
    python -m paper_1710_07358_b200 --op sum_exact --n 1000000 --check --json

Reduces one array on the current GPU through the C ABI and prints the result
(and, with --json, one JSON line with the timing). --check re-runs the
reduction through both kernel variants and a 4-way shard split (records) and
fails with exit code 1 unless every integer / min / max / arg / exact result
is bitwise identical and every float sum or product agrees within the
library's stated bound (include/b200reduce.h) -- a self-consistency check;
parity with the CPU oracle is the test suite's job (tests/).

Exit codes: 0 ok, 1 check failed, 2 usage (bad arguments, unknown or
unsupported dtype/op), 3 runtime (no CUDA device, CUDA/NCCL failure).
"""
from __future__ import annotations

import argparse
import json
import math
import sys


def _parse(argv):
    p = argparse.ArgumentParser(prog="python -m paper_1710_07358_b200", description=__doc__.split("\n\n")[0])
    p.add_argument("--op", required=True)
    p.add_argument("--dtype", default="float32")
    p.add_argument("--n", type=int, default=1 << 20, help="elements (synthetic input)")
    p.add_argument("--workload", default=None, help="synthetic input recipe (inputs/, DESIGN.md §5)")
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--input", default=None, help=".npy host array instead of a synthetic input")
    p.add_argument("--check", action="store_true", help="cross-check variants and a shard split")
    p.add_argument("--json", action="store_true", help="print one JSON line")
    return p.parse_args(argv)


def _scalar(v):
    if isinstance(v, tuple):
        return [_scalar(v[0]), int(v[1])]
    f = v.item() if hasattr(v, "item") else v
    if isinstance(f, float) and not math.isfinite(f):
        return str(f)
    return f


def main(argv=None) -> int:
    try:
        args = _parse(sys.argv[1:] if argv is None else argv)
    except SystemExit as e:                       # argparse: usage errors exit 2
        return int(e.code or 0)
    import numpy as np
    import torch

    import paper_1710_07358_b200 as rd
    if args.op not in rd.OPS or args.dtype not in rd.DTYPE_NAMES:
        print(f"unknown op {args.op!r} or dtype {args.dtype!r}; ops: {sorted(rd.OPS)}, "
              f"dtypes: {sorted(rd.DTYPE_NAMES)}", file=sys.stderr)
        return 2
    if not torch.cuda.is_available():
        print("no CUDA device", file=sys.stderr)
        return 3
    try:
        dev = torch.device("cuda", torch.cuda.current_device())
        if args.input:
            host = np.load(args.input)
            x = torch.from_numpy(np.ascontiguousarray(host.ravel())).to(dev)
            if str(x.dtype).replace("torch.", "") not in rd.DTYPE_NAMES:
                print(f"unsupported array dtype {host.dtype}", file=sys.stderr)
                return 2
        else:
            import inputs
            wl = args.workload or inputs.default_workload(args.dtype, args.op)
            if wl not in inputs.WORKLOADS or args.n < 0:
                print(f"unknown workload {wl!r} or n < 0", file=sys.stderr)
                return 2
            x = torch.empty(args.n, dtype=getattr(torch, args.dtype), device=dev)
            if args.n:
                inputs.fill_device(x, wl, seed=args.seed)
        rd.reduce(x, args.op)                     # warm-up (workspace, kernel load)
        torch.cuda.synchronize(dev)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = rd.reduce(x, args.op)
        b.record()
        torch.cuda.synchronize(dev)
        us = a.elapsed_time(b) * 1e3
        value = _scalar(r if not isinstance(r, tuple) else (r[0], r[1]))
        ok = True
        if args.check:
            ok = _check(rd, x, args.op, r)
    except rd.ReduceError as e:
        print(str(e), file=sys.stderr)
        return 2 if e.status in (1, 2, 3) else 3  # invalid / unsupported / misaligned: usage
    except (RuntimeError, OSError) as e:
        print(str(e), file=sys.stderr)
        return 3
    nbytes = x.numel() * x.element_size()
    if args.json:
        print(json.dumps({"op": args.op, "dtype": str(x.dtype).replace("torch.", ""), "n": x.numel(),
                          "result": value, "us": round(us, 3), "gbps": round(nbytes / us / 1e3, 2) if us else None,
                          "check": ("ok" if ok else "FAILED") if args.check else None}))
    else:
        print(value)
    return 0 if ok else 1


def _check(rd, x, op, r) -> bool:
    """Variants and a 4-way record split against the default result."""
    import numpy as np
    import torch

    def bits(t):
        if isinstance(t, tuple):
            return bits(t[0]) + bits(t[1])
        return t.detach().cpu().numpy().tobytes()

    got = [rd.reduce_ex(x, op, variant=v)[0] for v in ("vector", "bulk")]
    dt = str(x.dtype).replace("torch.", "")
    n = x.numel()
    if rd.OPS[op] == rd.OPS["sum_exact"] and x.is_floating_point():
        recs = torch.empty(4 * rd.EXACT_RECORD_BYTES, dtype=torch.uint8, device=x.device)
        for k in range(4):
            b, c = rd.shard_range(n, 4, k)
            rd.reduce_exact_partial(x[b:b + c], rec=recs[k * rd.EXACT_RECORD_BYTES:(k + 1) * rd.EXACT_RECORD_BYTES])
        got.append(rd.combine_exact_records(recs, dt))
    else:
        recs = torch.empty(4 * rd.RECORD_BYTES, dtype=torch.uint8, device=x.device)
        for k in range(4):
            b, c = rd.shard_range(n, 4, k)
            rd.reduce_partial(x[b:b + c], op, rec=recs[k * rd.RECORD_BYTES:(k + 1) * rd.RECORD_BYTES])
        got.append(rd.combine_records(recs, dt, op))
    exact_bits = (not x.is_floating_point()) or op in ("min", "max", "argmin", "argmax", "sum_exact")
    if exact_bits:
        return all(bits(g) == bits(r) for g in got)
    # float + / x: every evaluation order is a correct result; the
    # variants must agree within the stated bound of each other
    ref = float(r.item())
    vals = [float(g.item()) for g in got]
    if not math.isfinite(ref):
        return all((math.isnan(v) and math.isnan(ref)) or v == ref for v in vals)
    eps = float(np.finfo(np.dtype(dt)).eps)
    if op in ("sum", "sum_compensated"):
        scale = float(rd.reduce(torch.abs(x), "sum_compensated").item())   # sum |x_i| by this library
    else:
        scale = abs(ref)
    return all(abs(v - ref) <= 8 * eps * scale for v in vals)


if __name__ == "__main__":
    sys.exit(main())
