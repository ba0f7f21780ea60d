"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element for
element on the same seeded inputs. Needs a B200."""
from __future__ import annotations

import ctypes
import math

import numpy as np
import pytest

import inputs
import oracle
from tests import _brute, _parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

INT = ["int32", "uint32", "int64"]
FLT = ["float32", "float64"]
INT_OPS = ["sum", "prod", "min", "max", "and", "or", "xor"]
FLT_OPS = ["sum", "prod", "min", "max"]
EXTRA_OPS = ["argmin", "argmax", "sum_compensated", "sum_exact"]
PAIRS = [(d, o) for d in INT for o in INT_OPS + EXTRA_OPS] + [(d, o) for d in FLT for o in FLT_OPS + EXTRA_OPS]
SIZES = [0, 1, 2, 3, 7, 8, 9, 31, 32, 33, 255, 256, 257, 1023, 1025, 4097, 65535, 65537,
         (1 << 20) + 1, 5533214]


@pytest.fixture(scope="module")
def rd():
    from paper_1710_07358_b200.build import build_all
    build_all()
    import paper_1710_07358_b200 as m
    return m


def to_dev(x: np.ndarray, offset: int = 0):
    """Copy x to the GPU at an element offset from a 512-byte-aligned allocation."""
    dt = getattr(torch, x.dtype.name)
    carrier = {4: np.int32, 8: np.int64}[x.dtype.itemsize]
    buf = torch.empty(x.size + offset + 1, dtype=getattr(torch, np.dtype(carrier).name), device="cuda")
    if x.size:
        buf[offset:offset + x.size].copy_(torch.from_numpy(x.view(carrier)))
    return buf.view(dt)[offset:offset + x.size]


def val(t):
    """0-d CUDA tensor -> numpy scalar of the same dtype (bit-preserving);
    a (value, index) pair -> (numpy scalar, int)."""
    if isinstance(t, tuple):
        return val(t[0]), int(t[1].item())
    carrier = {4: torch.int32, 8: torch.int64}[t.element_size()]
    npdt = np.dtype(str(t.dtype).replace("torch.", ""))
    return np.array([t.view(carrier).item()], dtype=np.dtype(str(carrier).replace("torch.", ""))).view(npdt)[0]


# ------------------------------------------------------------------ C1
def test_c1_iota_int32_closed_form(rd):
    """BASELINE configs[0]: int32 sum of iota, n = 2^20 -> -524288 (= n(n-1)/2 mod 2^32)."""
    n = 1 << 20
    x = torch.empty(n, dtype=torch.int32, device="cuda")
    inputs.fill_device(x, "iota")
    assert int(val(rd.reduce(x, "sum"))) == -524288
    for seed in (1, 2, 3):
        xh = inputs.generate(n, "int32", "uniform_bits", seed=seed)
        _parity.check(val(rd.reduce(to_dev(xh), "sum")), xh, "sum")


# ------------------------------------------------------------------ C3/C4 matrix
@pytest.mark.parametrize("dtype,op", PAIRS, ids=[f"{d}-{o}" for d, o in PAIRS])
def test_matrix_sizes(rd, dtype, op):
    wl = inputs.default_workload(dtype, op)
    for n in SIZES:
        x = inputs.generate(n, dtype, wl, seed=n % 7 + 1)
        _parity.check(val(rd.reduce(to_dev(x), op)), x, op)


@pytest.mark.parametrize("dtype,op", PAIRS, ids=[f"{d}-{o}" for d, o in PAIRS])
def test_misaligned_bases(rd, dtype, op):
    """C4: element offsets 0..7 from an aligned allocation (head + body + tail)."""
    wl = inputs.default_workload(dtype, op)
    for n in (5, 13, 1000, 100003):
        x = inputs.generate(n, dtype, wl, seed=11)
        for off in range(8):
            _parity.check(val(rd.reduce(to_dev(x, off), op)), x, op)


@pytest.mark.parametrize("dtype,op", PAIRS, ids=[f"{d}-{o}" for d, o in PAIRS])
def test_bulk_variant_all_pairs(rd, dtype, op):
    """The bulk-copy pipeline (AUTO's choice for large inputs) on every pair, at
    sizes with partial stages/chunks and misaligned bases, forced on small n too."""
    wl = inputs.default_workload(dtype, op)
    for n in (0, 1, 7, 4099, 65536 + 3, (1 << 21) + 1, (1 << 23) + 5):
        x = inputs.generate(n, dtype, wl, seed=n % 3 + 1)
        for off in (0, 1):
            out, info = rd.reduce_ex(to_dev(x, off), op, variant="bulk")
            assert info["variant"] == "bulk"
            _parity.check(val(out), x, op)


def test_auto_planner_choice(rd):
    """The AUTO plan: one CTA up to 32 KB, one cluster of <= 16 CTAs
    up to 1 MiB, the vector grid (capped at 2 CTAs/SM from 12 MiB, the occupancy grid from
    48 MiB) below 128 MiB, the bulk ring from 128 MiB."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count

    def plan(nbytes):
        x = torch.zeros(nbytes // 4, dtype=torch.float32, device="cuda")
        return rd.reduce_ex(x, "sum")[1]

    p = plan(16 << 10)
    assert p["variant"] == "vector" and p["grid"] == 1
    p = plan(256 << 10)
    assert p["variant"] == "cluster" and 2 <= p["grid"] <= 16
    p = plan(1 << 20)
    assert p["variant"] == "cluster" and p["grid"] == 16
    assert plan(4 << 20)["variant"] == "vector"
    p = plan(16 << 20)
    assert p["variant"] == "vector" and p["grid"] == 2 * sms
    p = plan(64 << 20)
    assert p["variant"] == "vector" and p["grid"] == sms * p["ctas_per_sm"] and p["ctas_per_sm"] >= 2
    assert plan(128 << 20)["variant"] == "bulk"
    small = to_dev(inputs.generate(1 << 20, "float32", "u01"))
    assert rd.reduce_ex(small, "sum")[1]["variant"] == "vector"


@pytest.mark.parametrize("dtype,op", [("float32", "sum"), ("int64", "prod"), ("float64", "max"),
                                      ("uint32", "min"), ("float64", "prod"), ("int32", "xor")])
def test_forced_grids(rd, dtype, op):
    """a6 ticket combine for any grid size, including 1 (no ticket) and the cap."""
    wl = inputs.default_workload(dtype, op)
    x = inputs.generate((1 << 20) + 5, dtype, wl, seed=5)
    xd = to_dev(x, 3)
    for variant in ("vector", "bulk"):
        for g in (1, 2, 3, 7, 148, 593, 1000, 4096):
            out, info = rd.reduce_ex(xd, op, variant=variant, grid=g)
            assert info["grid"] == g
            _parity.check(val(out), x, op)


@pytest.mark.parametrize("dtype", ["float32", "int32"])
def test_ablation_configs(rd, dtype):
    """Every compiled configuration of the loads-in-flight sweep (Table 2 on B200)."""
    wl = "u01" if dtype == "float32" else "uniform_bits"
    x = inputs.generate(5533214, dtype, wl, seed=2)
    for off in (0, 1):
        xd = to_dev(x, off)
        for vb in (4, 8, 16, 32):
            for u in (1, 2, 3, 4, 5, 6, 7, 8, 16):
                out, info = rd.reduce_ex(xd, "sum", variant="vector", unroll=u, vec_bytes=vb)
                assert (info["unroll"], info["vec_bytes"]) == (u, vb)
                _parity.check(val(out), x, "sum")
        for f in (1, 2, 3, 4, 5, 6, 7, 8, 16):
            out, info = rd.reduce_ex(xd, "sum", variant="paper", unroll=f)
            assert info["variant"] == "paper" and info["unroll"] == f
            _parity.check(val(out), x, "sum")
        for st, sb in BULK_CONFIGS:
            out, info = rd.reduce_ex(xd, "sum", variant="bulk", unroll=st, vec_bytes=sb)
            assert info["variant"] == "bulk"
            _parity.check(val(out), x, "sum")


BULK_CONFIGS = [(4, 32768), (6, 32768), (3, 65536), (12, 16384), (8, 16384), (6, 16384), (24, 8192),
                (3, 32768), (5, 32768), (2, 65536), (4, 49152)]


@pytest.mark.parametrize("dtype", ["float32", "int32"])
def test_bulk_variant_sizes_and_alignment(rd, dtype):
    """Bulk-copy pipeline: partial stages, partial chunks, empty body, head/tail,
    and deterministic results (the per-chunk tree does not depend on scheduling)."""
    wl = "normalish" if dtype == "float32" else "uniform_bits"
    for n in (0, 1, 3, 4, 5, 17, 1000, 8191, 8193, 65536 + 5, (1 << 20) + 3, 5533214, (1 << 26) + 7):
        x = inputs.generate(n, dtype, wl, seed=n % 5 + 1)
        for off in (0, 1, 3):
            xd = to_dev(x, off)
            for st, sb in BULK_CONFIGS[:2] + BULK_CONFIGS[-1:]:
                outs = set()
                for rep in range(3):
                    out, info = rd.reduce_ex(xd, "sum", variant="bulk", unroll=st, vec_bytes=sb)
                    outs.add(val(out).tobytes())
                    _parity.check(val(out), x, "sum")
                assert len(outs) == 1, "bulk variant must be deterministic"


# ------------------------------------------------------------------ special values
@pytest.mark.parametrize("prec", FLT)
def test_absorption_example(rd, prec):
    """P:50 fn 2: 1.5 + 4^50 - 4^50 is 0 or 1.5 depending on the order; the GPU
    returns one of the tree results for every ordering and alignment."""
    big = 4.0 ** 50
    for order in ([1.5, big, -big], [big, -big, 1.5], [big, 1.5, -big]):
        x = np.array(order, dtype=prec)
        for off in range(4):
            g = float(val(rd.reduce(to_dev(x, off), "sum")))
            assert g in {0.0, 1.5}
            _parity.check(g, x, "sum")


@pytest.mark.parametrize("prec", FLT)
def test_small_n_float_sum_is_a_tree_result(rd, prec):
    """n <= 8: several results are correct (every evaluation tree); the
    GPU's must be one of them (set membership by brute force) -- trees whose nodes
    round to the element precision (block trees) or to the wide accumulator."""
    rng = np.random.default_rng(1)
    for n in range(1, 9):
        for trial in range(8):
            x = (rng.standard_normal(n) * 10.0 ** rng.integers(-3, 4, n)).astype(prec)
            trees = _brute.mixed_tree_results(list(x), prec)
            for off in (0, 3):
                g = float(val(rd.reduce(to_dev(x, off), "sum")))
                assert g in trees, (n, trial, off)


# ------------------------------------------------------------------ chain-order adversary
# with per-lane input-precision accumulators, an input that puts
# 1.0 at the head of every lane chain followed by 0.51-ulp(1) terms (each rounds up by
# 0.49 ulp) missed 4 eps sum|x| by up to 7x. The default sum now sums each thread's
# block of <= 32 loaded elements as a tree and adds block sums into fp64 / double-double
# (include/b200reduce.h), so the bound holds whatever the values.
def _bulk_chunks(body_bytes, s, stage=32768):
    """Chunk starts (body byte offsets) of the bulk schedule (rd_api.cu plan_bulk, plain ops)."""
    T = body_bytes
    C1 = stage
    R = min(T, 148 * 16 * C1)
    c0 = max(T // (148 * 16), T // 5000)
    c0 = (c0 + stage - 1) // stage * stage
    c0 = max(c0, 4 * stage)
    starts = list(range(0, T - R, c0)) + list(range(T - R, T, C1))
    return starts


def _chain_adversary(rd, n, prec, op, off):
    tiny = np.array([0.51 * float(np.finfo(prec).eps)], dtype=prec)[0]
    s = np.dtype(prec).itemsize
    _, info = rd.reduce_ex(to_dev(np.zeros(n, prec), off), op)
    x = np.full(n, tiny, dtype=prec)
    h = info["head"]
    if info["variant"] == "bulk":
        for c in _bulk_chunks(info["nvec"] * 16, s):
            e = h + c // s
            x[e:e + 256 * 16 // s] = 1.0          # every consumer thread's first vector of the chunk
    else:                                          # vector / cluster: the grid's first pass
        x[h:h + info["grid"] * 256 * 32 // s] = 1.0
    return x, info


ADV = [("float32", 1 << 17), ("float32", 1 << 22), ("float32", 1 << 24), ("float32", 1 << 26),
       ("float32", 1 << 28), ("float64", 1 << 16), ("float64", 1 << 21), ("float64", 1 << 23),
       ("float64", 1 << 25), ("float64", 1 << 27)]


@pytest.mark.parametrize("prec,n", ADV, ids=[f"{p}-2^{n.bit_length() - 1}" for p, n in ADV])
@pytest.mark.parametrize("op", ["sum", "sum_compensated"])
def test_chain_order_adversary(rd, prec, n, op):
    """The north-star bound 4 eps sum|x| on the chain-order adversary, through the AUTO
    planner's variant (cluster at 512 KB, vector at 16-64 MB, bulk at >= 256 MB), at an
    aligned and a misaligned base; the measured error must stay under the derived 3 eps."""
    for off in (0, 3):
        x, info = _chain_adversary(rd, n, prec, op, off)
        g = val(rd.reduce(to_dev(x, off), op))
        r = _parity.check(g, x, op)
        assert abs(float(g) - r.exact) <= 3.01 * _parity.EPS[prec] * r.sum_abs, info["variant"]


@pytest.mark.parametrize("prec", FLT)
def test_chain_order_adversary_forced_variants(rd, prec):
    """The same adversary (laid out for each variant's own schedule) on the vector and bulk
    kernels forced at one size, and on grids the planner does not pick."""
    n = (1 << 22) + 5 if prec == "float32" else (1 << 21) + 3
    tiny = np.array([0.51 * float(np.finfo(prec).eps)], dtype=prec)[0]
    s = np.dtype(prec).itemsize
    for variant, grid in (("vector", 0), ("vector", 1), ("vector", 4096), ("bulk", 0), ("bulk", 7)):
        _, info = rd.reduce_ex(to_dev(np.zeros(n, prec), 1), "sum", variant=variant, grid=grid)
        x = np.full(n, tiny, dtype=prec)
        h = info["head"]
        if variant == "bulk":
            for c in _bulk_chunks(info["nvec"] * 16, s):
                x[h + c // s:h + c // s + 256 * 16 // s] = 1.0
        else:
            x[h:h + info["grid"] * 256 * 32 // s] = 1.0
        out, _ = rd.reduce_ex(to_dev(x, 1), "sum", variant=variant, grid=grid)
        r = _parity.check(val(out), x, "sum")
        assert abs(float(val(out)) - r.exact) <= 3.01 * _parity.EPS[prec] * r.sum_abs, (variant, grid)


@pytest.mark.parametrize("prec", FLT)
def test_block_tree_worst_case(rd, prec):
    """Every 32-element block tree at its worst: 1.0 then 31 tiny terms in each block
    (and the reverse), so every block sum rounds, at vector, cluster and bulk sizes."""
    tiny = np.array([0.51 * float(np.finfo(prec).eps)], dtype=prec)[0]
    for n in (1 << 16, 1 << 20, (1 << 25) + 7):
        for first in (True, False):
            x = np.full(n, tiny, dtype=prec)
            if first:
                x[::32] = 1.0
            else:
                x[31::32] = 1.0
            r = _parity.check(val(rd.reduce(to_dev(x, 2), "sum")), x, "sum")


@pytest.mark.parametrize("prec", FLT)
def test_minmax_special_values(rd, prec):
    """IEEE minimum/maximum (NaN propagates, -0 < +0), bit-exact, in head, body and tail."""
    dom = [0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, 1e-45, -2.5]
    import itertools
    for k in (1, 2, 3):
        for combo in itertools.product(dom, repeat=k):
            x = np.array(combo, dtype=prec)
            for op in ("min", "max"):
                _parity.check(val(rd.reduce(to_dev(x, 1), op)), x, op)
    rng = np.random.default_rng(3)
    base = inputs.generate(100000, prec, "u01", seed=3) + 1
    for v in dom:
        for pos in (0, 5, 777, 50000, 99999):
            x = base.copy()
            x[pos] = v
            x[rng.integers(0, x.size)] = -0.0 if v == 0.0 else x[0]
            for op in ("min", "max"):
                _parity.check(val(rd.reduce(to_dev(x, pos % 8), op)), x, op)


@pytest.mark.parametrize("prec", FLT)
def test_signed_zero_and_nonfinite_sums(rd, prec):
    """Padding uses -0.0 (the additive identity): an all -0.0 input sums to -0.0
    at every size; empty input gives +0.0; inf/NaN classes follow IEEE."""
    for n in (1, 2, 9, 100, 4099, 1 << 20):
        x = np.full(n, -0.0, dtype=prec)
        g = val(rd.reduce(to_dev(x, n % 5), "sum"))
        assert _parity.to_bits(g, prec) == _parity.to_bits(-0.0, prec)
    g = val(rd.reduce(to_dev(np.zeros(0, prec)), "sum"))
    assert _parity.to_bits(g, prec) == _parity.to_bits(0.0, prec)
    # near-one data: no partial product under/overflows in any order, so the
    # class of the result (inf / NaN) is order-independent
    base = inputs.generate(10000, prec, "near_one", seed=4)
    for a, b in [(math.inf, 1.0), (math.inf, -math.inf), (math.nan, 0.0), (-math.inf, 2.0)]:
        x = base.copy()
        x[17], x[9000] = a, b
        for op in ("sum", "prod"):
            _parity.check(val(rd.reduce(to_dev(x, 2), op)), x, op)
    x = base.copy()
    x[123] = 0.0
    _parity.check(val(rd.reduce(to_dev(x), "prod")), x, "prod")


@pytest.mark.parametrize("dtype", INT)
def test_integer_wraparound(rd, dtype):
    """+ and x wrap mod 2^w; min/max respect signedness (values near the extremes)."""
    info = np.iinfo(dtype)
    x = np.array([info.max, 1, info.max, info.min, 3, -1 if dtype != "uint32" else 7] * 1001,
                 dtype=dtype)
    for op in INT_OPS:
        _parity.check(val(rd.reduce(to_dev(x, 1), op)), x, op)


# ------------------------------------------------------------------ generator twin
@pytest.mark.parametrize("dtype", INT + FLT)
def test_device_generator_matches_host(rd, dtype):
    for wl in inputs.WORKLOADS:
        try:
            h = inputs.generate(100003, dtype, wl, seed=9, offset=12345, n_total=10 ** 7)
        except ValueError:
            continue
        d = torch.empty(100003, dtype=getattr(torch, dtype), device="cuda")
        inputs.fill_device(d, wl, seed=9, offset=12345, n_total=10 ** 7)
        assert d.cpu().numpy().tobytes() == h.tobytes(), wl


# ------------------------------------------------------------------ determinism, graphs, streams
_ENV_SCRIPT = r"""
import sys, torch, numpy as np
sys.path.insert(0, sys.argv[1])
import inputs, paper_1710_07358_b200 as rd
out = []
for dt, n, op in (("float32", (1 << 26) + 3, "sum"), ("float64", (1 << 24) + 1, "sum"),
                  ("float32", 1 << 22, "sum"), ("float32", (1 << 25) + 5, "sum_exact"),
                  ("float64", (1 << 22) + 7, "sum_exact"), ("float32", (1 << 26) + 1, "argmin")):
    x = torch.empty(n, dtype=getattr(torch, dt), device="cuda")
    inputs.fill_device(x, "normalish", seed=5)
    r = rd.reduce(x, op)
    r = r if isinstance(r, tuple) else (r,)
    out.append(",".join(bytes(t.reshape(1).view(torch.uint8).cpu().numpy()).hex() for t in r))
    out.append(repr(rd.reduce_ex(x, op)[1]))
print("|".join(out))
"""


def test_environment_does_not_change_results(rd, tmp_path):
    """identical (x, n, alignment, dtype, op, device) give identical
    bits whatever the environment -- the tuning knobs of RD_TUNING builds and a library
    path override are ignored by the shipped library and its binding."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = tmp_path / "env_bits.py"
    script.write_text(_ENV_SCRIPT)
    base = dict(os.environ)
    for k in list(base):
        if k.startswith("RD_"):
            del base[k]
    tuned = dict(base, RD_TUNE_HEAD_PER_SM="3", RD_TUNE_TAIL_PER_SM="1", RD_TUNE_TAIL_STAGES="4",
                 RD_TUNE_VEC_CTAS_PER_SM="1000", RD_TUNE_EXACT="4,2,2", RD_TUNE_EXACT_BULK="8,2",
                 RD_LIB_PATH="/nonexistent/lib.so")
    outs = [subprocess.run([sys.executable, str(script), root], env=e, capture_output=True, text=True,
                           timeout=600) for e in (base, tuned)]
    for o in outs:
        assert o.returncode == 0, o.stderr[-2000:]
    assert outs[0].stdout == outs[1].stdout


def test_determinism(rd):
    x = torch.empty(1 << 24, dtype=torch.float32, device="cuda")
    inputs.fill_device(x, "normalish", seed=2)
    a = [val(rd.reduce(x, "sum")).tobytes() for _ in range(5)]
    assert len(set(a)) == 1


def test_cuda_graph_capture(rd):
    n = (1 << 22) + 3
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    inputs.fill_device(x, "u01", seed=5)
    s = torch.cuda.Stream()
    out = torch.empty((), dtype=torch.float64, device="cuda")
    with torch.cuda.stream(s):
        rd.reduce(x, "sum", out=out)            # creates the stream's workspace outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rd.reduce(x, "sum", out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    _parity.check(val(out), x.cpu().numpy(), "sum")


def test_concurrent_streams(rd):
    """Separate per-stream workspaces: concurrent reductions do not interfere."""
    xs = [inputs.generate((1 << 21) + i, "int64", "uniform_bits", seed=i) for i in range(4)]
    ds = [to_dev(x) for x in xs]
    streams = [torch.cuda.Stream() for _ in xs]
    outs = []
    for rep in range(3):
        outs = []
        for d, s in zip(ds, streams):
            with torch.cuda.stream(s):
                outs.append(rd.reduce(d, "sum"))
        torch.cuda.synchronize()
        for o, x in zip(outs, xs):
            _parity.check(val(o), x, "sum")


# ------------------------------------------------------------------ records / sharding
@pytest.mark.parametrize("dtype,op", [("float32", "sum"), ("float64", "sum"), ("int64", "prod"),
                                      ("float64", "prod"), ("float32", "max"), ("uint32", "and"),
                                      ("int32", "min"), ("float32", "prod")])
def test_shard_records_combine(rd, dtype, op):
    """Split one logical array into W contiguous shards (rd_shard_range), reduce
    each to a record, fold the records in rank order: parity with the oracle on
    the whole array (the exchange step of reduce_multi, without the transport)."""
    n = (1 << 22) + 3
    wl = inputs.default_workload(dtype, op)
    x = inputs.generate(n, dtype, wl, seed=7)
    xd = to_dev(x)
    for W in (1, 2, 3, 8, 17):
        recs = torch.empty(W * 32, dtype=torch.uint8, device="cuda")
        for r in range(W):
            b, c = rd.shard_range(n, W, r)
            rd.reduce_partial(xd[b:b + c], op, rec=recs[r * 32:(r + 1) * 32])
        out = rd.combine_records(recs, dtype, op)
        _parity.check(val(out), x, op)


def test_record_mismatch_detected(rd):
    x = to_dev(inputs.generate(1000, "float32", "u01"))
    recs = torch.empty(64, dtype=torch.uint8, device="cuda")
    rd.reduce_partial(x, "sum", rec=recs[:32])
    rd.reduce_partial(x, "max", rec=recs[32:])
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = rd.combine_records(recs, "float32", "sum", status=status)
    assert int(status.item()) == 6
    assert float(val(out)) == 0.0


def test_empty_shards(rd):
    recs = torch.empty(3 * 32, dtype=torch.uint8, device="cuda")
    x = inputs.generate(100, "float32", "u01")
    xd = to_dev(x)
    rd.reduce_partial(xd[:0], "sum", rec=recs[0:32])
    rd.reduce_partial(xd, "sum", rec=recs[32:64])
    rd.reduce_partial(xd[:0], "sum", rec=recs[64:96])
    _parity.check(val(rd.combine_records(recs, "float32", "sum")), x, "sum")


# ------------------------------------------------------------------ host entry point
@pytest.mark.parametrize("dtype,op", [("float32", "sum"), ("int32", "xor"), ("float64", "prod"),
                                      ("int64", "max"), ("uint32", "sum")])
def test_reduce_host(rd, dtype, op):
    n = (1 << 25) + 7   # several 32 MiB chunks
    wl = inputs.default_workload(dtype, op)
    x = inputs.generate(n, dtype, wl, seed=3)
    _parity.check(rd.reduce_host(x, op), x, op)                 # pageable
    pinned = torch.from_numpy(x.view({4: np.int32, 8: np.int64}[x.itemsize])).pin_memory()
    pinned = pinned.view(getattr(torch, dtype))
    _parity.check(rd.reduce_host(pinned, op), x, op)            # pinned
    for m in (0, 1, 5):
        _parity.check(rd.reduce_host(x[:m], op), x[:m], op)


# ------------------------------------------------------------------ NCCL path (1 rank)
def test_reduce_multi_single_rank(rd):
    from paper_1710_07358_b200 import _lib
    L = _lib.lib()
    uid = _lib.rd_unique_id()
    assert L.rd_get_unique_id(ctypes.byref(uid)) == 0
    h = ctypes.c_void_p()
    assert L.rd_comm_init(ctypes.byref(h), 1, 0, ctypes.byref(uid), torch.cuda.current_device()) == 0
    comm = rd.Comm(h.value, 1, 0, torch.cuda.current_device())
    try:
        for dtype, op in [("float32", "sum"), ("int32", "xor"), ("float64", "min")]:
            x = inputs.generate((1 << 20) + 9, dtype, inputs.default_workload(dtype, op), seed=1)
            _parity.check(val(comm.reduce(to_dev(x, 1), op)), x, op)
        comm.check()
    finally:
        comm.destroy()


# ------------------------------------------------------------------ full BASELINE sizes
def _device_input(n, dtype, wl, seed):
    x = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
    inputs.fill_device(x, wl, seed=seed)
    return x


@pytest.mark.parametrize("dtype", FLT)
@pytest.mark.parametrize("wl", ["u01", "normalish"])
def test_c2_full_size(rd, dtype, wl):
    """BASELINE configs[1]: float32 / float64 sum, n = 2^28, seeds 1-3, vs the fp64 oracle."""
    n = 1 << 28
    for seed in (1, 2, 3):
        x = _device_input(n, dtype, wl, seed)
        g = val(rd.reduce(x, "sum"))
        xh = x.cpu().numpy()
        del x
        _parity.check(g, xh, "sum")


def test_c2_exact_variants(rd):
    """Inputs whose sum is exact in any order: the GPU must return it bit-exactly."""
    n = 1 << 28
    x = _device_input(n, "float64", "int_small", 1)
    xi = _device_input(n, "int64", "int_small", 1)
    assert float(val(rd.reduce(x, "sum"))) == float(int(val(rd.reduce(xi, "sum"))))
    del x, xi
    x = _device_input(n, "float32", "sparse_pm1", 2)
    xi = _device_input(n, "int32", "sparse_pm1", 2)
    assert float(val(rd.reduce(x, "sum"))) == float(int(val(rd.reduce(xi, "sum"))))
    for prec in FLT:
        x = _device_input(n, prec, "pow2_sparse", 3)
        e = int((x == 2).sum().item()) - int((x == 0.5).sum().item())
        assert float(val(rd.reduce(x, "prod"))) == 2.0 ** e


@pytest.mark.parametrize("dtype", INT)
def test_closed_forms_2_30(rd, dtype):
    """iota at n = 2^30 (4-8 GiB): n(n-1)/2 mod 2^w, xor closed form, min/max."""
    n = 1 << 30
    x = _device_input(n, dtype, "iota", 1)
    w = 64 if dtype == "int64" else 32
    s = (n * (n - 1) // 2) % (1 << w)
    assert int(val(rd.reduce(x, "sum"))) & ((1 << w) - 1) == s
    assert int(val(rd.reduce(x, "xor"))) == [n - 1, 1, n, 0][(n - 1) % 4]
    assert int(val(rd.reduce(x, "min"))) == 0
    assert int(val(rd.reduce(x, "max"))) == n - 1


@pytest.mark.parametrize("dtype,op", [("float32", "sum"), ("int32", "sum"), ("float32", "max"),
                                      ("int32", "prod")])
def test_c3_2_30_vs_oracle(rd, dtype, op):
    """C3's largest size, n = 2^30, against the oracle on the whole array."""
    n = 1 << 30
    x = _device_input(n, dtype, inputs.default_workload(dtype, op), 1)
    g = val(rd.reduce(x, op))
    xh = x.cpu().numpy()
    del x
    _parity.check(g, xh, op)


def test_c5_sharded_layout_on_one_gpu(rd):
    """BASELINE configs[4] layout (float32 sum and max, sharded over W = 8 ranks)
    at n = 2^30 on one GPU: shard records folded in rank order == oracle."""
    n, W = 1 << 30, 8
    for op, wl in (("sum", "u01"), ("max", "planted")):
        x = _device_input(n, "float32", wl, 1)
        recs = torch.empty(W * 32, dtype=torch.uint8, device="cuda")
        for r in range(W):
            b, c = rd.shard_range(n, W, r)
            rd.reduce_partial(x[b:b + c], op, rec=recs[r * 32:(r + 1) * 32])
        g = val(rd.combine_records(recs, "float32", op))
        xh = x.cpu().numpy()
        del x
        _parity.check(g, xh, op)
        if op == "max":
            assert float(g) == 2.0 ** 20


# ------------------------------------------------------------------ f4: argmin / argmax
@pytest.mark.parametrize("prec", FLT)
def test_arg_ops_special_values(rd, prec):
    """Reading R6: NaN first (index of the first NaN), -0 < +0, lowest index on ties,
    in head, body and tail positions, for both kernel variants."""
    import itertools
    dom = [0.0, -0.0, 1.0, -1.0, math.inf, -math.inf, math.nan, 2.5]
    for k in (1, 2, 3):
        for combo in itertools.product(dom, repeat=k):
            x = np.array(combo, dtype=prec)
            for op in ("argmin", "argmax"):
                _parity.check(val(rd.reduce(to_dev(x, 1), op)), x, op)
    base = np.full(100003, 7.0, dtype=prec)
    for v in dom:
        for pos in (0, 3, 777, 50000, 100002):
            x = base.copy()
            x[pos] = v
            x[(pos * 7 + 13) % x.size] = v          # a tie later (or earlier) in the array
            for op in ("argmin", "argmax"):
                for variant in ("vector", "bulk"):
                    got = val(rd.reduce_ex(to_dev(x, pos % 4), op, variant=variant)[0])
                    _parity.check(got, x, op)


@pytest.mark.parametrize("prec", FLT)
def test_arg_ops_group_ties_and_zeros(rd, prec):
    """The group-best fold (rd_ops.cuh LaneOps): the best of a group of <= 8 elements by
    FMNMX, an improvement located at the group's FIRST position holding it, ties kept at
    the earliest group; a zero best (-0 vs +0, unordered by fmin/fmax) and NaN groups
    take the key path. Ties inside one vector, across vectors of one group, across
    groups of one thread and across threads, at every alignment, both variants."""
    rng = np.random.default_rng(7)
    n = 300007
    cases = []
    x = rng.uniform(-1, 1, n).astype(prec)
    for pos in ([5, 6], [8, 15], [64, 65, 70], [1000, 1003, 200000], [n - 3, n - 1]):
        y = x.copy()
        y[pos] = 3.0                                  # the max, tied
        z = y.copy()
        z[pos] = -3.0                                 # the min, tied
        cases += [y, z]
    zeros = np.full(n, -1.0, dtype=prec)              # max is a zero: -0 at 10, +0 at 90000
    zeros[10] = -0.0
    zeros[90000] = 0.0
    cases.append(zeros)
    zneg = np.full(n, 1.0, dtype=prec)                # min is a zero: +0 at 7, -0 at 5000
    zneg[7] = 0.0
    zneg[5000] = -0.0
    cases.append(zneg)
    only_negz = np.full(n, -0.0, dtype=prec)          # every element -0: index 0
    cases.append(only_negz)
    mixed0 = np.where(rng.random(n) < 0.5, 0.0, -0.0).astype(prec)
    cases.append(mixed0)
    nan_late = x.copy()
    nan_late[123456] = np.nan
    nan_late[123457] = np.nan
    cases.append(nan_late)
    for c in cases:
        for op in ("argmin", "argmax"):
            for off in (0, 1, 3):
                for variant in ("auto", "vector", "bulk"):
                    got = val(rd.reduce_ex(to_dev(c, off), op, variant=variant)[0])
                    _parity.check(got, c, op)


@pytest.mark.parametrize("dtype", INT + FLT)
def test_arg_ops_sharded_records(rd, dtype):
    """Shard records carry block-local indices; rd_combine_records shifts them by
    the elements of the records before (rank order) -> global index."""
    n = (1 << 22) + 9
    for op in ("argmin", "argmax"):
        x = inputs.generate(n, dtype, inputs.default_workload(dtype, op), seed=2)
        xd = to_dev(x)
        for W in (1, 2, 5, 8):
            recs = torch.empty(W * 32, dtype=torch.uint8, device="cuda")
            for r in range(W):
                b, c = rd.shard_range(n, W, r)
                rd.reduce_partial(xd[b:b + c], op, rec=recs[r * 32:(r + 1) * 32])
            _parity.check(val(rd.combine_records(recs, dtype, op)), x, op)


def test_arg_ops_full_size(rd):
    """2^28 float32 with the planted extremes: the planted indices come back."""
    n = 1 << 28
    x = _device_input(n, "float32", "planted", 4)
    pmax, pmin = inputs.planted_positions(4, n)
    v, i = val(rd.reduce(x, "argmax"))
    assert (float(v), i) == (2.0 ** 20, pmax)
    v, i = val(rd.reduce(x, "argmin"))
    assert (float(v), i) == (-(2.0 ** 20), pmin)
    xh = x.cpu().numpy()
    del x
    xd = _device_input(n, "float32", "u01", 5)   # 2^24-point grid: the extremes are tied
    for op in ("argmin", "argmax"):
        _parity.check(val(rd.reduce(xd, op)), xd.cpu().numpy(), op)
    del xh


# ------------------------------------------------------------------ f2: compensated sum
@pytest.mark.parametrize("dtype", FLT)
@pytest.mark.parametrize("wl", ["u01", "normalish"])
def test_compensated_sum_full_size(rd, dtype, wl):
    """n = 2^28: within 1/2 ulp + 4 u_acc sum|x| of the exact sum, and equal to the
    oracle's correctly rounded value; identical bits across kernel variants, grids
    and a sharded evaluation (reproducible in practice)."""
    n = 1 << 28
    x = _device_input(n, dtype, wl, 1)
    g = val(rd.reduce(x, "sum_compensated"))
    variants = {val(rd.reduce_ex(x, "sum_compensated", variant=v, grid=gr)[0]).tobytes()
                for v, gr in (("vector", 0), ("vector", 1000), ("bulk", 0), ("bulk", 37))}
    recs = torch.empty(8 * 32, dtype=torch.uint8, device="cuda")
    for r in range(8):
        b, c = rd.shard_range(n, 8, r)
        rd.reduce_partial(x[b:b + c], "sum_compensated", rec=recs[r * 32:(r + 1) * 32])
    variants.add(val(rd.combine_records(recs, dtype, "sum_compensated")).tobytes())
    xh = x.cpu().numpy()
    del x
    ref = _parity.check(g, xh, "sum_compensated")
    assert g.tobytes() == np.array([ref.value]).astype(dtype).tobytes()
    assert variants == {g.tobytes()}


# ------------------------------------------------------------------ f1: fused exchange
@pytest.mark.parametrize("W", [1, 2, 3, 8])
def test_fused_exchange_local_ranks(rd, W):
    """reduce_fused with W virtual ranks on one GPU (mailboxes connected by
    pointer, kernels on W concurrent streams): every rank returns the identical
    result, equal to the oracle on the whole array, over several epochs (the
    epoch-parity double buffering) and for plain, compensated, exact and arg ops."""
    comms = rd.FusedComm.local(W, torch.cuda.current_device())
    streams = [torch.cuda.Stream() for _ in range(W)]
    try:
        cases = [("float32", "sum", (1 << 20) + 7), ("float64", "argmax", 100003), ("int32", "xor", 5533214),
                 ("float64", "prod", (1 << 16) + 1), ("float32", "sum_compensated", 1 << 25), ("int64", "min", 7),
                 ("float32", "sum_exact", (1 << 20) + 7), ("float64", "sum_exact", (1 << 25) + 3)]
        for rep in range(3):
            for dtype, op, n in cases:
                x = inputs.generate(n, dtype, inputs.default_workload(dtype, op), seed=rep + 1)
                xd = to_dev(x, 1)
                outs = []
                for r in range(W):
                    b, c = rd.shard_range(n, W, r)
                    with torch.cuda.stream(streams[r]):
                        outs.append(comms[r].reduce(xd[b:b + c], op))
                torch.cuda.synchronize()
                for r in range(W):
                    comms[r].check(streams[r])
                vals = [val(o) for o in outs]
                for v in vals:
                    assert repr(v) == repr(vals[0])
                _parity.check(vals[0], x, op)
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()


def test_fused_exchange_mismatch_and_timeout(rd):
    comms = rd.FusedComm.local(2, torch.cuda.current_device())
    streams = [torch.cuda.Stream() for _ in range(2)]
    try:
        x = to_dev(inputs.generate(1000, "float32", "u01"))
        with torch.cuda.stream(streams[0]):
            comms[0].reduce(x, "sum")
        with torch.cuda.stream(streams[1]):
            comms[1].reduce(x, "max")
        torch.cuda.synchronize()
        for r in range(2):
            with pytest.raises(rd.ReduceError) as e:
                comms[r].check(streams[r])
            assert e.value.status == 6
        # rank 1 never calls: rank 0 gives up (RD_ERR_TIMEOUT) instead of hanging
        with torch.cuda.stream(streams[0]):
            comms[0].reduce(x, "sum")
        torch.cuda.synchronize()
        with pytest.raises(rd.ReduceError) as e:
            comms[0].check(streams[0])
        assert e.value.status == 7
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()


# ------------------------------------------------------------------ every pair at BASELINE's 2^28
@pytest.mark.parametrize("dtype,op", PAIRS, ids=[f"{d}-{o}" for d, o in PAIRS])
def test_all_pairs_full_size_2_28(rd, dtype, op):
    """Each (dtype, op) at n = 2^28 through `reduce` (the AUTO planner picks the
    bulk-copy kernel bench.py times) vs the oracle on the whole array."""
    n = 1 << 28
    x = _device_input(n, dtype, inputs.default_workload(dtype, op), 7)
    g = val(rd.reduce(x, op))
    assert rd.reduce_ex(x, op)[1]["variant"] == "bulk"
    xh = x.cpu().numpy()
    del x
    _parity.check(g, xh, op)


def _oracle_stream(x_dev, op, chunk=1 << 28):
    """The oracle's left fold streamed over device chunks (fold(A); fold(B) ==
    fold(A ++ B), pinned in test_streaming_fold_equals_one_shot)."""
    f = oracle.Fold(str(x_dev.dtype).replace("torch.", ""), op)
    for s in range(0, x_dev.numel(), chunk):
        f.fold(x_dev[s:s + chunk].cpu().numpy())
    return f.result()


@pytest.mark.slow
def test_c5_full_size_2_34(rd):
    """BASELINE configs[4] at its real size on ONE GPU: n = 2^34 float32 (64 GiB
    of HBM), sum and max; the whole array in one call, and the 8-way shard
    layout through records. argmax exercises element indices >= 2^32."""
    free, _ = torch.cuda.mem_get_info()
    if free < (70 << 30):
        pytest.skip("needs 70 GiB of free HBM")
    n = 1 << 34
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    for op, wl in (("max", "planted"), ("sum", "u01"), ("argmax", "planted")):
        inputs.fill_device(x, wl, seed=1)
        whole = val(rd.reduce(x, op))
        recs = torch.empty(8 * 32, dtype=torch.uint8, device="cuda")
        for r in range(8):
            b, c = rd.shard_range(n, 8, r)
            rd.reduce_partial(x[b:b + c], op, rec=recs[r * 32:(r + 1) * 32])
        sharded = val(rd.combine_records(recs, "float32", op))
        if op == "max":
            assert float(whole) == float(sharded) == 2.0 ** 20
        elif op == "argmax":
            pmax, _ = inputs.planted_positions(1, n)
            assert whole == sharded == (np.float32(2.0 ** 20), pmax)
        else:
            ref = _oracle_stream(x, "sum")
            _parity.check(whole, np.zeros(0, np.float32), "sum", ref=ref)
            _parity.check(sharded, np.zeros(0, np.float32), "sum", ref=ref)
            # the exact sum (reading R17): one result for the whole array, the
            # 8-shard exact records and another grid (bit-exact parity with the
            # exact oracle is checked at 2^28; streaming it over 2^34 terms
            # would take ~10 min), inside the plain sum's 4 eps sum|x| bound
            RB = rd.EXACT_RECORD_BYTES
            xrecs = torch.empty(8 * RB, dtype=torch.uint8, device="cuda")
            for r in range(8):
                b, c = rd.shard_range(n, 8, r)
                rd.reduce_exact_partial(x[b:b + c], rec=xrecs[r * RB:(r + 1) * RB])
            ex = {val(rd.reduce(x, "sum_exact")).tobytes(), val(rd.combine_exact_records(xrecs, "float32")).tobytes(),
                  val(rd.reduce_ex(x, "sum_exact", grid=777)[0]).tobytes()}
            assert len(ex) == 1
            _parity.check(np.frombuffer(ex.pop(), np.float32)[0], np.zeros(0, np.float32), "sum", ref=ref)
    del x


@pytest.mark.slow
@pytest.mark.parametrize("dtype", ["float32", "int64"])
def test_indices_past_2_32_every_variant(rd, dtype):
    """Element indices >= 2^32 through each variant's own index arithmetic (vector:
    head + (tid + step*stride)*L + lane; bulk: chunk offset + stage step; cluster
    and forced small grids make the per-thread step counts large): n = 2^32 + 12345
    'planted' data with the extremes moved past 2^32, a TIE for the minimum (the
    lower index must win) and an odd base offset; argmax / argmin / max / min
    against these closed forms, every variant and two grids."""
    s = 4 if dtype == "float32" else 8
    free, _ = torch.cuda.mem_get_info()
    if free < ((1 << 32) + 20000) * s + (8 << 30):
        pytest.skip("needs ~%d GiB of free HBM" % (((1 << 32) * s >> 30) + 8))
    n = (1 << 32) + 12345
    buf = torch.empty(n + 1, dtype=getattr(torch, dtype), device="cuda")
    x = buf[1:]                                    # element-aligned, not vector-aligned
    inputs.fill_device(x, "planted", seed=2)
    hi, lo = (2.0 ** 21, -2.0 ** 21) if dtype == "float32" else (1 << 40, -5)
    i_max, i_min, i_min2 = (1 << 32) + 777, (1 << 32) + 999, (1 << 32) + 5000
    x[i_max] = hi
    x[i_min] = lo
    x[i_min2] = lo                                 # tie: the lower index wins
    npdt = np.float32 if dtype == "float32" else np.int64
    for variant, grid in (("auto", 0), ("vector", 0), ("vector", 37), ("bulk", 0), ("bulk", 5), ("cluster", 16)):
        got = {op: val(rd.reduce_ex(x, op, variant=variant, grid=grid)[0])
               for op in ("argmax", "argmin", "max", "min")}
        assert got["argmax"] == (npdt(hi), i_max), (variant, grid, got["argmax"])
        assert got["argmin"] == (npdt(lo), i_min), (variant, grid, got["argmin"])
        assert got["max"] == npdt(hi) and got["min"] == npdt(lo), (variant, grid, got)
    del buf, x


def test_c_program_through_the_abi(rd, tmp_path):
    """A plain C99 program (examples/reduce_example.c) drives the library: exact
    sum of ones, argmax tie -> index 0, and back-to-back reduce() calls."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = tmp_path / "reduce_example"
    subprocess.check_call(["gcc", "-std=c99", "-O2", os.path.join(root, "examples", "reduce_example.c"),
                           "-I", os.path.join(root, "include"), "-I", "/usr/local/cuda/include",
                           "-L", os.path.join(root, "paper_1710_07358_b200"), "-lb200reduce",
                           f"-Wl,-rpath,{os.path.join(root, 'paper_1710_07358_b200')}",
                           "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", str(exe)])
    for log2n in ("10", "24"):
        r = subprocess.run([str(exe), log2n], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr
        print(r.stdout)


def test_cuda_graph_capture_bulk_and_args(rd):
    """The bulk-copy kernel (>= 128 MiB), an arg op and a shard record, captured
    in one CUDA graph and replayed twice."""
    n = (1 << 25) + 3                         # 128 MiB + 12 B of float32 -> bulk
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    inputs.fill_device(x, "u01", seed=8)
    s = torch.cuda.Stream()
    out = torch.empty((), dtype=torch.float32, device="cuda")
    arg = torch.empty(2, dtype=torch.int64, device="cuda")
    rec = torch.empty(32, dtype=torch.uint8, device="cuda")
    with torch.cuda.stream(s):
        assert rd.reduce_ex(x, "sum", out=out)[1]["variant"] == "bulk"
        rd.reduce(x, "argmax", out=arg)
        rd.reduce_partial(x[1:], "max", rec=rec)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rd.reduce(x, "sum", out=out)
        rd.reduce(x, "argmax", out=arg)
        rd.reduce_partial(x[1:], "max", rec=rec)
    xh = x.cpu().numpy()
    for _ in range(2):
        out.zero_()
        arg.zero_()
        g.replay()
        torch.cuda.synchronize()
        _parity.check(val(out), xh, "sum")
        _parity.check(val(rd._arg_view(arg, torch.float32)), xh, "argmax")
        _parity.check(val(rd.combine_records(rec, "float32", "max")), xh[1:], "max")


def test_host_threads_concurrently(rd):
    """Several host threads, each with its own stream, call the library at once
    (ctypes releases the GIL; the workspace map is locked)."""
    import threading
    xs = [inputs.generate((1 << 20) + 17 * i, "int64", "uniform_bits", seed=i + 1) for i in range(6)]
    ds = [to_dev(x, i % 3) for i, x in enumerate(xs)]
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(40):
                    o = rd.reduce(ds[i], "sum" if rep % 2 else "xor")
                    if rep % 10 == 9:
                        s.synchronize()
                        _parity.check(val(o), xs[i], "sum" if rep % 2 else "xor")
        except Exception as e:  # surfaced below
            errors.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(xs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors


# ------------------------------------------------------------------ cluster variant (small inputs)
@pytest.mark.parametrize("dtype,op", [("float32", "sum"), ("int32", "sum"), ("float64", "prod"), ("uint32", "min"),
                                      ("int64", "xor"), ("float32", "argmin"), ("float64", "argmax"),
                                      ("float32", "max"), ("float64", "sum_compensated"), ("int32", "argmax")])
def test_cluster_variant(rd, dtype, op):
    """The one-cluster kernel (2..16 CTAs combined over DSMEM): every forced grid size 1..16,
    misaligned bases, and AUTO's choice at 32 KB < n*s <= 512 KB."""
    wl = inputs.default_workload(dtype, op)
    s = np.dtype(dtype).itemsize
    for n in (1, 9, 4099, (1 << 15) // s + 1, (1 << 17) // s + 5, (1 << 19) // s, (1 << 20) // s - 3):
        x = inputs.generate(n, dtype, wl, seed=n % 5 + 1)
        for off in (0, 3):
            xd = to_dev(x, off)
            for g in (1, 2, 3, 8, 13, 16):
                out, info = rd.reduce_ex(xd, op, variant="cluster", grid=g)
                assert info["variant"] == "cluster" and info["grid"] == g
                _parity.check(val(out), x, op)
            out, info = rd.reduce_ex(xd, op)
            if (1 << 15) < n * s <= (1 << 20):
                assert info["variant"] == "cluster" and 1 <= info["grid"] <= 16, info
            _parity.check(val(out), x, op)
    with pytest.raises(rd.ReduceError):
        rd.reduce_ex(to_dev(inputs.generate(1000, dtype, wl)), op, variant="cluster", grid=17)


def test_cluster_variant_records_graph_and_fused(rd):
    """The cluster kernel writing records, captured in a CUDA graph, and inside the fused
    exchange (virtual ranks)."""
    n = (1 << 17) + 11                                # 512 KB of float32 -> AUTO: cluster
    x = inputs.generate(n, "float32", "u01", seed=4)
    xd = to_dev(x, 1)
    assert rd.reduce_ex(xd, "sum")[1]["variant"] == "cluster"
    recs = torch.empty(4 * 32, dtype=torch.uint8, device="cuda")
    for r in range(4):
        b, c = rd.shard_range(n, 4, r)
        rd.reduce_partial(xd[b:b + c], "sum", rec=recs[r * 32:(r + 1) * 32])
    _parity.check(val(rd.combine_records(recs, "float32", "sum")), x, "sum")
    out = torch.empty((), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        rd.reduce(xd, "sum", out=out)
    torch.cuda.synchronize()
    want = val(out)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rd.reduce(xd, "sum", out=out)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert val(out).tobytes() == want.tobytes()
    W = 3
    comms = rd.FusedComm.local(W, torch.cuda.current_device())
    streams = [torch.cuda.Stream() for _ in range(W)]
    try:
        for op in ("sum", "argmax", "xor"):
            dt = "int32" if op == "xor" else "float32"
            xx = inputs.generate(3 * (1 << 16) + 7, dt, inputs.default_workload(dt, op), seed=2)
            xdd = to_dev(xx)
            outs = []
            for r in range(W):
                b, c = rd.shard_range(xx.size, W, r)
                with torch.cuda.stream(streams[r]):
                    outs.append(comms[r].reduce(xdd[b:b + c], op))
            torch.cuda.synchronize()
            for r in range(W):
                comms[r].check(streams[r])
            vals = [val(o) for o in outs]
            assert all(repr(v) == repr(vals[0]) for v in vals)
            _parity.check(vals[0], xx, op)
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()
