"""Parity of the exact float sum (RD_SUM_EXACT, reading
R17) with the oracle: the exact sum rounded once is unique, so every
comparison is bit for bit -- across sizes, base offsets, grids, shard splits,
the host path, the NCCL path, specials and full BASELINE sizes. Needs a B200."""
from __future__ import annotations

import numpy as np
import pytest

import inputs
import oracle
from tests import _parity
from tests.test_gpu_parity import SIZES, to_dev, val

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FLT = ["float32", "float64"]
WLS = ["u01", "normalish", "wide", "wide_full"]


@pytest.fixture(scope="module")
def rd():
    from paper_1710_07358_b200.build import build_all
    build_all()
    import paper_1710_07358_b200 as m
    return m


def bits(v):
    return np.asarray(v).tobytes()


def same(g, want):
    g, want = np.asarray(g), np.asarray(want)
    if np.isnan(want):
        return bool(np.isnan(g))
    return g.tobytes() == want.tobytes()


@pytest.mark.parametrize("dtype", FLT)
@pytest.mark.parametrize("wl", WLS)
def test_exact_sizes(rd, dtype, wl):
    for n in SIZES:
        x = inputs.generate(n, dtype, wl, seed=n % 5 + 1)
        r = oracle.reduce(x, "sum_exact")
        assert same(val(rd.reduce(to_dev(x), "sum_exact")), r.value), (dtype, wl, n)


@pytest.mark.parametrize("dtype", FLT)
def test_exact_offsets_grids_and_shards(rd, dtype):
    """One result for every base offset, grid and split into records (reading R17)."""
    n = (1 << 20) + 13
    x = inputs.generate(n, dtype, "wide", seed=3)
    want = oracle.reduce(x, "sum_exact").value
    for off in range(8):
        xd = to_dev(x, off)
        assert same(val(rd.reduce(xd, "sum_exact")), want), off
        assert same(val(rd.reduce_ex(xd, "sum_exact", variant="bulk")[0]), want), off
    xd = to_dev(x, 3)
    for variant in ("vector", "bulk", "cluster"):
        for grid in ((1, 2, 3, 7, 16) if variant == "cluster" else (1, 2, 3, 7, 148, 296, 1000, 4096)):
            got, info = rd.reduce_ex(xd, "sum_exact", variant=variant, grid=grid)
            assert info["grid"] == grid and info["variant"] == variant and same(val(got), want), (variant, grid)
    RB = rd.EXACT_RECORD_BYTES
    for W in (1, 2, 3, 8, 17):
        recs = torch.empty(W * RB, dtype=torch.uint8, device="cuda")
        for r in range(W):
            b, c = rd.shard_range(n, W, r)
            rd.reduce_exact_partial(xd[b:b + c], rec=recs[r * RB:(r + 1) * RB])
        assert same(val(rd.combine_exact_records(recs, dtype)), want), W
        # records add in any order
        perm = torch.randperm(W).tolist()
        shuffled = torch.cat([recs[p * RB:(p + 1) * RB] for p in perm])
        assert same(val(rd.combine_exact_records(shuffled, dtype)), want)
        # a combined record combines again
        rec2 = torch.empty(RB, dtype=torch.uint8, device="cuda")
        rd.combine_exact_records(recs, dtype, rec_out=rec2)
        assert same(val(rd.combine_exact_records(rec2, dtype)), want)


@pytest.mark.parametrize("dtype", FLT)
def test_exact_host_and_multi(rd, dtype):
    n = (1 << 23) + 5                                   # several 32 MiB host chunks
    x = inputs.generate(n, dtype, "wide", seed=4)
    want = oracle.reduce(x, "sum_exact").value
    assert same(rd.reduce_host(x, "sum_exact"), want)
    assert same(rd.reduce_host(torch.from_numpy(x).pin_memory(), "sum_exact"), want)
    import ctypes
    from paper_1710_07358_b200 import _lib
    L = _lib.lib()
    uid = _lib.rd_unique_id()
    assert L.rd_get_unique_id(ctypes.byref(uid)) == 0
    h = ctypes.c_void_p()
    assert L.rd_comm_init(ctypes.byref(h), 1, 0, ctypes.byref(uid), torch.cuda.current_device()) == 0
    comm = rd.Comm(h.value, 1, 0, torch.cuda.current_device())
    try:
        assert same(val(comm.reduce(to_dev(x, 1), "sum_exact")), want)
        comm.check()
    finally:
        comm.destroy()


def _specials(dtype):
    f = np.finfo(dtype)
    big, tiny = f.max, f.smallest_subnormal
    return [
        [np.nan], [np.inf, 1.0], [-np.inf, 1.0], [np.inf, -np.inf], [1.0, np.nan, -np.inf],
        [-0.0], [-0.0, -0.0, -0.0], [-0.0, 0.0], [1.0, -1.0], [0.0],
        [big, big], [big, big, -big], [-big, -big], [big] * 5 + [-big] * 4,
        [tiny] * 7, [tiny, -tiny], [1.5, 2.0 ** 100, -(2.0 ** 100)],     # P:50 fn 2
        [1.0, 1e30, 1.0, -1e30], [1.0, 2.0 ** -24], [1.0, 2.0 ** -53], [1.0, 3 * 2.0 ** -24],
    ]


@pytest.mark.parametrize("dtype", FLT)
def test_exact_specials(rd, dtype):
    """Specials, signed zeros, overflow of the exact sum, subnormals, ties -- alone and
    buried in a larger array (so they sit in the body, head and tail of the kernel)."""
    with np.errstate(over="ignore"):
        cases = [np.array(c, dtype=dtype) for c in _specials(dtype)]
    for c in cases:
        assert same(val(rd.reduce(to_dev(c), "sum_exact")), oracle.reduce(c, "sum_exact").value), c
        for pos in (0, 5000, 10000 - c.size):
            x = np.zeros(10000, dtype=dtype)
            if c[0] == 0 and np.signbit(c[0]):
                x[:] = -0.0                             # keep "every term is -0.0" cases intact
            x[pos:pos + c.size] = c
            assert same(val(rd.reduce(to_dev(x, 1), "sum_exact")), oracle.reduce(x, "sum_exact").value), (c, pos)


@pytest.mark.parametrize("dtype", FLT)
@pytest.mark.parametrize("wl", ["u01", "normalish", "wide"])
def test_exact_full_size(rd, dtype, wl):
    """BASELINE configs[1] size, n = 2^28: bit-exact vs the oracle; the same bits from a
    forced grid and from an 8-way split (reading R17: reproducible across GPU counts)."""
    n = 1 << 28
    x = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
    inputs.fill_device(x, wl, seed=1)
    g = val(rd.reduce(x, "sum_exact"))
    RB = rd.EXACT_RECORD_BYTES
    recs = torch.empty(8 * RB, dtype=torch.uint8, device="cuda")
    for r in range(8):
        b, c = rd.shard_range(n, 8, r)
        rd.reduce_exact_partial(x[b:b + c], rec=recs[r * RB:(r + 1) * RB])
    alt = {bits(val(rd.combine_exact_records(recs, dtype))), bits(val(rd.reduce_ex(x, "sum_exact", grid=999)[0])),
           bits(val(rd.reduce_ex(x, "sum_exact", variant="vector")[0])),
           bits(val(rd.reduce_ex(x, "sum_exact", variant="bulk", grid=37)[0]))}
    xh = x.cpu().numpy()
    del x
    want = oracle.reduce(xh, "sum_exact").value
    assert same(g, want) and alt == {bits(g)}
    if wl != "wide":   # exact sum within the 4 eps sum|x| bound of the plain sum's contract too
        _parity.check(g, xh, "sum")


def test_exact_integers_are_sum(rd):
    for dt in ("int32", "uint32", "int64"):
        x = inputs.generate(100003, dt, "uniform_bits", seed=2)
        xd = to_dev(x, 1)
        assert bits(val(rd.reduce(xd, "sum_exact"))) == bits(val(rd.reduce(xd, "sum")))
        rec = rd.reduce_partial(xd, "sum_exact")
        assert bits(val(rd.combine_records(rec, dt, "sum_exact"))) == bits(oracle.reduce(x, "sum").value)


def test_exact_graph_capture(rd):
    x = to_dev(inputs.generate(1 << 22, "float32", "wide", seed=9), 2)
    want = val(rd.reduce(x, "sum_exact"))
    out = torch.empty((), dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        rd.reduce(x, "sum_exact", out=out)        # workspace for this stream outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        rd.reduce(x, "sum_exact", out=out)
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert bits(val(out)) == bits(want)


def test_exact_concurrent_streams_and_mixed_ops(rd):
    """Exact sums on concurrent streams (per-stream workspaces: slots, ticket, chunk counter),
    interleaved with plain sums and argmax on the same streams -- every result exact."""
    xs = [inputs.generate((1 << 21) + 7 * i, "float32" if i % 2 else "float64", "wide", seed=i + 1) for i in range(4)]
    ds = [to_dev(x, i) for i, x in enumerate(xs)]
    wants = [oracle.reduce(x, "sum_exact").value for x in xs]
    streams = [torch.cuda.Stream() for _ in xs]
    for rep in range(3):
        outs = []
        for d, s in zip(ds, streams):
            with torch.cuda.stream(s):
                rd.reduce(d, "sum")
                outs.append(rd.reduce(d, "sum_exact"))
                rd.reduce(d, "argmax")
                if rep == 1:                      # the bulk variant on the same stream too
                    outs[-1] = rd.reduce_ex(d, "sum_exact", variant="bulk")[0]
        torch.cuda.synchronize()
        for o, w in zip(outs, wants):
            assert same(val(o), w)


@pytest.mark.parametrize("dtype", FLT)
def test_exact_cluster_small_sizes(rd, dtype):
    """AUTO's one-cluster exact kernel at 48 KB < n*s <= 1 MiB (every grid 1..16 forced too),
    as a record, and through the fused exchange."""
    s = np.dtype(dtype).itemsize
    for n in ((1 << 16) // s + 3, (1 << 18) // s + 1, (1 << 20) // s):
        x = inputs.generate(n, dtype, "wide", seed=n % 7 + 1)
        want = oracle.reduce(x, "sum_exact").value
        xd = to_dev(x, 5)
        got, info = rd.reduce_ex(xd, "sum_exact")
        assert info["variant"] == "cluster" and same(val(got), want)
        for g in range(1, 17, 3):
            assert same(val(rd.reduce_ex(xd, "sum_exact", variant="cluster", grid=g)[0]), want)
        rec = rd.reduce_exact_partial(xd)
        assert same(val(rd.combine_exact_records(rec, dtype)), want)
    comms = rd.FusedComm.local(2, torch.cuda.current_device())
    streams = [torch.cuda.Stream() for _ in range(2)]
    try:
        n = (1 << 19) // s + 9
        x = inputs.generate(n, dtype, "wide", seed=3)
        xd = to_dev(x)
        outs = []
        for r in range(2):
            b, c = rd.shard_range(n, 2, r)
            with torch.cuda.stream(streams[r]):
                outs.append(comms[r].reduce(xd[b:b + c], "sum_exact"))
        torch.cuda.synchronize()
        for r in range(2):
            comms[r].check(streams[r])
        want = oracle.reduce(x, "sum_exact").value
        assert all(same(val(o), want) for o in outs)
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("dtype", FLT)
def test_exact_carry_chains(rd, dtype):
    """Totals whose carried words are long ripple chains (the warp carry-lookahead
    in rd_exact.cuh sacc_normalise_warp): a tiny negative total leaves a run of
    0xffffffff digits up to the top word; a huge value cancelled by its negative
    up to one subnormal crosses every word; both signs at once in one launch."""
    fi = np.finfo(dtype)
    tiny = fi.smallest_subnormal
    rng = np.random.default_rng(5)
    cases = []
    for n in (1, 33, 4099, (1 << 16) + 7, (1 << 20) + 3):
        for sgn in (-1.0, 1.0):
            x = np.zeros(n, dtype)
            x[n // 2] = sgn * tiny                                     # one subnormal unit
            cases.append(x)
            y = rng.standard_normal(n).astype(dtype) * np.asarray(2.0, dtype) ** rng.integers(-40, 40, n).astype(dtype)
            y = np.concatenate([y[:n // 2], [sgn * tiny], -y[::-1], y[n // 2:]]).astype(dtype)  # cancels up to +-tiny
            cases.append(y)
            z = np.zeros(n, dtype)
            z[0], z[-1] = fi.max, -fi.max
            if n > 2:
                z[1] = sgn * tiny
            cases.append(z)
    for x in cases:
        want = oracle.reduce(x, "sum_exact").value
        xd = to_dev(x, 1)
        for variant in ("auto", "vector", "bulk", "cluster"):
            got = rd.reduce_ex(xd, "sum_exact", variant=variant)[0]
            assert same(val(got), want), (dtype, len(x), variant)
        rec = rd.reduce_exact_partial(xd)
        assert same(val(rd.combine_exact_records(rec, dtype)), want)


def _ramp(n, dtype, lo, hi, rng, up=True):
    """Magnitudes that grow (or shrink) along the array: every thread's grid-stride
    share sees its maximum grow, so the bins re-anchor again and again (or, shrinking,
    terms fall below the last bin and are deposited)."""
    e = np.linspace(lo, hi, n) if up else np.linspace(hi, lo, n)
    m = rng.random(n) + 0.5
    return (rng.choice([-1.0, 1.0], n) * np.ldexp(m, np.floor(e).astype(int))).astype(dtype)


@pytest.mark.parametrize("dtype", FLT)
def test_exact_bins(rd, dtype):
    """The binned-extraction fallback (rd_exact.cuh bins_group): re-anchoring on a
    growing maximum, terms below the last bin, the 4096-addition limit (one CTA, long
    per-thread runs), groups that alternate between the group path and the bins in
    one thread -- bit-exact against the oracle on every variant."""
    rng = np.random.default_rng(11)
    big = 120 if dtype == "float32" else 1000
    small = -140 if dtype == "float32" else -1070
    cases = [
        _ramp((1 << 20) + 3, dtype, -60, 60, rng),
        _ramp((1 << 20) + 3, dtype, -60, 60, rng, up=False),
        _ramp((1 << 18) + 1, dtype, small, big, rng),
        _ramp((1 << 18) + 1, dtype, small, big, rng, up=False),
    ]
    mixed = inputs.generate((1 << 20) + 5, dtype, "u01", seed=2)
    idx = rng.integers(0, mixed.size, mixed.size // 97)
    mixed[idx] = inputs.generate(idx.size, dtype, "wide", seed=3)
    cases.append(mixed)
    for x in cases:
        want = oracle.reduce(x, "sum_exact").value
        xd = to_dev(x, 3)
        for variant in ("auto", "vector", "bulk"):
            assert same(val(rd.reduce_ex(xd, "sum_exact", variant=variant)[0]), want), (dtype, variant)
    # specials among groups that take the bins: the warp holding them goes per
    # element, every other warp stays in the bins
    base = inputs.generate((1 << 20) + 3, dtype, "wide", seed=6)
    for specials in ([np.inf], [-np.inf], [np.nan], [np.inf, -np.inf], [-0.0, np.inf]):
        y = base.copy()
        y[rng.integers(0, y.size, len(specials))] = specials
        want = oracle.reduce(y, "sum_exact").value
        yd = to_dev(y, 1)
        for variant in ("auto", "vector", "bulk"):
            assert same(val(rd.reduce_ex(yd, "sum_exact", variant=variant)[0]), want), (dtype, specials, variant)
    # long per-thread runs: one CTA over 2^22 wide terms -> > 4096 additions per bin
    x = inputs.generate(1 << 22, dtype, "wide", seed=8)
    want = oracle.reduce(x, "sum_exact").value
    xd = to_dev(x)
    for variant in ("vector", "bulk"):
        assert same(val(rd.reduce_ex(xd, "sum_exact", variant=variant, grid=1)[0]), want), variant


def test_exact_fp64_subnormal_high_word_zero(rd):
    """A subnormal double below 2^-1042 has a zero high word. The fp64 group path's
    exponent-spread test reads high words, so it must not take such a term for a zero:
    here 2^-900 + 2^-1060 + (2^-900 + 2^-952) makes the group's error tree inexact
    (2^-952 + 2^-1060 rounds), and the exact sum's last bit depends on the 2^-1060."""
    a, t, b = 2.0 ** -900, 2.0 ** -1060, 2.0 ** -900 + 2.0 ** -952
    rng = np.random.default_rng(4)
    for pos in ([0, 1, 2], [0, 1, 1024], [2, 0, 1], [1024, 1025, 0]):
        for n in (4096, 1 << 16, (1 << 20) + 8):
            x = np.zeros(n, np.float64)
            x[pos] = (a, t, b)
            want = oracle.reduce(x, "sum_exact").value
            xd = to_dev(x)
            for variant in ("auto", "vector", "bulk"):
                assert same(val(rd.reduce_ex(xd, "sum_exact", variant=variant)[0]), want), (pos, n, variant)
    # randomised: terms near 2^-900 with 52-bit mantissas and high-word-zero subnormals
    n = (1 << 20) + 3
    x = np.ldexp(rng.random(n) + 1.0, -900) * rng.choice([-1.0, 1.0], n)
    sub = rng.random(n) < 0.3
    x[sub] = np.ldexp(rng.integers(1, 1 << 30, sub.sum()).astype(np.float64), -1074)
    want = oracle.reduce(x, "sum_exact").value
    xd = to_dev(x, 1)
    for variant in ("auto", "vector", "bulk"):
        assert same(val(rd.reduce_ex(xd, "sum_exact", variant=variant)[0]), want), variant


@pytest.mark.parametrize("dtype", FLT)
def test_exact_bins_at_scale(rd, dtype):
    """2^31 `wide` terms (8 / 16 GiB): ~28k terms per thread on the bulk kernel, so
    every warp re-anchors on its addition limit several times, with different
    thread-to-term assignments per form -- the whole array, 8 shard records, a
    forced grid and the vector form must give the same bits (reading R17)."""
    n = 1 << 31
    free, _ = torch.cuda.mem_get_info()
    if free < n * np.dtype(dtype).itemsize + (8 << 30):
        pytest.skip("needs the array plus 8 GiB of free HBM")
    x = torch.empty(n, dtype=getattr(torch, dtype), device="cuda")
    inputs.fill_device(x, "wide", seed=2)
    RB = rd.EXACT_RECORD_BYTES
    recs = torch.empty(8 * RB, dtype=torch.uint8, device="cuda")
    for r in range(8):
        b, c = rd.shard_range(n, 8, r)
        rd.reduce_exact_partial(x[b:b + c], rec=recs[r * RB:(r + 1) * RB])
    got = {bits(val(rd.reduce(x, "sum_exact"))), bits(val(rd.combine_exact_records(recs, dtype))),
           bits(val(rd.reduce_ex(x, "sum_exact", grid=777)[0])),
           bits(val(rd.reduce_ex(x, "sum_exact", variant="vector")[0]))}
    del x
    assert len(got) == 1


def test_exact_auto_plan(rd):
    """The exact sum's AUTO variant (rd_api.cu, profiles/r02_exact_variants.json): the
    one-cluster form up to 1 MiB; above it fp64 terms take the bulk ring at every size,
    fp32 terms the vector form below 128 MiB and the bulk ring from there."""
    def plan(dtype, nbytes):
        x = torch.zeros(nbytes // np.dtype(dtype).itemsize, dtype=getattr(torch, dtype), device="cuda")
        return rd.reduce_ex(x, "sum_exact")[1]["variant"]

    for dtype in FLT:
        assert plan(dtype, 512 << 10) == "cluster"
        assert plan(dtype, 1 << 20) == "cluster"
        assert plan(dtype, 128 << 20) == "bulk"
    assert plan("float64", 2 << 20) == "bulk" and plan("float64", 64 << 20) == "bulk"
    assert plan("float32", 2 << 20) == "vector" and plan("float32", 64 << 20) == "vector"
