"""The seeded input generators (inputs/): deterministic, shard-consistent, and
with the value distributions DESIGN.md's input recipe states. CPU only."""
import numpy as np
import pytest

import inputs

DT = ["int32", "uint32", "int64", "float32", "float64"]


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("wl", list(inputs.WORKLOADS))
def test_deterministic_and_shard_consistent(dtype, wl):
    try:
        a = inputs.generate(5000, dtype, wl, seed=7)
    except ValueError:
        pytest.skip("workload undefined for dtype")
    b = inputs.generate(5000, dtype, wl, seed=7)
    assert a.tobytes() == b.tobytes()
    # generating a shard [lo, hi) of the logical array equals slicing it
    s = inputs.generate(1234, dtype, wl, seed=7, offset=1000, n_total=5000)
    assert s.tobytes() == a[1000:2234].tobytes()
    c = inputs.generate(5000, dtype, wl, seed=8)
    if wl not in ("iota", "sparse_clear", "sparse_set", "sparse_pm1", "pow2_sparse"):
        assert a.tobytes() != c.tobytes()


def test_distributions():
    u = inputs.generate(1 << 16, "float32", "u01")
    assert 0.0 <= u.min() and u.max() < 1.0 and abs(u.mean() - 0.5) < 0.01
    g = inputs.generate(1 << 16, "float64", "normalish")
    assert abs(g.mean()) < 0.01 and abs(g.std() - (4 / 12) ** 0.5) < 0.01
    k = inputs.generate(1 << 16, "float32", "near_one")
    assert np.all(np.abs(k - 1) <= 64 * 2.0 ** -23)
    p = inputs.generate(1 << 20, "float64", "pow2_sparse")
    assert 50 <= int((p != 1).sum()) <= 160
    o = inputs.generate(1 << 12, "int64", "odd")
    assert np.all(o & 1 == 1)
    sc = inputs.generate(1 << 16, "uint32", "sparse_clear")
    assert 0 < int((sc != 0xFFFFFFFF).sum()) < 64
    pm = inputs.generate(1 << 22, "float32", "sparse_pm1")
    assert 0 < int((pm != 0).sum()) <= (1 << 21)
    for dt, lo, hi in (("float32", -40, 40), ("float64", -40, 40)):
        w = inputs.generate(1 << 16, dt, "wide")
        e = np.frexp(w)[1] - 1
        assert e.min() == lo and e.max() == hi and abs((w < 0).mean() - 0.5) < 0.02
    wf = inputs.generate(1 << 16, "float32", "wide_full")
    assert np.isfinite(wf).all() and (np.abs(wf) < np.finfo(np.float32).tiny).any() and np.abs(wf).max() > 1e38
    wd = inputs.generate(1 << 16, "float64", "wide_full")
    assert np.isfinite(wd).all() and (np.abs(wd) < np.finfo(np.float64).tiny).any() and np.abs(wd).max() > 1e307


def test_undefined_workloads_rejected():
    with pytest.raises(ValueError):
        inputs.generate(4, "float32", "odd")
    with pytest.raises(ValueError):
        inputs.generate(4, "int32", "u01")
