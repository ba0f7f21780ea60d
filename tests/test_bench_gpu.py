"""bench.py on a GPU: the JSON line carries every key of the contract."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run("--steps", "20", "--warmup", "3", "--log2n", "26", "--cpu-seconds", "0.5", "--c5-log2n", "27")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 20 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["gpu_launches"] == 20
    assert d["value"] > 100 and d["unit"] == "GB/s" and d["dtype"] == "f32"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 2 and r["peak"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] == 1 and c["value"] > 0 and c["all_core"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == (1 << 26) * 4 and e["d2h_bytes_per_step"] == 4
    assert "workload" in d["config"]
    ctx = d["context"]
    assert ctx["check"]["ok"] is True and ctx["check"]["err_over_bound"] < 1   # the timed result vs the oracle
    assert ctx["int32_sum"]["check_bit_exact"] is True and ctx["int32_sum"]["gbs"] > 100
    assert ctx["cub_device_reduce_gbs"] > 100 and ctx["torch_sum_gbs"] > 100
    assert 0.5 < r["frac_of_read_probe"] < 1.2 and d["pct_read_probe"] > 50
    c5 = ctx["c5"]
    assert c5["n_total"] == 1 << 27 and c5["ranks"] == 1 and "fused_error" not in c5
    for k in ("sum_nccl_gbs", "sum_fused_gbs", "max_nccl_gbs", "max_fused_gbs"):
        assert c5[k] > 100, k
    assert c5["check"]["max_is_planted"] and c5["check"]["fused_equals_nccl"] and c5["check"]["sum_within_bound"]


def test_bench_force_comm_paths():
    for exch in ("fused", "nccl"):
        d = _run("--steps", "10", "--warmup", "3", "--log2n", "24", "--no-cpu", "--force-comm", "--exchange", exch,
                 "--no-c5")
        assert d["value"] > 100
        assert d["context"]["check"]["ok"] is True
        assert ("fused" in d["config"]["exchange"]) == (exch == "fused")
