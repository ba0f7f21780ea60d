"""bench.py helpers and the reference arm's JSON contract (CPU only)."""
import csv
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_gbps_reproduces_paper_table2():
    """tests/golden/table2.csv: GB/s = n * 4 bytes / time, decimal,
    with n = 5,533,214 -- the convention bench.py reports in."""
    n = 5533214
    with open(os.path.join(ROOT, "tests", "golden", "table2.csv")) as f:
        rows = [r for r in csv.DictReader(l for l in f if not l.startswith("#"))]
    assert len(rows) == 9
    t1 = float(rows[0]["time_ms"])
    for r in rows:
        t = float(r["time_ms"]) * 1e-3
        assert abs(bench.gbps(n * 4, t) - float(r["gbps"])) / float(r["gbps"]) < 1e-9
        assert abs(t1 / float(r["time_ms"]) - float(r["speedup"])) < 1e-6
        # the usage column implies one peak for every row (~332.8 GB/s)
        peak = float(r["gbps"]) / (float(r["usage_pct"]) / 100)
        assert 332.6 < peak < 333.0


def test_reference_arm_json_line():
    """`bench.py --impl reference` prints one JSON line with the contract's keys."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "3", "--warmup", "1", "--log2n", "20"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_table3_percentage_reading():
    """Reading R12: the printed 99.4 is 100*T_k7/T_new, not the
    100*T_new/T_k7 the text states, which would give 100.57."""
    with open(os.path.join(ROOT, "tests", "golden", "table3.txt")) as f:
        row = [l for l in f if l.strip() and not l.startswith("#")][0]
    t_k7, t_new, printed = (float(c) for c in row.split("|"))
    assert round(100 * t_k7 / t_new, 1) == printed
    assert round(100 * t_new / t_k7, 1) != printed
