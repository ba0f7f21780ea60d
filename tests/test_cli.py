"""The command line front end (exit codes 0 ok, 1 verification
failure, 2 usage, 3 runtime -- SPEC S:407)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def cli(*args, timeout=300):
    return subprocess.run([sys.executable, "-m", "paper_1710_07358_b200", *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout)


def test_usage_errors_exit_2():
    assert cli().returncode == 2                                  # --op missing
    assert cli("--op", "median").returncode == 2                  # unknown op
    assert cli("--op", "sum", "--dtype", "float16").returncode == 2


def test_no_gpu_exits_3():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert cli("--op", "sum").returncode == 3


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,op,n", [("float32", "sum", (1 << 20) + 3), ("int64", "xor", 5533214),
                                        ("float64", "argmax", 100003), ("float32", "sum_exact", 1 << 22),
                                        ("uint32", "min", 7)])
def test_cli_result_and_check(dtype, op, n):
    import inputs
    import oracle
    from tests import _parity
    r = cli("--op", op, "--dtype", dtype, "--n", str(n), "--check", "--json")
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["check"] == "ok" and d["n"] == n
    x = inputs.generate(n, dtype, inputs.default_workload(dtype, op), seed=1)
    got = d["result"]
    if op == "argmax":
        _parity.check((np.array([got[0]], dtype)[0], got[1]), x, op)
    else:
        _parity.check(np.array([got], dtype)[0], x, op)


@pytest.mark.gpu
def test_cli_npy_input_and_unsupported(tmp_path):
    x = np.arange(1000, dtype=np.int32)
    f = tmp_path / "x.npy"
    np.save(f, x)
    r = cli("--op", "sum", "--input", str(f))
    assert r.returncode == 0 and int(r.stdout.strip()) == 999 * 1000 // 2
    np.save(f, x.astype(np.float32))
    assert cli("--op", "xor", "--input", str(f)).returncode == 2    # bitwise on floats: unsupported
