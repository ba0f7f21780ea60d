"""The C-ABI library (CPU-only checks): it loads, exports every symbol that
include/*.h declares, and its host-side logic (argument validation, identity
table, shard split) behaves as the header states. No compute calls here."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

import oracle
import paper_1710_07358_b200 as rd
from paper_1710_07358_b200 import _lib
from paper_1710_07358_b200.build import build_library

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    build_library()


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z_0-9]*\s*\*?\s+\*?([A-Za-z_][A-Za-z_0-9]*)\s*\(",
                             src, flags=re.M):
            names.add(m.group(1))
    return names


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["reduce", "reduce_partial", "reduce_multi", "rd_combine_records", "reduce_host",
                 "rd_get_unique_id", "rd_comm_init", "rd_comm_destroy", "rd_comm_check",
                 "rd_identity", "rd_release_workspaces", "rd_status_string", "rd_last_error",
                 "rd_shard_range", "rd_reduce_ex", "reduce_fused", "rd_fused_create",
                 "rd_fused_connect", "rd_fused_connect_local", "rd_fused_mailbox", "rd_fused_check",
                 "rd_fused_destroy", "reduce_exact_partial", "rd_combine_exact_records"]:
        assert must in names, must


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_functions():
        assert hasattr(L, name), f"libb200reduce.so does not export {name}"
    assert set(_lib.SIGNATURES) == declared_functions()


def test_record_layout():
    assert ctypes.sizeof(_lib.rd_record) == 32 == rd.RECORD_BYTES
    assert ctypes.sizeof(_lib.rd_unique_id) == 128
    assert ctypes.sizeof(_lib.rd_exact_record) == 608 == rd.EXACT_RECORD_BYTES
    assert _lib.rd_exact_record.word.offset == 32


def test_status_strings():
    L = _lib.lib()
    for code, name in _lib.STATUS.items():
        assert L.rd_status_string(code).decode() == name


@pytest.mark.parametrize("dtype", ["int32", "uint32", "int64", "float32", "float64"])
@pytest.mark.parametrize("op", list(rd.OPS))
def test_identity_matches_oracle(dtype, op):
    """Two independent implementations of the empty-result table agree."""
    if dtype.startswith("float") and op in ("and", "or", "xor"):
        with pytest.raises(rd.ReduceError) as e:
            rd.identity(dtype, op)
        assert e.value.status == 2
        return
    if op in rd.ARG_OPS:
        v, i = rd.identity(dtype, op)
        assert i == -1 and v.tobytes() == oracle.identity(dtype, op).tobytes()
        assert oracle.reduce(np.zeros(0, dtype), op).index == -1
        return
    a = rd.identity(dtype, op)
    b = oracle.identity(dtype, op)
    assert a.tobytes() == b.tobytes()


def test_validation_before_any_device_work():
    """Bad calls fail synchronously with the documented status and touch nothing
    (no CUDA device needed: validation precedes every CUDA call)."""
    L = _lib.lib()
    buf = (ctypes.c_char * 64)()
    p = ctypes.addressof(buf)
    p = p + (-p) % 16
    out = ctypes.c_void_p(p)
    assert L.reduce(None, 5, 0, 0, out, None) == 1                 # x NULL, n > 0
    assert L.reduce(p, 5, 0, 0, None, None) == 1                   # out NULL
    assert L.reduce(p, 5, 9, 0, out, None) == 1                    # unknown dtype
    assert L.reduce(p, 5, 0, 11, out, None) == 1                   # unknown op
    assert L.reduce_partial(p, 5, 3, 10, out, None) == 2           # exact float partial needs a wide record
    assert L.rd_combine_records(p, 1, 4, 10, out, None, None, None) == 2
    assert L.reduce_fused(p, 4, 3, 10, out, None, None) == 1        # comm NULL
    assert L.reduce_exact_partial(p, 5, 0, out, None) == 2         # integer dtype: use reduce_partial
    assert L.reduce_exact_partial(None, 5, 3, out, None) == 1
    assert L.reduce_exact_partial(p + 2, 5, 3, out, None) == 3
    assert L.rd_combine_exact_records(p, 1, 2, out, None, None, None) == 2
    assert L.rd_combine_exact_records(None, 2, 3, out, None, None, None) == 1
    assert L.rd_combine_exact_records(p, 1, 3, None, None, None, None) == 1
    assert L.reduce(p, 5, 0, 7, ctypes.c_void_p(p + 4), None) == 3  # argmin result not 8-aligned
    for op in (4, 5, 6):
        assert L.reduce(p, 5, 3, op, out, None) == 2               # bitwise on float32
        assert L.reduce(p, 5, 4, op, out, None) == 2               # bitwise on float64
    assert L.reduce(p + 2, 5, 0, 0, out, None) == 3                # int32 base not 4-aligned
    assert L.reduce(p + 4, 5, 2, 0, out, None) == 3                # int64 base not 8-aligned
    assert L.reduce(p, 5, 2, 0, ctypes.c_void_p(p + 4), None) == 3  # out misaligned
    assert L.reduce(p, 1 << 41, 0, 0, out, None) == 1              # n too large
    assert "NULL" in L.rd_last_error().decode() or L.rd_last_error()
    assert L.reduce_host(None, 3, 0, 0, out) == 1
    assert L.rd_combine_records(None, 2, 0, 0, out, None, None, None) == 1
    assert L.rd_combine_records(None, -1, 0, 0, out, None, None, None) == 1
    assert L.reduce_multi(p, 4, 0, 0, out, None, None) == 1        # comm NULL
    h = ctypes.c_void_p()
    assert L.rd_fused_create(ctypes.byref(h), 33, 0, 0, None) == 1  # nranks > 32
    assert L.rd_fused_create(ctypes.byref(h), 2, 2, 0, None) == 1   # rank out of range
    assert L.reduce_fused(p, 4, 0, 0, out, None, None) == 1         # comm NULL
    cfg = _lib.rd_config(7, 0, 0, 0, 0)
    assert L.rd_reduce_ex(p, 4, 0, 0, out, None, ctypes.byref(cfg), None) == 1
    cfg = _lib.rd_config(1, 32, 3, 0, 0)                           # U=3 only for the ablation pairs
    assert L.rd_reduce_ex(p, 4, 2, 1, out, None, ctypes.byref(cfg), None) == 2


@pytest.mark.parametrize("n", [0, 1, 7, 8, 1000, 5533214, (1 << 34) + 5])
@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
def test_shard_range_partitions(n, W):
    """Contiguous blocks in rank order, covering [0, n) exactly, sizes differ by <= 1."""
    spans = [rd.shard_range(n, W, r) for r in range(W)]
    pos = 0
    for b, c in spans:
        assert b == pos
        pos += c
    assert pos == n
    sizes = [c for _, c in spans]
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(rd.ReduceError):
        rd.shard_range(n, W, W)


def test_header_is_plain_c_and_links(tmp_path):
    """include/b200reduce.h compiles as C99 (no C++ in the ABI) and a C program
    links against libb200reduce.so (examples/reduce_example.c)."""
    import subprocess
    exe = tmp_path / "reduce_example"
    cmd = ["gcc", "-std=c99", "-Wall", "-Werror", "-O2", os.path.join(ROOT, "examples", "reduce_example.c"),
           "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           "-L", os.path.join(ROOT, "paper_1710_07358_b200"), "-lb200reduce",
           f"-Wl,-rpath,{os.path.join(ROOT, 'paper_1710_07358_b200')}",
           "-L", "/usr/local/cuda/lib64", "-lcudart", "-o", str(exe)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert exe.exists()


def test_shipped_library_reads_no_tuning_environment():
    """the RD_TUNE_* knobs change the chunk schedule and grid (so the
    bits of float +); they exist only in RD_TUNING builds (build.py --tuning). The shipped
    library carries none of their names, and the binding loads only the in-tree build."""
    blob = open(_lib.LIB_PATH, "rb").read()
    for knob in (b"RD_TUNE_HEAD_PER_SM", b"RD_TUNE_TAIL_PER_SM", b"RD_TUNE_TAIL_STAGES",
                 b"RD_TUNE_VEC_CTAS_PER_SM", b"RD_TUNE_EXACT", b"RD_LIB_PATH"):
        assert knob not in blob, knob
    assert _lib.LIB_PATH == os.path.join(ROOT, "paper_1710_07358_b200", "libb200reduce.so")
    src = open(os.path.join(ROOT, "paper_1710_07358_b200", "_lib.py")).read()
    assert "os.environ" not in src and "getenv" not in src
