"""Multi-GPU parity of the sharded path: one process
per GPU under torch.distributed.run, NCCL and the fused in-kernel exchange, against
the oracle on the whole array (tests/_multi_worker.py). The W-rank cases run when
the box has W GPUs and are SKIPPED LOUDLY otherwise (a 1-GPU box still runs W = 1
through the same torchrun path). Plus the single-GPU checks of the communicator
set-up contract (include/b200reduce.h): the caller's device is kept, no other
stream is synchronised, plain/exact disagreement is a mismatch."""
from __future__ import annotations

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import inputs
from tests import _parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def rd():
    from paper_1710_07358_b200.build import build_all
    build_all()
    import paper_1710_07358_b200 as m
    return m


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _ngpus():
    return torch.cuda.device_count()


@pytest.mark.parametrize("W", [1, 2, 4, 8])
def test_torchrun_reduce_multi_and_fused(rd, W):
    if _ngpus() < W:
        pytest.skip(f"needs {W} GPUs for {W} ranks; this box has {_ngpus()} -- the {W}-rank NCCL and "
                    f"NVLink-fused exchange are NOT exercised here")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={W}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "_multi_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, (out.stdout[-4000:], out.stderr[-4000:])
    assert f"{W} rank(s)" in out.stdout and "0 failure(s)" in out.stdout


def test_fused_local_ranks_across_devices(rd):
    """rd_fused_connect_local with mailboxes on different devices: peer access is enabled
    by the library, one virtual rank per GPU, results identical to the oracle."""
    G = _ngpus()
    if G < 2:
        pytest.skip(f"needs >= 2 GPUs; this box has {G} -- cross-device peer stores NOT exercised here")
    comms = rd.FusedComm.local(G, devices=list(range(G)))
    try:
        for dtype, op, n in [("float32", "sum", (1 << 22) + 3), ("float64", "sum_exact", 100003),
                             ("int32", "max", 5533214)]:
            wl = inputs.default_workload(dtype, op) if op != "sum_exact" else "wide"
            xh = inputs.generate(n, dtype, wl, seed=2)
            outs = []
            for r in range(G):
                b, c = rd.shard_range(n, G, r)
                with torch.cuda.device(r):
                    xd = torch.from_numpy(xh[b:b + c].copy()).cuda(r)
                    st = torch.cuda.Stream(r)
                    with torch.cuda.stream(st):
                        outs.append((comms[r].reduce(xd, op), st, xd))
            for r in range(G):
                torch.cuda.synchronize(r)
                comms[r].check(outs[r][1])
            vals = [o[0].cpu().numpy().tobytes() for o in outs]
            assert all(v == vals[0] for v in vals)
            _parity.check(np.frombuffer(vals[0], dtype)[0], xh, op)
    finally:
        for r in range(G):
            torch.cuda.synchronize(r)
        for c in comms:
            c.destroy()


def test_comm_setup_keeps_device_and_other_streams(rd):
    """rd_comm_init / rd_fused_create / rd_fused_connect_local leave the caller's current
    device unchanged and do not wait for work on other streams."""
    import ctypes
    from paper_1710_07358_b200 import _lib
    dev = torch.cuda.current_device()
    warm = rd.FusedComm.local(2, dev)        # loads every kernel first (module loading may wait)
    for c in warm:
        c.destroy()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        torch.cuda._sleep(int(3e9))           # ~1.5 s of GPU time on another stream
    comms = rd.FusedComm.local(2, dev)
    assert not side.query(), "fused communicator set-up waited for another stream"
    assert torch.cuda.current_device() == dev
    L = _lib.lib()
    uid = _lib.rd_unique_id()
    assert L.rd_get_unique_id(ctypes.byref(uid)) == 0
    h = ctypes.c_void_p()
    assert L.rd_comm_init(ctypes.byref(h), 1, 0, ctypes.byref(uid), dev) == 0
    assert torch.cuda.current_device() == dev
    side.synchronize()
    rd.Comm(h.value, 1, 0, dev).destroy()
    for c in comms:
        c.destroy()


def test_fused_mismatch_plain_vs_exact(rd):
    """Ranks that disagree between a plain and an exact op (or two exact dtypes) report
    RD_ERR_MISMATCH, not RD_ERR_TIMEOUT: every record carries the common LL header
    (ADVICE r1)."""
    dev = torch.cuda.current_device()
    comms = rd.FusedComm.local(2, dev)
    streams = [torch.cuda.Stream() for _ in range(2)]
    try:
        x32 = torch.rand(5000, device="cuda")
        x64 = x32.double()
        for a, b in ((("sum", x32), ("sum_exact", x32)), (("sum_exact", x32), ("sum", x32)),
                     (("sum_exact", x32), ("sum_exact", x64)), (("max", x32), ("sum_exact", x32))):
            for r, (op, x) in enumerate((a, b)):
                with torch.cuda.stream(streams[r]):
                    comms[r].reduce(x, op)
            torch.cuda.synchronize()
            for r in range(2):
                with pytest.raises(rd.ReduceError) as e:
                    comms[r].check(streams[r])
                assert e.value.status == 6, (a[0], b[0], r, e.value)
        # and they agree again afterwards (epochs stay in step)
        for r in range(2):
            with torch.cuda.stream(streams[r]):
                comms[r].reduce(x32, "sum_exact")
        torch.cuda.synchronize()
        for r in range(2):
            comms[r].check(streams[r])
    finally:
        torch.cuda.synchronize()
        for c in comms:
            c.destroy()
