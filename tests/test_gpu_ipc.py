"""The fused exchange (reduce_fused) between two PROCESSES through
real CUDA IPC mappings -- rd_fused_create's exported handle, the gloo
all-gather of the handles, rd_fused_connect's cudaIpcOpenMemHandle -- with
both processes on the one GPU of the test box (the driver time-slices their
kernels; a rank's last CTA polls its mailbox until the peer's kernel has run).
On a multi-GPU box the same code maps a peer GPU's mailbox over NVLink; here
the mapping path itself is what is exercised. Needs a B200."""
from __future__ import annotations

import os
import pickle
import socket
import sys
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("float32", "sum", (1 << 20) + 7), ("float32", "sum_exact", (1 << 22) + 3), ("float64", "argmax", 100003),
         ("int32", "xor", 5533214), ("float64", "sum_exact", 4099)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import inputs
    import paper_1710_07358_b200 as rd
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = rd.FusedComm.from_process_group(device=0)
    out = {}
    try:
        for rep in range(2):                      # two epochs: both mailbox parities
            for dtype, op, n in CASES:
                b, c = rd.shard_range(n, world, rank)
                x = inputs.generate(c, dtype, inputs.default_workload(dtype, op), seed=rep + 1, offset=b, n_total=n)
                xd = torch.from_numpy(x).cuda()
                r = comm.reduce(xd, op)
                torch.cuda.synchronize()
                comm.check()
                if isinstance(r, tuple):
                    out[(rep, dtype, op)] = (r[0].cpu().numpy().tobytes(), int(r[1].item()))
                else:
                    out[(rep, dtype, op)] = r.cpu().numpy().tobytes()
    finally:
        dist.barrier()
        comm.destroy()
        dist.destroy_process_group()
    with open(os.path.join(outdir, f"ipc{rank}.pkl"), "wb") as f:
        pickle.dump(out, f)


def test_fused_exchange_two_processes_ipc():
    sys.path.insert(0, ROOT)
    import torch.multiprocessing as mp
    import inputs
    import oracle
    from tests import _parity
    from paper_1710_07358_b200.build import build_all
    build_all()
    with tempfile.TemporaryDirectory() as d:
        ctx = mp.start_processes(_worker, args=(2, _free_port(), d), nprocs=2, join=False, start_method="spawn")
        assert ctx.join(timeout=240) or ctx.join(timeout=60), "IPC ranks did not finish"
        outs = [pickle.load(open(os.path.join(d, f"ipc{r}.pkl"), "rb")) for r in range(2)]
    assert outs[0] == outs[1]                     # bitwise-identical on both ranks
    for (rep, dtype, op), v in outs[0].items():
        n = [c[2] for c in CASES if c[0] == dtype and c[1] == op][0]
        x = inputs.generate(n, dtype, inputs.default_workload(dtype, op), seed=rep + 1)
        if op == "argmax":
            _parity.check((np.frombuffer(v[0], dtype)[0], v[1]), x, op)
        else:
            _parity.check(np.frombuffer(v, dtype)[0], x, op)
